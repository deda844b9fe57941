"""Summarise an ncu --page source --print-source sass CSV: hot instructions,
stall reasons and instruction mix.  usage: ncu_sass_hot.py file.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
def _num(x):
    try:
        float(x)
        return True
    except ValueError:
        return False
data = [r for r in rows[2:] if len(r) == len(hdr) and _num(r[hdr.index("Warp Stall Sampling (All Samples)")])]
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
execd = ix["Instructions Executed"]
stall_cols = [h for h in hdr if h.startswith("stall_")]
tot = sum(float(r[samp]) for r in data)
print(f"instructions in SASS: {len(data)}, total samples {tot:.0f}, "
      f"executed {sum(float(r[execd]) for r in data):.0f}")
op = Counter()
ex = Counter()
for r in data:
    name = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if name.startswith("@"):
        name = r[ix["Source"]].split()[1]
    name = name.split(".")[0]
    op[name] += float(r[samp])
    ex[name] += float(r[execd])
print("samples by opcode:", [(k, int(v)) for k, v in op.most_common(15)])
print("executed by opcode:", [(k, int(v)) for k, v in ex.most_common(15)])
st = Counter()
for r in data:
    for h in stall_cols:
        try:
            st[h] += float(r[ix[h]])
        except ValueError:
            pass
print("stalls:", [(k, int(v)) for k, v in st.most_common(10)])
hot = sorted(data, key=lambda r: -float(r[samp]))[:top]
for r in hot:
    print(f"{float(r[samp]):7.0f} {float(r[execd]):8.0f}  {r[ix['Address']][-5:]}  {r[ix['Source']][:70]}")
