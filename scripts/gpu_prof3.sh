mkdir -p gpurun_out
timeout 300 python scripts/latency_probe.py --calls 30 > gpurun_out/lat_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_lat.csv python scripts/latency_probe.py --calls 30 > gpurun_out/ncu_lat.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/lat_plain.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_lat.csv')) if len(r)>10]
hdr=rows[0]; k=hdr.index('Kernel Name'); v=hdr.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]:
    try: d[r[k][:40]].append(float(r[v]))
    except: pass
for name,vals in d.items():
    vals=sorted(vals); print(name, len(vals), 'median', vals[len(vals)//2])
PY
