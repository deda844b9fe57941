mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/latency_probe.py --calls 300 > gpurun_out/lat_plain.log 2>&1; cat gpurun_out/lat_plain.log
timeout 300 python scripts/kernel_probe.py --slots 1024 > gpurun_out/probe_1024.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/probe_1024.json')); [print(s,k,round(v['p50_us'],2)) for s in d for k,v in d[s].items()]"
timeout 300 python scripts/latency_probe.py --calls 30 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_lat.csv python scripts/latency_probe.py --calls 30 > gpurun_out/ncu_lat.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/launches_lat.csv')) if len(r)>10]
hdr=rows[0]; k=hdr.index('Kernel Name'); v=hdr.index('Metric Value')
d=defaultdict(list)
for r in rows[1:]:
    try: d[r[k][:40]].append(float(r[v]))
    except: pass
for name,vals in d.items():
    vals=sorted(vals); print(name, len(vals), 'median ns', vals[len(vals)//2])
PY
