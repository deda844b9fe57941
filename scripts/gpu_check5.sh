mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 300
timeout 300 python scripts/latency_probe.py --calls 1000
CYR_ACTOR_CLUSTER=16 timeout 300 python scripts/latency_probe.py --calls 1000
timeout 300 python scripts/kernel_probe.py --slots 1024 > gpurun_out/probe_1024.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/probe_1024.json')); [print(s,k,round(v['p50_us'],2)) for s in d for k,v in d[s].items()]"
