mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/kernel_probe.py > gpurun_out/probe.json 2> gpurun_out/probe.err; echo "probe rc=$?"
cat gpurun_out/probe.json | python -c "import json,sys; d=json.load(sys.stdin); [print(s,k,round(v['p50_us'],2)) for s in d for k,v in d[s].items()]"
tail -3 gpurun_out/probe.err
