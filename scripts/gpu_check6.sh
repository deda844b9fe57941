timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/latency_probe.py --calls 2000
CYR_SLOT_GRAPH=0 timeout 300 python scripts/latency_probe.py --calls 2000
CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 300
