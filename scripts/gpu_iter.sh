# Quick GPU iteration: parity tests, latency trace, K3-heavy Mode-T probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 300 | head -30
timeout 300 python scripts/latency_probe.py --calls 2000 | head -3
timeout 600 python scripts/mode_t_probe.py --reps 3 --cfg cfg2 --slots 8 --precision bf16_tc
timeout 600 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc
