# GPU tests, then the K1 work-item sweep (scripts/k1_sweep.sh) on the bench workload
mkdir -p gpurun_out
[ -n "$NO_TESTS" ] || { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; }
bash scripts/k1_sweep.sh 2>&1 | tee gpurun_out/k1_sweep.txt
[ -n "$PROF" ] && NO_LAUNCH_LIST=1 NO_WP=1 bash scripts/gpu_prof_k1.sh
