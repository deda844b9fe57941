# GPU tests + Mode-T probe timings (cfg2 32-slot fp32 / bf16, cfg5 fp32 / bf16)
mkdir -p gpurun_out
[ -n "$NO_TESTS" ] || { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; }
P="python scripts/mode_t_probe.py --reps 3"
for c in "cfg2 32 fp32" "cfg2 32 bf16_tc" "cfg5 1 fp32" "cfg5 1 bf16_tc"; do
  set -- $c; timeout 600 $P --cfg $1 --slots $2 --precision $3 2>&1 | tail -1
done
