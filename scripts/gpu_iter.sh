# Quick GPU iteration: parity tests, Mode-T probes with launch lists (K3 focus).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for c in "cfg2 8 fp32" "cfg5 1 bf16_tc"; do
  set -- $c
  timeout 600 python scripts/mode_t_probe.py --reps 3 --cfg $1 --slots $2 --precision $3
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_k3_$1.csv python scripts/mode_t_probe.py --reps 1 --cfg $1 --slots $2 --precision $3 > /dev/null 2>&1
  python scripts/launch_table.py gpurun_out/launches_k3_$1.csv | grep -E "tree_level_kernel|total"
done
