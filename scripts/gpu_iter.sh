# Quick GPU iteration: parity tests, Mode-T probes (A/B of the layer-GEMM path), launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
P="python scripts/mode_t_probe.py --reps 2"
timeout 600 $P --cfg cfg5 --slots 1 --precision fp32
for g in wide all; do
  echo "CYR_ACTOR_GEMM=$g"; CYR_ACTOR_GEMM=$g timeout 600 $P --cfg cfg2 --slots 8 --precision fp32
done
CYR_ACTOR_GEMM=all timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_it_cfg2g.csv python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 8 --precision fp32 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_it_cfg2g.csv | tail -12
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_it_cfg5.csv python scripts/mode_t_probe.py --reps 1 --cfg cfg5 --slots 1 --precision fp32 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_it_cfg5.csv | tail -7
