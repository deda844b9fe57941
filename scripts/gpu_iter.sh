# Quick GPU iteration: parity tests, Mode-T probes (A/B), launch list, tiled-actor ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
P="python scripts/mode_t_probe.py --reps 3"
for v in 0 1; do
  echo "CYR_TILED16=$v"
  CYR_TILED16=$v timeout 300 $P --cfg cfg2 --slots 8 --precision fp32
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_iter.csv python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 8 --precision fp32 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_iter.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:actor_tiled_kernel -s 13 -c 1 \
  -o gpurun_out/prof_mt_tiled4 python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 8 --precision fp32 > gpurun_out/ncu_it.log 2>&1; echo "ncu tiled rc=$?"
