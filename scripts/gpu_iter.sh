# Quick GPU iteration: parity tests, Mode-T probes, launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bf16_agreement.json; echo
P="python scripts/mode_t_probe.py --reps 3"
timeout 600 $P --cfg cfg2 --slots 8 --precision bf16_tc
timeout 600 $P --cfg cfg5 --slots 1 --precision bf16_tc
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_it_cfg2b.csv python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 8 --precision bf16_tc > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_it_cfg2b.csv | tail -14
