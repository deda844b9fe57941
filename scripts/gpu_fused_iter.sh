#!/bin/bash
# fused narrow tcgen05 MLP: correctness (agreement tests), timing A/B, launch list
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -s > gpurun_out/tc.log 2>&1
echo "tc tests rc=$?"; grep "bf16_tc\]" gpurun_out/tc.log; tail -3 gpurun_out/tc.log
for f in 1 0; do
  CYR_TC_FUSED=$f timeout 300 python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_fused.csv python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_fused.csv | tail -25
