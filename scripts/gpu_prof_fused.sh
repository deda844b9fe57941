#!/bin/bash
# ncu --set full of the fused narrow tcgen05 MLP at the deepest cfg2 Mode-T level (2M columns)
cd "$GRAFT_REPO_ROOT"
P="python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1"
timeout 300 $P > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:actor_tc_fused \
  --launch-skip 4 --launch-count 1 -o gpurun_out/ncu_fused $P > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ncu_fused.ncu-rep --page details > gpurun_out/ncu_fused_details.txt 2>&1
ncu -i gpurun_out/ncu_fused.ncu-rep --page source --csv > gpurun_out/ncu_fused_source.csv 2>&1
grep -E "Duration|Throughput|Pipe|Issue|Warp Cycles|Eligible|Registers|Stall" gpurun_out/ncu_fused_details.txt | head -40
