#!/bin/bash
# source-level ncu of the lane-mapped K3 on the deepest cfg2 Mode-T level (32-slot bf16 tree)
cd "$GRAFT_REPO_ROOT"
P="python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 32 --precision bf16_tc"
timeout 300 $P > gpurun_out/mt.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_level_kernel -s 3 -c 1 \
  -o gpurun_out/prof_k3lane $P > gpurun_out/ncu_k3lane.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_k3lane.ncu-rep --page source --csv --print-source cuda > gpurun_out/k3lane_src.csv 2>/dev/null
ncu -i gpurun_out/prof_k3lane.ncu-rep --page source --csv --print-source sass > gpurun_out/k3lane_sass.csv 2>/dev/null
ncu -i gpurun_out/prof_k3lane.ncu-rep --page details > gpurun_out/k3lane_details.txt 2>/dev/null
grep -E "Duration|Issue Slots|Eligible|Warp Cycles Per Issued" gpurun_out/k3lane_details.txt | head
