#!/bin/bash
# lane K3 occupancy A/B (min blocks per SM): deepest cfg2 level time + tree
cd "$GRAFT_REPO_ROOT"
for mb in 5 6 7 8; do
  CYR_NVCC_EXTRA="-DCYR_LANE_MINB=$mb" python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
  echo "minblocks $mb"
  timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc
  timeout 300 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tree_level_kernel --csv \
    python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 2>/dev/null | grep 15625 | tail -3 | awk -F'","' '{print $(NF-2), $NF}'
done
