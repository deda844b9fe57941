#!/bin/bash
# fused-kernel launch times (ncu, clocks unlocked) + tree timing + bf16 agreement tests
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:actor_tc_fused --csv \
  python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 32 --precision bf16_tc 2>/dev/null \
  | grep fused | tail -5 | awk -F'","' '{print $8, $NF}'
