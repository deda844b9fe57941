#!/bin/bash
# same-box A/B of compile-time variants: each argument is one CYR_NVCC_EXTRA
# string ("" = default); per variant the cfg2 / cfg5 bf16 Mode-T trees and the
# deepest cfg2 level's lane K3 (ncu, serialised)
cd "$GRAFT_REPO_ROOT"
for round in 1 2; do
for v in "$@"; do
  CYR_NVCC_EXTRA="$v" python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
  echo "== variant [$v] round $round"
  timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc
  timeout 300 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tree_level_kernel --csv \
    python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 2>/dev/null | grep 15625 | tail -1 | awk -F'","' '{print "deepest K3 ns", $NF}'
done
done
