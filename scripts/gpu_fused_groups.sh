#!/bin/bash
# builder groups A/B: Mode-R probe, Mode-T tree and its deepest-level fused MLP
cd "$GRAFT_REPO_ROOT"
for g in 1 2 1 2; do
  CYR_NVCC_EXTRA="-DCYR_FUSED_GROUPS=$g" python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
  echo "== groups $g"
  timeout 300 python scripts/fused_probe.py 2097152 2>&1 | tail -1
  timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:actor_tc_fused --csv \
    python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 2>/dev/null | grep '"(148, 1, 1)"' | tail -1 | awk -F'","' '{print "deepest fused ns", $NF}'
done
