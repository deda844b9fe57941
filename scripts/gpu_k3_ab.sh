#!/bin/bash
# same-box A/B of the deepest-level lane K3 (tree_level_kernel) and the cfg2/cfg5 bf16 trees:
# in-tree .so vs paper_2506_00167_b200/libcyrus_b200_*.so.bak
cd "$GRAFT_REPO_ROOT"
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_tree.so
for r in 1 2; do
for f in /tmp/lib_tree.so paper_2506_00167_b200/libcyrus_b200_*.so.bak; do
  cp $f $L
  t=$(timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tree_level_kernel --csv \
    python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 32 --precision bf16_tc 2>/dev/null \
    | grep tree_level | tail -1 | awk -F'","' '{print $NF}')
  echo "$(basename $f): deepest K3 $t ns; $(timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc | cut -c1-50); $(timeout 300 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc | cut -c1-50)"
done
done
cp /tmp/lib_tree.so $L
