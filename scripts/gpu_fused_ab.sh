#!/bin/bash
# same-box A/B of library builds on the fused kernel's deepest-level launch time
cd "$GRAFT_REPO_ROOT"
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_tree.so
for f in /tmp/lib_tree.so paper_2506_00167_b200/libcyrus_b200_*.so.bak; do
  cp $f $L
  t=$(timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:actor_tc_fused --csv \
    python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 32 --precision bf16_tc 2>/dev/null \
    | grep fused | tail -1 | awk -F'","' '{print $NF}')
  echo "$(basename $f): deepest fused $t ns; $(timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc | cut -c1-60)"
done
cp /tmp/lib_tree.so $L
