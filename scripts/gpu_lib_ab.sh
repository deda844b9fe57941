# A/B of two library builds on one box: the in-tree .so (B) vs libcyrus_b200_head.so.bak (A)
P="python scripts/mode_t_probe.py --reps 3"
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_b.so
for round in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp paper_2506_00167_b200/libcyrus_b200_head.so.bak $L; else cp /tmp/lib_b.so $L; fi
    for c in "cfg2 32 fp32" "cfg5 1 fp32"; do set -- $c; echo "$v: $(timeout 600 $P --cfg $1 --slots $2 --precision $3 2>&1 | tail -1)"; done
  done
done
cp /tmp/lib_b.so $L
