# A/B of two library builds on one box for an arbitrary command: AB_CMD (run twice per build)
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_b.so
for round in 1 2; do for v in A B; do
  if [ $v = A ]; then cp paper_2506_00167_b200/libcyrus_b200_head.so.bak $L; else cp /tmp/lib_b.so $L; fi
  echo "$v: $(eval "$AB_CMD" 2>&1 | tail -1)"
done; done
cp /tmp/lib_b.so $L
