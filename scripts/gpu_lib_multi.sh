# Same-box comparison of several library builds: every paper_2506_00167_b200/libcyrus_b200_*.so.bak
# (plus the in-tree .so as "tree"), each timed with AB_CMD twice
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_tree.so
for round in 1 2; do
  for f in /tmp/lib_tree.so paper_2506_00167_b200/libcyrus_b200_*.so.bak; do
    cp $f $L
    echo "$(basename $f): $(eval "$AB_CMD" 2>&1 | tail -1)"
  done
done
cp /tmp/lib_tree.so $L
