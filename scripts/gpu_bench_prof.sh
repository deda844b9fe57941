mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 50"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench(default) rc=$?"
cat gpurun_out/bench_full.json
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 2 -c 1 -o gpurun_out/prof_tree $CMD > gpurun_out/ncu_tree.log 2>&1; echo "ncu tree rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"actor_kernel|codebook_kernel" -s 2 -c 2 -o gpurun_out/prof_k23 $CMD > gpurun_out/ncu_k23.log 2>&1; echo "ncu k2k3 rc=$?"
