# ncu --set full of K1 (tree_kernel) on the bench workload, plus the launch list.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 20 --no-mode-t"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 2 -c 1 \
  -o gpurun_out/prof_tree2 $CMD > gpurun_out/ncu_tree2.log 2>&1; echo "ncu tree rc=$?"
[ -n "$NO_LAUNCH_LIST" ] || { timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch list rc=$?"; }
[ -n "$NO_WP" ] || { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro/wp scripts/micro/write_patterns.cu && ./scripts/micro/wp > gpurun_out/write_patterns.txt 2>&1; echo "write patterns rc=$?"; }
