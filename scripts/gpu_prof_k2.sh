# ncu --set full of the bench step's K2 (actor_osplit_kernel / actor_tiled_kernel) with source
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 20 --no-mode-t"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"actor_osplit_kernel|actor_tiled_kernel" -s 4 -c 1 \
  -o gpurun_out/prof_k2 $CMD > gpurun_out/ncu_k2.log 2>&1; echo "ncu k2 rc=$?"
