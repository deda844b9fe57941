# ncu of the bench step's K2 (tiled actor) and K3 (codebook) kernels.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 20 --no-mode-t"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"actor_tiled_kernel|codebook_kernel" -s 4 -c 2 \
  -o gpurun_out/prof_k23b $CMD > gpurun_out/ncu_k23b.log 2>&1; echo "ncu rc=$?"
