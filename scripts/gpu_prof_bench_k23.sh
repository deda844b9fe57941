# ncu of the bench step's K2 (tiled actor, 4096 columns) and K3 (codebook) kernels.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 20 --no-mode-t"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"actor_tiled_kernel|codebook_kernel" -s 4 -c 2 \
  -o gpurun_out/prof_bench_k23 $CMD > gpurun_out/ncu_k23.log 2>&1; echo "ncu k2k3 rc=$?"
CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 200 > gpurun_out/trace8.log 2>&1
CYR_TRACE=1 CYR_ACTOR_CLUSTER=16 timeout 300 python scripts/latency_probe.py --calls 200 > gpurun_out/trace16.log 2>&1
tail -25 gpurun_out/trace8.log; tail -25 gpurun_out/trace16.log
