mkdir -p gpurun_out
export CYR_SLOT_SERVER=0  # profile the launched fused kernel (same body as the resident server)
timeout 300 python scripts/latency_probe.py --calls 12 > gpurun_out/lat_plain.log 2>&1 && \
timeout 600 ncu --set full --warp-sampling-interval 0 --cache-control none --clock-control none --import-source on -k regex:"actor_cluster" -s 10 -c 1 -o gpurun_out/prof_fused python scripts/latency_probe.py --calls 12 > gpurun_out/ncu_f.log 2>&1; echo "ncu rc=$?"
