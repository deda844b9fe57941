mkdir -p gpurun_out
timeout 300 python scripts/kernel_probe.py --slots 1 --reps 3 > gpurun_out/p2_plain.log 2>&1 && \
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"codebook_kernel|tree_kernel|actor_kernel" -s 12 -c 6 -o gpurun_out/prof_s1 python scripts/kernel_probe.py --slots 1 --reps 3 > gpurun_out/ncu_s1.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_s1.log
