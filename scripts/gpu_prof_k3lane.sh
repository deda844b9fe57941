# ncu (source-level) of the lane-mapped K3 on the deepest cfg2 Mode-T level (32-slot bf16 tree)
mkdir -p gpurun_out
P="python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 32 --precision bf16_tc"
timeout 300 $P > gpurun_out/mt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_level_kernel -s 3 -c 1 \
  -o gpurun_out/prof_k3lane $P > gpurun_out/ncu_k3lane.log 2>&1; echo "ncu rc=$?"
