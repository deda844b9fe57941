# ncu of the FFMA2 layer SGEMM: the 1024x1024 layer of cfg5's deepest Mode-T level (fp32)
mkdir -p gpurun_out
P="python scripts/mode_t_probe.py --reps 1 --cfg cfg5 --slots 1 --precision fp32"
timeout 600 $P > gpurun_out/mt5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgemm_layer_kernel -s 9 -c 1 \
  -o gpurun_out/prof_sgemm_ffma2 $P > gpurun_out/ncu_sg.log 2>&1; echo "ncu sgemm rc=$?"
