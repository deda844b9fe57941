# Round-end evidence: smoke, GPU tests, default bench, reference arm, launch list,
# ncu of K1 (bench step) and of the FFMA2 layer SGEMM (cfg5 Mode-T fp32)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash scripts/gpu_bench_launches.sh
[ -n "$NO_PROF" ] || {
NO_LAUNCH_LIST=1 NO_WP=1 bash scripts/gpu_prof_k1.sh
P="python scripts/mode_t_probe.py --reps 1 --cfg cfg5 --slots 1 --precision fp32"
timeout 600 $P > gpurun_out/mt5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgemm_layer_kernel -s 9 -c 1 \
  -o gpurun_out/prof_sgemm_ffma2 $P > gpurun_out/ncu_sg.log 2>&1; echo "ncu sgemm rc=$?"
}
