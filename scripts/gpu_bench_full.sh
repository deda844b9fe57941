# Round bench + profiles: plain bench, launch list of a short bench, ncu of
# the Mode-T kernels (each only after its command exited 0 without ncu).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 50 --no-mode-t"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch list rc=$?"
P="python scripts/mode_t_probe.py --reps 1 --cfg cfg2 --slots 8 --precision fp32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgemm_layer -s 9 -c 1 \
  -o gpurun_out/prof_sgemm_cfg2 $P > gpurun_out/ncu_sg2.log 2>&1; echo "ncu sgemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_level_kernel -s 5 -c 1 \
  -o gpurun_out/prof_level_deep $P > gpurun_out/ncu_lv.log 2>&1; echo "ncu level rc=$?"
