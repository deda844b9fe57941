#!/bin/bash
# Round-2 evidence: smoke, GPU tests, both bench arms (default commands), the
# launch list of a short bench, ncu --set full of K1 (bench step) and of the
# fused tcgen05 MLP (deepest cfg2 Mode-T level).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_full.err
CMD="python bench.py --steps 3 --warmup 3 --latency-slots 50 --no-mode-t"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch list rc=$?"
[ -n "$NO_PROF" ] || {
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 5 -c 1 \
  -o gpurun_out/prof_k1 python bench.py --steps 3 --warmup 3 --latency-slots 50 --no-mode-t > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
bash scripts/gpu_prof_fused.sh
}
