mkdir -p gpurun_out
set -x
timeout 300 python scripts/kernel_probe.py > gpurun_out/probe.json 2> gpurun_out/probe.err; echo "probe rc=$?"
cat gpurun_out/probe.json
timeout 600 python -m pytest tests -q -m gpu -s -k "codebooks_match or logits" > gpurun_out/neartie.log 2>&1; echo "neartie rc=$?"
grep -E "near-tie|logits" gpurun_out/neartie.log | head -60
timeout 300 python scripts/kernel_probe.py --slots 1 1024 --reps 3 > gpurun_out/probe_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_probe.csv python scripts/kernel_probe.py --slots 1 1024 --reps 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_kernel|codebook_kernel|actor_kernel" -s 0 -c 12 -o gpurun_out/prof_r01 python scripts/kernel_probe.py --slots 1 1024 --reps 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
tail -5 gpurun_out/ncu_full.log
