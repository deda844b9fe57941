#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (scripts/sanitize_probe.py); the resident slot server and the per-call
# graph path are both covered.  Summaries -> gpurun_out/sanitize_*.txt
cd "$GRAFT_REPO_ROOT"
CS=/usr/local/cuda/bin/compute-sanitizer
export CYR_SLOT_SERVER_IDLE_MS=2000   # instrumented kernels run ~100x slower
python scripts/sanitize_probe.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 python scripts/sanitize_probe.py \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
CYR_SLOT_SERVER=0 timeout 900 $CS --tool racecheck --print-limit 50 python scripts/sanitize_probe.py server \
  > gpurun_out/sanitize_racecheck_graphpath.txt 2>&1
echo "racecheck graph path rc=$?"; tail -3 gpurun_out/sanitize_racecheck_graphpath.txt
