#!/bin/bash
# one ncu --set full capture of the fused narrow MLP (2M Mode-R columns), with source counters
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:actor_tc_fused -s 3 -c 1 \
  -o gpurun_out/fused_full -f python scripts/fused_probe.py 524288 > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_fused.log
