#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_guards.py -x -q -s > gpurun_out/guards.log 2>&1
echo "guards rc=$?"; tail -5 gpurun_out/guards.log
bash scripts/gpu_modet_lists.sh
python scripts/launch_table.py gpurun_out/launches_mt32_cfg2_bf16_tc.csv > gpurun_out/lt_bf16.txt 2>&1
tail -40 gpurun_out/lt_bf16.txt
