#!/bin/bash
# CYR_FUSED_PROF trace of the fused MLP on the deepest cfg2 Mode-T level, plus the tree launch list
cd "$GRAFT_REPO_ROOT"
CYR_NVCC_EXTRA="-DCYR_FUSED_PROF" python -c "from paper_2506_00167_b200 import _build; _build.build()" 2>&1 | tail -2
timeout 300 python scripts/mode_t_probe.py --reps 2 --cfg cfg2 --slots 32 --precision bf16_tc 2>&1 | grep "TRACE" | head -4
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
for i in 1 2 3; do timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_modet_cfg2_bf16.csv python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_modet_cfg2_bf16.csv | tail -9
