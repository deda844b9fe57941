#!/bin/bash
# cfg5 bf16 Mode-T tree: per-launch times (ncu, clocks unlocked, serialised)
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_modet_cfg5_bf16.csv python scripts/mode_t_probe.py --cfg cfg5 --slots 1 --precision bf16_tc --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_modet_cfg5_bf16.csv | tail -40
