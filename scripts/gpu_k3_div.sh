#!/bin/bash
# shared-divisor K3: IEEE check, Mode-T parity, timing, launch list
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_numerics.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mode_t or tree or lane" 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc; done
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_modet_cfg2_bf16.csv python scripts/mode_t_probe.py --cfg cfg2 --slots 32 --precision bf16_tc --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_modet_cfg2_bf16.csv | grep "tree_level_kernel\|total"
