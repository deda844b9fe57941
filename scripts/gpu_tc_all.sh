#!/bin/bash
# all tcgen05 actor paths: agreement tests, then Mode-T tree timing (fused, layer, wide)
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc; done
CYR_TC_FUSED=0 timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 3 --cfg cfg5 --slots 1 --precision bf16_tc; done
timeout 300 python scripts/fused_probe.py
