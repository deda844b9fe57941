#!/bin/bash
# batched (4 K steps per asm, one elect) MMA issue: correctness + fused MLP timing + PROF phase split
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
timeout 300 python scripts/fused_probe.py
for i in 1 2; do timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc; done
CYR_NVCC_EXTRA="-DCYR_FUSED_PROF" python -c "from paper_2506_00167_b200 import _build; _build.build()" 2>&1 | tail -2
timeout 300 python scripts/fused_probe.py 2097152 2>&1 | grep "cta 0 \|fused=" | sort | uniq -c | sort -rn | head -8
