#!/bin/bash
# CYR_FUSED_PROF traces: 2M Mode-R columns and the deepest cfg2 Mode-T level
cd "$GRAFT_REPO_ROOT"
CYR_NVCC_EXTRA="-DCYR_FUSED_PROF ${EXTRA}" python -c "from paper_2506_00167_b200 import _build; _build.build()" 2>&1 | tail -2
echo "== Mode R"; timeout 300 python scripts/fused_probe.py 524288 2>&1 | grep "TRACE" | head -2
echo "== Mode T"; timeout 300 python scripts/mode_t_probe.py --reps 2 --cfg cfg2 --slots 32 --precision bf16_tc 2>&1 | grep TRACE | head -2
