#!/bin/bash
# CYR_FUSED_PROF phase split of the fused narrow MLP (printf, clock64)
cd "$GRAFT_REPO_ROOT"
CYR_NVCC_EXTRA="-DCYR_FUSED_PROF ${EXTRA}" python -c "from paper_2506_00167_b200 import _build; _build.build()" 2>&1 | tail -2
timeout 300 python scripts/fused_probe.py 2097152 2>&1 | grep "TRACE\|MMA cta 0\|BUILD cta 0" | head -8
