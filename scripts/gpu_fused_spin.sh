#!/bin/bash
# fused MLP: try_wait (default) vs test_wait spin on the critical-path barriers
cd "$GRAFT_REPO_ROOT"
for sp in 0 1 0 1; do
  CYR_NVCC_EXTRA="-DCYR_FUSED_SPIN=$sp" python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
  echo "spin $sp"; timeout 300 python scripts/fused_probe.py 2097152 2>&1 | tail -1
done
