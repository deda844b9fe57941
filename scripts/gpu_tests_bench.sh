#!/bin/bash
# full GPU test suite, then both bench arms (1 GPU)
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
echo "tests rc=$?"
tail -5 gpurun_out/gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.err
