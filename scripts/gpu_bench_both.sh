#!/bin/bash
# both bench arms as the driver runs them (reference first), 1 GPU
cd "$GRAFT_REPO_ROOT"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err
echo "ref rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 600 gpurun_out/bench.err
