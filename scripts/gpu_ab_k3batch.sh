#!/bin/bash
# same-box A/B of compile-time variants on the bench step's K2/K3/K1 split and the cfg2 tree
cd "$GRAFT_REPO_ROOT"
for round in 1 2; do
for v in "$@"; do
  CYR_NVCC_EXTRA="$v" python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
  echo "== variant [$v] round $round"
  timeout 600 python bench.py --steps 20 --warmup 5 --no-mode-t --latency-slots 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), [ (k['kernel'][:3], round(k['ms']*1e3,1)) for k in d['kernels']], 'lat p50', d['latency_us']['stochastic']['call_p50'])"
  timeout 300 python scripts/mode_t_probe.py --reps 5 --cfg cfg2 --slots 32 --precision bf16_tc
done
done
