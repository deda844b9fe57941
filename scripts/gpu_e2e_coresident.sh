#!/bin/bash
# CodebookStream e2e with the batch K2 at different column tiles (smaller tiles
# = less shared memory: can the next batch's actor co-reside with K1?)
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
for tc in 0 8 16 0 8 16; do
  if [ "$tc" = 0 ]; then unset CYR_OSPLIT_TC; else export CYR_OSPLIT_TC=$tc; fi
  echo "osplit tc=${tc} (0 = auto)"; timeout 300 python scripts/e2e_probe.py
done
unset CYR_OSPLIT_TC
for tc in 8 16; do
  CYR_OSPLIT_TC=$tc timeout 600 python bench.py --steps 10 --warmup 3 --no-mode-t --latency-slots 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tc', $tc, 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), [ (k['kernel'][:3], round(k['ms']*1e3,1)) for k in d['kernels']])"
done
