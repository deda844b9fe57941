# K1 work-item size / CTAs-per-SM sweep on the bench workload (K1 time from the bench's events).
for np in ${NPS:-128}; do for ps in ${PSS:-3 4 5 6 8}; do
  r=$(CYR_TREE_NP=$np CYR_TREE_PER_SM=$ps timeout 300 python bench.py --steps 10 --warmup 3 --latency-slots 20 --no-mode-t 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels'][-1]; print(round(k['ms']*1e3,1), round(k['achieved']), round(d['value']))")
  echo "NP=$np per_sm<=$ps: K1 us / GB/s / value: $r"
done; done
