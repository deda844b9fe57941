# K2 A/B on the bench workload: output-split tiled kernel (default) vs the first tiled mapping, tile sweep
mkdir -p gpurun_out
[ -n "$NO_TESTS" ] || { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; }
k2() { timeout 300 env "$@" python bench.py --steps 10 --warmup 3 --latency-slots 20 --no-mode-t 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels'][0]; print(round(k['ms']*1e3,1), 'us', round(k['frac'],3), 'of FMA peak; value', round(d['value']))"; }
echo "old mapping:      $(k2 CYR_TILED_OSPLIT=0)"
for tc in ${TCS:-32}; do echo "osplit TC=$tc: $(k2 CYR_OSPLIT_TC=$tc)"; done
echo "osplit default:   $(k2 CYR_X=1)"
