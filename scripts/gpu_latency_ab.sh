# Latency path A/B: persistent slot server (default) vs per-call graph launch, cluster sizes
mkdir -p gpurun_out
[ -n "$NO_TESTS" ] || { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log; }
for v in 0 1; do
  echo "CYR_SLOT_SERVER=$v: $(CYR_SLOT_SERVER=$v timeout 300 python scripts/latency_probe.py --calls 3000 2>&1 | tail -1)"
done
for g in ${CLUSTERS:-4 16}; do
  echo "server, cluster $g: $(CYR_ACTOR_CLUSTER=$g timeout 300 python scripts/latency_probe.py --calls 3000 2>&1 | tail -1)"
done
CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 300 2>&1 | tail -22
