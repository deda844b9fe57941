CYR_TRACE=1 timeout 300 python scripts/latency_probe.py --calls 200
CYR_TRACE=1 CYR_ACTOR_CLUSTER=16 timeout 300 python scripts/latency_probe.py --calls 200
