mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for G in 1 8 16; do
  CYR_ACTOR_CLUSTER=$G timeout 300 python scripts/kernel_probe.py --slots 1 2 > gpurun_out/probe_G$G.json 2> gpurun_out/probe_G$G.err; echo "probe G=$G rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/probe_G$G.json')); [print('G=$G', s,k,round(v['p50_us'],2)) for s in d for k,v in d[s].items()]"
  tail -2 gpurun_out/probe_G$G.err
done
timeout 300 python scripts/kernel_probe.py --slots 1024 > gpurun_out/probe_1024.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/probe_1024.json')); [print(s,k,round(v['p50_us'],2)) for s in d for k,v in d[s].items()]"
timeout 600 python bench.py --steps 10 --warmup 3 --latency-slots 1000 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], json.dumps(d['latency_us']), d['roofline']['frac'])"
tail -3 gpurun_out/bench.err
