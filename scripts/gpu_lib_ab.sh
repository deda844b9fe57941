# A/B of two library builds on one box: the in-tree .so (B) vs libcyrus_b200_head.so.bak (A).
# AB_WHAT=modet (default) | k3 : what to time.
L=paper_2506_00167_b200/libcyrus_b200.so
cp $L /tmp/lib_b.so
run() {
  case "${AB_WHAT:-modet}" in
    modet)
      for c in "cfg2 32 fp32" "cfg5 1 fp32"; do set -- $c
        echo "$v: $(timeout 600 python scripts/mode_t_probe.py --reps 3 --cfg $1 --slots $2 --precision $3 2>&1 | tail -1)"; done ;;
    k3)
      echo "$v latency: $(timeout 300 python scripts/latency_probe.py --calls 3000 2>&1 | tail -1)"
      echo "$v bench K3: $(timeout 300 python bench.py --steps 10 --warmup 3 --latency-slots 20 --no-mode-t 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernels'][1]['ms']*1e3,1), 'us; value', round(d['value']))")"
      echo "$v: $(timeout 600 python scripts/mode_t_probe.py --reps 3 --cfg cfg2 --slots 32 --precision bf16_tc 2>&1 | tail -1)" ;;
  esac
}
for round in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp paper_2506_00167_b200/libcyrus_b200_head.so.bak $L; else cp /tmp/lib_b.so $L; fi
    run
  done
done
cp /tmp/lib_b.so $L
