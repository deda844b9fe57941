# Mode-T cfg2 launch lists (fp32, bf16) of one 32-slot tree batch (the bench's Mode-T batch)
mkdir -p gpurun_out
P="python scripts/mode_t_probe.py --reps 1"
for pr in fp32 bf16_tc; do
  timeout 300 $P --cfg cfg2 --slots 32 --precision $pr > gpurun_out/mt_cfg2_$pr.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_mt32_cfg2_$pr.csv $P --cfg cfg2 --slots 32 --precision $pr > /dev/null 2>&1
  echo "cfg2 $pr rc=$?"; cat gpurun_out/mt_cfg2_$pr.log
done
