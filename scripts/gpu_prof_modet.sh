# Mode-T launch lists and ncu captures of the actor kernels (one GPU).
mkdir -p gpurun_out
P="python scripts/mode_t_probe.py --reps 1"
timeout 300 $P --cfg cfg2 --slots 8 --precision fp32 > gpurun_out/mt_cfg2_fp32.log 2>&1; echo "plain cfg2 fp32 rc=$?"
timeout 300 $P --cfg cfg2 --slots 8 --precision bf16_tc > gpurun_out/mt_cfg2_bf16.log 2>&1; echo "plain cfg2 bf16 rc=$?"
timeout 300 $P --cfg cfg5 --slots 1 --precision bf16_tc > gpurun_out/mt_cfg5_bf16.log 2>&1; echo "plain cfg5 bf16 rc=$?"
cat gpurun_out/mt_*.log
for c in "cfg2 8 fp32" "cfg2 8 bf16_tc" "cfg5 1 bf16_tc"; do
  set -- $c
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_mt_$1_$3.csv $P --cfg $1 --slots $2 --precision $3 > /dev/null 2>&1
  echo "launch list $c rc=$?"
done
# top kernels, one launch each (the deepest level = the last launches)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:actor_tiled_kernel -s 13 -c 1 \
  -o gpurun_out/prof_mt_tiled $P --cfg cfg2 --slots 8 --precision fp32 > gpurun_out/ncu_mt1.log 2>&1; echo "ncu tiled rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_level_kernel -s 13 -c 1 \
  -o gpurun_out/prof_mt_level $P --cfg cfg2 --slots 8 --precision fp32 > gpurun_out/ncu_mt2.log 2>&1; echo "ncu level rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:actor_tc_kernel -s 7 -c 1 \
  -o gpurun_out/prof_mt_tc $P --cfg cfg2 --slots 8 --precision bf16_tc > gpurun_out/ncu_mt3.log 2>&1; echo "ncu tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:actor_tc_wide -s 53 -c 1 \
  -o gpurun_out/prof_mt_wide $P --cfg cfg5 --slots 1 --precision bf16_tc > gpurun_out/ncu_mt4.log 2>&1; echo "ncu wide rc=$?"
