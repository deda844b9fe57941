#!/bin/bash
# ncu --set full of the bench step's batch K3 (codebook_kernel, warp per row)
cd "$GRAFT_REPO_ROOT"
python -c "from paper_2506_00167_b200 import _build; _build.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codebook_kernel -s 6 -c 1 \
  -o gpurun_out/prof_k3batch python bench.py --steps 3 --warmup 3 --latency-slots 20 --no-mode-t > gpurun_out/ncu_k3batch.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_k3batch.ncu-rep --page details > gpurun_out/k3batch_details.txt 2>&1
grep -E "Duration|Issue Slots|Registers|Achieved Occupancy|Warp Cycles Per Issued" gpurun_out/k3batch_details.txt | head
ncu -i gpurun_out/prof_k3batch.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
out=sorted([(float(x),k) for k,x in zip(h,v) if 'smsp__average_warps_issue_stalled_' in k and k.endswith('_per_issue_active.ratio') and x], reverse=True)[:8]
for x,k in out: print(round(x,3), k)"
