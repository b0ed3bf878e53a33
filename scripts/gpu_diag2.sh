#!/bin/bash
# after-fix evidence: ncu --set full of the BN-backward reduction and the BN final merges in the
# 4-stage VGG-16 bench (raw CSVs kept; summaries with the warp stall reasons)
out=gpurun_out/${RUN:-diag2}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
for k in bn_bwd_reduce_kernel bn_stats_final_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 8 \
      -o $out/prof_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-graphs > $out/ncu_$k.log 2>&1
  ncu -i $out/prof_$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  rm -f $out/prof_$k.ncu-rep
done
echo done > $out/summary.txt
