#!/bin/bash
# diagnosis call: fast-path tests, ncu launch lists of the C3/C4 bench lines, ncu --set full of the
# BN backward reduction and the batched wgrad in the 4-stage VGG-16 bench (raw CSVs kept)
out=gpurun_out/${RUN:-diag}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-900} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-4} $out/$name.log >> $out/summary.txt; }
[ -n "$TESTS" ] && T=1500 TL=6 run tests python -m pytest $TESTS -q --timeout=900
for wl in resnet101 inception; do
  T=900 TL=2 run ncu_launches_$wl ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 6000 --csv \
      --log-file $out/launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --minibatches 4 --no-cpu-baseline --no-e2e --no-sweep
  python scripts/ncu_summary.py launches $out/launches_$wl.csv $out/launches_$wl.md >> $out/summary.txt 2>&1
  rm -f $out/launches_$wl.csv
done
for k in bn_bwd_reduce_kernel bn_apply_kernel bn_bwd_apply_kernel; do
  T=600 TL=2 run ncu_$k ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 8 \
      -o $out/prof_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-graphs
done
T=600 TL=2 run ncu_wgrad ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)3" -s 40 -c 8 \
    -o $out/prof_wgrad python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-graphs
for k in bn_bwd_reduce_kernel bn_apply_kernel bn_bwd_apply_kernel wgrad; do
  [ -f $out/prof_$k.ncu-rep ] && python scripts/ncu_summary.py full $out/prof_$k.ncu-rep $out/${k}_full.md >> $out/summary.txt 2>&1
  ncu -i $out/prof_$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  ncu -i $out/prof_$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
  rm -f $out/prof_$k.ncu-rep
done
echo done >> $out/summary.txt
