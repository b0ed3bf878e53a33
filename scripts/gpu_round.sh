#!/bin/bash
# One evidence call: full GPU test suite, smoke, default bench line, per-layer conv timing,
# serialised ncu launch list of the bench, ncu --set full of the wgrad GEMM (dominant class)
# and of the sweep.  usage (under gpurun): RUN=r01x bash scripts/gpu_round.sh [notests]
out=gpurun_out/${RUN:-round}; mkdir -p $out
export PYTHONUNBUFFERED=1
export XPIPE_PARITY_LOG=$out/parity.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt 2>&1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-900} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-4} $out/$name.log >> $out/summary.txt; }
if [ "$1" != notests ]; then
  T=1800 TL=6 run tests python -m pytest tests -m gpu -q --timeout=900
  T=300 run smoke python -c "import __graft_entry__ as g; g.smoke()"
fi
T=600 TL=1 run bench python bench.py
T=300 TL=16 run conv python scripts/conv_bench.py
T=600 TL=2 run ncu_launches ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep
T=600 TL=2 run ncu_wgrad ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)3" -s 300 -c 6 \
    -o $out/prof_wgrad python bench.py --steps 1 --warmup 3 --stages 1 --no-cpu-baseline --no-e2e --no-sweep --no-graphs
T=600 TL=2 run ncu_fprop ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)1" -s 300 -c 6 \
    -o $out/prof_fprop python bench.py --steps 1 --warmup 3 --stages 1 --no-cpu-baseline --no-e2e --no-sweep --no-graphs
T=300 TL=2 run ncu_sweep ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
    -o $out/prof_sweep python bench.py --workload sweep --steps 1 --warmup 3
# summaries on the box (the .ncu-rep files stay there: gpurun copies back <= 64 MiB)
python scripts/ncu_summary.py launches $out/launches.csv $out/launches.md >> $out/summary.txt 2>&1
for k in wgrad fprop sweep; do
  [ -f $out/prof_$k.ncu-rep ] && python scripts/ncu_summary.py full $out/prof_$k.ncu-rep $out/${k}_full.md >> $out/summary.txt 2>&1
  ncu -i $out/prof_$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  rm -f $out/prof_$k.ncu-rep
done
echo done >> $out/summary.txt
