#!/bin/bash
# One gpurun call: parity tests, bench lines, ncu launch list + full captures.
# usage (under gpurun): bash scripts/gpu_check.sh [quick|full]
set -u
mode=${1:-full}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt 2>&1
python __graft_entry__.py > $out/build.log 2>&1
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-900} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -5 $out/$name.log >> $out/summary.txt; }
T=300 run mlp python -m pytest tests/test_gpu_mlp.py -q -k "stage_counts"
T=600 run mlp_all python -m pytest tests/test_gpu_mlp.py -q
T=300 run gemm python -m pytest tests/test_gpu_gemm.py -q
T=300 run sweep python -m pytest tests/test_gpu_sweep.py -q
T=600 run bf16 python -m pytest tests/test_gpu_bf16.py -q -k "not config2" -s
T=300 run smoke python -c "import __graft_entry__ as g; g.smoke()"
T=600 run bench python bench.py --steps 10 --warmup 3
T=300 run bench_sweep python bench.py --workload sweep --steps 20 --warmup 3
if [ "$mode" = full ]; then
  T=900 run config2 python -m pytest tests/test_gpu_bf16.py -q -k "config2" -s
  T=600 run ncu_launches ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv \
      --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e
  T=600 run ncu_conv ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 40 -c 3 \
      -o $out/prof_conv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
  T=300 run ncu_sweep ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
      -o $out/prof_sweep python bench.py --workload sweep --steps 1 --warmup 3
fi
echo done >> $out/summary.txt
