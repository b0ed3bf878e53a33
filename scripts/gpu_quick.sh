#!/bin/bash
out=gpurun_out/${RUN:-run}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-600} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-8} $out/$name.log >> $out/summary.txt; }
T=900 TL=6 run tests python -m pytest tests/test_gpu_mlp.py tests/test_gpu_gemm.py tests/test_gpu_sweep.py tests/test_gpu_bf16.py tests/test_multiprocess.py -q --timeout=300 -k "not config2" -x
T=600 TL=3 run bench_K1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
T=600 TL=3 run bench_K4 python bench.py --steps 10 --warmup 3 --stages 4 --no-cpu-baseline
T=600 TL=3 run ncu_launches ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv \
      --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graphs
T=1500 TL=12 run config2 python -m pytest tests/test_gpu_bf16.py -q -s --timeout=1400 -k config2
echo done >> $out/summary.txt
