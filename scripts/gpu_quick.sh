#!/bin/bash
# Quick GPU iteration: parity tests, smoke, bench variants, launch list.
out=gpurun_out; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-600} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-8} $out/$name.log >> $out/summary.txt; }
T=200 TL=12 run repro_fp32_K2T2 python scripts/repro_hang.py 2 2 8 2 fp32
T=900 TL=25 run tests python -m pytest tests/test_gpu_mlp.py tests/test_gpu_gemm.py tests/test_gpu_sweep.py tests/test_gpu_bf16.py tests/test_multiprocess.py -v --timeout=300 -k "not config2" -x
T=300 TL=5 run smoke python -c "import __graft_entry__ as g; g.smoke()"
T=600 run bench_K1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
T=600 run bench_K4 python bench.py --steps 10 --warmup 3 --stages 4 --no-cpu-baseline
T=600 run bench_K1_nographs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graphs
T=600 TL=3 run ncu_launches ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv \
      --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graphs
echo done >> $out/summary.txt
