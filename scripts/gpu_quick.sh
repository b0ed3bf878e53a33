#!/bin/bash
# Quick GPU iteration: hang repro, graph tests, bench variants.
out=gpurun_out; mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-600} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-8} $out/$name.log >> $out/summary.txt; }
export PYTHONUNBUFFERED=1
T=120 TL=60 XPIPE_VERBOSE=1 run repro_fp32_K2T2 python scripts/repro_hang.py 2 2 8 2 fp32
T=120 TL=30 run repro_fp32_K2T2_cudamalloc env TORCH_ALLOC=0 python scripts/repro_hang.py 2 2 8 2 fp32
T=120 TL=10 run repro_fp32_K2T1 python scripts/repro_hang.py 2 1 8 2 fp32
T=120 TL=10 run repro_bf16_K2T2 python scripts/repro_hang.py 2 2 8 2 bf16
T=300 TL=20 run graphs python -m pytest tests/test_gpu_mlp.py -v -x --timeout=120 -k "graph or stage_counts"
T=600 TL=40 run multiproc python -m pytest tests/test_multiprocess.py -v -x --timeout=300
T=600 run bench_K1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
T=600 run bench_K4 python bench.py --steps 10 --warmup 3 --stages 4 --no-cpu-baseline
T=600 run bench_K1_nographs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graphs
echo done >> $out/summary.txt
