#!/bin/bash
# per-layer evidence: conv GEMM timings (graph-replayed, warm), bench K=1/K=4, warm launch list
out=gpurun_out/${RUN:-layers}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
timeout 300 python scripts/conv_bench.py > $out/conv.log 2>&1; echo "conv rc=$?"; cat $out/conv.log
for K in 1 4; do timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e > $out/bench_K$K.log 2>&1; echo "K$K rc=$?"; tail -1 $out/bench_K$K.log | cut -c1-300; done
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -s 3000 -c 700 --csv --log-file $out/launches_warm_K1.csv \
  python bench.py --steps 1 --warmup 3 --stages 1 --no-cpu-baseline --no-e2e --no-graphs > $out/ncu.log 2>&1; echo "ncu rc=$?"
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
