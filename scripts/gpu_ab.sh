#!/bin/bash
# A/B of a bench flag: bench K=1/2/4 with and without "$1"
out=gpurun_out/ab; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
for K in 1 2 4; do for f in "" "$1"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --stages $K $f --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1
  echo "K$K [$f] rc=$? $(grep -o '"value": [0-9.]*' $out/b.log | head -1)"
done; done
