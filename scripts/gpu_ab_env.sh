#!/bin/bash
# A/B of an environment switch "$1" (e.g. XPIPE_NO_BNB_FUSE=1) on the same library, alternating runs
out=gpurun_out/${RUN:-abenv}; mkdir -p $out
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do for v in "" "$1"; do for K in ${KS:-4 1}; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1
  echo "rep$rep [$v] K$K rc=$? $(grep -o '"value": [0-9.]*' $out/b.log | head -1)" | tee -a $out/summary.txt
done; done; done
