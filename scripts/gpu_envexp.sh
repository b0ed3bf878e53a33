#!/bin/bash
# env-knob experiment without rebuilding: bench K=1/K=4 per setting.  usage: bash scripts/gpu_envexp.sh VAR v1 v2 ...
out=gpurun_out/envexp; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
var=$1; shift
for v in "$@"; do for K in ${KS:-1 4}; do
  env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e --no-sweep > $out/${var}_${v}_K$K.log 2>&1
  echo "$var=$v K$K rc=$? $(grep -o '"value": [0-9.]*' $out/${var}_${v}_K$K.log | head -1)"
done; done
