#!/bin/bash
# experiment: bench K=1/K=4 + conv_bench under env knobs; $1 = label, remaining env passed through
out=gpurun_out/exp; mkdir -p $out
export PYTHONUNBUFFERED=1
lab=$1
python -c "from paper_1911_04610_b200 import build as b; b.build(force=True)" > $out/build_$lab.log 2>&1 || { tail -20 $out/build_$lab.log; exit 1; }
for K in 1 4; do timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e > $out/bench_${lab}_K$K.log 2>&1; echo "$lab K$K rc=$? $(tail -1 $out/bench_${lab}_K$K.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))' 2>&1)"; done
if [ -n "$CONV" ]; then timeout 200 python scripts/conv_bench.py 2>&1 | tail -1; fi
