#!/bin/bash
# A/B of two prebuilt libraries (libxpipe_old.so vs libxpipe_new.so), alternating runs
out=gpurun_out/${RUN:-abso}; mkdir -p $out
export PYTHONUNBUFFERED=1
P=paper_1911_04610_b200
for v in old new; do
  cp $P/libxpipe_$v.so $P/libxpipe.so
  timeout 300 python scripts/params_dump.py /tmp/params_$v.npy > $out/dump_$v.log 2>&1
done
python -c "import numpy as np, sys; a, b = (np.load(sys.argv[i]) for i in (1, 2)); print('params bit-identical:', a.shape == b.shape and bool(np.array_equal(a, b)))" /tmp/params_old.npy /tmp/params_new.npy | tee -a $out/summary.txt
for rep in 1 2 3; do for v in old new; do for K in ${KS:-4 1}; do
  cp $P/libxpipe_$v.so $P/libxpipe.so
  timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1
  echo "rep$rep $v K$K rc=$? $(grep -o '"value": [0-9.]*' $out/b.log | head -1)" | tee -a $out/summary.txt
done; done; done
cp $P/libxpipe_new.so $P/libxpipe.so
