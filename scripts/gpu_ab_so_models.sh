#!/bin/bash
# A/B of two prebuilt libraries (paper_1911_04610_b200/libxpipe_{old,new}.so) on the VGG-16 /
# ResNet-101 / Inception-V3 bench lines, alternating runs; optional test suite on the new one first
out=gpurun_out/${RUN:-abso}; mkdir -p $out
export PYTHONUNBUFFERED=1
P=paper_1911_04610_b200
cp $P/libxpipe_new.so $P/libxpipe.so
if [ -n "$TESTS" ]; then
  timeout ${TT:-1500} python -m pytest $TESTS -q --timeout=900 > $out/tests.log 2>&1
  echo "tests rc=$?" >> $out/summary.txt; tail -${TL:-6} $out/tests.log >> $out/summary.txt
fi
for rep in $(seq ${REPS:-2}); do for wl in ${WLS:-vgg16 resnet101 inception}; do for v in old new; do
  cp $P/libxpipe_$v.so $P/libxpipe.so
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b_$v.log 2>&1
  echo "rep$rep $wl $v rc=$? $(grep -o '"value": [0-9.]*' $out/b_$v.log | head -1)" >> $out/summary.txt
done; done; done
cp $P/libxpipe_new.so $P/libxpipe.so
echo done >> $out/summary.txt
