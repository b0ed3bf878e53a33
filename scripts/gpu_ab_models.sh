#!/bin/bash
# A/B of an environment switch $AB on the VGG-16 / ResNet-101 / Inception-V3 bench lines (one GPU)
out=gpurun_out/${RUN:-abm}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout ${TT:-1500} python -m pytest $TESTS -q --timeout=900 > $out/tests.log 2>&1
  echo "tests rc=$?" >> $out/summary.txt; tail -${TL:-6} $out/tests.log >> $out/summary.txt
fi
for rep in $(seq ${REPS:-2}); do for wl in "" "--workload resnet101" "--workload inception"; do for v in "" $AB; do
  env $v timeout 600 python bench.py $wl --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1
  echo "[$wl] [$v] $(tail -1 $out/b.log | grep -o '"value": [0-9.]*' | head -1)" >> $out/summary.txt
done; done; done
echo done >> $out/summary.txt
