#!/bin/bash
# A/B/C... of (library, environment) variants on the bench lines, alternating runs.
# VARIANTS="name=lib[,ENV=V...][,--bench-arg...] ..." (lib: old|new -> paper_1911_04610_b200/libxpipe_<lib>.so)
out=gpurun_out/${RUN:-abv}; mkdir -p $out
export PYTHONUNBUFFERED=1
P=paper_1911_04610_b200
cp $P/libxpipe_new.so $P/libxpipe.so
if [ -n "$TESTS" ]; then
  timeout ${TT:-1500} python -m pytest $TESTS -q --timeout=900 > $out/tests.log 2>&1
  echo "tests rc=$?" >> $out/summary.txt; tail -${TL:-6} $out/tests.log >> $out/summary.txt
fi
for rep in $(seq ${REPS:-2}); do for wl in ${WLS:-vgg16 resnet101 inception}; do for var in $VARIANTS; do
  name=${var%%=*}; rest=${var#*=}; lib=${rest%%,*}; envs=""; args=""
  if [ "$rest" != "$lib" ]; then for t in $(echo ${rest#*,} | tr ',' ' '); do
    case $t in --*) args="$args $t";; *) envs="$envs $t";; esac; done; fi
  cp $P/libxpipe_$lib.so $P/libxpipe.so
  env $envs timeout 600 python bench.py --workload $wl --steps ${STEPS:-8} --warmup 3 ${BASE_ARGS:---no-cpu-baseline --no-e2e --no-sweep} $BARGS $args > $out/b_$name.log 2>&1
  echo "rep$rep $wl $name rc=$? $(tail -1 $out/b_$name.log | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); e=d.get("e2e") or {}; print("value", round(d["value"]), "e2e", e.get("value") and round(e["value"]))
except Exception as ex: print("failed", ex)')" >> $out/summary.txt
done; done; done
cp $P/libxpipe_new.so $P/libxpipe.so
echo done >> $out/summary.txt
