#!/bin/bash
# Development call: build, the GPU tests named in $TESTS (pytest node ids / files), then an A/B of
# the environment switch(es) in $AB against the default, alternating, $REPS times, over the
# stage counts in $KS (VGG-16 bench lines, no CPU baseline / sweep / e2e).
# usage (under gpurun): RUN=r02b TESTS="tests/test_x.py" AB="XPIPE_BN_FUSED=0" bash scripts/gpu_dev.sh
out=gpurun_out/${RUN:-dev}; mkdir -p $out
export PYTHONUNBUFFERED=1
export XPIPE_PARITY_LOG=$out/parity.jsonl
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout ${TT:-1500} python -m pytest $TESTS -q --timeout=900 > $out/tests.log 2>&1
  echo "tests rc=$?" >> $out/summary.txt; tail -${TL:-8} $out/tests.log >> $out/summary.txt
fi
for rep in $(seq ${REPS:-2}); do for v in "" $AB; do for K in ${KS:-4 1}; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline --no-e2e --no-sweep $BENCH_ARGS > $out/b.log 2>&1
  python - $out/b.log "rep$rep [$v] K$K" >> $out/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b=d.get("bubble") or {}
    ks={k:round(v["ms_per_step"],2) for k,v in (d.get("kernel_shares") or {}).items()}
    print("AB", sys.argv[2], round(d["value"]), "launches/step", d.get("gpu_launches",0)//max(1,d["steps"]), "prof_ms", round(d.get("profiled_step_ms") or 0,1), "bubble", b.get("bubble_fraction") and round(b["bubble_fraction"],3), ks)
except Exception as e:
    print("AB", sys.argv[2], "failed", e, open(sys.argv[1]).read()[-500:])
PY
done; done; done
echo done >> $out/summary.txt
