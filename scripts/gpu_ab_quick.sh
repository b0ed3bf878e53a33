#!/bin/bash
# Quick A/B lines after a gpu_run: bench without timing stamps, and without batched wgrad.
out=gpurun_out/${RUN:-r02}; mkdir -p $out
for v in "notiming|--no-timing" "nowbatch|XPIPE_NO_WGRAD_BATCH=1" "default|"; do
  name=${v%%|*}; arg=${v#*|}
  if [[ "$arg" == XPIPE_* ]]; then env $arg timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-e2e > $out/ab_$name.log 2>&1
  else timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-e2e $arg > $out/ab_$name.log 2>&1; fi
  python - $out/ab_$name.log $name >> $out/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b=d.get("bubble") or {}
    print("AB", sys.argv[2], round(d["value"]), "ms/step", round(d["ms_per_step"],2), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"],3), "bubble", b.get("bubble_fraction"), "steady", b.get("steady_samples_per_s"))
except Exception as e:
    print("AB", sys.argv[2], "failed", e)
PY
done
