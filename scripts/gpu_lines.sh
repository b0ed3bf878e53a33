#!/bin/bash
# bench lines of the BASELINE configs and partition variants (one GPU), one LINE per run
out=gpurun_out/${RUN:-lines}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
j() { python - "$1" "$2" >> $out/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b=d.get("bubble") or {}
    r=d.get("roofline") or {}
    print("LINE", sys.argv[2], round(d["value"]), "e2e", d.get("e2e") and round(d["e2e"]["value"]), "launches/step", d.get("gpu_launches",0)//max(1,d["steps"]), "bubble", b.get("bubble_fraction") and round(b["bubble_fraction"],3), "ideal", b.get("ideal_uniform") and round(b["ideal_uniform"],3), "roof", r.get("kernel"), r.get("frac") and round(r["frac"],3), "proof", (d.get("pipeline_roofline") or {}).get("frac"), "split", d["config"].get("stage_first_layer"))
except Exception as e:
    print("LINE", sys.argv[2], "failed", e, open(sys.argv[1]).read()[-600:])
PY
}
b() { name=$1; shift; timeout 900 python bench.py --no-sweep --no-cpu-baseline "$@" > $out/$name.log 2>&1; j $out/$name.log $name; }
DEFAULT_LINES="vgg_K4
vgg_K4_bal --partition balanced
vgg_K2 --stages 2
vgg_K1 --stages 1
vgg_K8 --stages 8
vgg_K8_bal --stages 8 --partition balanced
resnet_K8 --workload resnet101
resnet_K8_bal --workload resnet101 --partition balanced
inception_K4 --workload inception
inception_K8 --workload inception --stages 8
mlp_K2 --workload mlp
vgg_gpipe_K4 --schedule gpipe
resnet_gpipe_K8 --workload resnet101 --schedule gpipe
inception_gpipe_K4 --workload inception --schedule gpipe"
while read -r spec; do
  [ -n "$spec" ] && b $spec
done <<< "${LINES:-$DEFAULT_LINES}"
echo done >> $out/summary.txt
