#!/bin/bash
# r02d: linear + residual-fusion tests, ResNet A/B, measured-cost partition, 2-rank dry run
out=gpurun_out/${RUN:-r02d}; mkdir -p $out
export PYTHONUNBUFFERED=1
export XPIPE_PARITY_LOG=$out/parity.jsonl
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fastpaths.py tests/test_gpu_bf16.py tests/test_gpu_benched.py tests/test_gpu_recompute.py tests/test_gpu_mlp.py -q --timeout=900 > $out/tests.log 2>&1
echo "tests rc=$?" >> $out/summary.txt; tail -8 $out/tests.log >> $out/summary.txt
j() { python - "$1" "$2" >> $out/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b=d.get("bubble") or {}
    print("LINE", sys.argv[2], round(d["value"]), "launches/step", d.get("gpu_launches",0)//max(1,d["steps"]), "replays", d.get("graph_replays"), "bubble", b.get("bubble_fraction") and round(b["bubble_fraction"],3), "split", d["config"].get("stage_first_layer"), "cost", d["config"].get("unit_cost"))
except Exception as e:
    print("LINE", sys.argv[2], "failed", e, open(sys.argv[1]).read()[-800:])
PY
}
for v in "" "XPIPE_NO_ADD_FUSE=1" "" "XPIPE_NO_ADD_FUSE=1"; do
  env $v timeout 600 python bench.py --workload resnet101 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1; j $out/b.log "resnet_K8 [$v]"
done
for v in "" "XPIPE_NO_CONCAT_VIEWS=1" "" "XPIPE_NO_CONCAT_VIEWS=1"; do
  env $v timeout 600 python bench.py --workload inception --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1; j $out/b.log "inception_K4 [$v]"
done
timeout 600 python bench.py --stages 8 --partition balanced --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1; j $out/b.log "vgg_K8_balanced"
timeout 600 python bench.py --stages 8 --partition macs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1; j $out/b.log "vgg_K8_macs"
XPIPE_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --no-sweep > $out/mp.log 2>&1
echo "mp rc=$?" >> $out/summary.txt; j $out/mp.log "mp_dry_run_2ranks"
echo done >> $out/summary.txt
