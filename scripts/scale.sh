#!/bin/bash
# SURVEY 8d/8e scaling run on one 8xB200 node: VGG-16 (BASELINE configs[1] shapes) with K = 1, 2,
# 4, 8 pipeline stages, one stage per GPU (one process per GPU, torchrun), with the layer-count
# and the measured cost-balanced partitions; one JSON line per run in $OUT/scale.jsonl.
# usage: bash scripts/scale.sh [steps] [warmup]      (needs 8 GPUs; OUT defaults to gpurun_out/scale)
OUT=${OUT:-gpurun_out/scale}; mkdir -p $OUT
STEPS=${1:-10}; WARM=${2:-3}
export PYTHONUNBUFFERED=1
for part in layer-count balanced; do for K in 1 2 4 8; do
  if [ $K = 1 ]; then
    [ $part = balanced ] && continue
    timeout 900 python bench.py --gpus 1 --stages 1 --steps $STEPS --warmup $WARM --no-cpu-baseline > $OUT/K1.log 2>&1
    tail -1 $OUT/K1.log >> $OUT/scale.jsonl
  else
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 \
      --master-port $((29600 + K)) bench.py --gpus $K --partition $part --steps $STEPS --warmup $WARM \
      --no-cpu-baseline > $OUT/K${K}_$part.log 2>&1
    tail -1 $OUT/K${K}_$part.log >> $OUT/scale.jsonl
  fi
  echo "K=$K $part rc=$? $(tail -1 $OUT/scale.jsonl | grep -o '"value": [0-9.]*' | head -1)"
done; done
