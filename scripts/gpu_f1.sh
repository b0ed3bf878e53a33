#!/bin/bash
# f1 (SURVEY 8f, P:338 / P:394): XPipe vs GPipe-flush through the same kernels on the paper's
# throughput grid -- Inception-V3 and ResNet-101 on Tiny-ImageNet upscaled to 224x224, K in {2, 4},
# T in {1, 2, 4}, mini-batch 50T (K=2) / 100T (K=4).  One GPU: all K stages share the device.
# usage (under gpurun): RUN=r02f bash scripts/gpu_f1.sh
out=gpurun_out/${RUN:-f1}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
for model in ${MODELS:-inception resnet101}; do for K in 2 4; do for T in 1 2 4; do for sch in xpipe gpipe; do
  mb=$([ $K = 2 ] && echo 50 || echo 100)
  name=${model}_K${K}_T${T}_${sch}
  timeout 900 python bench.py --workload $model --stages $K --image 224 --micro-batch $mb --micro-batches $T \
      --minibatches ${MB:-4} --steps 3 --warmup 3 --schedule $sch --no-cpu-baseline --no-e2e --no-sweep \
      > $out/$name.log 2>&1
  echo "$name rc=$?" >> $out/summary.txt
  tail -1 $out/$name.log > $out/$name.json
done; done; done; done
echo done >> $out/summary.txt
