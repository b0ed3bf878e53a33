#!/bin/bash
# bench lines of the other BASELINE configs and the GPipe-flush comparison (f1)
out=gpurun_out/${RUN:-wl}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
b() { name=$1; shift; timeout 900 python bench.py --no-e2e --no-sweep "$@" > $out/$name.log 2>&1; echo "$name rc=$? $(grep -o '"value": [0-9.]*' $out/$name.log | head -1) $(grep -o '"bubble_fraction": [0-9.]*, "ideal_uniform": [0-9.]*' $out/$name.log)"; }
b vgg_xpipe_K4 --no-cpu-baseline
b vgg_gpipe_K4 --no-cpu-baseline --schedule gpipe
b vgg_xpipe_K2 --no-cpu-baseline --stages 2
b vgg_gpipe_K2 --no-cpu-baseline --stages 2 --schedule gpipe
b vgg_xpipe_K1 --no-cpu-baseline --stages 1
b resnet_K8 --workload resnet101
b resnet_gpipe_K8 --workload resnet101 --no-cpu-baseline --schedule gpipe
b inception_K4 --workload inception
b inception_gpipe_K4 --workload inception --no-cpu-baseline --schedule gpipe
b inception_K8 --workload inception --no-cpu-baseline --stages 8
b mlp_K2 --workload mlp
b vgg_sgd_K4 --no-cpu-baseline --optimizer sgd
b vgg_recompute_K4 --no-cpu-baseline --recompute
b resnet224_K2_T2 --workload resnet101 --no-cpu-baseline --stages 2 --image 224 --micro-batch 50 --micro-batches 2 --minibatches 2 --steps 5
b resnet224_gpipe_K2_T2 --workload resnet101 --no-cpu-baseline --stages 2 --image 224 --micro-batch 50 --micro-batches 2 --minibatches 2 --steps 5 --schedule gpipe
b inception224_K4_T4 --workload inception --no-cpu-baseline --stages 4 --image 224 --micro-batch 100 --micro-batches 4 --minibatches 2 --steps 5
b inception224_gpipe_K4_T4 --workload inception --no-cpu-baseline --stages 4 --image 224 --micro-batch 100 --micro-batches 4 --minibatches 2 --steps 5 --schedule gpipe
