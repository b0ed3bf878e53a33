#!/bin/bash
# GEMM iteration: conv tests + per-layer timing, per-CTA phase probes, bench K=1/4, warm ncu launch list
RUN=${RUN:-probe} bash scripts/gpu_conv.sh
timeout 900 python -m pytest tests/test_gpu_bf16.py -q -x --timeout=600 > gpurun_out/${RUN:-probe}/bf16_tests.log 2>&1; echo "bf16 tests rc=$?"; tail -3 gpurun_out/${RUN:-probe}/bf16_tests.log
out=gpurun_out/${RUN:-probe}
for lm in ${PROBES:-1:1 1:3 0:3 8:1 8:3 10:1}; do XPIPE_GEMM_DBG=1 timeout 120 python scripts/gemm_probe.py --layer ${lm%%:*} --mode ${lm##*:} 2>&1 | tail -18; done
for K in 1 4; do timeout 300 python bench.py --steps 10 --warmup 3 --stages $K --no-cpu-baseline > $out/bench_K$K.log 2>&1; echo "K$K rc=$?"; tail -1 $out/bench_K$K.log | cut -c1-200; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 6000 -c 2500 --csv --log-file $out/launches_warm.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graphs > $out/ncu.log 2>&1; echo "ncu rc=$?"
