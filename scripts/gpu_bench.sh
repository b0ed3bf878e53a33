#!/bin/bash
# quick perf iteration: build, bf16 pipeline parity subset, bench K=1 / K=4, ncu launch list
out=gpurun_out/${RUN:-bench}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_gemm.py -q -x --timeout=300 -k "not config2" > $out/tests.log 2>&1; echo "tests rc=$?"; tail -3 $out/tests.log
timeout 300 python scripts/conv_bench.py > $out/conv.log 2>&1; tail -1 $out/conv.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_K1.log 2>&1; echo "K1 rc=$?"; tail -1 $out/bench_K1.log | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 --stages 4 --no-cpu-baseline > $out/bench_K4.log 2>&1; echo "K4 rc=$?"; tail -1 $out/bench_K4.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graphs > $out/ncu.log 2>&1; echo "ncu rc=$?"
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
