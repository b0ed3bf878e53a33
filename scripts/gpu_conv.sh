#!/bin/bash
# quick GEMM iteration: build, GEMM parity tests, per-layer conv timing (TMA on / off)
out=gpurun_out/${RUN:-conv}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout=300 > $out/gemm_tests.log 2>&1; echo "gemm tests rc=$?"; tail -5 $out/gemm_tests.log
timeout 300 python scripts/conv_bench.py --check > $out/conv.log 2>&1; echo "conv rc=$?"; cat $out/conv.log
XPIPE_NO_TMA=1 timeout 300 python scripts/conv_bench.py > $out/conv_notma.log 2>&1; echo "conv notma rc=$?"; tail -1 $out/conv_notma.log
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
