#!/bin/bash
# per-layer conv GEMM timings under development knobs (what bounds the main loop)
out=gpurun_out/${RUN:-probe}; mkdir -p $out
export PYTHONUNBUFFERED=1
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
for v in "" "XPIPE_BN_FILL=8" "XPIPE_PERSIST_STAGES=6" "XPIPE_PERSIST_STAGES=2" "XPIPE_NO_KPAIR=1" "XPIPE_NO_TMA_A=1" "XPIPE_PERSIST_MULT=2" "XPIPE_NO_SPLITK=1"; do
  echo "=== [$v]" >> $out/summary.txt
  env $v timeout 300 python scripts/conv_bench.py --modes ${MODES:-12} > $out/p.log 2>&1
  cat $out/p.log >> $out/summary.txt
done
echo done >> $out/summary.txt
