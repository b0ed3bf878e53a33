#!/bin/bash
# One gpurun call of this round: build, GPU tests (parity curves to parity.jsonl), smoke,
# bench line.  usage (under gpurun): RUN=r02x bash scripts/gpu_run.sh [tests|notests] [extra bench args]
out=gpurun_out/${RUN:-r02}; mkdir -p $out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt 2>&1
nproc > $out/nproc.txt; lscpu | grep "Model name" >> $out/nproc.txt
python __graft_entry__.py > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
run() { name=$1; shift; echo "=== $name" >> $out/summary.txt; timeout ${T:-900} "$@" > $out/$name.log 2>&1; echo "rc=$?" >> $out/summary.txt; tail -${TL:-4} $out/$name.log >> $out/summary.txt; }
mode=${1:-tests}; shift
if [ "$mode" = tests ]; then
  XPIPE_PARITY_LOG=$out/parity.jsonl T=2400 TL=30 run tests python -m pytest tests -m gpu -q --timeout=1500 -rf --durations=25 ${PYTEST_K:+-k "$PYTEST_K"}
  T=300 run smoke python -c "import __graft_entry__ as g; g.smoke()"
fi
T=900 TL=1 run bench python bench.py "$@"
echo done >> $out/summary.txt
