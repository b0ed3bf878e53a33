out=gpurun_out/r02n; mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1
for rep in 1 2; do for wl in "--workload resnet101" "--workload inception" ""; do for v in "" "XPIPE_BN_FUSE=1" "XPIPE_BN_FUSE=1 XPIPE_BN_FUSE_MT=4"; do
  env $v timeout 600 python bench.py $wl --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $out/b.log 2>&1
  echo "[$wl] [$v] $(tail -1 $out/b.log | grep -o '"value": [0-9.]*' | head -1) $(tail -1 $out/b.log | grep -o '"gpu_launches": [0-9]*')" >> $out/summary.txt
done; done; done
