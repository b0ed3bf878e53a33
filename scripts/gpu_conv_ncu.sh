RUN=conv5 bash scripts/gpu_conv.sh
out=gpurun_out/conv5
for L in 8 10; do
timeout 600 ncu --set full --import-source on -k regex:tc_gemm -c 3 -o $out/ncu_L$L python scripts/conv_bench.py --only $L --iters 2 > $out/ncu_L$L.log 2>&1; echo "ncu L$L rc=$?"
done
