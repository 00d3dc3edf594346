OUT=gpurun_out/${1:-n2}; mkdir -p $OUT
timeout 300 python tools/kernel_bench.py --only ectgemm > $OUT/kb.txt 2>&1; cat $OUT/kb.txt
# 4th shape (gate|up SILU 13824x2048, ECT): skip warm-up/graph launches of the first 7 benches
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 325 -c 1 -o $OUT/gemm_gu_ect python tools/kernel_bench.py --only ectgemm > $OUT/l1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 280 -c 1 -o $OUT/gemm_gu_plain python tools/kernel_bench.py --only ectgemm > $OUT/l2.log 2>&1
for f in gemm_gu_ect gemm_gu_plain; do echo "== $f"; python tools/ncu_kv.py $OUT/$f.ncu-rep; done
