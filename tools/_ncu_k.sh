OUT=gpurun_out/${1:-n1}; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 6 -c 1 -o $OUT/gemv_plain python tools/kernel_bench.py --only gemv > $OUT/l1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 6 -c 1 -o $OUT/gemv_ect python tools/kernel_bench.py --only ect > $OUT/l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o $OUT/gemm_o python tools/kernel_bench.py --only splitk > $OUT/l3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 80 -c 1 -o $OUT/gemm_o_split python tools/kernel_bench.py --only splitk > $OUT/l4.log 2>&1
for f in gemv_plain gemv_ect gemm_o gemm_o_split; do echo "== $f"; python tools/ncu_kv.py $OUT/$f.ncu-rep "Stall Long Scoreboard" "Stall Barrier" "Stall Wait" "Stall Short Scoreboard" "Stall Math Pipe Throttle" "Stall MIO Throttle" "Stall LG Throttle" "Stall Not Selected" "Stall Selected" 2>&1 | head -40; done
