#!/bin/bash
# ncu --set full captures of the kernels VERDICT r1 names (one launch each,
# eager, after 3 warm-up launches) + CUDA-graph timings of the same shapes.
OUT=${1:-gpurun_out/prof}
mkdir -p $OUT
cap() {  # name only-mode kernel-regex
  KB_EAGER=5 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$3" -s 3 -c 1 \
     -o $OUT/$1 python tools/kernel_bench.py --only $2 > $OUT/$1.log 2>&1
  python tools/ncu_kv.py $OUT/$1.ncu-rep "Duration" "DRAM Throughput" > $OUT/$1_summary.txt 2>&1
  ncu -i $OUT/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed > $OUT/$1_raw.csv 2>&1
}
for m in ${MODES:-attn16 flash4 ectgemm_gu ectgemm_qkv prefill_gemm}; do
  timeout 300 python tools/kernel_bench.py --only $m > $OUT/time_$m.jsonl 2>&1
done
cap attn16 attn16 decode_attn
cap flash4 flash4 flash_kernel
cap ectgemm_gu ectgemm_gu gemm_kernel
cap ectgemm_qkv ectgemm_qkv gemm_kernel
cap prefill_gu prefill_gemm gemm_kernel
ls -la $OUT
