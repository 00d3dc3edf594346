#!/bin/bash
# ncu evidence for one round: launch list (durations, one planned inference)
# and full captures of the dominant kernels.  Run under gpurun.
set -x
OUT=${1:-gpurun_out/ncu}
mkdir -p $OUT
KRE='regex:gemv_kernel|gemm_kernel|flash_kernel|decode_attn|rmsnorm|layernorm|qk_norm|embed_rows|add_rows|argmax_to|time_embed|action_|silu_kernel|fill_u64'
# launches of the second (profiled) inference: skip the warm-up inference
N=$(python tools/profile_step.py --runs 1 2>/dev/null | sed -n 's/.*kernel_launches.: \([0-9]*\).*/\1/p' | head -1)
echo "launches per inference: $N"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -s $N -c $N --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py --runs 2 > $OUT/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:gemv_kernel<.int.2>' -s 40 -c 2 -o $OUT/gemv_silu python tools/profile_step.py --runs 1 > $OUT/full_gemv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:gemm_kernel<.int.128, .int.0>' -s 4 -c 2 -o $OUT/gemm_qkv python tools/profile_step.py --runs 1 > $OUT/full_gemm.log 2>&1
ls -la $OUT
