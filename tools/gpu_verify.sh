#!/bin/bash
# Round verification on one B200: GPU tests, smoke, both bench arms, ncu launch
# list of one planned inference + a full capture of the dominant decode GEMV.
OUT=${1:-gpurun_out/verify}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 1200 python bench.py --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 400 $OUT/bench.err; cat $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cat $OUT/bench_ref.json
PROF=$OUT/profile_alpamayo-r1-10b-shape.json
if [ -f "$PROF" ] && [ -z "$SKIP_NCU" ]; then
  KRE='regex:gemv_kernel|gemv_ect_kernel|gemm_kernel|flash_kernel|decode_attn|rmsnorm|layernorm|qk_norm|embed_rows|add_rows|argmax_to|time_embed|action_|silu_kernel|fill_u64|ecf'
  N=$(python tools/profile_step.py --profile $PROF --runs 1 2>/dev/null | sed -n "s/.*kernel_launches.: \([0-9]*\).*/\1/p" | head -1)
  echo "launches per inference: $N"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -s $N -c $N --csv \
      --log-file $OUT/launches.csv python tools/profile_step.py --profile $PROF --runs 2 > $OUT/launches.log 2>&1
  python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1; head -30 $OUT/launches_summary.txt
  # the dominant decode kernel as launched in the step: gate|up GEMV over ECT pages
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:gemv_ect_kernel<.int.2' -s 40 -c 1 -o $OUT/gemv_silu_ect python tools/profile_step.py --profile $PROF --runs 1 > $OUT/full_gemv.log 2>&1
  ncu -i $OUT/gemv_silu_ect.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $OUT/gemv_silu_ect_dram.csv 2>&1
  cat $OUT/gemv_silu_ect_dram.csv | tail -3
  python tools/ncu_kv.py $OUT/gemv_silu_ect.ncu-rep > $OUT/gemv_silu_ect_summary.txt 2>&1
  # the prefill gate|up tcgen05 GEMM as launched in the step: tensor-pipe utilisation
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:gemm_kernel<.int.256, .int.3' -s 2 -c 1 -o $OUT/gemm_gu_prefill python tools/profile_step.py --profile $PROF --runs 1 > $OUT/full_gemm.log 2>&1
  ncu -i $OUT/gemm_gu_prefill.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum > $OUT/gemm_gu_prefill_raw.csv 2>&1
  tail -1 $OUT/gemm_gu_prefill_raw.csv
  python tools/ncu_kv.py $OUT/gemm_gu_prefill.ncu-rep > $OUT/gemm_gu_prefill_summary.txt 2>&1
  # the ViT flash attention (hd 72, per-image blocks) as launched in the step
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:flash_kernel<.int.72' -s 2 -c 1 -o $OUT/flash_vit python tools/profile_step.py --profile $PROF --runs 1 > $OUT/full_flash_vit.log 2>&1
  python tools/ncu_kv.py $OUT/flash_vit.ncu-rep > $OUT/flash_vit_summary.txt 2>&1
  ncu -i $OUT/flash_vit.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct >> $OUT/flash_vit_summary.txt 2>&1; head -20 $OUT/flash_vit_summary.txt
fi
ls -la $OUT
