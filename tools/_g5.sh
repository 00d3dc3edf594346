OUT=gpurun_out/${1:-v10}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
timeout 1200 python bench.py --no-cpu-baseline --no-sweep --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 800 $OUT/bench.err; cat $OUT/bench.json
PROF=$OUT/profile_alpamayo-r1-10b-shape.json
KRE='regex:gemv_kernel|gemm_kernel|flash_kernel|decode_attn|rmsnorm|layernorm|qk_norm|embed_rows|add_rows|argmax_to|time_embed|action_|silu_kernel|fill_u64|ecf|ect'
N=$(python tools/profile_step.py --profile $PROF --runs 1 2>/dev/null | sed -n "s/.*kernel_launches.: \([0-9]*\).*/\1/p" | head -1)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -s $N -c $N --csv --log-file $OUT/launches.csv python tools/profile_step.py --profile $PROF --runs 2 > $OUT/launches.log 2>&1
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1; head -24 $OUT/launches_summary.txt
