OUT=gpurun_out/${1:-v6}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 $OUT/pytest_gpu.log
for o in gemv ect splitk attn; do timeout 300 python tools/kernel_bench.py --only $o >> $OUT/kb.txt 2>&1; done; cat $OUT/kb.txt
timeout 1200 python bench.py --no-cpu-baseline --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 1500 $OUT/bench.err; cat $OUT/bench.json
