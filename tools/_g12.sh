OUT=gpurun_out/${1:-v25}; mkdir -p $OUT
timeout 600 python tools/kernel_bench.py --only ectprefill > $OUT/kb.txt 2>&1; cat $OUT/kb.txt
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "graph" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
