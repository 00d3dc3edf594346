OUT=gpurun_out/${1:-v9}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
timeout 1200 python bench.py --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 800 $OUT/bench.err; cat $OUT/bench.json
timeout 1500 python tools/sweep.py --trials 3 --out $OUT/sweep.json > $OUT/sweep.log 2>&1; echo "sweep rc=$?"; tail -5 $OUT/sweep.log
