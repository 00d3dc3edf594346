OUT=gpurun_out/${1:-v20}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
for o in gemv ect; do timeout 300 python tools/kernel_bench.py --only $o >> $OUT/kb.txt 2>&1; done; cat $OUT/kb.txt
timeout 1200 python bench.py --no-cpu-baseline --no-sweep --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.err; python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['lower_bound'], d['config']['placement'], d['roofline']['achieved'], d['roofline']['decode_layer_gbs_live'])"
