OUT=gpurun_out/${1:-v29}; mkdir -p $OUT
timeout 600 python tools/kernel_bench.py --only ect > $OUT/kb.txt 2>&1; cat $OUT/kb.txt | head -3
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 1200 python bench.py --no-cpu-baseline --no-sweep --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.err; python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['e2e']['value'], d['lower_bound'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['decode_layer_gbs_live'])"
