OUT=gpurun_out/${1:-v22}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --no-cpu-baseline --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.err; python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['e2e']['value'], d['host_enqueue_ms_per_step'], d['lower_bound'], d['config']['placement'], d['predictor']['dfbsim_max_abs_error_pct'])"
