OUT=gpurun_out/${1:-v21}; mkdir -p $OUT
timeout 1200 python bench.py --no-cpu-baseline --no-sweep --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.err; python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['host_enqueue_ms_per_step'], d['gpu_launches'])"
