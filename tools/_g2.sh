OUT=gpurun_out/${1:-v7}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 $OUT/pytest_gpu.log
for o in gemv ect splitk attn; do timeout 300 python tools/kernel_bench.py --only $o >> $OUT/kb.txt 2>&1; done; cat $OUT/kb.txt
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 6 -c 1 -o $OUT/gemv_ect python tools/kernel_bench.py --only ect > $OUT/l2.log 2>&1
python tools/ncu_kv.py $OUT/gemv_ect.ncu-rep
timeout 1200 python bench.py --no-cpu-baseline --no-sweep --dump $OUT > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 1500 $OUT/bench.err; cat $OUT/bench.json
