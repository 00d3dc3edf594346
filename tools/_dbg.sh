OUT=gpurun_out/${1:-d1}; mkdir -p $OUT
timeout 300 python -X faulthandler -m pytest tests/test_kernels_gpu.py -k "gemm_ect or split_k" -v -x > $OUT/p1.log 2>&1; echo "rc=$?"; grep -E "PASS|FAIL|Fatal|Error|line" $OUT/p1.log | head -30
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_kernels_gpu.py -k "gemm_ect" -x -q > $OUT/p2.log 2>&1; echo "rc=$?"; grep -v "^$" $OUT/p2.log | head -40
