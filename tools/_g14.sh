OUT=gpurun_out/${1:-v28}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 1500 python tools/blind_offload.py --out $OUT/blind_offload.json > $OUT/blind.log 2>&1; echo "blind rc=$?"; tail -5 $OUT/blind.log
