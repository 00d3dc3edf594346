#!/bin/bash
mkdir -p gpurun_out/r3
timeout 300 python -m pytest -q tests/test_kernels_gpu.py tests/test_engine_gpu.py 2>&1 | tail -4
timeout 200 python tools/kernel_bench.py 2>&1 | tail -12
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 12 -c 1 -o gpurun_out/r3/gemv_silu python tools/kernel_bench.py --only gemv > gpurun_out/r3/ncu_gemv.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 10 -c 1 -o gpurun_out/r3/gemm_qkv python tools/kernel_bench.py --only gemm > gpurun_out/r3/ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 35 -c 1 -o gpurun_out/r3/gemm_silu python tools/kernel_bench.py --only gemm > gpurun_out/r3/ncu_gemm2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 30 -c 1 -o gpurun_out/r3/dattn python tools/kernel_bench.py --only attn > gpurun_out/r3/ncu_attn.log 2>&1
ls gpurun_out/r3
timeout 900 python bench.py --no-cpu-baseline --dump gpurun_out/r3 > gpurun_out/r3/bench.json 2> gpurun_out/r3/bench.err
echo bench rc=$?; tail -c 600 gpurun_out/r3/bench.err; cat gpurun_out/r3/bench.json
