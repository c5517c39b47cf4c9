#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_remap.py tests/test_gpu_bilinear.py tests/test_gpu_halo.py tests/test_gpu_output.py \
  -k "not o1280 and not cfg2 and not second_order and not O160" -x -q > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
