#!/bin/bash
# Signalled-exchange session: the step/exchange tests, the multi-process tests, one bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_halo.py tests/test_gpu_dist.py tests/test_gpu_nccl.py -q -x > gpurun_out/pytest_step.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_step.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err
echo "bench rc=$?" >> gpurun_out/bench_step.err
