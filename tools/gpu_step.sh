#!/bin/bash
# Exchange-kernel session: halo / step / multi-process tests, one bench line, first-call timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_halo.py tests/test_gpu_dist.py tests/test_gpu_output.py tests/test_gpu_gather.py -q -x > gpurun_out/pytest_step.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_step.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err
echo "bench rc=$?" >> gpurun_out/bench_step.err
for k in 1 2 3; do timeout 300 python tools/first_call_plan.py 2>/dev/null | head -2; done > gpurun_out/first_call.log
