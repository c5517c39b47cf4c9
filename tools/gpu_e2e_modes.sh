#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_remap.py -q -x -k "execute_host or fallback" > gpurun_out/pytest_e2e.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_e2e.log
for mode in dma compact; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode $mode > gpurun_out/bench_e2e_$mode.json 2> gpurun_out/bench_e2e_$mode.err
done
