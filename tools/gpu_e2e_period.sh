#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_remap.py -q -x -k "execute_host" > gpurun_out/pytest_e2e.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_e2e.log
for p in 0 8 5 3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode compact --e2e-period $p > gpurun_out/bench_period_$p.json 2> gpurun_out/bench_period_$p.err
done
