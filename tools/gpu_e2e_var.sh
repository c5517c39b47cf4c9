#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
for i in 1 2; do
for mode in compact dma; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode $mode > gpurun_out/bench_var_${mode}_$i.json 2> gpurun_out/bench_var_${mode}_$i.err
done
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config cfg5 > gpurun_out/bench_var_cfg5.json 2> gpurun_out/bench_var_cfg5.err
