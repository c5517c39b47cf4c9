#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for ch in 16 32 64 128 256; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode gather --e2e-chunks $ch > gpurun_out/bench_gch_${ch}.json 2> gpurun_out/bench_gch_${ch}.err
done
