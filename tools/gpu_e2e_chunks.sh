#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 8 16 32 64 128; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/bench_chunks_$c.json 2> gpurun_out/bench_chunks_$c.err
done
