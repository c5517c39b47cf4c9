#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2; do
for mode in compact dma; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode $mode > gpurun_out/bench_var_${mode}_$i.json 2> gpurun_out/bench_var_${mode}_$i.err
done
done
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|Socket|NUMA" >> gpurun_out/nproc.txt
