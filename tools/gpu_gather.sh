#!/bin/bash
# gather host-execute mode: parity tests, then the cfg3 e2e per mode on one box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_remap.py -q -m gpu -k "execute_host" > gpurun_out/pytest_gather.log 2>&1
for mode in ${MODES:-gather gather_warp dma auto}; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode $mode > gpurun_out/bench_mode_${mode}.json 2> gpurun_out/bench_mode_${mode}.err
done
