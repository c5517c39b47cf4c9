#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_locate.py > gpurun_out/prof_locate_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"locate_kernel|tri_bins_kernel|pull_rows|pack_rows|unpack_rows" -c 8 \
   -o gpurun_out/prof_locate python tools/prof_locate.py > gpurun_out/ncu_locate.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/ncu_locate.log
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_cfg5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply4 -s 3 -c 1 \
   -o gpurun_out/prof_apply4 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_apply4.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_apply4.log
