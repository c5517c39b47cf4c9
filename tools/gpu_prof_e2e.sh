#!/bin/bash
# e2e pipeline kernels under ncu: launch list of one gather-mode call + a full capture of one
# gather_tma launch (PCIe / sysmem traffic) and one compact-source apply launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_e2e.py 1 > gpurun_out/prof_e2e_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/e2e_launches.csv python tools/prof_e2e.py 2 > gpurun_out/prof_e2e_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_tma -s 70 -c 1 \
  -o gpurun_out/prof_gather python tools/prof_e2e.py 2 > gpurun_out/prof_e2e_ncu2.log 2>&1
echo "rc=$?" >> gpurun_out/prof_e2e_ncu2.log
