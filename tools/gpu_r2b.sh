#!/bin/bash
# Round-2 session: full GPU suite, default bench, step-kernel ncu, gather timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python tools/fused_step_emulated.py > gpurun_out/fstep.json 2> gpurun_out/fstep.err && \
REPS=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
  -o gpurun_out/r02_step_kernel python tools/fused_step_emulated.py > gpurun_out/ncu_step.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_step.log
timeout 900 python tools/gather_timing.py > gpurun_out/gather_timing.jsonl 2> gpurun_out/gather_timing.err
