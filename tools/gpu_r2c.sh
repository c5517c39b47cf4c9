#!/bin/bash
# Round-2 session: full GPU suite, default bench, cfg4 signalled-exchange sweep (emulated).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for h in 1 2 3; do HALO=$h timeout 300 python tools/xchg_sweep.py; done > gpurun_out/xchg_sweep.jsonl 2> gpurun_out/xchg_sweep.err
for h in 1 2 3; do HALO=$h PART=blocks timeout 300 python tools/xchg_sweep.py; done >> gpurun_out/xchg_sweep.jsonl 2>> gpurun_out/xchg_sweep.err
