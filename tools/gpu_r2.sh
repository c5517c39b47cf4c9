#!/bin/bash
# Round-2 GPU session: smoke, gpu tests, bench (product arm then reference arm).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; nvidia-smi -L >> gpurun_out/nproc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [ "${REF:-1}" = "1" ]; then
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?" >> gpurun_out/bench_ref.err
fi
