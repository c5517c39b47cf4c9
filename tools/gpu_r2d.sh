#!/bin/bash
# Round-2 evidence session: smoke, full GPU suite, bench (both arms), ncu launch list + full
# capture of the apply kernel of the bench, and of the step kernel (emulated P=8).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_bench_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-halo > /dev/null 2>&1; echo "ncu list rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_warp_v1 -s 3 -c 1 -o gpurun_out/r02_apply \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-halo > /dev/null 2>&1; echo "ncu full rc=$?" >> gpurun_out/bench.err
REPS=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:xchg_kernel -s 2 -c 1 \
  -o gpurun_out/r02_xchg_kernel python tools/xchg_sweep.py > /dev/null 2>&1; echo "ncu xchg rc=$?" >> gpurun_out/bench.err
