#!/bin/bash
# Round-2 final evidence: smoke, full GPU suite, bench cfg3 (both arms), cfg2 / cfg5 / cfg5fe
# lines, ncu launch list of the bench command, emulated fused step and exchange sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
for c in cfg2 cfg5 cfg5fe; do
  timeout 1200 python bench.py --steps 20 --warmup 5 --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?" >> gpurun_out/bench_cfgs.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_bench_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-halo > /dev/null 2>&1; echo "ncu list rc=$?" >> gpurun_out/bench.err
REPS=20 timeout 300 python tools/fused_step_emulated.py > gpurun_out/fstep.json 2> gpurun_out/fstep.err
for p in equal_regions blocks; do for h in 1 2 3; do PART=$p HALO=$h timeout 300 python tools/xchg_sweep.py; done; done > gpurun_out/xchg_sweep.jsonl 2> gpurun_out/xchg_sweep.err
