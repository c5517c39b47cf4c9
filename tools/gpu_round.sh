#!/bin/bash
# One GPU session: tests, bench (both arms), launch list, full ncu capture of the apply kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${REF:-1}" = "1" ]; then
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
for extra in ${EXTRA:-}; do
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $extra > gpurun_out/bench_$extra.json 2> gpurun_out/bench_$extra.err
done
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply -s 3 -c 2 \
      -o gpurun_out/prof_apply python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu2.log
fi
