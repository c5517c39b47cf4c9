#!/bin/bash
# The torchrun (one process per rank) bench path on ONE GPU: 2 ranks share device 0 and
# exchange halos through CUDA-IPC + the pull kernel (host-barrier synchronised; no kernel
# waits on another).  Validates the multi-process plumbing; not a scaling number.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --transport ipc --config cfg2 \
  > gpurun_out/bench_multi_ipc.json 2> gpurun_out/bench_multi_ipc.err
echo "rc=$?" >> gpurun_out/bench_multi_ipc.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29519 bench.py --gpus 2 --steps 5 --warmup 3 --transport ipc --fused --config cfg2 \
  > gpurun_out/bench_multi_fused.json 2> gpurun_out/bench_multi_fused.err
echo "rc=$?" >> gpurun_out/bench_multi_fused.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 --config cfg1 \
  > gpurun_out/bench_multi_ref.json 2> gpurun_out/bench_multi_ref.err
echo "rc=$?" >> gpurun_out/bench_multi_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29520 bench.py --gpus 4 --steps 5 --warmup 3 --transport ipc --fused --partitioner equal_regions \
  --config cfg2 > gpurun_out/bench_multi_fused_eq4.json 2> gpurun_out/bench_multi_fused_eq4.err
echo "rc=$?" >> gpurun_out/bench_multi_fused_eq4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29521 bench.py --gpus 2 --steps 5 --warmup 3 --transport ipc --config cfg3 \
  > gpurun_out/bench_multi_cfg3.json 2> gpurun_out/bench_multi_cfg3.err
echo "rc=$?" >> gpurun_out/bench_multi_cfg3.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29522 bench.py --gpus 2 --steps 5 --warmup 3 --transport ipc --config cfg5 \
  > gpurun_out/bench_multi_cfg5.json 2> gpurun_out/bench_multi_cfg5.err
echo "rc=$?" >> gpurun_out/bench_multi_cfg5.err
