#!/bin/bash
# Fused peer-memory halo: tests, the 2-rank bench on one GPU (gloo for the
# plumbing, IPC for the halo), and the 1-GPU headline bench.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest -q -x tests/test_dist_gpu.py -k fused > gpurun_out/p2p_test.log 2>&1; echo "fused rc=$?" >> gpurun_out/p2p_test.log
PSM_HALO=p2p PSM_DIST_BACKEND=gloo timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --shape 512 512 512 --no-cpu-baseline \
  > gpurun_out/p2p_bench_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/p2p_bench_p2p.log
for i in 1 2 3; do timeout -s KILL 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/p2p_bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/p2p_bench_n1.log; done
