#!/bin/bash
# multi-rank bench path on one GPU (2 ranks on cuda:0, gloo): path check only
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LFB_BENCH_ONE_DEVICE=1 LFB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-nelt 65536 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "rc=$?" >> gpurun_out/bench_2rank.err
LFB_BENCH_ONE_DEVICE=1 LFB_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_2rank_ref.json 2>> gpurun_out/bench_2rank.err; echo "rc=$?" >> gpurun_out/bench_2rank.err
