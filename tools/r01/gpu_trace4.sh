#!/bin/bash
# 4 GPUs: CUPTI traces of c3 graph replays at N=4 (all ranks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/trace
TAG=${1:-t4}
mkdir -p gpurun_out/trace/c3_$TAG
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 4 --config c3 --no-cpu-baseline --trace-iters 6 --trace-dir gpurun_out/trace/c3_$TAG > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
echo "bench c3 rc=$?"
gzip -f gpurun_out/trace/c3_$TAG/*.json
