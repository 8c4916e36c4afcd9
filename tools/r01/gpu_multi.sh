#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
echo "gpus=$N" > gpurun_out/multi_summary.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -x > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> gpurun_out/multi_summary.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29500 bench.py --gpus $N --profile-json gpurun_out/prof_c2_n$N.json > gpurun_out/bench_c2_n$N.json 2> gpurun_out/bench_c2_n$N.err; echo "bench c2 n$N rc=$?" >> gpurun_out/multi_summary.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29501 bench.py --gpus $N --config c3 --profile-json gpurun_out/prof_c3_n$N.json > gpurun_out/bench_c3_n$N.json 2> gpurun_out/bench_c3_n$N.err; echo "bench c3 n$N rc=$?" >> gpurun_out/multi_summary.txt
cat gpurun_out/multi_summary.txt; tail -n 5 gpurun_out/pytest_multi.log; cat gpurun_out/bench_c2_n$N.json; tail -n 5 gpurun_out/bench_c2_n$N.err
