#!/bin/bash
# 2-GPU box: P=2 parity with the current kernels, then CUPTI traces of c2/c3 graph replays (N=1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/trace
TAG=${1:-tr}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?" >> $S
for c in c2 c3; do
  mkdir -p gpurun_out/trace/$c
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $c --no-cpu-baseline --trace-iters 6 --trace-dir gpurun_out/trace/$c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  echo "bench $c rc=$?" >> $S
done
gzip -f gpurun_out/trace/*/*.json
cat $S; tail -3 gpurun_out/pytest2_$TAG.log; ls -la gpurun_out/trace/*
