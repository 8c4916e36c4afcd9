#!/bin/bash
# 1 GPU: CUPTI traces of c2/c3 graph replays (N=1) for critical-path analysis
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/trace
TAG=${1:-t1}
for c in c2 c3; do
  mkdir -p gpurun_out/trace/${c}_$TAG
  timeout 600 python bench.py --config $c --no-cpu-baseline --trace-iters 6 --trace-dir gpurun_out/trace/${c}_$TAG > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  echo "bench $c rc=$?"
done
gzip -f gpurun_out/trace/*_$TAG/*.json
