#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-a}
S=gpurun_out/summary_$TAG.txt
: > $S
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_parity or routing" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest parity rc=$?" >> $S
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all_$TAG.log 2>&1; echo "pytest all rc=$?" >> $S
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  [ $c != c2 ] && extra="$extra --no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_$TAG.json > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?" >> $S
done
cat $S; tail -n 30 gpurun_out/pytest_$TAG.log; tail -n 3 gpurun_out/pytest_all_$TAG.log
for c in c2 c3 c4; do head -c 300 gpurun_out/bench_${c}_$TAG.json; echo; done
