#!/bin/bash
# validate + measure: pytest -m gpu, bench c2/c3/c4 with per-kernel profile, warm ncu launch list of c2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v}
S=gpurun_out/summary_$TAG.txt
: > $S
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  [ $c != c2 ] && extra="$extra --no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_$TAG.json > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?" >> $S
done
K='regex:gemm_tc|attn|gate|route|permute|unpermute|combine|gather|colsum'
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k "$K" -s 1200 -c 1200 --csv --log-file gpurun_out/launches_c2_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?" >> $S
cat $S; tail -n 3 gpurun_out/pytest_$TAG.log
for c in c2 c3 c4; do head -c 400 gpurun_out/bench_${c}_$TAG.json; echo; done
