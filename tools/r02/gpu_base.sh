#!/bin/bash
# Round-2 baseline on one B200: dsv2s and c4 bench lines (with the per-kernel profile
# and the CUPTI timeline), before any round-2 change.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/base; mkdir -p $O
for c in dsv2s c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline \
    --profile-json $O/prof_$c.json --trace-dir $O > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"; tail -c 600 $O/bench_$c.json
done
