#!/bin/bash
# DRAM traffic + device time of every kernel of one steady-state eager iteration (lightweight metrics)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-t}
S=gpurun_out/summary_$TAG.txt; : > $S
K='regex:gemm_tc|attn|gate|route|permute|unpermute|combine|gather|colsum'
for c in c2 c3; do
  B="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --trace-iters 0"
  SKIP=1200; [ $c = c3 ] && SKIP=110; CNT=1000; [ $c = c3 ] && CNT=110
  timeout 600 $B > gpurun_out/plain_${c}_$TAG.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s $SKIP -c $CNT --csv --log-file gpurun_out/traffic_${c}_$TAG.csv $B > gpurun_out/ncu_traffic_${c}_$TAG.log 2>&1; echo "traffic $c rc=$?" >> $S
done
cat $S
