#!/bin/bash
# ncu --set full (with source) of the attention forward and backward at the dsv2s chunk
# shape, from the bench command (after it exited 0 without ncu).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-ncu_attn}; mkdir -p $O
CMD="python bench.py --config ${C:-dsv2s} --steps 1 --warmup 3 --no-cpu-baseline --trace-iters 0 --no-graph"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"attn_fwd_tc|attn_bwd_tc" --launch-skip 16 -c 2 \
  -o $O/attn_${C:-dsv2s} $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $O/ncu.log
