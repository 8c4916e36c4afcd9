#!/bin/bash
# ncu --set full captures of the top kernels (one GPU; each command first runs clean without ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-n1}
S=gpurun_out/summary_$TAG.txt; : > $S
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --trace-iters 0"
timeout 600 $B > gpurun_out/plain_$TAG.log 2>&1; echo "plain c2 rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 700 -c 4 -o gpurun_out/ncu_c2_gemm_$TAG $B > gpurun_out/ncu_c2_gemm_$TAG.log 2>&1; echo "ncu c2 gemm rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_.*_tc_kernel|gate_topk|gather_gate" -s 20 -c 5 -o gpurun_out/ncu_c2_attn_$TAG $B > gpurun_out/ncu_c2_attn_$TAG.log 2>&1; echo "ncu c2 attn rc=$?" >> $S
B4="python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --trace-iters 0 --layers 1"
timeout 600 $B4 > gpurun_out/plain4_$TAG.log 2>&1; echo "plain c4 rc=$?" >> $S
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 13 -c 13 -o gpurun_out/ncu_c4_gemm_$TAG $B4 > gpurun_out/ncu_c4_gemm_$TAG.log 2>&1; echo "ncu c4 gemm rc=$?" >> $S
cat $S; ls -la gpurun_out/*.ncu-rep
