#!/bin/bash
# 2-GPU box: P=2 parity; then (GPU 0 only) the c2 bench launch list under ncu
# (gpu__time_duration, --clock-control none, same bench command), and ncu --set full
# captures of the c2 attention / gate / expert GEMM kernels.  Each ncu command runs
# first without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-n2}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?" >> $S
export CUDA_VISIBLE_DEVICES=0
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --trace-iters 0"
timeout 600 $B > gpurun_out/plain_$TAG.log 2>&1; echo "plain c2 rc=$?" >> $S
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_tc|attn_bwd_tc|gate_topk" -s 60 -c 6 -o gpurun_out/ncu_c2_attn_$TAG $B > gpurun_out/ncu_c2_attn_$TAG.log 2>&1; echo "ncu c2 attn rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 200 -c 8 -o gpurun_out/ncu_c2_gemm_$TAG $B > gpurun_out/ncu_c2_gemm_$TAG.log 2>&1; echo "ncu c2 gemm rc=$?" >> $S
cat $S; tail -2 gpurun_out/pytest2_$TAG.log; ls -la gpurun_out/*$TAG*
