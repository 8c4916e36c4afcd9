#!/bin/bash
# Round-1 profile set (one GPU; every ncu command runs first without ncu):
#  1. launch list of the bench command (gpu__time_duration, --clock-control none)
#  2. DRAM traffic per kernel (dram__bytes_read/write) of c2/c3/c4 steady-state iterations
#  3. ncu --set full captures of the top kernels (c2 GEMM, c3 attention, c4 expert GEMM)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
O=gpurun_out/prof
S=$O/summary.txt; : > $S
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --trace-iters 0"
timeout 600 $B > $O/plain_c2.log 2>&1; echo "plain c2 rc=$?" >> $S
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c2.csv $B > $O/ncu_launches_c2.log 2>&1; echo "launch list c2 rc=$?" >> $S
K='regex:gemm_tc|attn|gate|route|permute|unpermute|combine|gather|colsum'
for c in c2 c3 c4; do
  BC="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --trace-iters 0"
  [ $c = c4 ] && BC="$BC --layers 1"
  SKIP=1400; CNT=700
  [ $c = c3 ] && { SKIP=300; CNT=150; }
  [ $c = c4 ] && { SKIP=80; CNT=40; }
  timeout 600 $BC > $O/plain_$c.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s $SKIP -c $CNT --csv --log-file $O/traffic_$c.csv $BC > $O/ncu_traffic_$c.log 2>&1; echo "traffic $c rc=$?" >> $S
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 600 -c 6 -o $O/full_c2_gemm $B > $O/full_c2_gemm.log 2>&1; echo "full c2 gemm rc=$?" >> $S
B3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --trace-iters 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_tc|attn_fwd_tc" -s 40 -c 4 -o $O/full_c3_attn $B3 > $O/full_c3_attn.log 2>&1; echo "full c3 attn rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_topk -s 40 -c 4 -o $O/full_c3_gate $B3 > $O/full_c3_gate.log 2>&1; echo "full c3 gate rc=$?" >> $S
B4="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --trace-iters 0 --layers 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 30 -c 10 -o $O/full_c4_gemm $B4 > $O/full_c4_gemm.log 2>&1; echo "full c4 gemm rc=$?" >> $S
cat $S; ls -la $O
