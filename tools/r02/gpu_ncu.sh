#!/bin/bash
# ncu launch list (device time, DRAM bytes, UTCHMMA count per launch) of the default bench
# command, after the same command exited 0 without ncu.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-ncu}; mkdir -p $O
C=${CONFIG:-dsv2s}
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --trace-iters 0"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 1500 ncu --clock-control none -c ${NLAUNCH:-320} --csv -k regex:"gemm_tc|attn_|gate_|permute|combine|gather|colsum|a2a_|route_scan" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__cycles_elapsed.avg.per_second \
  --log-file $O/launches_$C.csv $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $O/ncu.log
python tools/r02/ncu_groups.py $O/launches_$C.csv $C > $O/groups_$C.md; cat $O/groups_$C.md
