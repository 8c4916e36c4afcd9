#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-fix1}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > $O/parity.log 2>&1; echo "parity rc=$?"; grep -E "^FAILED|passed|failed" $O/parity.log | head -5
# tcgen05 activity counters of one GEMM (dsv2s E2 shape) on CTA pairs and on single CTAs
cat > /tmp/one_gemm.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"]); sys.path.insert(0, os.path.join(os.environ["GRAFT_REPO_ROOT"], "tools"))
import gemm_microbench as gm
cg = int(sys.argv[1]); gm.run("dsv2s_e2", 2, 256, 1, cg)
PY
for cg in 2 1; do
  timeout 120 python /tmp/one_gemm.py $cg > $O/plain_cg$cg.log 2>&1 && \
  timeout 600 ncu --clock-control none -k regex:gemm_tc_kernel -s 2 -c 1 \
    --metrics gpu__time_duration.sum,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc_scope_2cta.sum,sm__inst_executed_pipe_tc_scope_1cta.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_2cta.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum,sm__cycles_elapsed.avg.per_second \
    --csv python /tmp/one_gemm.py $cg > $O/ncu_cg$cg.csv 2> $O/ncu_cg$cg.err; echo "ncu cg$cg rc=$?"
done
tail -20 $O/ncu_cg2.csv
