#!/bin/bash
# first GPU validation run
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -k gemm -q -p no:cacheprovider > gpurun_out/t_gemm.log 2>&1; echo "gemm rc=$?" >> gpurun_out/summary.txt
FLOWMOE_DEBUG_SWAP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc_layouts and 200" -q -p no:cacheprovider > gpurun_out/t_gemm_swap.log 2>&1; echo "gemm swap rc=$?" >> gpurun_out/summary.txt
FLOWMOE_DEBUG_SIMT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "not gemm" -q -p no:cacheprovider > gpurun_out/t_simt.log 2>&1; echo "simt blocks rc=$?" >> gpurun_out/summary.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -k "not gemm" -q -p no:cacheprovider > gpurun_out/t_tc.log 2>&1; echo "tc blocks rc=$?" >> gpurun_out/summary.txt
tail -5 gpurun_out/*.log
cat gpurun_out/summary.txt
