#!/bin/bash
# First run of the CTA-pair GEMM: one small case under a short timeout, then the GEMM
# tests, the forced-pair block tests, and the dsv2s GEMM microbenchmark (1-CTA vs pairs).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-cg2}; mkdir -p $O
timeout 120 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "test_gemm_tc_layouts_vs_fp64 and 2-256 and shape0 and 0-0" > $O/first.log 2>&1; rc=$?
echo "first rc=$rc"; tail -5 $O/first.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -k "gemm or cta_pair" > $O/gemm.log 2>&1; echo "gemm tests rc=$?"; tail -15 $O/gemm.log
timeout 600 python tools/gemm_microbench.py dsv2s c4_qkv c4_e1 > $O/micro.jsonl 2> $O/micro.err; echo "micro rc=$?"; cat $O/micro.jsonl; tail -3 $O/micro.err
