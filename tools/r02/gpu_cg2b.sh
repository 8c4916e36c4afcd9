#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-cg2b}; mkdir -p $O
timeout 300 bash tools/r02/gpu_cg2probe.sh > /dev/null 2>&1; cat gpurun_out/r02/cg2probe/probe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 120 -x -k "gemm or cta_pair or routing or block_parity" > $O/gemm.log 2>&1; echo "tests rc=$?"; tail -5 $O/gemm.log
timeout 600 python tools/gemm_microbench.py dsv2s > $O/micro.jsonl 2> $O/micro.err; echo "micro rc=$?"; cat $O/micro.jsonl; tail -3 $O/micro.err
timeout 120 build/route_probe 512 5120 16 8 1.0 2; timeout 120 build/route_probe 1024 4096 16 2 1.0 2
