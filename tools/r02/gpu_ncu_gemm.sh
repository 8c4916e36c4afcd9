#!/bin/bash
# ncu --set full of GEMM launches (microbench shape $SHAPE, variants $ONLY = "cg,bn,sk;...",
# each launched twice without a graph), after the same command exited 0 without ncu.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-ncugemm}; mkdir -p $O
N=$(( $(echo "$ONLY" | tr ';' '\n' | wc -l) * 2 ))
ONLY="$ONLY" timeout 300 python tools/gemm_microbench.py $SHAPE > $O/plain.log 2>&1 && \
ONLY="$ONLY" timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -c $N \
    -o $O/$SHAPE python tools/gemm_microbench.py $SHAPE > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $O/ncu.log
