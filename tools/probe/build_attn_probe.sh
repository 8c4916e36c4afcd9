#!/bin/bash
# attn_probe against the library objects; variant "lin" builds k_attn_tc.cu with -DFM_ATTN_LINEAR
set -e
cd "$(dirname "$0")/../.."
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include"
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
OBJS="build/flowmoe.cu.o build/k_attn.cu.o build/k_gemm_simt.cu.o build/k_gemm_tc.cu.o build/k_optim.cu.o build/k_p2p.cu.o build/k_route.cu.o"
for v in lpt lin; do
  D=""; [ $v = lin ] && D="-DFM_ATTN_LINEAR"
  $NV $D -I $NCCL/include -c paper_2510_00207_b200/csrc/k_attn_tc.cu -o build/attn_tc_$v.o
  $NV tools/probe/attn_probe.cu build/attn_tc_$v.o $OBJS -L $NCCL/lib -l:libnccl.so.2 -lcuda -Xlinker -rpath=$NCCL/lib -o build/attn_probe_$v
done
