#!/bin/bash
# A/B at N GPUs: SMs the backward GEMMs leave to the NCCL all-reduce (FLOWMOE_BWD_SM_RESERVE).
cd $GRAFT_REPO_ROOT
for r in ${RESERVES:-0 32 16 0}; do
  FLOWMOE_BWD_SM_RESERVE=$r SUFFIX=_res$r BT=420 TAG=${TAG:-reserve} CONFIGS="${CONFIGS:-dsv2s}" bash tools/r02/gpu_n2dsv.sh
done
