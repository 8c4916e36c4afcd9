#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-bisect}; mkdir -p $O
i=0
while read -r k; do
  i=$((i+1))
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$k" > $O/run$i.log 2>&1; echo "[$k] rc=$?"; grep -E "^FAILED|passed|failed" $O/run$i.log | head -3
done <<'LIST'
stack_api
stack_api_matches
unsplit or tok-True
chain or tok-True
cta_pair or tok-True
gemm or tok-True
LIST
