#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-flaky}; mkdir -p $O
for i in 1 2 3 4 5 6 7 8; do
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "${KEXPR:-stack_api_matches_per_block and tok}" > $O/run$i.log 2>&1; echo "run $i rc=$?"; grep -E "AssertionError: |passed|failed" $O/run$i.log | head -3
done
