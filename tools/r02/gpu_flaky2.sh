#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-flaky2}; mkdir -p $O
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_schedule.py -q -p no:cacheprovider > $O/run$i.log 2>&1; echo "run $i rc=$?"; grep -E "^FAILED|passed|failed" $O/run$i.log | head -5
done
