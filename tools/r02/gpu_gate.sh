#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-gate}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_schedule.py -q -s -p no:cacheprovider > $O/sched.log 2>&1; echo "sched rc=$?"; grep -E "priority|passed|failed|Error" $O/sched.log | head
