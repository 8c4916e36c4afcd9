#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-gate2}; mkdir -p $O
timeout 120 build/gate_probe > $O/gate_probe.txt 2>&1; echo "gate probe rc=$?"; grep -A1 "dsv2s\|c4 \|c2 " $O/gate_probe.txt | tail -6
timeout 120 build/route_probe 512 5120 16 8 1.0 2 | grep -E "gate|scan"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py tests/test_gpu_group.py -q -s -p no:cacheprovider -x > $O/tests.log 2>&1; echo "tests rc=$?"; grep -E "priority|passed|failed|Error" $O/tests.log | tail -8
