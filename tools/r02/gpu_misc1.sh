#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-misc1}; mkdir -p $O
timeout 120 build/gate_probe > $O/gate_probe.txt 2>&1; echo "gate probe rc=$?"; grep -A1 "dsv2s\|c4 " $O/gate_probe.txt | tail -4
timeout 600 python tools/gemm_microbench.py dsv2s_e1gelu dsv2s_dgelu_mul dsv2s_oproj dsv2s_dctx > $O/micro.jsonl 2> $O/micro.err; echo "micro rc=$?"; cat $O/micro.jsonl
timeout 600 python -m pytest tests/test_gpu_schedule.py -q -s -p no:cacheprovider > $O/sched.log 2>&1; echo "sched rc=$?"; grep -E "priority|passed|failed" $O/sched.log
