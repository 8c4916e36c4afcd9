#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-sched}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_parity.py -k "schedule or crafted" -q -s -p no:cacheprovider --timeout 400 > $O/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "priority|passed|failed|Error|assert" $O/pytest.log | head -30
timeout 900 python bench.py --steps 20 --warmup 5 --profile-json $O/prof_dsv2s.json --trace-dir $O > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 3000 $O/bench.json; tail -3 $O/bench.err
