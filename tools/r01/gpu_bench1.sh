#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/summary.txt
timeout 600 python bench.py --profile-json gpurun_out/prof_c2.json > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --config c3 --no-cpu-baseline --profile-json gpurun_out/prof_c3.json > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/prof_c4.json > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_c2.json gpurun_out/bench_c3.json gpurun_out/bench_c4.json
tail -3 gpurun_out/bench_c2.err gpurun_out/bench_c3.err gpurun_out/bench_c4.err
