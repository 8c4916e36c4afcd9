#!/bin/bash
# Copy-engine A2A exchanges (FLOWMOE_CE_A2A) vs the SM peer-memory kernel at N GPUs: multi-GPU
# parity tests with it on, the A2A bus bandwidth, and dsv2s / c3 bench lines with and without.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/${TAG:-ceA2A}_n$N; mkdir -p $O
FLOWMOE_CE_A2A=1 timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider --timeout 1400 > $O/pytest.log 2>&1; echo "multi pytest (CE A2A) rc=$?"; tail -3 $O/pytest.log
FLOWMOE_CE_A2A=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29750 tools/r02/busbw.py > $O/busbw.jsonl 2> $O/busbw.err; echo "busbw rc=$?"; grep A2A $O/busbw.jsonl | cut -c1-160; tail -2 $O/busbw.err
for c in ${CONFIGS:-dsv2s c3}; do
  for v in "" 1 "" 1; do
    env ${v:+FLOWMOE_CE_A2A=1} timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29760 \
      bench.py --gpus $N --config $c --steps 20 --warmup 5 --no-cpu-baseline --trace-iters 0 > $O/bench_${c}_ceA2A$v.json 2> $O/bench_${c}_ceA2A$v.err
    echo "bench $c ceA2A=$v rc=$?"; python -c "
import json
d=[json.loads(l) for l in open('$O/bench_${c}_ceA2A$v.json') if l.startswith('{')][-1]
print('$c ceA2A=$v', round(d['ms_per_step'],3), 'ms', round(d['value']))" 2>&1 | tail -1
  done
done
