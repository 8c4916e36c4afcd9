#!/bin/bash
# 2-GPU check: the multi-GPU parity tests and the default bench at N=1 and N=2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/m2
O=gpurun_out/m2
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 $O/pytest_multi.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "bench n2 rc=$?"
for f in $O/bench_n1.json $O/bench_n2.json; do python -c "
import json
d=[json.loads(l) for l in open('$f') if l.startswith('{')][0]
print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']), 'e2e', round(d['e2e']['value']), 'exposed', (d.get('exposed_comm') or {}).get('exposed_ms'))
"; done
