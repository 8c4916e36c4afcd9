#!/bin/bash
# End-of-round check on a 2-GPU box: smoke, the full GPU suite (P=1 and P=2), the default
# bench at N=1 (as the driver runs it) and N=2, and the reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "bench n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?"
for f in $O/bench_n1.json $O/bench_n2.json $O/bench_ref.json; do python -c "
import json
d=[json.loads(l) for l in open('$f') if l.startswith('{')][0]
print('$f', d.get('impl','flowmoe'), round(d['ms_per_step'],3), 'ms', round(d['value']), 'e2e', round(d['e2e']['value']), 'launches', d.get('gpu_launches'), 'clocks', d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
"; done
