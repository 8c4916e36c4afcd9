#!/bin/bash
# full validation + scaling on a 4-GPU box: pytest -m gpu (incl. P=2,4 parity), bench c2/c3/c4 at N=1,2,4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-s}
N=$(nvidia-smi -L | wc -l)
S=gpurun_out/summary_$TAG.txt; echo "gpus=$N" > $S
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
P=29700
for n in 1 2 4; do
  [ $n -gt $N ] && continue
  for c in c2 c3 c4; do
    extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
    P=$((P+1))
    if [ $n = 1 ]; then
      CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_${TAG}_n1.json > gpurun_out/bench_${c}_${TAG}_n1.json 2> gpurun_out/bench_${c}_${TAG}_n1.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --config $c $extra --profile-json gpurun_out/prof_${c}_${TAG}_n$n.json > gpurun_out/bench_${c}_${TAG}_n$n.json 2> gpurun_out/bench_${c}_${TAG}_n$n.err
    fi
    echo "bench $c n$n rc=$?" >> $S
  done
done
cat $S; tail -n 3 gpurun_out/pytest_$TAG.log
for f in gpurun_out/bench_*_${TAG}_n*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'exposed_ms', e.get('exposed_ms'), 'frac', e.get('frac_of_comm'))
except Exception as ex: print(f, 'ERR', ex)
"; done
