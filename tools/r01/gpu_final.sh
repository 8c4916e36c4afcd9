#!/bin/bash
# End-of-round validation on a 4-GPU box: smoke, full pytest -m gpu (P=1,2,4), the default
# bench line (N=1, as the driver runs it), the reference arm, and c2/c3/c4 at N=1,2,4.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
TAG=${1:-f}
S=$O/summary_$TAG.txt; echo "gpus=$(nvidia-smi -L | wc -l)" > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err; echo "bench default rc=$?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "bench reference rc=$?" >> $S
P=29500
for n in 2 4; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > $O/bench_default_n${n}_$TAG.json 2> $O/bench_default_n${n}_$TAG.err; echo "bench default n$n rc=$?" >> $S
done
for c in c3 c4; do
  for n in 1 2 4; do
    extra="--no-cpu-baseline"; [ $c = c4 ] && extra="$extra --steps 10 --warmup 3"
    P=$((P+1))
    if [ $n = 1 ]; then
      CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config $c $extra > $O/bench_${c}_n1_$TAG.json 2> $O/bench_${c}_n1_$TAG.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --config $c $extra > $O/bench_${c}_n${n}_$TAG.json 2> $O/bench_${c}_n${n}_$TAG.err
    fi
    echo "bench $c n$n rc=$?" >> $S
  done
done
cat $S; tail -n 3 $O/pytest_$TAG.log; tail -n 2 $O/smoke_$TAG.log
for f in $O/bench_*_$TAG.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  r=d.get('roofline') or {}
  print(f.split('/')[-1], d.get('impl','flowmoe'), round(d['ms_per_step'],3), 'ms', round(d['value']), d['unit'], 'e2e', round((d.get('e2e') or {}).get('value',0)), 'roof', r.get('bound'), round(r.get('frac',0),3), 'exposed', e.get('exposed_ms'), e.get('frac_of_comm'), e.get('ranks_valid'))
except Exception as ex: print(f, 'ERR', ex)
"; done
