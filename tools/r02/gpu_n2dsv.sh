#!/bin/bash
# dsv2s at N GPUs with the CUPTI trace kept per config (exposure analysis), then the GEMM
# microbench on GPU 0.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/${TAG:-n2dsv}; mkdir -p $O
for c in ${CONFIGS:-dsv2s}; do
timeout ${BT:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29760 \
  bench.py --gpus $N --config $c --steps 20 --warmup 5 --trace-dir $O $BENCH_EXTRA > $O/bench_${c}_n$N${SUFFIX}.json 2> $O/bench_${c}_n$N${SUFFIX}.err
echo "bench $c rc=$?"; rm -f $O/flowmoe_trace_*_r[1-9].json; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_${c}_n$N${SUFFIX}.json") if l.startswith("{")][-1]
x=d.get("exposed_comm") or {}
print("$c$SUFFIX N=$N", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), "exposed/comm", x.get("frac_of_comm"), "exposed ms", x.get("exposed_ms"), d["clocks"]["reasons"])
PY
done
if [ -n "$SHAPES" ]; then SHAPES="$SHAPES" TAG=$TAG/micro bash tools/r02/gpu_micro.sh; fi
