#!/bin/bash
# N-GPU: multi-GPU parity + schedule test, then bench lines under AR communicator CTA caps.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/${TAG:-arcap}_n$N; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 1400 -rs > $O/pytest.log 2>&1; echo "multi pytest rc=$?"; tail -3 $O/pytest.log; grep -E "AssertionError" $O/pytest.log | head -3
for cap in ${CAPS:-16 32 64}; do
for c in ${CONFIGS:-dsv2s c3}; do
  FLOWMOE_AR_MAX_CTAS=$cap timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29760 \
    bench.py --gpus $N --config $c --steps 20 --warmup 5 --no-cpu-baseline --trace-dir $O > $O/bench_${c}_cap$cap.json 2> $O/bench_${c}_cap$cap.err
  python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_${c}_cap$cap.json") if l.startswith("{")][-1]
x=d.get("exposed_comm") or {}
print("$c N=$N cap=$cap", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s", "exposed/comm", x.get("frac_of_comm"), "of iter", x.get("frac_of_iteration"), "comm ms", x.get("comm_busy_ms"))
PY
done; done
