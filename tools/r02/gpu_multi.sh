#!/bin/bash
# Multi-GPU pass (N = number of visible GPUs): parity + schedule properties vs the oracle
# (tests/test_gpu_multi.py), NVLink busBW table, and bench lines at N for c2 / c3 / dsv2s.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/${TAG:-multi}_n$N; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 1400 -rs > $O/pytest.log 2>&1; echo "multi pytest rc=$?"; tail -4 $O/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29750 tools/r02/busbw.py > $O/busbw.jsonl 2> $O/busbw.err; echo "busbw rc=$?"; cp profiles/r02/busbw_n$N.md $O/ 2>/dev/null; cat profiles/r02/busbw_n$N.md; tail -3 $O/busbw.err
for c in ${CONFIGS:-c2 c3 dsv2s}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29760 \
    bench.py --gpus $N --config $c --steps 20 --warmup 5 --trace-dir $O > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"; rm -f $O/flowmoe_trace_*_r[1-9].json; gzip -f $O/flowmoe_trace_*_r0.json 2>/dev/null; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$c.json") if l.startswith("{")][-1]
x=d.get("exposed_comm") or {}
print("$c N=$N", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), "exposed/comm", x.get("frac_of_comm"), "transfer-only", (x.get("transfer_only") or {}).get("frac_of_transfer"), d["clocks"]["reasons"])
PY
done
