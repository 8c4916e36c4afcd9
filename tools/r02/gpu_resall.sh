#!/bin/bash
# A/B at N=1: SMs every GEMM leaves to the other lane's kernels (FLOWMOE_SM_RESERVE).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-resall}; mkdir -p $O
for r in ${RESERVES:-0 8 16 24 32 0}; do
  FLOWMOE_SM_RESERVE=$r timeout 600 python bench.py --config ${C:-dsv2s} --steps 20 --warmup 5 --no-cpu-baseline --trace-iters 0 > $O/bench_res$r.json 2> $O/bench_res$r.err
  python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_res$r.json") if l.startswith("{")][-1]
print("reserve $r", round(d["ms_per_step"],3), "ms", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
