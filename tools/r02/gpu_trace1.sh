#!/bin/bash
# dsv2s at N=1 with the CUPTI trace kept (in-graph kernel durations), two lanes vs one.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-trace1}; mkdir -p $O
for cs in 2 1; do
  mkdir -p $O/cs$cs
  timeout 600 python bench.py --config dsv2s --steps 20 --warmup 5 --no-cpu-baseline --compute-streams $cs --trace-dir $O/cs$cs > $O/bench_cs$cs.json 2> $O/bench_cs$cs.err
  echo "bench cs=$cs rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_cs$cs.json") if l.startswith("{")][-1]
r=d["roofline"]; print("cs=$cs", round(d["ms_per_step"],3), "ms", r["kernel"], round(r["achieved"]), round(r["frac"],3), d["clocks"]["sm_mhz"], d["timeline"])
PY
done
