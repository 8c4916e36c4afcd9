#!/bin/bash
# dsv2s / c4 / c3 bench lines with the PDL-off trace for the roofline.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-bench2}; mkdir -p $O
for c in ${CONFIGS:-dsv2s c4 c3}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --trace-dir $O > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"; tail -2 $O/bench_$c.err | cut -c1-300; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$c.json") if l.startswith("{")][-1]
r=d["roofline"]; print("$c", round(d["ms_per_step"],3), "ms", round(d["value"]), r["kernel"], round(r["achieved"]), round(r["frac"],3), "busy", round(r["busy_ms_per_step"],3), "pdl-trace busy", r.get("busy_ms_per_step_pdl_trace"), r["timing"][:60], d["clocks"]["sm_mhz"])
for g in r["groups"][:8]: print("   ", g["group"], round(g["achieved"]), g["unit"], round(g["frac"],3), round(g["busy_ms_per_step"],3))
PY
done
rm -f $O/*.json.gz
