#!/bin/bash
# Round-2 pass on one B200: routing probe, smoke, GPU suite, dsv2s bench (+c4, c2).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-round2}; mkdir -p $O
timeout 120 build/route_probe 512 5120 16 8 1.0 2 > $O/route.txt 2>&1; timeout 120 build/route_probe 1024 4096 16 2 1.0 2 >> $O/route.txt 2>&1; grep -E "gather|T_r" $O/route.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
for spec in "dsv2s:" "c4:" "c2:"; do
  c=${spec%%:*}; extra=${spec#*:}; tag=$c$(echo $extra | tr -d ' -')
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline $extra \
    --profile-json $O/prof_$tag.json --trace-dir $O > $O/bench_$tag.json 2> $O/bench_$tag.err
  echo "bench $tag rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$tag.json") if l.startswith("{")][-1]
r=d["roofline"]; print("$tag", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), r["kernel"], r["bound"], round(r["achieved"]), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for g in r["groups"][:8]: print("   ", g["group"], round(g["achieved"]), g["unit"], round(g["frac"],3), round(g["busy_ms_per_step"],3))
PY
done
