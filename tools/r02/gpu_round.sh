#!/bin/bash
# Round-2 GPU pass: smoke, the GPU suite, dsv2s bench (default lanes and one lane), c4, c2.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-round}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
if [ -z "$NOTESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
fi
for spec in "dsv2s:" "dsv2s:--compute-streams 1" "c4:" "c2:"; do
  c=${spec%%:*}; extra=${spec#*:}; tag=$c$(echo $extra | tr -d ' -')
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline $extra \
    --profile-json $O/prof_$tag.json --trace-dir $O > $O/bench_$tag.json 2> $O/bench_$tag.err
  echo "bench $tag rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$tag.json") if l.startswith("{")][-1]
r=d["roofline"]; print("$tag", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), r["kernel"], r["bound"], round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
