#!/bin/bash
# GEMM change check: GEMM parity tests, microbench (auto vs forced vs cuBLAS), the full GPU
# suite, and the dsv2s / c4 / c3 bench lines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-gemmround}; mkdir -p $O
SHAPES="${SHAPES:-dsv2s c4_ c3_}" TAG=$TAG bash tools/r02/gpu_micro.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for c in ${CONFIGS:-dsv2s c4 c3 dsv2s}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --profile-json $O/prof_$c.json > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$c.json") if l.startswith("{")][-1]
r=d["roofline"]; print("$c", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), r["kernel"], r["bound"], round(r["achieved"]), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
