#!/bin/bash
# 192-column GEMM tiles + the wave-quantised tiling choice: GEMM parity, microbench of the
# dsv2s / c3 / c4 shapes (automatic choice vs each forced tiling), dsv2s / c4 / c3 bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-bn192}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -k "gemm" > $O/pytest_gemm.log 2>&1; echo "gemm tests rc=$?"; tail -3 $O/pytest_gemm.log
timeout 900 python tools/gemm_microbench.py dsv2s c3_ c4_ > $O/micro.jsonl 2> $O/micro.err; echo "micro rc=$?"; cat $O/micro.jsonl | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
by={}
for r in rows: by.setdefault(r['shape'], []).append(r)
for k, v in by.items():
    auto=[r for r in v if r['bn']==0][0]['us_per_launch']; best=min(v[1:], key=lambda r: r['us_per_launch'])
    print(f\"{k:18s} auto {auto:8.2f} us  best {best['us_per_launch']:8.2f} (cg{best['cg']} bn{best['bn']})  \" + ' '.join(f\"{r['cg']}/{r['bn']}:{r['us_per_launch']:.1f}\" for r in v[1:]))
"
for c in dsv2s c4 c3 dsv2s; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --profile-json $O/prof_$c.json > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open("$O/bench_$c.json") if l.startswith("{")][-1]
r=d["roofline"]; print("$c", round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), r["kernel"], r["bound"], round(r["achieved"]), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
