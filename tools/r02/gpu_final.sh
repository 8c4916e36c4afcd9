#!/bin/bash
# Final one-GPU pass: smoke, the full GPU suite, the default bench (as the driver runs it:
# dsv2s, CPU baseline included), the reference arm, c4 / c3 / c2 lines, then the ncu launch
# list of the default bench command (after that command exited 0 without ncu).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-final}; mkdir -p $O
mkdir -p $O; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench reference rc=$?"; tail -1 $O/bench_reference.json | cut -c1-400
for c in c4 c3 c2 dsv2s; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --profile-json $O/prof_$c.json > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?"
done
python - <<PY
import json
for f in ["default", "c4", "c3", "c2", "dsv2s"]:
    d=[json.loads(l) for l in open("$O/bench_%s.json" % f) if l.startswith("{")][-1]
    r=d["roofline"]; cb=d.get("cpu_baseline") or {}
    print(f, d["config"]["workload"][:12], round(d["ms_per_step"],3), "ms", round(d["value"]), "tok/s e2e", round(d["e2e"]["value"]), r["kernel"], round(r["achieved"]), r["unit"], round(r["frac"],3), "traffic", r.get("traffic"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "cpu", cb.get("value"), cb.get("cores"), "launches", d.get("gpu_launches"))
PY
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --trace-iters 0"
timeout 600 $CMD > $O/ncu_plain.log 2>&1 && \
timeout 1500 ncu --clock-control none -c 400 --csv -k regex:"gemm_tc|attn_|gate_|permute|combine|gather|colsum|a2a_|route_scan" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__cycles_elapsed.avg.per_second \
  --log-file $O/launches_dsv2s.csv $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $O/ncu.log
