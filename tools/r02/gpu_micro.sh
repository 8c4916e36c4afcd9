#!/bin/bash
# GEMM microbench (automatic tiling vs each forced tiling vs cuBLAS through torch.bmm) on
# the shape prefixes in $SHAPES.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-micro}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -k "gemm" -x > $O/pytest_gemm.log 2>&1; echo "gemm tests rc=$?"; tail -2 $O/pytest_gemm.log
timeout 1200 python tools/gemm_microbench.py ${SHAPES:-dsv2s} > $O/micro.jsonl 2> $O/micro.err; echo "micro rc=$?"; tail -3 $O/micro.err; cat $O/micro.jsonl | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
by={}
for r in rows: by.setdefault(r['shape'], []).append(r)
for k, v in by.items():
    ours=[r for r in v if 'impl' not in r]; cb=[r for r in v if 'impl' in r]
    auto=[r for r in ours if r['bn']==0][0]['us_per_launch']; best=min(ours[1:], key=lambda r: r['us_per_launch'])
    print(f\"{k:18s} auto {auto:8.2f} us  best {best['us_per_launch']:8.2f} (cg{best['cg']} bn{best['bn']} sk{best.get('sk',0)})  cublas {cb[0]['us_per_launch'] if cb else float('nan'):8.2f}  \" + ' '.join(f\"{r['cg']}/{r['bn']}{'sk' if r.get('sk')==2 else ''}:{r['us_per_launch']:.1f}\" for r in ours[1:]))
"
