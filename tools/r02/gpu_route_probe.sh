#!/bin/bash
# Routing-kernel microbenchmarks at the dsv2s / c4 / c3 / c2 chunk shapes, then one ncu
# --set full capture of the gather and gate kernels at the dsv2s shape.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-route}; mkdir -p $O
for shape in "512 5120 16 8 1.0 2" "1024 4096 16 2 1.0 2" "1024 1024 16 2 1.0 2" "256 256 8 2 1.0 4"; do
  timeout 120 build/route_probe $shape
done > $O/probe.txt 2>&1; echo "probe rc=$?"; cat $O/probe.txt
if [ -n "$NCU" ]; then
timeout 120 build/route_probe 512 5120 16 8 1.0 2 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 10 -c 3 -o $O/route_ncu build/route_probe 512 5120 16 8 1.0 2 > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $O/ncu.log
fi
