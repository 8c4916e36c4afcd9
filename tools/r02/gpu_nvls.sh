#!/bin/bash
# Is NVLink SHARP (NVLS) available to NCCL on this box, and what does it do to the AR?
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/${TAG:-nvls}_n$N; mkdir -p $O
nvidia-smi -q | grep -i -A3 "fabric" | head -20 > $O/fabric.txt
for alg in default NVLS; do
  if [ $alg = default ]; then E=""; else E="NCCL_ALGO=allreduce:NVLS"; fi
  env $E NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,NVLS timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29770 tools/r02/busbw.py > $O/busbw_$alg.jsonl 2> $O/busbw_$alg.err
  echo "busbw $alg rc=$?"; grep -i "nvls" $O/busbw_$alg.err | sort | uniq -c | sort -rn | head -8
  grep allreduce $O/busbw_$alg.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('  ', d.get('op'), round(d.get('bytes',0)/2**20), 'MiB', round(d.get('us',0),1), 'us', round(d.get('busbw_gbs',0)), 'GB/s')
"
done
cat $O/fabric.txt
