#!/bin/bash
# A/B of the fused per-rank kernels over NVLink (bench.py at N GPUs, 1024^3)
# usage: tools/gpu/ab_dd4.sh N "ENV=.. ENV2=.." ["..."]
N=$1; shift
out=gpurun_out/ab_dd$N.log
rm -f $out
for v in "$@"; do
  echo "== $v" >> $out
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 200 --warmup 5 \
      --no-t1 --e2e-steps 1 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks'])" >> $out
done
