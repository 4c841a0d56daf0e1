#!/bin/bash
# the m = 128 per-rank block of BASELINE config 3 at N = 8, reached with 512^3
# on 4 GPUs (bench.py --size 512): per-rank kernel A/B
out=gpurun_out/ab_m128.log
rm -f $out
for v in "$@"; do
  echo "== $v" >> $out
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --size 512 --steps 300 \
      --warmup 5 --no-t1 --no-transport --e2e-steps 1 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['partition'], d['clocks'])" >> $out
done
