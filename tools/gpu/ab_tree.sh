#!/bin/bash
# A/B of this tree against build/base (the previous commit, built there) with
# bench.py on `ngpu` GPUs at `size` (512 on 4 GPUs = the m = 128 block of
# 1024^3 on 8), alternating trees
ngpu=$1; size=$2; reps=${3:-2}
out=gpurun_out/ab_tree_n${ngpu}_s$size.log
rm -f $out
for rep in $(seq 1 $reps); do
  for d in build/base .; do
    echo "== $d" >> $out
    (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ngpu \
        --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus $ngpu --size $size \
        --steps 300 --warmup 5 --no-t1 --no-transport --e2e-steps 1 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['partition'][:2], d['clocks'])") >> $out
  done
done
