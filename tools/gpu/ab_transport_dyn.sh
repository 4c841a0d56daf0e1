#!/bin/bash
# dynamic item schedule A/B for the transport RHS (config 5): this tree
# against a baseline tree built under build/base (git archive of the previous
# commit), on `ngpu` GPUs (1: evaluate_transport_rhs; > 1: SlabTransport)
ngpu=${1:-1}
out=gpurun_out/ab_transport_dyn_n$ngpu.log
rm -f $out
run() {
  if [ "$ngpu" = 1 ]; then timeout 300 python tools/bench_transport.py --grid $1 --reps 5
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ngpu \
       --master-addr 127.0.0.1 --master-port 29541 tools/bench_transport.py --grid $1 --reps 5
  fi
}
grids="512 1024"
[ "$ngpu" != 1 ] && grids="1024"
for g in $grids; do
  for rep in 1 2; do
    for d in build/base .; do
      echo "== $g $d" >> $out
      (cd $d && run $g 2>&1 | grep '^{') >> $out
    done
  done
done
