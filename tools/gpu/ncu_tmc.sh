# ncu --set full of k_tmc (n=2048) and the production k_tma (n=512), one launch each
set -x
python tools/sweep_n.py 2048 4096 8192 --iters 100 2>&1 | tail -3
ncu --set full --clock-control none --import-source on -k regex:k_tmc -s 3 -c 1 -o gpurun_out/k_tmc_n2048 python tools/sweep_n.py 2048 --iters 5 > gpurun_out/ncu_tmc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 3 -c 1 -o gpurun_out/k_tma_n512 python tools/sweep_n.py 512 --iters 5 > gpurun_out/ncu_tma.log 2>&1
tail -3 gpurun_out/ncu_tmc.log gpurun_out/ncu_tma.log
