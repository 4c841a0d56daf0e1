# ncu --set full: k_tma on open d/dx vs open d2/dx2 (512^3-sized x solve)
ncu --set full --clock-control none -k regex:k_tma -s 3 -c 1 -o gpurun_out/k_tma_open_d1 python tools/sweep_n.py 512 --open --iters 5 > gpurun_out/ncu_o1.log 2>&1
ncu --set full --clock-control none -k regex:k_tma -s 3 -c 1 -o gpurun_out/k_tma_open_d2 python tools/sweep_n.py 512 --open --op d2 --iters 5 > gpurun_out/ncu_o2.log 2>&1
python tools/sweep_n.py 512 --op d2 --iters 100 | tail -1
