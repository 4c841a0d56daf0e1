# ncu --set full of the fused per-rank kernel in loopback (m=512, 1 GPU)
ncu --set full --clock-control none --import-source on -k regex:k_dd -s 2 -c 1 -o gpurun_out/k_dd2_m512_loop python tools/dd_loopback.py --m 512 --iters 3 > gpurun_out/ncu_dd.log 2>&1
tail -2 gpurun_out/ncu_dd.log
