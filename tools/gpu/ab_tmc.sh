set -x
python tools/sweep_n.py 2048 4096 8192 --iters 100 2>&1 | tail -3
for tl in 32 16 8; do for q in 2 4 8 16; do python tools/sweep_n.py 2048 4096 8192 --iters 60 TDS_TMC_TL=$tl TDS_TMC_Q=$q 2>&1 | grep -v staged | sed "s/^/tl=$tl q=$q /"; done; done
python -m pytest tests/test_gpu_parity.py -q -x -k "long_lines" 2>&1 | tail -2
