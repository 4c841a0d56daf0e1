set -x
python tools/sweep_n.py 512 1024 --iters 200 2>&1 | tail -2
python tools/sweep_n.py 512 1024 --iters 200 TDS_BULK_ST=1 2>&1 | tail -2
python tools/sweep_n.py 512 1024 --iters 200 2>&1 | tail -2
python tools/sweep_n.py 512 1024 --iters 200 TDS_BULK_ST=1 2>&1 | tail -2
python tools/sweep_n.py 512 --open --iters 200 TDS_BULK_ST=1 2>&1 | tail -1
python tools/sweep_n.py 512 --open --iters 200 2>&1 | tail -1
TDS_BULK_ST=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
