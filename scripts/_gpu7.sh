python scripts/diag_norm.py
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python scripts/ktime.py 4194304 16 3 | head -6
python scripts/ktime_rmat.py 18
