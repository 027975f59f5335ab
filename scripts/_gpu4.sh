timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python scripts/ktime.py 4194304 16 3 | head -3
for v in w1792m3 nt128w1024 w2560; do SPG_LIB_PATH=$PWD/var/$v/libspgb200.so timeout 120 python scripts/ktime.py 4194304 16 3 | head -3; done
