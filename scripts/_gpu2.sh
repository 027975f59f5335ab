timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python scripts/ktime.py
SPG_LIB_PATH=$PWD/var/nb0/libspgb200.so python scripts/ktime.py
SPG_LIB_PATH=$PWD/var/m16_2/libspgb200.so python scripts/ktime.py
