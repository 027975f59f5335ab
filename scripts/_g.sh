python scripts/ktime.py 4194304 16 3 | head -3
SPG_LIB_PATH=var/nolb/libspgb200.so python scripts/ktime.py 4194304 16 3 | head -3
