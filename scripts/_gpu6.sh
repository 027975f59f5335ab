SPG_LIB_PATH=$PWD/var/prof/libspgb200.so timeout 120 python scripts/ktime.py 4194304 16 2
