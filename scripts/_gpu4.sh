for v in minb2 nolb2 nolb3; do SPG_LIB_PATH=$PWD/var/$v/libspgb200.so timeout 120 python scripts/ktime.py 4194304 16 3; done
