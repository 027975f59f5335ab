for v in n512w3072 n512w4096 n256w2560; do SPG_LIB_PATH=$PWD/var/$v/libspgb200.so timeout 120 python scripts/ktime.py 4194304 16 3; done
