"""k_tile phase profile on R-MAT (dev tool): a library built with
-DSPG_TILE_PROF (scripts/build_variant.sh tprof -DSPG_TILE_PROF) via
SPG_LIB_PATH=var/tprof/libspgb200.so. usage: tprof_rmat.py [scale]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402
from paper_2603_21444_b200 import _capi  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 18
a = spg.gen_rmat(s, 16, 1, 2) if s > 0 else spg.gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1)
dev = spg.Device(0)
da = dev.upload(a)
c = dev.spgemm(da, da)
del c
dev.synchronize()
f = _capi.lib().spg_dev_tile_prof
buf = (C.c_ulonglong * 16)()
f(buf)
c = dev.spgemm(da, da)
dev.synchronize()
f(buf)
names = ["loop-top", "process(rest)", "publish+sync", "prologue(rest)", "gather-issue", "look-back", "crp+copy-out",
         "final sync", "p:mul+count", "p:count barrier", "p:scan", "p:place", "p:place barrier", "p:pairs+lists",
         "p:or-barrier", "pro:loads"]
tot = sum(buf[i] for i in range(16)) or 1
print(f"scale {s}: thread-0 cycles {tot}")
for i, nm in enumerate(names):
    print(f"      {nm:20s} {100 * buf[i] / tot:5.1f}%")
