"""k_merge phase profile (dev tool): run with a library built with
-DSPG_MERGE_PROF (scripts/build_variant.sh mprof -DSPG_MERGE_PROF) via
SPG_LIB_PATH=var/mprof/libspgb200.so. usage: mprof.py [n] [d]"""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402
from paper_2603_21444_b200 import _capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
d = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
a = spg.gen_erdos_renyi(n, d / n, 1)
dev = spg.Device(0)
da = dev.upload(a)
dev.timing(True)
c = dev.spgemm(da, da)
del c
dev.synchronize()
f = _capi.lib().spg_dev_merge_prof
buf = (C.c_ulonglong * 28)()
f(buf)
dev.timing_reset()
t0 = time.perf_counter()
c = dev.spgemm(da, da)
dev.synchronize()
print(f"n={n} d={d} nnzC={c.nnz} wall={1e3 * (time.perf_counter() - t0):.2f} ms")
for k, (cnt, ms) in sorted(dev.timing_read().items()):
    print(f"   {k:22s} {ms / max(cnt, 1):8.3f} ms")
f(buf)
names = ["c:wait-next", "c:pre", "c:cp-wait", "c:sort", "c:tiles", "s:wait-freed", "s:stage", "s:tiles",
         "e:wait-ready+done", "e:look-back", "e:rest", "e:tiles"]
for i, nm in enumerate(names):
    print(f"   {nm:20s} {buf[i]:16d}")
print(f"   lb:windows {buf[24]}  sum n {buf[25]}  overflow products: total {buf[26]} max n {buf[27]}")
rows0 = buf[4] or 1
print(f"   compute per tile (cycles, summed over compute warps / tiles): pre={buf[1] / rows0:.0f} "
      f"gather-issue={buf[13] / rows0:.0f} cp-wait={buf[2] / rows0:.0f} sort={buf[3] / rows0:.0f} "
      f"wait-next={buf[0] / rows0:.0f}")
sp = [buf[16 + i] for i in range(6)]
rows = buf[4] or 1
print("   sort phases (cycles/tile-warp): " + " ".join(f"{nm}={v / rows:.0f}" for nm, v in
                                               zip(["P1", "P2+P3", "P5", "compact-count", "compact-write", "P4"], sp)))
w = sum(buf[i] for i in (0, 1, 2, 3)) or 1
print("   worker split: " + " ".join(f"{names[i]}={100 * buf[i] / w:.1f}%" for i in (0, 1, 2, 3)))
e = sum(buf[i] for i in (8, 9, 10)) or 1
print("   epilogue split: " + " ".join(f"{names[i]}={100 * buf[i] / e:.1f}%" for i in (8, 9, 10)))
s = sum(buf[i] for i in (5, 6)) or 1
print("   setup split: " + " ".join(f"{names[i]}={100 * buf[i] / s:.1f}%" for i in (5, 6)))
