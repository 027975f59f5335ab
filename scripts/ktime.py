"""Per-kernel CUDA-event times of C = A*A on ER(n, d) (dev tool).
usage: ktime.py [n] [d] [reps]; SPG_LIB_PATH selects a variant library."""
import os
import sys
import time
sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
d = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
a = spg.gen_erdos_renyi(n, d / n, 1)
dev = spg.Device(0)
da = dev.upload(a)
prods = dev.products(da, da)
dev.timing(True)
for _ in range(2):
    c = dev.spgemm(da, da)
    del c
dev.synchronize()
dev.timing_reset()
t0 = time.perf_counter()
for _ in range(reps):
    c = dev.spgemm(da, da)
    nnz = c.nnz
    del c
dev.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
kt = dev.timing_read()
tag = os.environ.get("SPG_LIB_PATH", "default")
print(f"[{tag}] n={n} d={d} products={prods} nnzC={nnz} wall/step={wall:.3f} ms "
      f"GFLOP/s={2*prods/wall/1e6:.1f}")
for k, (cnt, ms) in sorted(kt.items()):
    print(f"   {k:22s} {ms/max(cnt,1):8.3f} ms")

# phase profile of the tile kernel when the library was built with -DSPG_TILE_PROF
try:
    import ctypes as C
    from paper_2603_21444_b200 import _capi
    L = _capi.lib()
    f = L.spg_dev_tile_prof
    buf = (C.c_ulonglong * 16)()
    f(buf)  # reset after the timed loop; run one more multiply and read
    c = dev.spgemm(da, da)
    dev.synchronize()
    f(buf)
    names = ["loop-top->process", "process(rest)", "publish+sync", "prologue(rest)", "gather-issue", "look-back",
             "crp+copy-out", "final sync", "p:mul+count(wait data)", "p:count barrier", "p:scan", "p:place",
             "p:place barrier", "p:pairs+lists", "p:or-barrier", "pro:loads(RT2)"]
    tot = sum(buf[i] for i in range(16)) or 1
    print("   tile phases (thread 0 of every CTA, % of CTA time):")
    for i, nm in enumerate(names):
        print(f"      {nm:24s} {100 * buf[i] / tot:5.1f}%")
except AttributeError:
    pass
