"""Per-kernel times of config 5 (k-mer A*A^T), or config 2 with argument `er`, or
`rand`: config 5's shapes with a random B (2^18 x 2^22, 64/row: long B rows like
A^T's, but no structural duplicates) (dev tool)."""
import sys
import time
sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "er":  # config 2 instead
    a = spg.gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1)
    at = a
elif len(sys.argv) > 1 and sys.argv[1] == "rand":
    a = spg.gen_erdos_renyi_rect(1 << 22, 1 << 18, 2.0 ** -16, 5)
    at = spg.gen_erdos_renyi_rect(1 << 18, 1 << 22, 2.0 ** -16, 6)
else:
    a = spg.gen_erdos_renyi_rect(1 << 22, 1 << 18, 2.0 ** -16, 5)
    at = spg.transpose(a)
dev = spg.Device(0)
da, db = dev.upload(a), dev.upload(at)
dev.timing(True)
for _ in range(2):
    c = dev.spgemm(da, db)
    del c
dev.synchronize()
dev.timing_reset()
t0 = time.perf_counter()
for _ in range(3):
    c = dev.spgemm(da, db)
    nnz = c.nnz
    del c
dev.synchronize()
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'config5'} wall/step {1e3 * (time.perf_counter() - t0) / 3:.2f} ms nnz {nnz}")
for k, (n, ms) in sorted(dev.timing_read().items()):
    print(f"   {k:20s} {ms / max(n, 1):10.3f} ms x{n}")

try:  # phase profile when built with -DSPG_TILE_PROF
    import ctypes as C
    from paper_2603_21444_b200 import _capi
    f = _capi.lib().spg_dev_tile_prof
    buf = (C.c_ulonglong * 16)()
    f(buf)
    c = dev.spgemm(da, db)
    dev.synchronize()
    f(buf)
    names = ["loop-top", "process(rest)", "publish+sync", "prologue(rest)", "gather-issue", "look-back",
             "crp+copy-out", "final sync", "p:mul+count", "p:count barrier", "p:scan", "p:place",
             "p:place barrier", "p:pairs+lists", "p:or-barrier", "pro:loads"]
    tot = sum(buf[i] for i in range(16)) or 1
    for i, nm in enumerate(names):
        print(f"      {nm:20s} {100 * buf[i] / tot:5.1f}%")
except AttributeError:
    pass
