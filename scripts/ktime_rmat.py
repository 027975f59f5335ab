"""Per-kernel times of C = A*A on R-MAT(scale) (dev tool).
usage: ktime_rmat.py SCALE [ROW0 ROW1]  (a row range of A times A: scale 22 does not fit whole)"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2603_21444_b200 as spg  # noqa: E402
sys.path.insert(0, "scripts")
from configs import row_products  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 16
a = spg.gen_rmat(s, 16, 1, 2)
rp = row_products(a, a)
ne = np.diff(np.asarray(a.rowptr))
print(f"scale {s}: n={a.nrows} nnz={a.nnz} products={rp.sum()} rows>512: {(rp > 512).sum()} >4096: {(rp > 4096).sum()}"
      f" prod in >4096: {rp[rp > 4096].sum()} in 513..4096: {rp[(rp > 512) & (rp <= 4096)].sum()} max ne {ne.max()}")
dev = spg.Device(0)
da = dev.upload(a)
dl = da
if len(sys.argv) > 3:
    r0, r1 = int(sys.argv[2]), int(sys.argv[3])
    dl = dev.extract(da, r0, r1, 0, int(a.ncols))
    print(f"rows {r0}..{r1}: products {rp[r0:r1].sum()}")
dev.timing(True)
c = dev.spgemm(dl, da)
dev.synchronize()
dev.timing_reset()
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    del c
    c = dev.spgemm(dl, da)
    dev.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0) / reps:.1f} ms/step nnzC={c.nnz}")
for k, (n, ms) in sorted(dev.timing_read().items()):
    print(f"   {k:20s} {ms / reps:10.3f} ms/step ({n // reps} launches)")
