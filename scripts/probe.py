"""Quick device timing probe of the local multiply (dev tool, not the bench)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2603_21444_b200 as spg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
d = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
t0 = time.time()
a = spg.gen_erdos_renyi(n, d / n, 1)
print(f"gen {time.time()-t0:.2f}s nnz={a.nnz}", flush=True)
dev = spg.Device(0)
da = dev.upload(a)
prods = dev.products(da, da)
print("products", prods, flush=True)
dev.timing(True)
for it in range(4):
    dev.timing_reset()
    t0 = time.time()
    c = dev.spgemm(da, da)
    dev.synchronize()
    wall = time.time() - t0
    tm = dev.timing_read()
    tot = sum(v[1] for v in tm.values())
    print(f"iter {it}: wall {wall*1e3:.2f} ms, kernels {tot:.2f} ms, nnzC={c.nnz}, GFLOP/s(wall)={2*prods/wall/1e9:.1f}",
          {k: round(v[1], 3) for k, v in tm.items()}, flush=True)
    del c
