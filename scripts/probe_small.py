"""One spgemm on ER(n, d) for profiling (dev tool)."""
import sys
sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
d = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
a = spg.gen_erdos_renyi(n, d / n, 1)
dev = spg.Device(0)
da = dev.upload(a)
for _ in range(reps):
    c = dev.spgemm(da, da)
    dev.synchronize()
    print("nnzC", c.nnz)
    del c
