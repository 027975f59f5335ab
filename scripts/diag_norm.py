import sys, time
sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg
n = 1 << 21
m = spg.gen_erdos_renyi(n, 16.0 / n, 1)
dev = spg.Device(0)
dm = dev.upload(m)
dev.column_normalize(dm)
c = dev.spgemm(dm, dm)
dev.synchronize()
dev.timing(True)
for it in range(3):
    dev.timing_reset()
    cc = dev.copy(c)
    dev.synchronize()
    t0 = time.perf_counter()
    dev.column_normalize(cc)
    dev.synchronize()
    t1 = time.perf_counter()
    p = dev.prune(cc, 0.002)
    dev.synchronize()
    t2 = time.perf_counter()
    print(f"normalize {1e3*(t1-t0):.2f} ms prune {1e3*(t2-t1):.2f} ms nnz {p.nnz}", dev.timing_read())
    del cc, p
