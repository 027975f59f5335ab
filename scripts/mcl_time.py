"""Kernel timers of the device MCL post-step at config-4 size (C = M*M, M =
column_normalize(ER 2^21, 16/row)): fused spg_mcl_poststep vs the unfused
device steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21444_b200 as spg  # noqa: E402


def main():
    dev = spg.Device(0)
    m = spg.gen_erdos_renyi(1 << 21, 16.0 / (1 << 21), 1)
    dm = dev.upload(m)
    dev.column_normalize(dm)
    c = dev.spgemm(dm, dm)
    dev.synchronize()
    dev.timing(True)
    for rep in range(3):
        dev.timing_reset()
        t0 = time.perf_counter()
        s = dev.mcl_poststep(c, 0.002, 2.0)
        dev.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(f"fused rep {rep}: wall {wall:.2f} ms nnz {s.nnz}",
              {k: (v[0], round(v[1], 3)) for k, v in dev.timing_read().items()})
        del s
    for rep in range(2):
        dev.timing_reset()
        t0 = time.perf_counter()
        x = dev.copy(c)
        dev.column_normalize(x)
        p = dev.prune(x, 0.002)
        dev.elementwise_power(p, 2.0)
        dev.column_normalize(p)
        dev.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(f"unfused rep {rep}: wall {wall:.2f} ms",
              {k: (v[0], round(v[1], 3)) for k, v in dev.timing_read().items()})
        del x, p


if __name__ == "__main__":
    main()
