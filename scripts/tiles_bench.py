import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""Device tile store timing (spg_partition / spg_reassemble) at config-2 size:
ER n=2^22, 16/row. Partition A into the trident tiles of (P, lambda) on the
GPUs of the box (tile r on device r % ndev), multiply-free; then reassemble.
Prints ms and effective GB/s (bytes read + written)."""
import sys
import time

import numpy as np

import paper_2603_21444_b200 as spg


def main():
    P, lam = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 2)
    a = spg.gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1)
    devs = [spg.default_device(d) for d in range(spg.Device.count())]
    d0 = devs[0]
    da = d0.upload(a)
    csr_bytes = lambda rows, nnz: (rows + 1) * 8 + nnz * 12  # noqa: E731
    for rep in range(4):
        for d in devs:
            d.synchronize()
        t0 = time.perf_counter()
        tiles, tm = d0.partition(da, "trident", P, lam, devices=devs)
        for d in devs:
            d.synchronize()
        t1 = time.perf_counter()
        back = d0.reassemble(tiles, tm)
        d0.synchronize()
        t2 = time.perf_counter()
        moved = csr_bytes(a.nrows, a.nnz) + sum(csr_bytes(t.shape3[0], t.nnz) for t in tiles)
        print(f"P={P} lam={lam} ndev={len(devs)} partition {1e3 * (t1 - t0):.2f} ms ({moved / (t1 - t0) / 1e9:.0f} GB/s)"
              f"  reassemble {1e3 * (t2 - t1):.2f} ms ({moved / (t2 - t1) / 1e9:.0f} GB/s)")
        if rep == 3:
            b = back.download()
            print("roundtrip bit-exact:", np.array_equal(b.rowptr, a.rowptr) and np.array_equal(b.colind, a.colind)
                  and np.array_equal(b.values, a.values))
        del tiles, back
    d0.timing(True)
    for rep in range(2):  # second pass: allocations warm
        d0.timing_reset()
        tiles, tm = d0.partition(da, "trident", P, lam, devices=[d0])
        back = d0.reassemble(tiles, tm)
        del tiles, back
    print("one device, kernel ms (warm):", {k: round(v[1], 3) for k, v in d0.timing_read().items()})


if __name__ == "__main__":
    main()
