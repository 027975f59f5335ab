"""One small C = A*A through the product path for compute-sanitizer runs
(dev tool): config 1 (ER 16384, 8/row) or R-MAT scale 11 (skewed rows, BIG-row
side path). Checks the result against the oracle; exits non-zero on mismatch.
usage: sanitize_case.py er|rmat"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2603_21444_b200 as spg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "er"
a = spg.gen_erdos_renyi(16384, 8.0 / 16384, 1) if which == "er" else spg.gen_rmat(11, 16, 1, 2)
dev = spg.Device(0)
da = dev.upload(a)
c = dev.spgemm(da, da).download()
ref = O.port_spgemm(a, a)
ok = (np.array_equal(c.rowptr, ref.rowptr) and np.array_equal(c.colind, ref.colind)
      and np.array_equal(c.values, ref.values))
print(f"{which}: nnz(C)={c.nnz} parity={'bit-exact' if ok else 'MISMATCH'}")
sys.exit(0 if ok else 1)
