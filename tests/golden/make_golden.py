"""Generates the golden fixtures in tests/golden/ by running the REFERENCE
itself (oracle/_ref/libspgref.so, built from /root/reference/proj sources by
oracle/Makefile). Run in the build container:  python tests/golden/make_golden.py [small|configs|all]

small   : the reference's own known-answer cases (test_csr.cpp:24-109,182-200)
          plus small random products, spgeam, vconcat, partition tiles and
          trident/SUMMA ledgers  -> small.npz  (full arrays)
mcl4    : adds one MCL post-step digest of config 4 to config4.json
configs : digests of the benchmark configs' C = A*B (nnz, sha256 of rowptr /
          colind / values, sampled rows) -> config<k>.json
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def csr_arrays(prefix, m, out):
    out[prefix + "_shape"] = np.array([m.nrows, m.ncols], np.int64)
    out[prefix + "_rowptr"] = np.asarray(m.rowptr, np.int64)
    out[prefix + "_colind"] = np.asarray(m.colind, np.int64)
    out[prefix + "_values"] = np.asarray(m.values, np.float64)


def mat2x2(a00, a01, a10, a11):
    t = [(0, 0, a00), (0, 1, a01), (1, 0, a10), (1, 1, a11)]
    t = [x for x in t if x[2] != 0]
    return O.ref_from_triplets(2, 2, [x[0] for x in t], [x[1] for x in t], [x[2] for x in t])


def crop_cols(m, nc):
    rp = [0]
    ci, va = [], []
    for i in range(m.nrows):
        for t in range(m.rowptr[i], m.rowptr[i + 1]):
            if m.colind[t] < nc:
                ci.append(m.colind[t])
                va.append(m.values[t])
        rp.append(len(ci))
    return O.Csr(m.nrows, nc, np.array(rp, np.int64), np.array(ci, np.int64), np.array(va))


def small():
    out = {}
    cases = []
    # test_csr.cpp:24-34
    a = O.ref_gen_erdos_renyi(3, 0.7, 11)
    cases.append(("identity3", O.ref_identity(3), a))
    cases.append(("frozen2x2", mat2x2(1, 0, 0, 2), mat2x2(0, 3, 4, 0)))
    # :36-41 empty row
    cases.append(("emptyrow", O.ref_from_triplets(3, 3, [0, 2], [1, 0], [2.0, 1.0]), O.ref_gen_erdos_renyi(3, 1.0, 5)))
    # :48-72 dense-oracle ER and rectangular crop
    for s in (1, 2, 3):
        cases.append((f"er40_s{s}", O.ref_gen_erdos_renyi(40, 0.15, s), O.ref_gen_erdos_renyi(40, 0.15, s + 100)))
    cases.append(("rect24x17", O.ref_gen_erdos_renyi(24, 0.2, 9), crop_cols(O.ref_gen_erdos_renyi(24, 0.2, 10), 17)))
    # :74-81 explicit zero from cancellation
    cases.append(("cancel", O.ref_from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0]),
                  O.ref_from_triplets(2, 1, [0, 1], [0, 0], [1.0, -1.0])))
    # larger random / skewed products
    cases.append(("er1024_s3", O.ref_gen_erdos_renyi(1024, 0.004, 3), O.ref_gen_erdos_renyi(1024, 0.004, 4)))
    cases.append(("dense20", O.ref_gen_erdos_renyi(20, 1.0, 4), O.ref_gen_erdos_renyi(20, 1.0, 5)))
    cases.append(("er300_p3", O.ref_gen_erdos_renyi(300, 0.03, 3), O.ref_gen_erdos_renyi(300, 0.03, 4)))
    names = []
    for name, a, b in cases:
        c = O.ref_spgemm_local(a, b)
        csr_arrays(f"{name}_A", a, out)
        csr_arrays(f"{name}_B", b, out)
        csr_arrays(f"{name}_C", c, out)
        names.append(name)
    out["spgemm_cases"] = np.array(names)
    # spgeam (test_csr.cpp:83-109)
    x, y = O.ref_gen_erdos_renyi(30, 0.2, 1), O.ref_gen_erdos_renyi(30, 0.2, 2)
    csr_arrays("geam_X", x, out)
    csr_arrays("geam_Y", y, out)
    csr_arrays("geam_Z", O.ref_spgeam(x, y), out)
    f = O.ref_spgeam(mat2x2(1, 0, 0, 1), mat2x2(0, 2, 0, 1))
    csr_arrays("geam_frozen", f, out)
    # vconcat (test_csr.cpp:182-200)
    v = O.ref_gen_erdos_renyi(17, 0.3, 8)
    csr_arrays("vcat_A", v, out)
    # distributed drivers on ER(300) and rectangular A*A^T: C and ledgers
    a, b = O.ref_gen_erdos_renyi(300, 0.03, 3), O.ref_gen_erdos_renyi(300, 0.03, 4)
    grids = [(1, 1), (2, 2), (4, 1), (4, 4), (8, 2), (16, 4)]
    for P, lam in grids:
        r = O.ref_run_algo("trident", a, b, P, lam)
        out[f"trident_P{P}_L{lam}_ledger"] = r["ledger"]
        out[f"trident_P{P}_L{lam}_events"] = r["events"]
        out[f"trident_P{P}_L{lam}_Cvalues"] = r["c"].values
        tiles, rects = O.ref_partition(a, "trident", P, lam)
        out[f"part_P{P}_L{lam}_rects"] = rects
        out[f"part_P{P}_L{lam}_nnz"] = np.array([t.nnz for t in tiles], np.int64)
    for P in (1, 4):
        r = O.ref_run_algo("summa", a, b, P, 2)
        out[f"summa_P{P}_ledger"] = r["ledger"]
        out[f"summa_P{P}_Cvalues"] = r["c"].values
    out["grids"] = np.array(grids, np.int64)
    # Prop. 1 exactness case: uniform stride is in the reference,
    # generated here via triplets of the same rule
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz:", len(out), "arrays")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def digest(c, seconds, nsample=256):
    rng = np.random.default_rng(12345)
    rows = np.sort(rng.choice(c.nrows, size=min(nsample, c.nrows), replace=False)) if c.nrows else np.zeros(0, np.int64)
    samples = {}
    for i in rows:
        lo, hi = int(c.rowptr[i]), int(c.rowptr[i + 1])
        samples[int(i)] = {"cols": c.colind[lo:hi].tolist(), "vals": c.values[lo:hi].tolist()}
    return {"nrows": int(c.nrows), "ncols": int(c.ncols), "nnz": int(c.nnz),
            "sha_rowptr": sha(np.asarray(c.rowptr, np.int64)), "sha_colind": sha(np.asarray(c.colind, np.int64)),
            "sha_values": sha(np.asarray(c.values, np.float64)), "ref_seconds_1core": seconds,
            "sample_rows": samples}


def config(k):
    t0 = time.time()
    if k == 1:
        a = O.ref_gen_erdos_renyi(16384, 8.0 / 16384, 1, handle=True)
        b = a
        desc = "gen_erdos_renyi(16384, 8/16384, 1); C=A*A"
    elif k == 2:
        a = O.ref_gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1, handle=True)
        b = a
        desc = "gen_erdos_renyi(2^22, 2^-18, 1); C=A*A"
    elif k == 4:
        m = O.ref_gen_erdos_renyi(1 << 21, 16.0 / (1 << 21), 1, handle=True)
        a = O.ref_column_normalize(m, handle=True)
        b = a
        desc = "M=column_normalize(gen_erdos_renyi(2^21, 16/2^21, 1)); C=M*M"
    elif k == 5:
        r = O.port_gen_erdos_renyi_rect(1 << 22, 1 << 18, 2.0 ** -16, 5)
        import paper_2603_21444_b200 as spg  # host transpose only (no device)
        rt = spg.transpose(r)
        a, b = O.RefHandle.from_csr(r), O.RefHandle.from_csr(rt)
        desc = "A=ER_rect(2^22 x 2^18, 2^-16, seed 5) (oracle_gen_erdos_renyi_rect); C=A*A^T"
    gen_s = time.time() - t0
    secs, nnz, c = O.ref_spgemm_local_timed(a, b, keep=True)
    d = digest(c, secs)
    d["desc"] = desc
    d["gen_seconds"] = gen_s
    d["products"] = int(O.port_products(a.to_csr(), b.to_csr()) if k != 2 else 1074038175)
    if k == 4:
        cn = O.ref_column_normalize(c, handle=True)
        p = O.ref_prune(cn, 0.002)
        d["pruned"] = {k2: v for k2, v in digest(p, 0.0, 64).items() if k2 != "ref_seconds_1core"}
    with open(os.path.join(HERE, f"config{k}.json"), "w") as f:
        json.dump(d, f)
    print(f"config{k}: nnz={d['nnz']} ref {secs:.1f}s")


def _views(h):
    """rowptr/colind/values of a reference matrix handle as numpy views (no copy)."""
    import ctypes as C
    L = O._R()
    nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
    L.ref_csr_info(h.ptr, C.byref(nr), C.byref(nc), C.byref(nz))
    nr, nc, nz = nr.value, nc.value, nz.value
    rp = np.ctypeslib.as_array(L.ref_csr_rowptr(h.ptr), shape=(nr + 1,))
    ci = np.ctypeslib.as_array(L.ref_csr_colind(h.ptr), shape=(nz,)) if nz else np.zeros(0, np.int64)
    va = np.ctypeslib.as_array(L.ref_csr_values(h.ptr), shape=(nz,)) if nz else np.zeros(0, np.float64)
    return nr, nc, nz, rp, ci, va


def config3():
    """Config 3 (R-MAT Graph500, edge factor 16, (a,b,c)=(0.57,0.19,0.19),
    SplitMix64 draw order of SURVEY.md §8(d), duplicates summed by
    from_triplets, symmetric random permutation): at scale 18 the digest of
    the full C = A*A from the reference's spgemm_local (csr.cpp:132-165); at
    scale 22 (full C ~7.2e10 entries: no host holds it) the reference rows of
    C for the heaviest row of A*A and 50 random rows with products, each
    computed as spgemm_local(A[rows, :], A) — exact, since a row of C depends
    only on its row of A."""
    import ctypes as C
    import paper_2603_21444_b200 as spg  # host generator (bit-identical to the reference's from_triplets rules)
    out = {}
    # ---- scale 18, full product
    t0 = time.time()
    a = spg.gen_rmat(18, 16, 1, 2)
    ha = O.RefHandle.from_csr(a)
    gen_s = time.time() - t0
    secs, nz, o = C.c_double(), C.c_int64(), C.c_void_p()
    O._chk(O._R().ref_spgemm_local_timed(ha.ptr, ha.ptr, C.byref(secs), C.byref(nz), C.byref(o)))
    hc = O.RefHandle(o.value)
    nr, nc, nnz, rp, ci, va = _views(hc)
    rng = np.random.default_rng(12345)
    rows = np.sort(rng.choice(nr, size=256, replace=False))
    samples = {int(i): {"cols": ci[rp[i]:rp[i + 1]].tolist(), "vals": va[rp[i]:rp[i + 1]].tolist()}
               for i in rows if rp[i + 1] - rp[i] <= 4096}
    out["s18"] = {"nrows": int(nr), "ncols": int(nc), "nnz": int(nnz), "nnz_A": int(a.nnz),
                  "products": int(O.port_products(a, a)), "sha_rowptr": sha(rp), "sha_colind": sha(ci),
                  "sha_values": sha(va), "ref_seconds_1core": secs.value, "gen_seconds": gen_s,
                  "sample_rows": samples,
                  "desc": "gen_rmat(18, 16, seed 1, perm seed 2); C = A*A; reference spgemm_local"}
    print(f"config3 s18: nnz(A)={a.nnz} nnz(C)={nnz} ref {secs.value:.1f}s")
    del hc, ha, a, ci, va, rp
    # ---- scale 22, sampled rows
    a = spg.gen_rmat(22, 16, 1, 2)
    _, prod = O.port_products(a, a, per_row=True)
    heavy = int(np.argmax(prod))
    rng = np.random.default_rng(22)
    cand = np.nonzero(prod > 0)[0]
    rows = np.unique(np.concatenate([[heavy], rng.choice(cand, size=50, replace=False)]))
    rp = np.asarray(a.rowptr)
    sub_rp = [0]
    sub_ci, sub_va = [], []
    for i in rows:
        sub_ci.append(np.asarray(a.colind[rp[i]:rp[i + 1]], np.int64))
        sub_va.append(np.asarray(a.values[rp[i]:rp[i + 1]], np.float64))
        sub_rp.append(sub_rp[-1] + rp[i + 1] - rp[i])
    sub = O.Csr(len(rows), a.ncols, np.array(sub_rp, np.int64), np.concatenate(sub_ci), np.concatenate(sub_va))
    t0 = time.time()
    cs = O.ref_spgemm_local(sub, a)
    secs22 = time.time() - t0
    srows = {}
    for t, i in enumerate(rows):
        lo, hi = int(cs.rowptr[t]), int(cs.rowptr[t + 1])
        cols, vals = np.asarray(cs.colind[lo:hi], np.int64), np.asarray(cs.values[lo:hi], np.float64)
        e = {"products": int(prod[i]), "nnz": hi - lo, "sha_cols": sha(cols), "sha_vals": sha(vals)}
        if hi - lo <= 4096:
            e["cols"], e["vals"] = cols.tolist(), vals.tolist()
        srows[int(i)] = e
    out["s22"] = {"nrows": int(a.nrows), "nnz_A": int(a.nnz), "products_total": int(prod.sum()),
                  "heaviest_row": heavy, "ref_seconds_rows": secs22, "rows": srows,
                  "desc": "gen_rmat(22, 16, seed 1, perm seed 2); rows of C = A*A by spgemm_local(A[rows,:], A)"}
    print(f"config3 s22: heaviest row {heavy} products {int(prod[heavy])} nnz {srows[heavy]['nnz']}; "
          f"{len(rows)} rows in {secs22:.1f}s")
    with open(os.path.join(HERE, "config3.json"), "w") as f:
        json.dump(out, f)


def mcl4():
    """Adds to config4.json the digest of one MCL post-step of config 4's
    product with the reference's own functions (apps.cpp:79-82: normalize,
    prune 0.002, elementwise_power 2, normalize)."""
    m = O.ref_gen_erdos_renyi(1 << 21, 16.0 / (1 << 21), 1, handle=True)
    a = O.ref_column_normalize(m, handle=True)
    _, _, c = O.ref_spgemm_local_timed(a, a, keep=True)
    t0 = time.time()
    s = O.ref_mcl_poststep(c, 0.002, 2.0)
    secs = time.time() - t0
    path = os.path.join(HERE, "config4.json")
    with open(path) as f:
        d = json.load(f)
    d["mcl_step"] = {k2: v for k2, v in digest(s, secs, 64).items()}
    d["mcl_step"]["params"] = {"prune_threshold": 0.002, "inflation": 2.0}
    with open(path, "w") as f:
        json.dump(d, f)
    print(f"config4 mcl step: nnz={s.nnz} ref {secs:.1f}s")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        small()
    if what in ("configs", "all"):
        for k in (1, 4, 5, 2):
            config(k)
    if what == "mcl4":
        mcl4()
    if what == "config3":
        config3()
    elif what.startswith("config") and what != "configs":
        config(int(what[6:]))
