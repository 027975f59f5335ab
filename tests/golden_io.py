"""Helpers to read tests/golden/small.npz (reference-generated fixtures)."""
import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small.npz")
_z = None


def z():
    global _z
    if _z is None:
        _z = dict(np.load(GOLDEN))
    return _z


def csr(prefix) -> O.Csr:
    g = z()
    nr, nc = (int(x) for x in g[prefix + "_shape"])
    return O.Csr(nr, nc, g[prefix + "_rowptr"], g[prefix + "_colind"], g[prefix + "_values"])


def spgemm_cases():
    return [str(x) for x in z()["spgemm_cases"]]


def grids():
    return [tuple(int(v) for v in g) for g in z()["grids"]]
