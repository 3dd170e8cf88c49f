"""Test helpers (no method arithmetic beyond densification / mask gathering)."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def to_dense(A) -> np.ndarray:
    D = np.zeros((A.nrows, A.ncols), dtype=np.float64)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.indptr))
    D[rows, A.indices] = A.values
    return D


def pattern_dense(A) -> np.ndarray:
    P = np.zeros((A.nrows, A.ncols), dtype=bool)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.indptr))
    P[rows, A.indices] = True
    return P


def gather_mask(D: np.ndarray, indptr, indices) -> np.ndarray:
    """Values of dense D at the stored positions of a pattern, in CSR order ((.) mask)."""
    rows = np.repeat(np.arange(len(indptr) - 1), np.diff(indptr))
    return D[rows, indices]


def assert_S_close(got, ref, S, rtol, what=""):
    """SURVEY 8(c) c.2 / DESIGN reading A6: |got - ref| <= rtol * S elementwise (S = sum |terms|).
    S = 0 forces exact equality."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    assert got.shape == ref.shape == S.shape, (what, got.shape, ref.shape, S.shape)
    err = np.abs(got - ref)
    bad = err > rtol * S
    if bad.any():
        i = np.flatnonzero(bad.ravel())[0]
        raise AssertionError(f"{what}: {bad.sum()} elements out of tolerance; first flat idx {i}: "
                             f"got {got.ravel()[i]!r} ref {ref.ravel()[i]!r} S {S.ravel()[i]!r}")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_fig3():
    """Parse tests/golden/fig3_spgemm.txt -> dict of 0-based boolean patterns + flows."""
    mats, flows, cur = {}, [], None
    with open(os.path.join(GOLDEN, "fig3_spgemm.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] in ("A", "B", "C") and len(tok) == 3:
                cur = tok[0]
                mats[cur] = np.zeros((int(tok[1]), int(tok[2])), bool)
            elif tok[0] == "FLOW":
                ci, cj = int(tok[2]) - 1, int(tok[3]) - 1
                ia, ib = tok.index("A"), tok.index("B")
                a = [tuple(int(v) - 1 for v in t.split("/")) for t in tok[ia + 1:ib]]
                b = [tuple(int(v) - 1 for v in t.split("/")) for t in tok[ib + 1:]]
                flows.append(((ci, cj), a, b))
            else:
                for t in tok:
                    r, c = (int(v) - 1 for v in t.split("/"))
                    mats[cur][r, c] = True
    return mats, flows


def csr_from_pattern(P: np.ndarray, values=None, dtype=np.float64):
    import synth
    m, n = P.shape
    counts = P.sum(axis=1).astype(np.int64)
    indptr = np.zeros(m + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.nonzero(P)[1].astype(np.int32)
    if values is None:
        vals = np.ones(indices.shape[0], dtype)
    else:
        vals = np.asarray(values, dtype)
    return synth.CSR(m, n, indptr, indices, vals)
