"""Where does SpMM time go?  spmm_fwd / spmm_bwd (fused) on n = 2048^2 rows, k = 32 fp64, for
patterns of increasing gather spread: identity, tridiagonal (1D Poisson), 2D 5-point Poisson,
and a 5-point band with +-b offsets for several b.  CUDA events, L2 flushed, median.

    python tools/spmm_probe.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2212_05159_b200 import csrk as ck  # noqa: E402
from tools.micro import timeit  # noqa: E402


def band(n, offs):
    i = np.arange(n, dtype=np.int64)
    cols = np.stack([i + o for o in sorted(offs)], 1)
    ok = (cols >= 0) & (cols < n)
    cnt = ok.sum(1)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=indptr[1:])
    idx = cols[ok].astype(np.int32)
    return synth.CSR(n, n, indptr, idx, np.ones(len(idx)))


def main():
    n, k = 2048 * 2048, 32
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    X = torch.rand((n, k), dtype=torch.float64, device="cuda")
    dY = torch.rand((n, k), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    dX = torch.empty_like(X)
    cases = {
        "diag": [0], "tri": [-1, 0, 1], "b5_64": [-64, -1, 0, 1, 64], "b5_2048": [-2048, -1, 0, 1, 2048],
        "b5_65536": [-65536, -1, 0, 1, 65536], "b3_far": [-2048, 0, 2048],
    }
    res = {}
    for name, offs in cases.items():
        A = ck.CSR.from_host(band(n, offs))
        plan = ck.csr_transpose(A, with_values=False)
        dA = torch.empty(A.nnz, dtype=torch.float64, device="cuda")
        f = timeit(lambda: ck.spmm_fwd(A, X, out=Y), 10, flush)
        b = timeit(lambda: ck.spmm_bwd(A, X, dY, plan=plan, dA=dA, dX=dX), 10, flush)
        res[name] = {"nnz": A.nnz, "fwd_us": round(f, 1), "bwd_us": round(b, 1)}
        del A, plan, dA
    res["copy_2GB"] = round(timeit(lambda: Y.copy_(X), 10, flush), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
