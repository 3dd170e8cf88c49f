"""Run each listed op ONCE on BASELINE config 2 (2D Poisson 2048^2, fp64, k = 32) -- a target
for `ncu --set full` captures (one launch per kernel, cold caches).

    ncu --set full --import-source on -o gpurun_out/x python tools/ncu_ops.py spmm_fwd spmm_bwd
"""
from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2212_05159_b200 import csrk as ck  # noqa: E402


def main(ops):
    A = synth.poisson2d(2048)
    Ad = ck.CSR.from_host(A)
    n, nnz, k = A.nrows, A.nnz, 32
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.rand(*s, dtype=torch.float64, device="cuda", generator=g)
    x, dy, X, dY = r(n), r(n), r(n, k), r(n, k)
    plan = ck.csr_transpose(Ad, with_values=False)
    C = ck.spgemm_symbolic(Ad, Ad) if any(o.startswith("spgemm") for o in ops) else None
    torch.cuda.synchronize()
    for op in ops:
        if op == "transpose":
            ck.csr_transpose(Ad, with_values=False, out=plan)
        elif op == "spmv_fwd":
            ck.spmv_fwd(Ad, x)
        elif op == "spmv_bwd":
            ck.spmv_bwd(Ad, x, dy)
        elif op == "spmv_bwd_plan":
            ck.spmv_bwd(Ad, x, dy, plan=plan)
        elif op == "spmm_fwd":
            ck.spmm_fwd(Ad, X)
        elif op == "spmm_bwd":
            ck.spmm_bwd(Ad, X, dY, plan=plan)
        elif op == "spgemm_symbolic":
            ck.spgemm_symbolic(Ad, Ad)
        elif op == "spgemm_numeric":
            ck.spgemm_numeric(Ad, Ad, C)
        elif op == "spgemm_bwd":
            ck.spgemm_bwd(Ad, Ad, C, r(C.nnz))
        else:
            raise SystemExit(f"unknown op {op}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1:])
