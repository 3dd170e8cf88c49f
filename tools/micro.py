"""Per-op micro-benchmarks on BASELINE config 2 (2D Poisson 2048^2, fp64) -- CUDA events,
L2 flushed between reps, median of `--reps`.  Used to iterate on kernels; bench.py is the
number of record.

    python tools/micro.py [--ops spmv,spmm,gemm,transpose] [--reps 20] [--grid 2048] [--dim 2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2212_05159_b200 import csrk as ck  # noqa: E402


def timeit(fn, reps, flush):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="spmv,spmm,gemm,transpose")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", type=int, default=2048)
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--k", type=int, default=32)
    args = ap.parse_args()
    A = synth.poisson2d(args.grid) if args.dim == 2 else synth.poisson3d(args.grid)
    Ad = ck.CSR.from_host(A)
    n, nnz, k = A.nrows, A.nnz, args.k
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    dev = "cuda"
    res = {}
    x = torch.rand(n, dtype=torch.float64, device=dev)
    dy = torch.rand(n, dtype=torch.float64, device=dev)
    plan = ck.csr_transpose(Ad, with_values=False)
    ops = args.ops.split(",")
    if "transpose" in ops:
        res["transpose"] = timeit(lambda: ck.csr_transpose(Ad, with_values=False, out=plan), args.reps, flush)
    if "spmv" in ops:
        y = torch.empty(n, dtype=torch.float64, device=dev)
        dA = torch.empty(nnz, dtype=torch.float64, device=dev)
        dx = torch.empty(n, dtype=torch.float64, device=dev)
        res["spmv_fwd"] = timeit(lambda: ck.spmv_fwd(Ad, x, out=y), args.reps, flush)
        res["spmv_bwd_plan"] = timeit(lambda: ck.spmv_bwd(Ad, x, dy, plan=plan, dA=dA, dx=dx), args.reps, flush)
        res["spmv_bwd_atomic"] = timeit(lambda: ck.spmv_bwd(Ad, x, dy, dA=dA, dx=dx), args.reps, flush)
        res["spmv_bwd_dA_only"] = timeit(lambda: ck.spmv_bwd(Ad, x, dy, dA=dA, need_dx=False), args.reps, flush)
        res["spmv_bwd_dx_only"] = timeit(lambda: ck.spmv_bwd(Ad, x, dy, dx=dx, need_dA=False), args.reps, flush)
        res["spmv_fwd_T_atomic"] = timeit(lambda: ck.spmv_fwd(Ad, x, op=ck.OP_T, out=y), args.reps, flush)
    if "spmm" in ops:
        X = torch.rand((n, k), dtype=torch.float64, device=dev)
        dY = torch.rand((n, k), dtype=torch.float64, device=dev)
        Y = torch.empty((n, k), dtype=torch.float64, device=dev)
        dA = torch.empty(nnz, dtype=torch.float64, device=dev)
        dX = torch.empty((n, k), dtype=torch.float64, device=dev)
        res["spmm_fwd"] = timeit(lambda: ck.spmm_fwd(Ad, X, out=Y), args.reps, flush)
        res["spmm_bwd_fused"] = timeit(lambda: ck.spmm_bwd(Ad, X, dY, plan=plan, dA=dA, dX=dX), args.reps, flush)
        res["spmm_bwd_dX_only"] = timeit(lambda: ck.spmm_bwd(Ad, X, dY, plan=plan, need_dA=False, dX=dX),
                                         args.reps, flush)
        res["spmm_bwd_sddmm_only"] = timeit(lambda: ck.spmm_bwd(Ad, X, dY, need_dX=False, dA=dA), args.reps, flush)
        res["copy_2GB"] = timeit(lambda: Y.copy_(X), args.reps, flush)
    if "gemm" in ops:
        C = ck.spgemm_symbolic(Ad, Ad)
        Cv = torch.empty(C.nnz, dtype=torch.float64, device=dev)
        dC = torch.rand(C.nnz, dtype=torch.float64, device=dev)
        dA = torch.empty(nnz, dtype=torch.float64, device=dev)
        dB = torch.empty(nnz, dtype=torch.float64, device=dev)
        res["gemm_symbolic"] = timeit(lambda: ck.spgemm_symbolic(Ad, Ad), args.reps, flush)
        res["gemm_numeric"] = timeit(lambda: ck.spgemm_numeric(Ad, Ad, C, out=Cv), args.reps, flush)
        res["gemm_bwd"] = timeit(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, dB=dB), args.reps, flush)
        res["gemm_bwd_dA_only"] = timeit(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, need_dB=False), args.reps, flush)
        res["gemm_bwd_dB_only"] = timeit(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, need_dA=False, dB=dB), args.reps, flush)
        res["gemm_bwd_plan"] = timeit(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, dB=dB, plan=plan), args.reps, flush)
        res["gemm_bwd_dB_plan"] = timeit(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, need_dA=False, dB=dB, plan=plan),
                                         args.reps, flush)
    print(json.dumps({kk: round(v, 1) for kk, v in res.items()}))


if __name__ == "__main__":
    main()
