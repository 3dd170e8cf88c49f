"""Config-4 SpGEMM micro-benchmark (power-law n = 2^23, fp32, C = A A): symbolic / numeric /
backward op times with CUDA events, L2 flushed before each rep, median of --reps.  For A/B runs
and ncu captures of single phases; bench.py --workload cfg4 is the number of record.

    python tools/gemm4.py [--ops sym,num,bwd,bwdplan] [--reps 3] [--n 23]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="sym,num,bwd")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=23)
    args = ap.parse_args()
    A = synth.powerlaw(n=1 << args.n)
    dev = torch.device("cuda", 0)
    Ad = ck.CSR.from_host(A)
    nnz = A.nnz
    del A
    C = ck.spgemm_symbolic(Ad, Ad)
    q = torch.arange(C.nnz, device=dev, dtype=torch.int64)
    dC = (((q * 2654435761 + 12345) % 1000003).to(torch.float64) / 500001.5 - 1.0).to(torch.float32)
    del q
    Cv = torch.empty(C.nnz, dtype=torch.float32, device=dev)
    dA, dB = torch.empty(nnz, dtype=torch.float32, device=dev), torch.empty(nnz, dtype=torch.float32, device=dev)
    plan = ck.csr_transpose(Ad, with_values=False) if "bwdplan" in args.ops else None
    fns = {
        "sym": lambda: ck.spgemm_symbolic(Ad, Ad),
        "num": lambda: ck.spgemm_numeric(Ad, Ad, C, out=Cv),
        "bwd": lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, dB=dB),
        "bwdplan": lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, dB=dB, plan=plan),
    }
    flush = torch.empty(1 << 27, dtype=torch.float32, device=dev)
    out = {"nnzC": C.nnz}
    for op in args.ops.split(","):
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fns[op]()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[op] = round(float(np.median(ts)), 2)
    if "num" in args.ops:
        out["Cv_sum"] = float(Cv.double().sum())
    if "bwd" in args.ops:
        out["dA_sum"], out["dB_sum"] = float(dA.double().sum()), float(dB.double().sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
