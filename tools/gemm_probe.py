"""Probe: SpGEMM backward cost split (dA only / dB only / both) and numeric on config 2."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2212_05159_b200 import csrk as ck


def t(fn, reps=20):
    fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        fl.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


dim = int(sys.argv[1]) if len(sys.argv) > 1 else 2
A = synth.poisson2d(2048) if dim == 2 else synth.poisson3d(160)
Ad = ck.CSR.from_host(A)
C = ck.spgemm_symbolic(Ad, Ad)
dC = torch.rand(C.nnz, dtype=torch.float64, device="cuda")
dA = torch.empty_like(Ad.values); dB = torch.empty_like(Ad.values); Cv = torch.empty(C.nnz, dtype=torch.float64, device="cuda")
print("numeric", t(lambda: ck.spgemm_numeric(Ad, Ad, C, out=Cv)))
print("bwd both", t(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA, dB=dB)))
print("bwd dA only", t(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, need_dB=False, dA=dA)))
print("bwd dB only", t(lambda: ck.spgemm_bwd(Ad, Ad, C, dC, need_dA=False, dB=dB)))
print("symbolic", t(lambda: ck.spgemm_symbolic(Ad, Ad)))
