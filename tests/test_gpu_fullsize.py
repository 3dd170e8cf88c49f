"""GPU parity at BASELINE.json's full sizes (configs 2, 3, 4), in the launch configuration
bench.py times, checked on SAMPLED outputs that the oracle computes one by one (row subsets
of A, of A^T for column-indexed outputs, of the rows of A referencing sampled rows of B), plus
properties that hold at any size (exact closed forms of the Poisson products, full transpose
equality).  Tolerance rule as in test_gpu_parity.py (S-scaled, 1e-12 fp64 / 1e-5 fp32)."""
import os
import sys

import numpy as np
import pytest
import torch

import synth
from util import assert_S_close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RTOL = {np.float64: 1e-12, np.float32: 1e-5}


@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def sub_rows(A, rows):
    """Rows `rows` (sorted) of A as a CSR with global column indices, plus the position of
    each kept entry in A."""
    rows = np.asarray(rows, np.int64)
    lens = A.indptr[rows + 1] - A.indptr[rows]
    indptr = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=indptr[1:])
    pos = np.concatenate([np.arange(A.indptr[r], A.indptr[r + 1]) for r in rows]) if len(rows) else np.zeros(0, np.int64)
    vals = None if A.values is None else A.values[pos]
    return synth.CSR(len(rows), A.ncols, indptr, A.indices[pos], vals), pos


def sample_rows(n, k, seed):
    rng = np.random.default_rng(seed)
    r = np.unique(np.concatenate([[0, 1, n // 2, n - 2, n - 1], rng.choice(n, k, replace=False)]))
    return r[(r >= 0) & (r < n)]


def close(got, ref, S, dt, what):
    assert_S_close(np.asarray(got, np.float64), ref, S, RTOL[dt], what)


def check_spmv(orc, A, x, dy, y, dA, dx, dt, rows, cols, AT):
    As, pos = sub_rows(A, rows)
    r = orc.spmv_fwd(As, x)
    close(y[rows], r.value, r.S, dt, "y sampled rows")
    dA_ref, _ = orc.spmv_bwd(As, x, dy[rows], want_dx=False)
    np.testing.assert_array_equal(dA[pos], dA_ref, err_msg="dA sampled rows (bit-exact)")
    ATs, _ = sub_rows(AT, cols)
    r = orc.spmv_fwd(ATs, dy)        # dx_j = sum_i A_ij dy_i = (A^T dy)_j
    close(dx[cols], r.value, r.S, dt, "dx sampled cols")


def check_spgemm(orc, A, B, AT, C_p, C_i, C_v, dC, dA, dB, dt, rows, brows):
    # C rows: pattern bit-exact, values S-scaled
    As, apos = sub_rows(A, rows)
    Cp, Ci = orc.spgemm_symbolic(As, B)
    got_len = C_p[rows + 1] - C_p[rows]
    np.testing.assert_array_equal(got_len, np.diff(Cp), err_msg="C row lengths")
    cpos = np.concatenate([np.arange(C_p[r], C_p[r + 1]) for r in rows])
    np.testing.assert_array_equal(C_i[cpos], Ci, err_msg="C indices")
    r = orc.spgemm_numeric(As, B, Cp, Ci)
    close(C_v[cpos], r.value, r.S, dt, "C values")
    dA_ref, _ = orc.spgemm_bwd(As, B, Cp, Ci, dC[cpos], want_dB=False)
    close(dA[apos], dA_ref.value, dA_ref.S, dt, "dA sampled rows")
    # dB rows k: every row i of A with A_ik != 0 contributes; take those rows of A
    irows = np.unique(np.concatenate([AT.indices[AT.indptr[k]:AT.indptr[k + 1]] for k in brows]))
    As2, _ = sub_rows(A, irows)
    Cp2, Ci2 = orc.spgemm_symbolic(As2, B)
    cpos2 = np.concatenate([np.arange(C_p[r], C_p[r + 1]) for r in irows])
    _, dB_ref = orc.spgemm_bwd(As2, B, Cp2, Ci2, dC[cpos2], want_dA=False)
    bpos = np.concatenate([np.arange(B.indptr[k], B.indptr[k + 1]) for k in brows])
    close(dB[bpos], dB_ref.value[bpos], dB_ref.S[bpos], dt, "dB sampled rows")


def test_config2_bench_step(ck, orc):
    """BASELINE config 2 through bench.Workload.step (the timed launch configuration)."""
    sys.path.insert(0, ROOT)
    import bench
    W = bench.Workload(torch, ck)
    W.step()
    torch.cuda.synchronize()
    A = W.A_host
    n = A.nrows
    assert A.nnz == 20963328 and W.nnzC == 13 * 2048 ** 2 - 20 * 2048 + 4   # closed forms
    h = lambda t: t.cpu().numpy()
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    # the step's transpose plan: bit-exact over the whole matrix
    np.testing.assert_array_equal(h(W.plan.AT.indptr), ATp)
    np.testing.assert_array_equal(h(W.plan.AT.indices), ATi)
    np.testing.assert_array_equal(h(W.plan.perm), perm)
    AT = synth.CSR(n, n, ATp, ATi, ATv)
    rows = sample_rows(n, 3000, 1)
    cols = sample_rows(n, 3000, 2)
    x, dy = h(W.x), h(W.dy)
    check_spmv(orc, A, x, dy, h(W.y), h(W.dA_v), h(W.dx), np.float64, rows, cols, AT)
    # SpMM k = 32
    X, dY = h(W.X), h(W.dY)
    As, pos = sub_rows(A, rows)
    r = orc.spmm_fwd(As, X)
    close(h(W.Y)[rows], r.value, r.S, np.float64, "Y sampled rows")
    dA_ref, _ = orc.spmm_bwd(As, X, dY[rows], want_dX=False)
    close(h(W.dA_m)[pos], dA_ref.value, dA_ref.S, np.float64, "spmm dA sampled rows")
    ATs, _ = sub_rows(AT, cols)
    r = orc.spmm_fwd(ATs, dY)
    close(h(W.dX)[cols], r.value, r.S, np.float64, "dX sampled cols")
    # SpGEMM C = A A
    check_spgemm(orc, A, A, AT, h(W.C.indptr), h(W.C.indices), h(W.Cv), h(W.dC), h(W.dA_g), h(W.dB_g),
                 np.float64, sample_rows(n, 500, 3), sample_rows(n, 200, 4))


def test_config3_spgemm_3d(ck, orc):
    """BASELINE config 3: 3D 7-point Poisson 160^3, fp64, C = A A forward + backward."""
    N = 160
    A = synth.poisson3d(N)
    assert A.nnz == 7 * N ** 3 - 6 * N ** 2
    Ad = ck.CSR.from_host(A)
    C = ck.spgemm_symbolic(Ad, Ad)
    assert C.nnz == 25 * N ** 3 - 42 * N ** 2 + 12 * N
    Cv = ck.spgemm_numeric(Ad, Ad, C)
    dC = synth.dense(C.nnz, synth.seed_of(3, 5))
    dA, dB = ck.spgemm_bwd(Ad, Ad, C, torch.from_numpy(dC).cuda())
    h = lambda t: t.cpu().numpy()
    C_p, C_i, C_v = h(C.indptr), h(C.indices), h(Cv)
    # integer stencil: every value of A^2 is an exact integer of the closed form (A^2 diag =
    # 36 + degree); check all diagonals exactly
    rows_all = np.repeat(np.arange(A.nrows), np.diff(C_p))
    diag = C_v[rows_all == C_i]
    deg = np.diff(A.indptr) - 1
    np.testing.assert_array_equal(diag, 36.0 + deg)
    ATp, ATi, ATv, _ = orc.csr_transpose(A)
    AT = synth.CSR(A.ncols, A.nrows, ATp, ATi, ATv)
    check_spgemm(orc, A, A, AT, C_p, C_i, C_v, dC, h(dA), h(dB), np.float64,
                 sample_rows(A.nrows, 400, 5), sample_rows(A.nrows, 150, 6))
    # Euler identity at full size: <dC, C> = <dA, A> = <dB, A>
    lhs = float(np.dot(dC, C_v))
    assert abs(lhs - float(np.dot(h(dA), A.values))) <= 1e-9 * np.abs(dC * C_v).sum()
    assert abs(lhs - float(np.dot(h(dB), A.values))) <= 1e-9 * np.abs(dC * C_v).sum()


def test_config4_powerlaw(ck, orc):
    """BASELINE config 4: power-law n = 2^23, 16 nnz/row, fp32: SpMV fwd/bwd, transpose,
    SpGEMM A A forward + backward on sampled rows (nnz(C) ~ 2.1e9)."""
    A = synth.powerlaw()
    assert A.nnz == 1 << 27
    n = A.nrows
    dt = np.float32
    Ad = ck.CSR.from_host(A)
    x = synth.dense(n, synth.seed_of(4, 3), dt)
    dy = synth.dense(n, synth.seed_of(4, 4), dt)
    xt, dyt = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
    y = ck.spmv_fwd(Ad, xt)
    dA, dx = ck.spmv_bwd(Ad, xt, dyt)
    plan = ck.csr_transpose(Ad)
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    np.testing.assert_array_equal(plan.AT.indptr.cpu().numpy(), ATp)
    np.testing.assert_array_equal(plan.AT.indices.cpu().numpy(), ATi)
    np.testing.assert_array_equal(plan.perm.cpu().numpy(), perm)
    AT = synth.CSR(n, n, ATp, ATi, ATv)
    h = lambda t: t.cpu().numpy()
    # long rows (up to 32,769) and short rows both sampled
    lens = np.diff(A.indptr)
    rows = np.unique(np.concatenate([sample_rows(n, 2000, 7), np.argsort(lens)[-50:]]))
    check_spmv(orc, A, x, dy, h(y), h(dA), h(dx), dt, rows, sample_rows(n, 2000, 8), AT)
    _, dx_plan = ck.spmv_bwd(Ad, xt, dyt, plan=plan, need_dA=False)
    ATs, _ = sub_rows(AT, rows)
    r = orc.spmv_fwd(ATs, dy)
    close(h(dx_plan)[rows], r.value, r.S, dt, "dx (plan) sampled cols")
    # with dA too: scattered pattern -> dA by the row traversal, dx by the transposed gather
    dA_plan, dx_plan2 = ck.spmv_bwd(Ad, xt, dyt, plan=plan)
    np.testing.assert_array_equal(h(dA_plan), h(dA))          # single products: bit-exact
    np.testing.assert_array_equal(h(dx_plan2), h(dx_plan))     # same gather, same order
    del dx_plan, dx_plan2, dA_plan
    torch.cuda.empty_cache()
    # SpGEMM
    C = ck.spgemm_symbolic(Ad, Ad)
    prod = int(lens[A.indices].sum())
    assert 0 < C.nnz <= prod
    Cv = ck.spgemm_numeric(Ad, Ad, C)
    # dC from a counter-based generator (too large to build on the host): value(q) in [-1, 1)
    q = torch.arange(C.nnz, device="cuda", dtype=torch.int64)
    dCd = (((q * 2654435761 + 12345) % 1000003).to(torch.float32) / 500001.5 - 1.0)
    dAg, dBg = ck.spgemm_bwd(Ad, Ad, C, dCd)
    C_p = h(C.indptr)
    srows = np.unique(np.concatenate([sample_rows(n, 120, 9), np.argsort(lens)[-3:]]))
    brows = sample_rows(n, 30, 10)
    irows = np.unique(np.concatenate([AT.indices[AT.indptr[k]:AT.indptr[k + 1]] for k in brows]))
    need = np.unique(np.concatenate([srows, irows]))
    cpos = np.concatenate([np.arange(C_p[r], C_p[r + 1]) for r in need])
    dC_host = np.zeros(C.nnz, np.float32)
    cpos_t = torch.from_numpy(cpos).cuda()
    dC_host[cpos] = dCd[cpos_t].cpu().numpy()
    C_i = np.zeros(C.nnz, np.int32)
    C_i[cpos] = C.indices[cpos_t].cpu().numpy()
    C_v = np.zeros(C.nnz, np.float32)
    C_v[cpos] = Cv[cpos_t].cpu().numpy()
    check_spgemm(orc, A, A, AT, C_p, C_i, C_v, dC_host, h(dAg), h(dBg), dt, srows, brows)
    # deterministic dB (flat per-entry gather on this scattered pattern) on the same samples, twice
    _, dBp = ck.spgemm_bwd(Ad, Ad, C, dCd, need_dA=False, plan=plan)
    _, dBp2 = ck.spgemm_bwd(Ad, Ad, C, dCd, need_dA=False, plan=plan)
    np.testing.assert_array_equal(h(dBp), h(dBp2))
    check_spgemm(orc, A, A, AT, C_p, C_i, C_v, dC_host, h(dAg), h(dBp), dt, srows, brows)
