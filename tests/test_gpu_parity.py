"""GPU parity: every hot-path op through the C-ABI (paper_2212_05159_b200.csrk -> libcsrk.so)
against the CPU oracle, element by element, on seeded synthetic inputs.

Bar (BASELINE.json north_star): patterns (indptr / indices / perm)
bit-exact; values |gpu - oracle| <= rtol * S with S = sum |terms| (rtol 1e-12 fp64, 1e-5
fp32); integer-valued inputs and the single-product masked gradient bit-exact.
"""
import numpy as np
import pytest
import torch

import synth
from util import assert_S_close

pytestmark = pytest.mark.gpu

RTOL = {np.float64: 1e-12, np.float32: 1e-5}


@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def skew(n, long_row, seed, dtype=np.float64, values="real"):
    """Row 0 holds `long_row` entries and column 0 is full (a dense column): exercises
    multi-chunk tiles, the huge-column transpose sort and the large-row SpGEMM bins."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        if i == 0:
            cols = np.sort(rng.choice(n, long_row, replace=False))
            cols = np.union1d([0], cols)
        else:
            cols = np.union1d([0, i], rng.choice(n, 2))
        rows.append(cols)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum([len(c) for c in rows], out=indptr[1:])
    indices = np.concatenate(rows).astype(np.int32)
    vr = np.random.default_rng(seed + 1)
    vals = synth.real_values(vr, len(indices), dtype) if values == "real" else synth.int_values(vr, len(indices), dtype)
    return synth.CSR(n, n, indptr, indices, vals)


def empty_matrix(m, n, dtype=np.float64):
    return synth.CSR(m, n, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, dtype))


CASES = {
    "config1_poisson16": lambda dt, v: synth.poisson2d(16, dtype=dt),
    "poisson2d_70": lambda dt, v: synth.poisson2d(70, dtype=dt),
    "poisson3d_17": lambda dt, v: synth.poisson3d(17, dtype=dt),
    "rand_rect_empty_rows": lambda dt, v: synth.random_csr(3001, 2003, 0.004, 11, dt, v, empty_rows=True),
    "powerlaw_16k": lambda dt, v: synth.powerlaw(1 << 14, seed=41, dtype=dt, values=v),
    "skew_mid": lambda dt, v: skew(3000, 700, 5, dt, v),
    "tiny_3x3": lambda dt, v: synth.poisson1d(3, dtype=dt),
    "one_row": lambda dt, v: synth.random_csr(1, 50, 0.5, 3, dt, v),
    "nnz0": lambda dt, v: empty_matrix(40, 30, dt),
    "skew_huge": lambda dt, v: skew(9000, 8500, 8, dt, v),   # one row > kHugeRow (CTA-wide pass)
}


def make(case, dt, values="real"):
    A = CASES[case](dt, values)
    if values == "int" and case.startswith(("config1", "poisson", "tiny")):
        A = A.with_values(synth.int_values(np.random.default_rng(9), A.nnz, dt))
    return A


def dev(ck, A):
    return ck.CSR.from_host(A)


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def close(got, ref, S, dt, what, exact=False):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    if exact:
        np.testing.assert_array_equal(got, ref, err_msg=what)
    else:
        assert_S_close(got, ref, S, RTOL[dt], what)


DTS = [np.float64, np.float32]


# ---------------------------------------------------------------- SpMV
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("values", ["real", "int"])
def test_spmv_fwd_bwd(ck, orc, case, dt, values):
    A = make(case, dt, values)
    m, n = A.nrows, A.ncols
    x = synth.dense(n, 3, dt, values)
    xt = synth.dense(m, 4, dt, values)
    dy = synth.dense(m, 5, dt, values)
    dyt = synth.dense(n, 6, dt, values)
    exact = values == "int"
    Ad = dev(ck, A)
    plan = ck.csr_transpose(Ad)
    # forward, op N and op T (with and without the transpose plan)
    r = orc.spmv_fwd(A, x)
    close(ck.spmv_fwd(Ad, t(x)), r.value, r.S, dt, "y=Ax", exact)
    r = orc.spmv_fwd(A, xt, op=1)
    close(ck.spmv_fwd(Ad, t(xt), op=ck.OP_T), r.value, r.S, dt, "y=A^T x atomic", exact)
    close(ck.spmv_fwd(Ad, t(xt), op=ck.OP_T, plan=plan), r.value, r.S, dt, "y=A^T x plan", exact)
    # backward op N: dA bit-exact (one product), dx = A^T dy
    dA_ref, dx_ref = orc.spmv_bwd(A, x, dy)
    for p in (None, plan):
        dA, dx = ck.spmv_bwd(Ad, t(x), t(dy), plan=p)
        np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref, err_msg=f"dA plan={p is not None}")
        close(dx, dx_ref.value, dx_ref.S, dt, f"dx plan={p is not None}", exact)
    dA, _ = ck.spmv_bwd(Ad, t(x), t(dy), need_dx=False)
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref)
    _, dx = ck.spmv_bwd(Ad, t(x), t(dy), plan=plan, need_dA=False)
    close(dx, dx_ref.value, dx_ref.S, dt, "dx only", exact)
    # backward op T
    dA_ref, dx_ref = orc.spmv_bwd(A, xt, dyt, op=1)
    dA, dx = ck.spmv_bwd(Ad, t(xt), t(dyt), op=ck.OP_T)
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref)
    close(dx, dx_ref.value, dx_ref.S, dt, "dx op T", exact)
    dA, _ = ck.spmv_bwd(Ad, t(xt), t(dyt), op=ck.OP_T, need_dx=False)
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref)


WIN_CASES = {
    # square operators of ~10^6 rows (several waves of the scatter kernel): banded, odd order,
    # scattered power-law columns with a few long rows
    "poisson2d_1024": lambda dt, v: synth.poisson2d(1024, dtype=dt),
    "poisson2d_1023": lambda dt, v: synth.poisson2d(1023, dtype=dt),
    "powerlaw_2p20": lambda dt, v: synth.powerlaw(1 << 20, seed=17, dtype=dt, values=v),
}


@pytest.mark.parametrize("case", list(WIN_CASES))
@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("values", ["real", "int"])
def test_spmv_bwd_large(ck, orc, case, dt, values):
    """SpMV backward without a plan (atomic dx scatter) at ~10^6 rows: dA bit-exact, dx within
    the S rule (exact for integer data), also dx only."""
    A = WIN_CASES[case](dt, values)
    if values == "int" and case.startswith("poisson"):
        rng = np.random.default_rng(9)
        A = A.with_values(synth.int_values(rng, A.nnz, dt))
    assert A.nrows == A.ncols and A.nrows >= 148 * 4096
    x = synth.dense(A.ncols, 13, dt, values)
    dy = synth.dense(A.nrows, 14, dt, values)
    dA_ref, dx_ref = orc.spmv_bwd(A, x, dy)
    Ad = dev(ck, A)
    dA, dx = ck.spmv_bwd(Ad, t(x), t(dy))
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref)
    close(dx, dx_ref.value, dx_ref.S, dt, "dx", values == "int")
    _, dx2 = ck.spmv_bwd(Ad, t(x), t(dy), need_dA=False)
    close(dx2, dx_ref.value, dx_ref.S, dt, "dx only", values == "int")


def test_spmv_deterministic(ck):
    A = synth.powerlaw(1 << 14, seed=3, dtype=np.float64)
    Ad = dev(ck, A)
    x = t(synth.dense(A.ncols, 1))
    dy = t(synth.dense(A.nrows, 2))
    plan = ck.csr_transpose(Ad)
    y0 = ck.spmv_fwd(Ad, x)
    dA0, dx0 = ck.spmv_bwd(Ad, x, dy, plan=plan)
    for _ in range(3):
        assert torch.equal(ck.spmv_fwd(Ad, x), y0)
        dA, dx = ck.spmv_bwd(Ad, x, dy, plan=plan)
        assert torch.equal(dA, dA0) and torch.equal(dx, dx0)


# ---------------------------------------------------------------- transpose
@pytest.mark.parametrize("case", list(CASES))
def test_csr_transpose(ck, orc, case):
    A = make(case, np.float64)
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    plan = ck.csr_transpose(dev(ck, A))
    np.testing.assert_array_equal(plan.AT.indptr.cpu().numpy(), ATp)
    np.testing.assert_array_equal(plan.AT.indices.cpu().numpy(), ATi)
    np.testing.assert_array_equal(plan.perm.cpu().numpy(), perm)
    np.testing.assert_array_equal(plan.AT.values.cpu().numpy(), ATv)
    # involution
    back = ck.csr_transpose(plan.AT)
    np.testing.assert_array_equal(back.AT.indptr.cpu().numpy(), A.indptr)
    np.testing.assert_array_equal(back.AT.indices.cpu().numpy(), A.indices)
    np.testing.assert_array_equal(back.AT.values.cpu().numpy(), A.values)


def _symmetrized(A, drop=None, seed=3):
    """pattern(A) U pattern(A^T) with seeded values (structurally symmetric, unsymmetric values);
    drop = index of one stored entry to remove (then the pattern is no longer symmetric)."""
    import scipy.sparse as sp
    M = sp.csr_matrix((np.ones(A.nnz), A.indices, A.indptr), shape=(A.nrows, A.ncols))
    S = (M + M.T).tocsr()
    S.sort_indices()
    indptr, indices = S.indptr.astype(np.int64), S.indices.astype(np.int32)
    if drop is not None:
        row = int(np.searchsorted(indptr, drop, side="right") - 1)
        indices = np.delete(indices, drop)
        indptr = indptr.copy()
        indptr[row + 1:] -= 1
    vals = synth.real_values(np.random.default_rng(seed), len(indices))
    return synth.CSR(A.nrows, A.ncols, indptr, indices, vals)


@pytest.mark.parametrize("case", ["sym_powerlaw", "sym_skew", "sym_drop_first", "sym_drop_mid", "sym_drop_last",
                                  "poisson3d_17"])
def test_csr_transpose_symmetric_path(ck, orc, case):
    """Structurally symmetric patterns take the one-search-per-entry path (k_tr_sym: long rows by
    the warp); patterns one entry short of symmetric must be detected and fall back, bit-exact."""
    base = synth.powerlaw(1 << 12, seed=5)
    if case == "sym_powerlaw":
        A = _symmetrized(base)
    elif case == "sym_skew":
        A = _symmetrized(skew(3000, 2500, 4))
    elif case == "poisson3d_17":
        A = make(case, np.float64)
    else:
        S = _symmetrized(base)
        A = _symmetrized(base, drop={"sym_drop_first": 0, "sym_drop_mid": S.nnz // 2,
                                     "sym_drop_last": S.nnz - 1}[case])
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    plan = ck.csr_transpose(dev(ck, A))
    np.testing.assert_array_equal(plan.AT.indptr.cpu().numpy(), ATp)
    np.testing.assert_array_equal(plan.AT.indices.cpu().numpy(), ATi)
    np.testing.assert_array_equal(plan.perm.cpu().numpy(), perm)
    np.testing.assert_array_equal(plan.AT.values.cpu().numpy(), ATv)


# ---------------------------------------------------------------- SpMM
@pytest.mark.parametrize("case", ["config1_poisson16", "poisson2d_70", "rand_rect_empty_rows", "skew_mid",
                                  "tiny_3x3", "nnz0", "powerlaw_16k"])
@pytest.mark.parametrize("dt,k", [(np.float64, 32), (np.float32, 32), (np.float64, 5), (np.float32, 7),
                                  (np.float64, 200), (np.float64, 300), (np.float32, 16),
                                  (np.float64, 16)])
def test_spmm_fwd_bwd(ck, orc, case, dt, k):
    values = "int" if k in (5, 16) else "real"
    A = make(case, dt, values)
    if case == "powerlaw_16k" and k > 32:
        pytest.skip("large k on the power-law case is covered by smaller cases")
    m, n = A.nrows, A.ncols
    X = synth.dense((n, k), 3, dt, values)
    dY = synth.dense((m, k), 4, dt, values)
    exact = values == "int"
    Ad = dev(ck, A)
    r = orc.spmm_fwd(A, X)
    close(ck.spmm_fwd(Ad, t(X)), r.value, r.S, dt, "Y", exact)
    dA_ref, dX_ref = orc.spmm_bwd(A, X, dY)
    plan = ck.csr_transpose(Ad)
    for p in (plan, None):
        dA, dX = ck.spmm_bwd(Ad, t(X), t(dY), plan=p)
        close(dA, dA_ref.value, dA_ref.S, dt, f"dA plan={p is not None}", exact)
        close(dX, dX_ref.value, dX_ref.S, dt, f"dX plan={p is not None}", exact)
    dA, _ = ck.spmm_bwd(Ad, t(X), t(dY), need_dX=False)
    close(dA, dA_ref.value, dA_ref.S, dt, "dA only (SDDMM)", exact)
    _, dX = ck.spmm_bwd(Ad, t(X), t(dY), plan=plan, need_dA=False)
    close(dX, dX_ref.value, dX_ref.S, dt, "dX only", exact)


@pytest.mark.parametrize("case", ["poisson2d_150", "powerlaw_32k", "rand_rect_40k"])
@pytest.mark.parametrize("dt,k", [(np.float64, 32), (np.float32, 32), (np.float64, 16)])
@pytest.mark.parametrize("values", ["real", "int"])
def test_spmm_pipelined_path(ck, orc, case, dt, k, values):
    """Matrices of >= 148 x 128 rows take the persistent TMA-pipelined wide kernel (k_spmm_pipe):
    every mode (fwd, fused dA + dX, dA only, dX only) against the oracle, ragged last tile."""
    A = {"poisson2d_150": lambda: synth.poisson2d(150, dtype=dt),
         "powerlaw_32k": lambda: synth.powerlaw(1 << 15, seed=43, dtype=dt, values=values),
         "rand_rect_40k": lambda: synth.random_csr(40001, 30011, 0.0002, 12, dt, values, empty_rows=True)}[case]()
    if values == "int" and case.startswith("poisson"):
        A = A.with_values(synth.int_values(np.random.default_rng(9), A.nnz, dt))
    exact = values == "int"
    m, n = A.nrows, A.ncols
    X = synth.dense((n, k), 3, dt, values)
    dY = synth.dense((m, k), 4, dt, values)
    Ad = dev(ck, A)
    r = orc.spmm_fwd(A, X)
    close(ck.spmm_fwd(Ad, t(X)), r.value, r.S, dt, "Y", exact)
    dA_ref, dX_ref = orc.spmm_bwd(A, X, dY)
    plan = ck.csr_transpose(Ad)
    dA, dX = ck.spmm_bwd(Ad, t(X), t(dY), plan=plan)
    close(dA, dA_ref.value, dA_ref.S, dt, "dA", exact)
    close(dX, dX_ref.value, dX_ref.S, dt, "dX", exact)
    dA, _ = ck.spmm_bwd(Ad, t(X), t(dY), need_dX=False)
    close(dA, dA_ref.value, dA_ref.S, dt, "dA only (SDDMM)", exact)
    _, dX = ck.spmm_bwd(Ad, t(X), t(dY), plan=plan, need_dA=False)
    close(dX, dX_ref.value, dX_ref.S, dt, "dX only", exact)


def test_spmm_strided_operands(ck, orc):
    """Leading dimensions > k (row-major with padding, reading A10)."""
    A = synth.poisson2d(20)
    k, ld = 6, 9
    Xf = synth.dense((A.ncols, ld), 1)
    dYf = synth.dense((A.nrows, ld), 2)
    Ad = dev(ck, A)
    Xt, dYt = t(Xf)[:, :k], t(dYf)[:, :k]
    r = orc.spmm_fwd(A, Xf[:, :k])
    close(ck.spmm_fwd(Ad, Xt), r.value, r.S, np.float64, "Y strided")
    dA_ref, dX_ref = orc.spmm_bwd(A, Xf[:, :k], dYf[:, :k])
    dA, dX = ck.spmm_bwd(Ad, Xt, dYt, plan=ck.csr_transpose(Ad))
    close(dA, dA_ref.value, dA_ref.S, np.float64, "dA strided")
    close(dX, dX_ref.value, dX_ref.S, np.float64, "dX strided")


# ---------------------------------------------------------------- SpGEMM
GEMM_CASES = ["config1_poisson16", "poisson2d_70", "poisson3d_17", "rand_rect_empty_rows", "powerlaw_16k",
              "skew_mid", "tiny_3x3", "one_row", "nnz0", "skew_big", "clustered",
              "wide_huge"]


def clustered_operands(dt, values):
    """Warp-path rows (l in {20, 40, 60, 70}: W, W2 and CTA classes) times B rows whose 12 columns
    sit in one of three 24-column clusters: ~3 products per C column and ~25 per bucket of the
    FILL bucket sort -- the buckets overflow, so FILL takes its shared-memory bitonic fallback, and
    the numeric / backward position index sees long, clustered buckets."""
    rng = np.random.default_rng(515)
    n = 3000
    la = rng.choice([20, 40, 60, 70], size=n)
    a_cols = [np.sort(rng.choice(n, size=int(l), replace=False)) for l in la]
    b_cols = [np.sort(rng.choice(24, size=12, replace=False) + 1000 * (k % 3)) for k in range(n)]

    def csr(cols):
        indptr = np.zeros(n + 1, np.int64)
        indptr[1:] = np.cumsum([len(c) for c in cols])
        idx = np.concatenate(cols).astype(np.int32)
        vals = synth.real_values(rng, idx.size, dt) if values == "real" else synth.int_values(rng, idx.size, dt)
        return synth.CSR(n, n, indptr, idx, vals)
    return csr(a_cols), csr(b_cols)


def gemm_operands(case, dt, values):
    if case == "wide_huge":
        # huge rows (w = 10,000 > 8192 products) over 2*10^7 columns: the cluster kernel's eight
        # 1.6M-column windows and a second super-window (columns beyond 8 x 1,638,400)
        A = synth.random_csr(24, 3000, 1 / 3, 31, dt, values)
        rng = np.random.default_rng(32)
        cols = np.sort(rng.choice(20_000_000, size=(3000, 12), replace=True), axis=1)
        keep = np.concatenate([np.ones((3000, 1), bool), cols[:, 1:] != cols[:, :-1]], axis=1)
        indptr = np.zeros(3001, np.int64)
        indptr[1:] = np.cumsum(keep.sum(1))
        idx = cols[keep].astype(np.int32)
        vals = synth.real_values(rng, idx.size, dt) if values == "real" else synth.int_values(rng, idx.size, dt)
        return A, synth.CSR(3000, 20_000_000, indptr, idx, vals)
    if case == "clustered":
        return clustered_operands(dt, values)
    if case == "skew_big":
        A = skew(9000, 8500, 21, dt, values)
        return A, A
    A = make(case, dt, values)
    if case in ("rand_rect_empty_rows", "one_row"):
        B = synth.random_csr(A.ncols, 777, 0.01 if case != "one_row" else 0.2, 12, dt, values)
        return A, B
    if case == "nnz0":
        return A, synth.random_csr(A.ncols, 20, 0.3, 2, dt, values)
    return A, A


@pytest.mark.parametrize("case", GEMM_CASES)
@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("values", ["real", "int"])
def test_spgemm(ck, orc, case, dt, values):
    if case == "skew_big" and (dt == np.float32 or values == "int"):
        pytest.skip("one dtype suffices for the big skewed case")
    A, B = gemm_operands(case, dt, values)
    exact = values == "int"
    Ad, Bd = dev(ck, A), dev(ck, B)
    Cp, Ci = orc.spgemm_symbolic(A, B)
    C = ck.spgemm_symbolic(Ad, Bd)
    np.testing.assert_array_equal(C.indptr.cpu().numpy(), Cp)
    np.testing.assert_array_equal(C.indices.cpu().numpy(), Ci)
    r = orc.spgemm_numeric(A, B, Cp, Ci)
    close(ck.spgemm_numeric(Ad, Bd, C), r.value, r.S, dt, "C values", exact)
    dC = synth.dense(len(Ci), 7, dt, values)
    dA_ref, dB_ref = orc.spgemm_bwd(A, B, Cp, Ci, dC)
    dA, dB = ck.spgemm_bwd(Ad, Bd, C, t(dC))
    close(dA, dA_ref.value, dA_ref.S, dt, "dA", exact)
    close(dB, dB_ref.value, dB_ref.S, dt, "dB", exact)
    dA2, _ = ck.spgemm_bwd(Ad, Bd, C, t(dC), need_dB=False)
    close(dA2, dA_ref.value, dA_ref.S, dt, "dA only", exact)
    _, dB2 = ck.spgemm_bwd(Ad, Bd, C, t(dC), need_dA=False)
    close(dB2, dB_ref.value, dB_ref.S, dt, "dB only", exact)
    # deterministic dB: gather over A's columns through A's transpose plan
    plan = ck.csr_transpose(Ad, with_values=False)
    dA3, dB3 = ck.spgemm_bwd(Ad, Bd, C, t(dC), plan=plan)
    close(dA3, dA_ref.value, dA_ref.S, dt, "dA (plan)", exact)
    close(dB3, dB_ref.value, dB_ref.S, dt, "dB (plan)", exact)
    _, dB4 = ck.spgemm_bwd(Ad, Bd, C, t(dC), need_dA=False, plan=plan)
    close(dB4, dB_ref.value, dB_ref.S, dt, "dB only (plan)", exact)


@pytest.mark.parametrize("dt", DTS)
def test_spgemm_bwd_plan_narrow_C(ck, dt):
    """csrk.h: with A's transpose plan, entries of C_i missing for some j of B_k count as
    dC_ij = 0.  C = the structural product of a 20x20 Poisson A with every third entry of each row
    dropped; dA and dB against the dense definition (dC_dense B^T) o mask(A), (A^T dC_dense) o
    mask(B), exact for integer data."""
    A = synth.poisson2d(20, dtype=dt)
    rng = np.random.default_rng(21)
    A = A.with_values(synth.int_values(rng, A.nnz, dt))
    Ad = dev(ck, A)
    C = ck.spgemm_symbolic(Ad, Ad)
    Cp, Ci = C.indptr.cpu().numpy(), C.indices.cpu().numpy()
    keep = np.ones(Ci.size, bool)
    for r in range(A.nrows):
        keep[Cp[r] + 1:Cp[r + 1]:3] = False
    Cp2 = np.zeros_like(Cp)
    Cp2[1:] = np.cumsum([keep[Cp[r]:Cp[r + 1]].sum() for r in range(A.nrows)])
    Ci2 = Ci[keep]
    C2 = ck.CSR.from_host(synth.CSR(A.nrows, A.ncols, Cp2, Ci2, np.zeros(Ci2.size, dt)))
    dC = synth.int_values(rng, Ci2.size, dt)
    n = A.nrows
    Dd = np.zeros((n, n))
    Dd[np.repeat(np.arange(n), np.diff(Cp2)), Ci2] = dC
    Ad_dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(A.indptr))
    Ad_dense[rows, A.indices] = A.values
    dA_ref = (Dd @ Ad_dense.T)[rows, A.indices]
    dB_ref = (Ad_dense.T @ Dd)[rows, A.indices]
    plan = ck.csr_transpose(Ad, with_values=False)
    dA, dB = ck.spgemm_bwd(Ad, Ad, C2, t(dC), plan=plan)
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref.astype(dt))
    np.testing.assert_array_equal(dB.cpu().numpy(), dB_ref.astype(dt))


@pytest.mark.parametrize("case", ["powerlaw_16k", "skew_big", "poisson3d_17"])
@pytest.mark.parametrize("dt", DTS)
def test_spgemm_dB_plan_bitwise_reproducible(ck, orc, case, dt):
    """The plan dB has no atomics: ten runs give the same bits (reading A7/A9), and they agree
    with the oracle; the atomic path is only required to agree within the S rule."""
    A, B = gemm_operands(case, dt, "real")
    Ad, Bd = dev(ck, A), dev(ck, B)
    C = ck.spgemm_symbolic(Ad, Bd)
    dC = synth.dense(C.nnz, 17, dt)
    plan = ck.csr_transpose(Ad, with_values=False)
    runs = [ck.spgemm_bwd(Ad, Bd, C, t(dC), need_dA=False, plan=plan)[1].cpu().numpy() for _ in range(10)]
    for r in runs[1:]:
        np.testing.assert_array_equal(r, runs[0])
    _, dB_ref = orc.spgemm_bwd(A, B, C.indptr.cpu().numpy(), C.indices.cpu().numpy(), dC)
    close(runs[0], dB_ref.value, dB_ref.S, dt, "dB (plan)")


def test_spgemm_fig3(ck, orc):
    """PAPER Fig. 3: the printed 9x3 product pattern, on the GPU."""
    from util import csr_from_pattern, load_fig3, pattern_dense
    mats, _ = load_fig3()
    A, B = csr_from_pattern(mats["A"]), csr_from_pattern(mats["B"])
    C = ck.spgemm_symbolic(dev(ck, A), dev(ck, B))
    got = synth.CSR(9, 3, C.indptr.cpu().numpy(), C.indices.cpu().numpy(), np.ones(C.nnz))
    np.testing.assert_array_equal(pattern_dense(got), mats["C"])


def test_launch_counter_advances(ck):
    before = ck.launch_count()
    A = dev(ck, synth.poisson2d(8))
    ck.spmv_fwd(A, torch.ones(64, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    assert ck.launch_count() > before


def test_spgemm_symbolic_interleaved_calls(ck, orc):
    """The fill call reuses the columns its count call left in the workspace only when it is
    the fill of the LAST count on that workspace (csrk.h): count(A1), count(A2), fill(A1),
    fill(A2), fill(A2) on one workspace must all equal the oracle (A1's fill and the second
    fill of A2 merge again; the first fill of A2 copies)."""
    import ctypes
    from paper_2212_05159_b200.csrk import _check, _ptr, _stream, _workspace, lib
    A1, A2 = synth.poisson2d(40), synth.random_csr(1600, 1600, 0.002, 5)
    d1, d2 = dev(ck, A1), dev(ck, A2)
    ws, wsb = _workspace("spgemm_symbolic", 0, d1, d1)
    ws2, wsb2 = _workspace("spgemm_symbolic", 0, d2, d2)
    assert ws.value == ws2.value and wsb >= wsb2
    out = {}
    for name, D in (("A1", d1), ("A2", d2)):
        Cp = torch.empty(D.nrows + 1, dtype=torch.int64, device="cuda")
        nnz = ctypes.c_int64(0)
        _check(lib().csrk_spgemm_symbolic(D.pattern(), D.pattern(), _ptr(Cp), None, ctypes.byref(nnz), ws, wsb,
                                          _stream()), "count")
        out[name] = (Cp, int(nnz.value))
    for name, D, H in (("A1", d1, A1), ("A2", d2, A2), ("A2", d2, A2)):
        Cp, nnz = out[name]
        Ci = torch.full((nnz,), -1, dtype=torch.int32, device="cuda")
        _check(lib().csrk_spgemm_symbolic(D.pattern(), D.pattern(), _ptr(Cp), _ptr(Ci), None, ws, wsb, _stream()),
               "fill")
        rp, ri = orc.spgemm_symbolic(H, H)
        np.testing.assert_array_equal(Cp.cpu().numpy(), rp)
        np.testing.assert_array_equal(Ci.cpu().numpy(), ri)
