"""GPU parity for SpTRSV (PAPER 3.1.5 P:477-488) through the C-ABI against
the oracle: x within |gpu - orc| <= rtol S, S = M(T)^{-1}|T||x| (DESIGN reading R-TRSV);
integer systems built as b = T x_int solve exactly; db like x (on T^T); dT = -(db) x^T (.) mask(T)
within rtol S_db |x|.  Covers both device paths: the chain scan (bidiagonal L of PAPER 4.3
P:857, the triangle of A_N of Table 2) across many tiles, and the sync-free solve
(random, banded, wavefront Poisson triangles), lower and upper, unit and stored diagonals,
with and without a transpose plan, fp64 and fp32, plus config-5's full 4096^2 L."""
import numpy as np
import pytest
import torch

import synth
from util import assert_S_close, to_dense

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


def flip_T(orc, T):
    """T^T as a synth.CSR (values kept) -- lower <-> upper."""
    p, i, v, _ = orc.csr_transpose(T)
    return synth.CSR(T.ncols, T.nrows, p, i, v)


def cases(orc):
    P2 = synth.lower_part(synth.poisson2d(96))              # IC(0) pattern: wavefront, sync-free
    PL = synth.lower_part(synth.poisson1d(2048 * 5 + 77))   # chain across 6 tiles
    BL = synth.bidiag_lower(2048 * 3 + 5, "seeded")         # PCG L
    return {
        "random_dense_rows": synth.tri_random(700, 0.05, 1),
        "banded": synth.tri_banded(20000, 6, 300, 2),
        "banded_long_band": synth.tri_banded(5000, 3, 5000, 3),
        "poisson2d_lower": P2,
        "poisson1d_chain": PL,
        "bidiag_chain": BL,
        "chain_then_general": _chain_then_general(),
        "single": synth.CSR(1, 1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([-2.5])),
    }


def _chain_then_general():
    """Bidiagonal for the first 5000 rows, one long-range dependency afterwards: the chain
    pass must abort and the sync-free pass must solve everything."""
    B = synth.bidiag_lower(9000, "seeded")
    D = synth.tri_banded(9000, 1, 4000, 4)
    rows_b = np.repeat(np.arange(9000), np.diff(B.indptr))
    rows_d = np.repeat(np.arange(9000), np.diff(D.indptr))
    keep_d = (rows_d == 7000) & (D.indices < rows_d - 1)
    r = np.concatenate([rows_b, rows_d[keep_d]])
    c = np.concatenate([B.indices, D.indices[keep_d]])
    v = np.concatenate([B.values, D.values[keep_d] * 0.05])
    o = np.lexsort((c, r))
    indptr = np.zeros(9001, np.int64)
    np.cumsum(np.bincount(r, minlength=9000), out=indptr[1:])
    return synth.CSR(9000, 9000, indptr, c[o].astype(np.int32), v[o])


def as_dtype(T, dt):
    return T.with_values(T.values.astype(dt))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("case", ["random_dense_rows", "banded", "banded_long_band", "poisson2d_lower",
                                  "poisson1d_chain", "bidiag_chain", "chain_then_general", "single"])
def test_sptrsv_parity(ck, orc, case, upper, dt):
    T = cases(orc)[case]
    if upper:
        T = flip_T(orc, T)
    T = as_dtype(T, dt)
    n = T.nrows
    b = synth.dense(n, 11, dt)
    v = synth.dense(n, 12, dt)
    Td = ck.CSR.from_host(T)
    x = ck.sptrsv_fwd(Td, torch.from_numpy(b).cuda(), upper=upper)
    r = orc.sptrsv(T, b, upper=upper)
    xg = x.cpu().numpy()
    assert_S_close(xg, r.value, r.S, RTOL[dt], f"{case} x")
    # backward from the same x on both sides (the GPU's own forward output)
    for plan in (None, ck.csr_transpose(Td)):
        dT, db = ck.sptrsv_bwd(Td, x, torch.from_numpy(v).cuda(), upper=upper, plan=plan)
        dT_ref, db_ref = orc.sptrsv_bwd(T, xg, v, upper=upper)
        assert_S_close(db.cpu().numpy(), db_ref.value, db_ref.S, RTOL[dt], f"{case} db")
        rows = np.repeat(np.arange(n), np.diff(T.indptr))
        scale = db_ref.S[rows] * np.abs(xg[T.indices].astype(np.float64))
        # reading R-TRSV: dT = -db_i x_j with x an exact input; the GPU forms it from db already
        # rounded to dtype (u |db_i||x_j| = u |dT|) plus the product's own rounding (u |dT|), so
        # fp32 adds 2 u32 |dT| = 2^-23 |dT| to rtol S_db,i |x_j| (fp64: 2 u64 |dT|, below rtol S)
        u2 = 2.0 ** -23 if dt == np.float32 else 2.0 ** -52
        assert_S_close(dT.cpu().numpy(), dT_ref, scale + (u2 / RTOL[dt]) * np.abs(dT_ref), RTOL[dt],
                       f"{case} dT")


@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("unit", [False, True])
@pytest.mark.parametrize("gen", ["random", "banded"])
def test_sptrsv_integer_exact(ck, orc, gen, upper, unit):
    """b = T x_int with integer T (diagonal in {+-1, +-2, +-4} or unit): exact on both sides."""
    if gen == "random":
        T = synth.tri_random(600, 0.02, 21, upper=upper, values="int", unit=unit)
    else:
        T = synth.tri_banded(30000, 2, 40, 22, upper=upper, values="int", unit=unit)
    xi = synth.dense(T.nrows, 23, values="int")
    rows = np.repeat(np.arange(T.nrows), np.diff(T.indptr))
    vals = T.values.copy()
    if unit:
        vals[rows == T.indices] = 1.0
    b = np.zeros(T.nrows)
    np.add.at(b, rows, vals * xi[T.indices])
    if unit:
        b += xi * (1 - np.bincount(rows[rows == T.indices], minlength=T.nrows))
    Td = ck.CSR.from_host(T)
    x = ck.sptrsv_fwd(Td, torch.from_numpy(b).cuda(), upper=upper, unit=unit).cpu().numpy()
    np.testing.assert_array_equal(x, orc.sptrsv(T, b, upper=upper, unit=unit).value)
    np.testing.assert_array_equal(x, xi)


def test_sptrsv_poisson1d_closed_form(ck):
    """Triangle of A_N at the size of the paper's Table 2 (32768): b = 1 gives
    x_i = 1 - 2^-(i+1) (exact dyadic; 1.0 once i >= 53) -- through the chain pass."""
    n = 32768
    L = synth.lower_part(synth.poisson1d(n))
    x = ck.sptrsv_fwd(ck.CSR.from_host(L), torch.ones(n, dtype=torch.float64, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(x, 1.0 - 2.0 ** -(np.arange(n) + 1.0))


def test_sptrsv_unit_and_wrong_side(ck, orc):
    """unit_diag ignores a stored diagonal (and gives it zero gradient); entries on the wrong side
    of the diagonal are ignored by the solve."""
    T = synth.tri_random(300, 0.05, 31)
    b, v = synth.dense(300, 32), synth.dense(300, 33)
    Td = ck.CSR.from_host(T)
    x = ck.sptrsv_fwd(Td, torch.from_numpy(b).cuda(), unit=True)
    r = orc.sptrsv(T, b, unit=True)
    assert_S_close(x.cpu().numpy(), r.value, r.S, 1e-12, "unit x")
    dT, _ = ck.sptrsv_bwd(Td, x, torch.from_numpy(v).cuda(), unit=True)
    rows = np.repeat(np.arange(300), np.diff(T.indptr))
    assert not dT.cpu().numpy()[rows == T.indices].any()
    # add an upper entry to every 7th row: the lower solve must not change
    D = to_dense(T)
    for i in range(0, 299, 7):
        D[i, i + 1] = 5.0
    rr, cc = np.nonzero(D)
    W = synth.CSR(300, 300, np.concatenate([[0], np.cumsum(np.bincount(rr, minlength=300))]).astype(np.int64),
                  cc.astype(np.int32), D[rr, cc])
    xw = ck.sptrsv_fwd(ck.CSR.from_host(W), torch.from_numpy(b).cuda())
    r = orc.sptrsv(T, b)
    assert_S_close(xw.cpu().numpy(), r.value, r.S, 1e-12, "wrong-side entries ignored")


def test_sptrsv_empty(ck):
    T = synth.CSR(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    Td = ck.CSR.from_host(T)
    x = ck.sptrsv_fwd(Td, torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert x.numel() == 0


def test_sptrsv_config5_L_full(ck, orc):
    """Config 5's lower-bidiagonal L (PAPER 4.3 P:857; 4096^2 = 16,777,216 rows) and its L^T --
    the solves that apply M^{-1} = (L L^T)^{-1} exactly -- against the oracle on every row."""
    n = 4096 * 4096
    L = synth.bidiag_lower(n, "seeded")
    b = synth.dense(n, synth.seed_of(5, 3))
    Ld = ck.CSR.from_host(L)
    bt = torch.from_numpy(b).cuda()
    x = ck.sptrsv_fwd(Ld, bt)
    r = orc.sptrsv(L, b)
    assert_S_close(x.cpu().numpy(), r.value, r.S, 1e-12, "L x = b")
    dT, db = ck.sptrsv_bwd(Ld, x, bt)  # db = L^{-T} b through the upper chain
    _, db_ref = orc.sptrsv_bwd(L, x.cpu().numpy(), b, want_dT=False)
    assert_S_close(db.cpu().numpy(), db_ref.value, db_ref.S, 1e-12, "L^T w = v")
