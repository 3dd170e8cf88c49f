"""SPAI workload (PAPER 4.6 P:1071-1102).

CPU pins of the oracle (oracle/spai.py): the paper's column decomposition of the loss
(P:1079-1082), closed forms (A = I and A = diag(d)), the classical per-row
least-squares SPAI at which the gradient must vanish, and exact central
finite differences (the loss is quadratic in M.values).  GPU parity of csrk_spai_loss_grad
against the oracle is at the bottom (marked gpu).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import spai as osp
from util import assert_S_close, gather_mask, pattern_dense, to_dense


def ones_on(A):
    """M = mask(A): all stored entries 1 (the paper's initialisation)."""
    return A.with_values(np.ones(A.nnz))


def test_spai_identity_and_diagonal_closed_forms():
    n = 7
    I = np.eye(n)
    loss, g = osp.spai_loss_grad(I, I.astype(bool), I)          # A = I: M = I is exact
    assert loss == 0.0 and not g.any()
    d = np.array([2.0, -4.0, 0.5, 8.0, 1.0, -0.25, 16.0])        # powers of 2: exact inverses
    D = np.diag(d)
    loss, g = osp.spai_loss_grad(D, D != 0, np.diag(1.0 / d))   # A = diag(d): M = diag(1/d)
    assert loss == 0.0 and not g.any()
    np.testing.assert_array_equal(osp.spai_reference(D, D != 0), np.diag(1.0 / d))


@pytest.mark.parametrize("N", [4, 8])
def test_spai_loss_column_decomposition(N):
    A = synth.poisson2d(N)
    Ad, P = to_dense(A), pattern_dense(A)
    M = to_dense(A.with_values(np.random.default_rng(N).uniform(-1, 1, A.nnz)))
    loss, _ = osp.spai_loss_grad(Ad, P, M)
    assert abs(loss - osp.spai_loss_by_columns(Ad, M)) <= 1e-12 * loss


def test_spai_gradient_vanishes_at_least_squares_reference():
    """The per-row least-squares solution minimises the loss over the pattern, so the
    autodiff gradient there is zero (up to rounding)."""
    A = synth.poisson2d(8)                                       # the paper's 64 x 64
    Ad, P = to_dense(A), pattern_dense(A)
    Mref = osp.spai_reference(Ad, P)
    loss_ref, g = osp.spai_loss_grad(Ad, P, Mref)
    assert np.abs(g).max() < 1e-10
    loss0, _ = osp.spai_loss_grad(Ad, P, to_dense(ones_on(A)))  # the paper's start point
    assert loss_ref < loss0


def test_spai_S_bounds_the_oracle_against_a_reordered_evaluation():
    """The S-scales bound the difference between two evaluation orders of the same quantities:
    the oracle (autograd of M A) and the column decomposition / explicit -2 (R A^T) form."""
    A = synth.poisson2d(8)
    Ad, P = to_dense(A), pattern_dense(A)
    M = to_dense(A.with_values(np.random.default_rng(3).uniform(-1, 1, A.nnz)))
    loss, g = osp.spai_loss_grad(Ad, P, M)
    S_loss, S_dM = osp.spai_S(Ad, P, M)
    assert abs(loss - osp.spai_loss_by_columns(Ad, M)) <= 1e-14 * S_loss
    R = np.eye(Ad.shape[0]) - M @ Ad
    g2 = np.where(P, -2.0 * (R @ Ad.T), 0.0)
    assert np.all(np.abs(g - g2) <= 1e-14 * S_dM)
    assert np.all(np.abs(g) <= S_dM * (1 + 1e-12)) and abs(loss) <= S_loss


def test_spai_gradient_exact_fd():
    """l is quadratic in M.values: the central difference at h = 1 is exact on integer data."""
    A = synth.poisson2d(4)
    Ad, P = to_dense(A), pattern_dense(A)
    Mv = np.random.default_rng(2).integers(-3, 4, A.nnz).astype(np.float64)
    M = to_dense(A.with_values(Mv))
    _, g = osp.spai_loss_grad(Ad, P, M)
    gv = gather_mask(g, A.indptr, A.indices)
    for q in range(A.nnz):
        e = np.zeros(A.nnz)
        e[q] = 1.0
        lp, _ = osp.spai_loss_grad(Ad, P, to_dense(A.with_values(Mv + e)))
        lm, _ = osp.spai_loss_grad(Ad, P, to_dense(A.with_values(Mv - e)))
        assert (lp - lm) / 2 == gv[q]


# ---------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["poisson8_ones", "poisson8_random", "poisson16_random", "poisson3d_6_random",
                                  "random_diag", "lstsq_reference"])
def test_spai_gpu_parity(ck, case):
    if case.startswith("poisson3d"):
        A = synth.poisson3d(6)
    elif case == "random_diag":
        R = synth.random_csr(200, 200, 0.03, 5, np.float64, "real")
        A = synth.CSR(200, 200, *_with_diag(R))
    else:
        A = synth.poisson2d(16 if "16" in case else 8)
    Ad, P = to_dense(A), pattern_dense(A)
    if case.endswith("ones"):
        Mv = np.ones(A.nnz)
    elif case == "lstsq_reference":
        Mv = gather_mask(osp.spai_reference(Ad, P), A.indptr, A.indices)
    else:
        Mv = np.random.default_rng(7).uniform(-1, 1, A.nnz)
    loss_ref, g = osp.spai_loss_grad(Ad, P, to_dense(A.with_values(Mv)))
    gref = gather_mask(g, A.indptr, A.indices)
    A_d = ck.CSR.from_host(A)
    M_d = ck.CSR.from_host(A.with_values(Mv))
    plan = ck.spai_plan(M_d, A_d)
    loss, dM = ck.spai_loss_grad(plan, M_d, A_d)
    # elementwise S-rule of reading A6 with the composed magnitudes of oracle.spai.spai_S
    S_loss, S_dM = osp.spai_S(Ad, P, to_dense(A.with_values(Mv)))
    assert abs(loss - loss_ref) <= 1e-12 * S_loss
    assert_S_close(dM.cpu().numpy(), gref, gather_mask(S_dM, A.indptr, A.indices), 1e-12, f"{case} dM")


def _with_diag(R):
    """R + I pattern (a diagonal entry in every row), values: R's, diagonal 4."""
    rows = []
    for i in range(R.nrows):
        c = list(R.indices[R.indptr[i]:R.indptr[i + 1]])
        v = list(R.values[R.indptr[i]:R.indptr[i + 1]])
        if i not in c:
            c.append(i)
            v.append(4.0)
        o = np.argsort(c)
        rows.append((np.array(c)[o], np.array(v)[o]))
    indptr = np.zeros(R.nrows + 1, np.int64)
    np.cumsum([len(c) for c, _ in rows], out=indptr[1:])
    return indptr, np.concatenate([c for c, _ in rows]).astype(np.int32), np.concatenate([v for _, v in rows])
