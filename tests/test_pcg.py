"""Config-5 composition (PAPER 4.3 P:825-862): the learned-preconditioner
PCG training step.  CPU pins of the oracle (oracle/pcg.py: dense torch autograd of the
algorithm) and GPU parity of csrk_pcg_loss_grad (hand adjoint over the CUDA kernels)."""
import numpy as np
import pytest
import scipy.sparse as sps
import scipy.sparse.linalg as spla
import torch

import synth
from util import pattern_dense, to_dense


def problem(N, init):
    A = synth.poisson2d(N)
    L = synth.bidiag_lower(A.nrows, init)
    b = np.full(A.nrows, 1.0 / np.sqrt(A.nrows))     # b = 1/||1||
    return A, L, b


# ---------------------------------------------------------------- CPU pins of the oracle
def test_loss_weights_paper_values():
    from oracle import pcg
    w = pcg.loss_weights(4, 0.6)       # N_it = 4, gamma = 0.6
    np.testing.assert_allclose(w, [0.0993, 0.1654, 0.2757, 0.4596], atol=5e-5)
    assert abs(w.sum() - 1.0) < 1e-15


def test_identity_preconditioner_is_cg():
    """L = I  =>  PCG == CG: residual history equals scipy's CG."""
    from oracle import pcg
    A, L, b = problem(8, "identity")   # the paper's 8x8 grid, A in R^{64x64}
    loss, res, _ = pcg.pcg_loss_grad(to_dense(A), pattern_dense(L), to_dense(L), b, 6, 0.6)
    As = sps.csr_matrix((A.values, A.indices, A.indptr), shape=(64, 64))
    xs = []
    spla.cg(As, b, x0=np.zeros(64), rtol=1e-30, maxiter=6, callback=lambda xk: xs.append(xk.copy()))
    ref = [np.linalg.norm(b - As @ xk) for xk in xs]
    np.testing.assert_allclose(res, ref[:6], rtol=1e-10)


def test_oracle_gradient_finite_differences():
    """Central differences of the oracle loss on stored entries of L (h = 1e-6 max(1,|theta|))."""
    from oracle import pcg
    A, L, b = problem(6, "seeded")
    Ad, P, Lv = to_dense(A), pattern_dense(L), to_dense(L)
    _, _, g = pcg.pcg_loss_grad(Ad, P, Lv, b, 4, 0.6)
    rows = np.repeat(np.arange(L.nrows), np.diff(L.indptr))
    rng = np.random.default_rng(0)
    for e in rng.choice(L.nnz, 8, replace=False):
        i, j = rows[e], L.indices[e]
        h = 1e-6 * max(1.0, abs(Lv[i, j]))
        Lp, Lm = Lv.copy(), Lv.copy()
        Lp[i, j] += h
        Lm[i, j] -= h
        fd = (pcg.pcg_loss_grad(Ad, P, Lp, b, 4, 0.6)[0] - pcg.pcg_loss_grad(Ad, P, Lm, b, 4, 0.6)[0]) / (2 * h)
        assert abs(fd - g[i, j]) <= 1e-6 * max(1.0, abs(g[i, j])), (e, fd, g[i, j])
    assert np.all(g[~P] == 0)


# ---------------------------------------------------------------- CPU pins (orientation, sparse oracle)
def _inverse_factor_case(N=5):
    """L = chol(A^{-1}) (lower, dense lower pattern) so that L L^T = A^{-1} exactly."""
    from util import csr_from_pattern
    A = synth.poisson2d(N)
    Ad = to_dense(A)
    Lc = np.linalg.cholesky(np.linalg.inv(Ad))
    P = np.tril(np.ones_like(Ad)).astype(bool)
    return A, Ad, P, Lc, csr_from_pattern(P, Lc[P])


def test_pcg_mult_inverse_factor_converges_in_one_step(orc):
    """P:838 M = L L^T.  With L = chol(A^{-1}) the preconditioner is A^{-1}, so the first PCG step
    solves A x = b: ||r^(1)|| vanishes to rounding.  An oracle that applied L^T L instead would
    not converge (checked: same L passed transposed gives ||r^(1)|| / ||b|| ~ 0.17).  Pins both the
    dense and the sparse oracle."""
    from oracle import pcg
    A, Ad, P, Lc, Ls = _inverse_factor_case()
    b = synth.dense(A.nrows, 3)
    nb = np.linalg.norm(b)
    _, res, _ = pcg.pcg_loss_grad(Ad, P, Lc, b, 3, 0.6)
    assert res[0] <= 1e-13 * nb
    _, res_s, _, _ = pcg.pcg_loss_grad_sparse(A, Ls, b, 3, 0.6)
    assert res_s[0] <= 1e-13 * nb
    _, res_t, _ = pcg.pcg_loss_grad(Ad, P.T, Lc.T, b, 3, 0.6)     # L^T L: the wrong orientation
    assert res_t[0] >= 1e-2 * nb


@pytest.mark.parametrize("precond", ["mult", "solve"])
@pytest.mark.parametrize("N,init,n_it", [(6, "seeded", 4), (8, "identity", 6), (16, "seeded", 50),
                                         (24, "seeded", 30)])
def test_sparse_oracle_matches_dense_oracle(orc, N, init, n_it, precond):
    """The CSR oracle (C oracle products under torch autograd) against the dense torch oracle:
    loss, residual history and dL elementwise on the S-scale of the sparse oracle."""
    from oracle import pcg
    A, L, b = problem(N, init)
    l1, r1, g1 = pcg.pcg_loss_grad(to_dense(A), pattern_dense(L), to_dense(L), b, n_it, 0.6, precond=precond)
    l2, r2, g2, S = pcg.pcg_loss_grad_sparse(A, L, b, n_it, 0.6, precond=precond)
    rows = np.repeat(np.arange(L.nrows), np.diff(L.indptr))
    assert abs(l1 - l2) <= 1e-11 * abs(l1)
    np.testing.assert_allclose(r2, r1, rtol=1e-10)
    assert np.all(np.abs(g1[rows, L.indices] - g2) <= 1e-11 * S)
    assert np.all(np.abs(g2) <= S * (1 + 1e-12))          # S bounds the gradient it scales


def test_sparse_oracle_identity_is_cg(orc):
    """L = I: the sparse oracle's residual history equals scipy's CG."""
    from oracle import pcg
    A, L, b = problem(10, "identity")
    _, res, _, _ = pcg.pcg_loss_grad_sparse(A, L, b, 8, 0.6)
    As = sps.csr_matrix((A.values, A.indices, A.indptr), shape=(A.nrows, A.nrows))
    xs = []
    spla.cg(As, b, x0=np.zeros(A.nrows), rtol=1e-30, maxiter=8, callback=lambda xk: xs.append(xk.copy()))
    np.testing.assert_allclose(res, [np.linalg.norm(b - As @ xk) for xk in xs][:8], rtol=1e-10)


def test_sparse_oracle_finite_differences(orc):
    """Central differences of the sparse oracle's loss on stored entries of L."""
    from oracle import pcg
    A, L, b = problem(7, "seeded")
    _, _, g, _ = pcg.pcg_loss_grad_sparse(A, L, b, 5, 0.6)
    for q in range(0, L.nnz, 7):
        h = 1e-6
        Lp, Lm = L.values.copy(), L.values.copy()
        Lp[q] += h
        Lm[q] -= h
        fd = (pcg.pcg_loss_grad_sparse(A, L.with_values(Lp), b, 5, 0.6, want_S=False)[0]
              - pcg.pcg_loss_grad_sparse(A, L.with_values(Lm), b, 5, 0.6, want_S=False)[0]) / (2 * h)
        assert abs(fd - g[q]) <= 1e-6 * max(1.0, abs(fd)), (q, fd, g[q])


# ---------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def _pcg_parity(ck, A, L, b, n_it, precond, rtol=1e-12, margin=20.0):
    """GPU csrk_pcg_loss_grad vs the sparse oracle (DESIGN reading R-PCG):
      dL elementwise:  |gpu - orc| <= tau * S_dL,    loss / residuals: relative tau_l / tau_r,
      tau = max(rtol, margin * kappa), kappa = the oracle's own response to b perturbed by
      ~5 ulps (relative 1e-15 N(0,1)), measured on the same rule -- n_it chained CG steps amplify
      rounding-level differences, so both sides agree to the extent the algorithm is stable."""
    from oracle import pcg
    loss_ref, res_ref, g_ref, S = pcg.pcg_loss_grad_sparse(A, L, b, n_it, 0.6, precond=precond)
    bp = b * (1.0 + 1e-15 * np.random.default_rng(1).standard_normal(b.shape))
    loss_alt, res_alt, g_alt, _ = pcg.pcg_loss_grad_sparse(A, L, bp, n_it, 0.6, want_S=False, precond=precond)
    res_ref, res_alt = np.array(res_ref), np.array(res_alt)
    Sg = np.where(S > 0, S, 1.0)
    tau_g = max(rtol, margin * float(np.max(np.abs(g_alt - g_ref) / Sg)))
    tau_l = max(rtol, margin * abs(loss_alt - loss_ref) / abs(loss_ref))
    tau_r = max(rtol, margin * float(np.max(np.abs(res_alt - res_ref) / res_ref)))
    del g_alt
    Ad, Ld = ck.CSR.from_host(A), ck.CSR.from_host(L)
    loss, res, dL = ck.pcg_loss_grad(Ad, Ld, torch.from_numpy(b).cuda(), n_it, 0.6, precond=precond)
    assert abs(loss - loss_ref) <= tau_l * abs(loss_ref), (loss, loss_ref, tau_l)
    np.testing.assert_allclose(res, res_ref, rtol=tau_r)
    got = dL.cpu().numpy()
    err = np.abs(got - g_ref)
    assert np.all(err <= tau_g * S), (float(np.max(err / Sg)), tau_g)
    return tau_g, tau_l, tau_r


@pytest.mark.gpu
@pytest.mark.parametrize("precond", ["mult", "solve"])
@pytest.mark.parametrize("N,init,n_it", [(8, "identity", 4), (8, "seeded", 4), (16, "seeded", 50),
                                         (32, "identity", 50), (40, "seeded", 50), (128, "seeded", 50)])
def test_pcg_gpu_vs_oracle(ck, N, init, n_it, precond):
    """Elementwise S-rule parity of the loss, the residual history and dL (R-PCG)."""
    A, L, b = problem(N, init)
    _pcg_parity(ck, A, L, b, n_it, precond)


@pytest.mark.gpu
def test_pcg_gpu_inverse_factor_one_step(ck):
    """The orientation pin on the GPU: L = chol(A^{-1}) => ||r^(1)|| ~ 0 (M = L L^T = A^{-1})."""
    A, Ad, P, Lc, Ls = _inverse_factor_case()
    b = synth.dense(A.nrows, 3)
    _, res, _ = ck.pcg_loss_grad(ck.CSR.from_host(A), ck.CSR.from_host(Ls), torch.from_numpy(b).cuda(), 3, 0.6)
    assert res[0] <= 1e-13 * np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("precond", ["mult", "solve"])
def test_pcg_config5_vs_sparse_oracle(ck, precond):
    """BASELINE config 5 at full size (2D Poisson 4096^2, lower-bidiagonal L, 50 iterations) against
    the sparse oracle on the host (all cores): loss, residual history and dL elementwise (R-PCG)."""
    import oracle
    oracle.set_threads(len(__import__("os").sched_getaffinity(0)))
    A, L, b = problem(4096, "seeded")
    assert A.nnz == 83869696 and L.nnz == 33554431
    try:
        tau_g, tau_l, tau_r = _pcg_parity(ck, A, L, b, 50, precond)
    finally:
        oracle.set_threads(1)
    assert tau_g < 1e-9 and tau_l < 1e-9 and tau_r < 1e-9, (tau_g, tau_l, tau_r)   # a well-posed case


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("precond", ["mult", "solve"])
def test_pcg_config5_directional_derivative(ck, precond):
    """Config 5 at full size: the gradient also agrees with a central difference of the GPU loss
    along a random direction of L.values (a second, oracle-free check of the hand adjoint)."""
    A, L, b = problem(4096, "seeded")
    Ad, Ld = ck.CSR.from_host(A), ck.CSR.from_host(L)
    bt = torch.from_numpy(b).cuda()
    loss, res, dL = ck.pcg_loss_grad(Ad, Ld, bt, 50, 0.6, precond=precond)
    assert np.isfinite(loss) and all(np.isfinite(res))
    V = torch.from_numpy(synth.dense(L.nnz, 77)).cuda()
    h = 1e-6
    base = Ld.values.clone()
    Ld.values.copy_(base + h * V)
    lp, _, _ = ck.pcg_loss_grad(Ad, Ld, bt, 50, 0.6, precond=precond)
    Ld.values.copy_(base - h * V)
    lm, _, _ = ck.pcg_loss_grad(Ad, Ld, bt, 50, 0.6, precond=precond)
    fd = (lp - lm) / (2 * h)
    dd = float((dL * V).sum())
    assert abs(fd - dd) <= 1e-6 * max(abs(dd), 1e-12), (fd, dd)


# ---------------------------------------------------------------- precond="solve"
from oracle import pcg  # noqa: E402
def test_pcg_solve_identity_is_cg(orc):
    """L = I: M = (L L^T)^{-1} = I, the same CG as the multiplicative form with L = I."""
    A = synth.poisson2d(6)
    L = synth.bidiag_lower(A.nrows, "identity")
    b = np.full(A.nrows, 1.0 / np.sqrt(A.nrows))
    args = (to_dense(A), pattern_dense(L), to_dense(L), b, 5, 0.6)
    l1, r1, _ = pcg.pcg_loss_grad(*args)
    l2, r2, _ = pcg.pcg_loss_grad(*args, precond="solve")
    assert abs(l1 - l2) <= 1e-14 * abs(l1)
    np.testing.assert_allclose(r2, r1, rtol=1e-13)


def test_pcg_solve_exact_cholesky_converges_in_one_step(orc):
    """L = chol(A) (dense lower pattern): M = A^{-1}, so the first PCG step solves A x = b and the
    residual after it vanishes (to rounding) -- exact preconditioning."""
    A = synth.poisson2d(5)
    Ad = to_dense(A)
    Lc = np.linalg.cholesky(Ad)
    P = np.tril(np.ones_like(Ad)).astype(bool)
    b = synth.dense(A.nrows, 3)
    _, res, _ = pcg.pcg_loss_grad(Ad, P, Lc, b, 3, 0.6, precond="solve")
    assert res[0] <= 1e-12 * np.linalg.norm(b)


def test_pcg_solve_diagonal_matches_mult(orc):
    """L = D diagonal: (L L^T)^{-1} = D^{-2} = (D^{-1})(D^{-1})^T, so precond="solve" with D and the
    multiplicative form with D^{-1} run the same PCG."""
    A = synth.poisson2d(6)
    n = A.nrows
    d = np.random.default_rng(4).uniform(0.5, 2.0, n)
    P = np.eye(n, dtype=bool)
    b = synth.dense(n, 5)
    l1, r1, _ = pcg.pcg_loss_grad(to_dense(A), P, np.diag(d), b, 6, 0.6, precond="solve")
    l2, r2, _ = pcg.pcg_loss_grad(to_dense(A), P, np.diag(1.0 / d), b, 6, 0.6)
    assert abs(l1 - l2) <= 1e-12 * abs(l1)
    np.testing.assert_allclose(r1, r2, rtol=1e-11)


def test_pcg_solve_finite_differences(orc):
    """Central differences of the solve-preconditioned loss in the stored entries of a seeded
    bidiagonal L (nonlinear: h = 1e-6, rel 1e-6)."""
    A = synth.poisson2d(5)
    L = synth.bidiag_lower(A.nrows, "seeded")
    b = np.full(A.nrows, 1.0 / np.sqrt(A.nrows))
    Ad, P, Lv = to_dense(A), pattern_dense(L), to_dense(L)
    _, _, g = pcg.pcg_loss_grad(Ad, P, Lv, b, 4, 0.6, precond="solve")
    rows = np.repeat(np.arange(L.nrows), np.diff(L.indptr))
    h = 1e-6
    for q in range(0, L.nnz, 5):
        i, j = rows[q], L.indices[q]
        Lp, Lm = Lv.copy(), Lv.copy()
        Lp[i, j] += h
        Lm[i, j] -= h
        fd = (pcg.pcg_loss_grad(Ad, P, Lp, b, 4, 0.6, precond="solve")[0]
              - pcg.pcg_loss_grad(Ad, P, Lm, b, 4, 0.6, precond="solve")[0]) / (2 * h)
        assert abs(fd - g[i, j]) <= 1e-6 * max(1.0, abs(fd)), (i, j)
