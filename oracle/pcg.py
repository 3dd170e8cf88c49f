"""oracle.pcg -- TEST INFRASTRUCTURE ONLY.

Config-5 composition: the learned-preconditioner PCG training step of
PAPER 4.3, written as the algorithm step by step in plain dense PyTorch (CPU,
float64) and differentiated by torch autograd -- no hand-derived adjoint, so it checks the
CUDA path's hand adjoint independently.  Dense, so only for small n (n <= ~4096).

    M = L L^T, L lower triangular (bidiagonal in P:857)
    PCG on A x = b, x0 = 0: r0 = b, z0 = M r0, p0 = z0, rho0 = r0.z0
      q = A p; alpha = rho / (p.q); x += alpha p; r -= alpha q; record ||r||
      z = M r; rho' = r.z; p = z + (rho'/rho) p; rho = rho'
    loss = sum_{i=1}^{N_it} w_i ||r^(i)|| / ||b||,  w_i = gamma^(N_it - i) / sum_j gamma^(N_it - j)

pcg_loss_grad_sparse (below) is the same algorithm on CSR operands, for the full config-5 size
(4096^2 x 50 iterations): the sparse products are torch.autograd.Functions over the C oracle and
the reverse pass is torch autograd's; it also returns S_dL, the sum of |terms| added into each
dL entry (the S-scale of the elementwise rule, DESIGN reading R-PCG).

Pins (tests/test_pcg.py): the P:844 weights for N_it = 4, gamma = 0.6; L = I gives scipy's
CG history; L = chol(A^{-1}) (lower) makes M = L L^T = A^{-1}, so PCG converges in ONE step
-- the pin that fixes the orientation L L^T (an L^T L oracle does not converge); central finite
differences; the sparse and dense oracles agree elementwise; |dL| <= S_dL.

precond="solve" is the SpTRSV extension of SURVEY 8(f) row f3: M = (L L^T)^{-1} applied exactly by
two triangular solves, z = L^{-T} (L^{-1} r) (an incomplete-Cholesky-type preconditioner whose
factor L is learned with the same loss); the algorithm is otherwise unchanged.
"""
from __future__ import annotations

import numpy as np
import torch


def loss_weights(n_it: int, gamma: float) -> np.ndarray:
    """w_i, i = 1..N_it of P:844 (normalised geometric weights, later iterates heavier)."""
    raw = np.array([gamma ** (n_it - i) for i in range(1, n_it + 1)], dtype=np.float64)
    return raw / raw.sum()


def pcg_loss_grad(A_dense: np.ndarray, L_pattern_dense: np.ndarray, L_vals_dense: np.ndarray, b: np.ndarray,
                  n_it: int, gamma: float, reassociate: bool = False, precond: str = "mult"):
    """Returns (loss, residual norms [n_it], dL dense masked to L's pattern).
    reassociate=True applies M as (L L^T) v instead of L (L^T v): the same mathematics in a
    different rounding order, used by the tests to measure how strongly n_it chained CG steps
    amplify rounding (parity of the composition is judged against that sensitivity)."""
    A = torch.tensor(A_dense, dtype=torch.float64)
    mask = torch.tensor(L_pattern_dense.astype(np.float64))
    Lfull = torch.tensor(L_vals_dense, dtype=torch.float64, requires_grad=True)
    L = Lfull * mask                                   # gradient lives on mask(L)
    bt = torch.tensor(b, dtype=torch.float64)
    if precond == "solve":
        tri = torch.linalg.solve_triangular
        if reassociate:
            M = lambda v: torch.linalg.solve(L @ L.T, v)
        else:
            M = lambda v: tri(L.T, tri(L, v[:, None], upper=False), upper=True)[:, 0]
    elif reassociate:
        M = lambda v: (L @ L.T) @ v
    else:
        M = lambda v: L @ (L.T @ v)
    x = torch.zeros_like(bt)
    r = bt - A @ x
    z = M(r)
    p = z
    rho = r @ z
    res = []
    for _ in range(n_it):
        q = A @ p
        alpha = rho / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        res.append(torch.linalg.norm(r))
        z = M(r)
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    w = torch.tensor(loss_weights(n_it, gamma))
    loss = (w * torch.stack(res)).sum() / torch.linalg.norm(bt)
    loss.backward()
    grad = (Lfull.grad * mask).numpy()
    return float(loss.detach()), [float(v.detach()) for v in res], grad


# ------------------------------------------------------------------------------------------------
# Sparse composition oracle (full config-5 size): the same algorithm, step by step, in CPU torch
# float64 autograd whose sparse products are torch.autograd.Functions over the C oracle
# (csr_oracle.c: long-double row sums, the stable counting-sort transpose).  No hand adjoint: the
# reverse pass is torch autograd's.  Memory: autograd keeps ~5 n-vectors per iteration (~34 GB at
# 4096^2 x 50 iterations); time ~1-2 min on 16 cores.
# ------------------------------------------------------------------------------------------------
class SparseMat:
    """Fixed pattern M (m x n) plus the oracle's own transpose of it (stable counting sort,
    oracle.csr_transpose), so that M^T v is evaluated as the row sums of M^T: entries of each
    M^T row come in ascending row order of M, i.e. the serial scatter order of orc_spmv op 1."""

    def __init__(self, M):
        import oracle as _o
        from synth import CSR
        self.CSR = CSR
        self.M = M
        pat = CSR(M.nrows, M.ncols, M.indptr, M.indices, None)
        self.ATp, self.ATi, _, self.perm = _o.csr_transpose(pat)
        self._o = _o

    def with_vals(self, vals: np.ndarray):
        M = self.M
        return self.CSR(M.nrows, M.ncols, M.indptr, M.indices, vals)

    def mul(self, vals: np.ndarray, v: np.ndarray, op: int) -> np.ndarray:
        """op 0: M v;  op 1: M^T v (row sums of the transpose, values gathered through perm)."""
        M = self.M
        if op == 0:
            return self._o.spmv_fwd(self.with_vals(vals), v).value
        MT = self.CSR(M.ncols, M.nrows, self.ATp, self.ATi, np.ascontiguousarray(vals[self.perm]))
        return self._o.spmv_fwd(MT, v).value

    def outer(self, v: np.ndarray, g: np.ndarray, op: int) -> np.ndarray:
        """Masked outer product on M's pattern (the VJP w.r.t. M.values):
        op 0 (y = M v): g_i v_j;  op 1 (y = M^T v): v_i g_j -- one multiply per stored entry."""
        dA, _ = self._o.spmv_bwd(self.with_vals(np.zeros(self.M.nnz)), v, g, op=op, want_dx=False)
        return dA


class _SpMV(torch.autograd.Function):
    """y = op(M) v with M's values `vals` (VJP Table 1).  If S is given,
    backward also accumulates S += |g_i||v_j| (the magnitude of each term it adds to dvals), the
    S-scale of the elementwise tolerance rule (DESIGN reading R-PCG)."""

    @staticmethod
    def forward(ctx, vals, v, mat, op, S):
        ctx.mat, ctx.op, ctx.S = mat, op, S
        ctx.save_for_backward(vals, v)
        return torch.from_numpy(mat.mul(vals.detach().numpy(), v.detach().contiguous().numpy(), op))

    @staticmethod
    def backward(ctx, gy):
        vals, v = ctx.saved_tensors
        g = gy.detach().contiguous().numpy()
        vn = v.detach().contiguous().numpy()
        dvals = dv = None
        if ctx.needs_input_grad[1]:
            dv = torch.from_numpy(ctx.mat.mul(vals.detach().numpy(), g, 1 - ctx.op))
        if ctx.needs_input_grad[0]:
            dvals = torch.from_numpy(ctx.mat.outer(vn, g, ctx.op))
            if ctx.S is not None:
                ctx.S += ctx.mat.outer(np.abs(vn), np.abs(g), ctx.op)
        return dvals, dv, None, None, None


class _SpTRSV(torch.autograd.Function):
    """x = T^{-1} rhs with T = L (trans = 0, forward substitution) or T = L^T (trans = 1, the
    oracle's transpose of L, backward substitution) -- PAPER 3.1.5.  VJP:
    d rhs = T^{-T} g, dT = -(T^{-T} g) x^T (.) mask(T) (oracle.sptrsv_bwd); for trans = 1 the dT
    entries are mapped back to L's positions through perm.  S += |d rhs_i||x_j| per stored entry."""

    @staticmethod
    def forward(ctx, vals, rhs, mat, trans, S):
        import oracle as _o
        v = vals.detach().numpy()
        if trans:
            M = mat.M
            T = mat.CSR(M.ncols, M.nrows, mat.ATp, mat.ATi, np.ascontiguousarray(v[mat.perm]))
        else:
            T = mat.with_vals(v)
        x = _o.sptrsv(T, rhs.detach().contiguous().numpy(), upper=bool(trans)).value
        ctx.T, ctx.trans, ctx.mat, ctx.S, ctx.x = T, trans, mat, S, x
        return torch.from_numpy(x)

    @staticmethod
    def backward(ctx, g):
        import oracle as _o
        T, x = ctx.T, ctx.x
        dT, db = _o.sptrsv_bwd(T, x, g.detach().contiguous().numpy(), upper=bool(ctx.trans))
        rows = np.repeat(np.arange(T.nrows), np.diff(T.indptr))
        s = np.abs(db.value[rows]) * np.abs(x[T.indices])
        if ctx.trans:                                   # entry q of L^T is entry perm[q] of L
            d2, s2 = np.empty_like(dT), np.empty_like(s)
            d2[ctx.mat.perm], s2[ctx.mat.perm] = dT, s
            dT, s = d2, s2
        if ctx.S is not None:
            ctx.S += s
        return torch.from_numpy(dT), torch.from_numpy(db.value), None, None, None


def pcg_loss_grad_sparse(A, L, b: np.ndarray, n_it: int, gamma: float, want_S: bool = True,
                         precond: str = "mult"):
    """The config-5 training step on CSR A (constant) and L (learned values, fixed
    pattern), M = L L^T applied as z = L (L^T r), x0 = 0.  Returns (loss, [||r^(i)||],
    dL[nnz(L)], S_dL[nnz(L)] or None).  S_dL[p] = sum over every term autograd adds into dL[p]
    of |term| (the masked outer products of the L and L^T products, one per application of M).
    precond="solve": M = (L L^T)^{-1}, z = L^{-T} (L^{-1} r) by the oracle's substitutions (the
    SpTRSV extension)."""
    Am, Lm = SparseMat(A), SparseMat(L)
    Av = torch.from_numpy(np.asarray(A.values, np.float64))
    Lv = torch.tensor(np.asarray(L.values, np.float64), requires_grad=True)
    S = np.zeros(L.nnz) if want_S else None
    spmv = _SpMV.apply
    Amul = lambda v: spmv(Av, v, Am, 0, None)                      # A v
    if precond == "solve":
        M = lambda v: _SpTRSV.apply(Lv, _SpTRSV.apply(Lv, v, Lm, 0, S), Lm, 1, S)   # L^{-T} (L^{-1} v)
    else:
        M = lambda v: spmv(Lv, spmv(Lv, v, Lm, 1, S), Lm, 0, S)     # L (L^T v)
    bt = torch.from_numpy(np.asarray(b, np.float64))
    x = torch.zeros_like(bt)
    r = bt - Amul(x)
    z = M(r)
    p = z
    rho = r @ z
    res = []
    for _ in range(n_it):
        q = Amul(p)
        alpha = rho / (p @ q)
        with torch.no_grad():                                       # x never reaches the loss
            x = x + alpha * p
        r = r - alpha * q
        res.append(torch.linalg.norm(r))
        z = M(r)
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    w = torch.tensor(loss_weights(n_it, gamma))
    loss = (w * torch.stack(res)).sum() / torch.linalg.norm(bt)
    loss.backward()
    return float(loss.detach()), [float(v.detach()) for v in res], Lv.grad.numpy().copy(), S
