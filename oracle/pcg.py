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
