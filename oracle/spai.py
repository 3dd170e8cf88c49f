"""oracle.spai -- TEST INFRASTRUCTURE ONLY.

SPAI workload (PAPER 4.6): the loss

    l = || I - M A ||_F^2                                         (Eq. spai_loss)

over the stored entries of M, with pattern(M) = pattern(A) fixed ("we force the sparsity
pattern of M to remain static ... mask(M) = mask(A)"), and its gradient
dl/dM.values = -2 ((I - M A) A^T) (.) mask(M), here obtained by torch autograd (CPU, float64,
dense) -- no hand-derived adjoint.  Dense, so for small N only (N <= ~4096).

Also the classical reference the paper compares against: the loss
"decomposed into parallel least squares problems" -- row i of M minimises
|| e_i^T - m_i^T A ||_2 over the stored columns of row i, solved here with numpy lstsq.
"""
from __future__ import annotations

import numpy as np
import torch


def spai_loss_grad(A_dense: np.ndarray, M_pattern: np.ndarray, M_dense: np.ndarray):
    """Returns (loss, dM dense with zeros off the pattern).  P:1075-1078."""
    N = A_dense.shape[0]
    A = torch.tensor(A_dense, dtype=torch.float64)
    mask = torch.tensor(M_pattern, dtype=torch.bool)
    Mv = torch.tensor(M_dense, dtype=torch.float64, requires_grad=True)
    M = torch.where(mask, Mv, torch.zeros_like(Mv))          # only stored entries are variables
    R = torch.eye(N, dtype=torch.float64) - M @ A
    loss = (R * R).sum()
    loss.backward()
    return float(loss.detach()), torch.where(mask, Mv.grad, torch.zeros_like(Mv.grad)).numpy()


def spai_S(A_dense: np.ndarray, M_pattern: np.ndarray, M_dense: np.ndarray):
    """S-scales of the elementwise tolerance rule (reading A6) for the composed evaluation
    C = M A, R = I - C, loss = sum R^2, dM = -2 (R A^T) (.) mask(M): first-order magnitudes of
    the rounding of each stage, S_R = |I| + |M| |A| (the terms of R), then
        S_loss = sum_ij (2 |R_ij| S_R,ij + R_ij^2),
        S_dM   = 2 (S_R + |R|) |A|^T (.) mask(M)     (the error of R times |A|, plus the terms).
    Returns (S_loss, S_dM dense)."""
    N = A_dense.shape[0]
    M = np.where(M_pattern, M_dense, 0.0)
    R = np.eye(N) - M @ A_dense
    SR = np.eye(N) + np.abs(M) @ np.abs(A_dense)
    S_loss = float((2.0 * np.abs(R) * SR + R * R).sum())
    S_dM = np.where(M_pattern, 2.0 * (SR + np.abs(R)) @ np.abs(A_dense).T, 0.0)
    return S_loss, S_dM


def spai_loss_by_columns(A_dense: np.ndarray, M_dense: np.ndarray) -> float:
    """sum_i ||(I - M A) e_i||_2^2 -- the column decomposition of P:1079-1082, column by column."""
    N = A_dense.shape[0]
    total = 0.0
    for i in range(N):
        e = np.zeros(N)
        e[i] = 1.0
        r = e - M_dense @ (A_dense @ e)
        total += float(r @ r)
    return total


def spai_reference(A_dense: np.ndarray, M_pattern: np.ndarray) -> np.ndarray:
    """Classical static-pattern SPAI: row i of M solves the least-squares
    problem min || e_i^T - m_i^T A ||_2 with m_i supported on row i of the pattern."""
    N = A_dense.shape[0]
    M = np.zeros_like(A_dense)
    for i in range(N):
        J = np.nonzero(M_pattern[i])[0]
        e = np.zeros(N)
        e[i] = 1.0
        # m_i^T A = (A^T m_i)^T: least squares in the unknowns m_i[J] with matrix A[J, :]^T
        sol, *_ = np.linalg.lstsq(A_dense[J, :].T, e, rcond=None)
        M[i, J] = sol
    return M
