"""oracle.gcn -- TEST INFRASTRUCTURE ONLY.

GCN layer (PAPER 4.4): the graph convolution

    X^(i+1) = D~^{-1/2} A~ D~^{-1/2} X^(i) Theta^(i+1),   A~ = A + I,  D~ = diag of A~'s row sums
                                                               (Eq. gcn_update)

computed exactly as the paper's reference listing does it (Fig. 12), right to left:

    D       = (graph.row_sum() + 1.) ** -0.5
    XTheta  = X @ weights
    DXTheta = D[:, None] * XTheta
    C       = D[:, None] * (graph @ DXTheta + DXTheta)
    return C + bias

in plain PyTorch on the CPU in float64 (graph as a torch CSR tensor), differentiated by torch
autograd -- no hand-derived adjoint.  `gcn_prop` is the same listing from XTheta on (the part
csrk_gcn_fwd / csrk_gcn_bwd compute); `gcn_layer` is the whole listing.  Alongside each
output element the magnitude S = D_i (sum_p |a_p D_j Z_jc| + |D_i Z_ic|) + |b_c| is returned
for the S-scaled tolerance (DESIGN reading A6).  Pinned by tests/test_gcn.py.
"""
from __future__ import annotations

import numpy as np
import torch


def _graph(A):
    return torch.sparse_csr_tensor(torch.from_numpy(np.asarray(A.indptr, np.int64)),
                                   torch.from_numpy(np.asarray(A.indices, np.int64)),
                                   torch.from_numpy(np.asarray(A.values, np.float64)),
                                   size=(A.nrows, A.ncols))


def row_sum(A) -> torch.Tensor:
    """graph.row_sum() of Fig. 12: sum of the stored values of each row (float64)."""
    rows = np.repeat(np.arange(A.nrows), np.diff(A.indptr))
    return torch.from_numpy(np.bincount(rows, weights=np.asarray(A.values, np.float64), minlength=A.nrows))


def gcn_prop(A, Z, bias=None, want_grad=None):
    """Fig. 12 from XTheta on: Y = D (A (D Z) + D Z) + bias, D = (row_sum + 1)^-1/2.
    want_grad = dY (n x F) -> also returns (dZ, dbias) by autograd.
    Returns dict(Y, S, D[, dZ, dbias])."""
    graph = _graph(A)
    Zt = torch.tensor(np.asarray(Z, np.float64), requires_grad=want_grad is not None)
    bt = None if bias is None else torch.tensor(np.asarray(bias, np.float64), requires_grad=want_grad is not None)
    D = (row_sum(A) + 1.0) ** -0.5
    DXTheta = D[:, None] * Zt
    C = D[:, None] * (graph @ DXTheta + DXTheta)
    Y = C + bt if bt is not None else C
    absg = torch.sparse_csr_tensor(graph.crow_indices(), graph.col_indices(), graph.values().abs(), size=graph.shape)
    aD = D.abs()[:, None] * Zt.detach().abs()
    S = D.abs()[:, None] * (absg @ aD + aD)
    if bt is not None:
        S = S + bt.detach().abs()
    out = {"Y": Y.detach().numpy(), "S": S.numpy(), "D": D.numpy()}
    if want_grad is not None:
        dY = torch.tensor(np.asarray(want_grad, np.float64))
        Y.backward(dY)
        out["dZ"] = Zt.grad.numpy()
        out["dbias"] = None if bt is None else bt.grad.numpy()
        # magnitudes of the adjoint's terms: S_dZ = D (|A|^T |D dY| + |D dY|), S_dbias = sum_i |dY_i|
        absgT = absg.to_dense().t().to_sparse_csr() if A.nrows <= 4096 else \
            torch.sparse_coo_tensor(torch.stack([graph.col_indices(), torch.repeat_interleave(
                torch.arange(A.nrows), graph.crow_indices().diff())]), graph.values().abs(), graph.shape).coalesce()
        aG = D.abs()[:, None] * dY.abs()
        out["S_dZ"] = (D.abs()[:, None] * (absgT @ aG + aG)).numpy()
        out["S_dbias"] = dY.abs().sum(0).numpy()
    return out


def gcn_layer(A, X, Theta, bias, want_grad=None):
    """The whole Fig. 12 listing (X @ weights first).  want_grad = dY -> (dX, dTheta, dbias)."""
    graph = _graph(A)
    req = want_grad is not None
    Xt = torch.tensor(np.asarray(X, np.float64), requires_grad=req)
    Wt = torch.tensor(np.asarray(Theta, np.float64), requires_grad=req)
    bt = torch.tensor(np.asarray(bias, np.float64), requires_grad=req)
    D = (row_sum(A) + 1.0) ** -0.5
    XTheta = Xt @ Wt
    DXTheta = D[:, None] * XTheta
    C = D[:, None] * (graph @ DXTheta + DXTheta)
    Y = C + bt
    out = {"Y": Y.detach().numpy()}
    if req:
        Y.backward(torch.tensor(np.asarray(want_grad, np.float64)))
        out.update(dX=Xt.grad.numpy(), dTheta=Wt.grad.numpy(), dbias=bt.grad.numpy())
    return out


def gcn_dense_formula(A_dense: np.ndarray, X, Theta, bias) -> np.ndarray:
    """Eq. gcn_update written out densely: D~^-1/2 (A + I) D~^-1/2 X Theta + bias with D~ the
    diagonal of (A + I)'s row sums -- a different evaluation order than Fig. 12."""
    n = A_dense.shape[0]
    At = A_dense + np.eye(n)
    Dm = np.diag(At.sum(axis=1) ** -0.5)
    return Dm @ At @ Dm @ np.asarray(X) @ np.asarray(Theta) + np.asarray(bias)
