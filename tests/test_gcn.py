"""Pins for the GCN-layer oracle (PAPER 4.4 Eq. gcn_update, Fig. 12
P:905-925): SPEC's worked examples, the dense Eq. gcn_update against the Fig. 12
right-to-left evaluation, the closed form on a cycle graph, torch gradcheck, and the S bound.
CPU only.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import gcn
from util import to_dense


def graph(n, p, seed, weighted=False):
    """Random symmetric adjacency (no self loops), values 1 or U[0.5, 2) (nonnegative)."""
    rng = np.random.default_rng(seed)
    M = np.triu(rng.random((n, n)) < p, 1)
    M = M | M.T
    W = np.where(M, rng.uniform(0.5, 2.0, (n, n)) if weighted else 1.0, 0.0)
    W = np.triu(W, 1) + np.triu(W, 1).T
    r, c = np.nonzero(W)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    return synth.CSR(n, n, indptr, c.astype(np.int32), W[r, c])


def test_spec_zero_adjacency():
    """adj = 0 -> output = X Theta + bias (D~ = I)."""
    A = synth.CSR(5, 5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0))
    X, W, b = synth.dense((5, 3), 1), synth.dense((3, 4), 2), synth.dense(4, 3)
    np.testing.assert_allclose(gcn.gcn_layer(A, X, W, b)["Y"], X @ W + b, rtol=0, atol=1e-15)


def test_spec_two_node_edge():
    """2-node single-edge graph, Theta = I, bias = 0, X = I_2 -> [[.5, .5], [.5, .5]]."""
    A = synth.CSR(2, 2, np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), np.array([1.0, 1.0]))
    Y = gcn.gcn_layer(A, np.eye(2), np.eye(2), np.zeros(2))["Y"]
    np.testing.assert_allclose(Y, [[0.5, 0.5], [0.5, 0.5]], rtol=4e-16, atol=0)


@pytest.mark.parametrize("seed", range(6))
def test_fig12_equals_eq_gcn_update(seed):
    """Fig. 12's right-to-left evaluation equals Eq. gcn_update's dense formula."""
    A = graph(40, 0.1, seed, weighted=seed % 2 == 1)
    X, W, b = synth.dense((40, 6), 10 + seed), synth.dense((6, 5), 20 + seed), synth.dense(5, 30 + seed)
    ref = gcn.gcn_dense_formula(to_dense(A), X, W, b)
    np.testing.assert_allclose(gcn.gcn_layer(A, X, W, b)["Y"], ref, rtol=1e-13, atol=1e-13)
    r = gcn.gcn_prop(A, X @ W, b)
    np.testing.assert_allclose(r["Y"], ref, rtol=1e-13, atol=1e-13)


def test_cycle_closed_form():
    """Cycle graph C_n (degree 2): D~ = 3 I, so Y = (A + I) Z / 3 + b; with Z = 1 1^T every output
    entry is 1 + b (to rounding: (1/sqrt 3)^2 (1 + 1 + 1))."""
    n = 12
    i = np.arange(n)
    cols = np.sort(np.stack([(i - 1) % n, (i + 1) % n], 1), axis=1)
    A = synth.CSR(n, n, np.arange(0, 2 * n + 1, 2, dtype=np.int64), cols.ravel().astype(np.int32), np.ones(2 * n))
    Z = np.ones((n, 4))
    b = np.array([0.0, 0.5, -1.0, 2.0])
    Y = gcn.gcn_prop(A, Z, b)["Y"]
    np.testing.assert_allclose(Y, np.broadcast_to(1.0 + b[None, :], Y.shape), rtol=0, atol=1e-15)
    D = gcn.gcn_prop(A, Z, b)["D"]
    np.testing.assert_allclose(D, 3.0 ** -0.5, rtol=4e-16)


def test_gradcheck_layer():
    """gradients of Theta, bias, X pass gradcheck through the whole layer (torch autograd
    of the Fig. 12 listing against central finite differences)."""
    A = graph(12, 0.25, 7, weighted=True)
    g = torch.sparse_csr_tensor(torch.from_numpy(A.indptr), torch.from_numpy(A.indices.astype(np.int64)),
                                torch.from_numpy(A.values), size=(12, 12))
    D = (gcn.row_sum(A) + 1.0) ** -0.5

    def f(X, W, b):
        XT = X @ W
        DX = D[:, None] * XT
        return D[:, None] * (g @ DX + DX) + b

    X = torch.tensor(synth.dense((12, 3), 1), requires_grad=True)
    W = torch.tensor(synth.dense((3, 2), 2), requires_grad=True)
    b = torch.tensor(synth.dense(2, 3), requires_grad=True)
    assert torch.autograd.gradcheck(f, (X, W, b), eps=1e-6, atol=1e-8)


def test_prop_vjp_is_transpose_propagation():
    """dZ of Y = D (A + I) D Z + b is D (A + I)^T D dY (the adjoint), dbias = column sums of dY:
    checked against the dense transposed operator on a non-symmetric weighted graph."""
    rng = np.random.default_rng(5)
    n = 30
    Ad = np.where(rng.random((n, n)) < 0.15, rng.uniform(0.5, 2.0, (n, n)), 0.0)
    np.fill_diagonal(Ad, 0.0)
    r, c = np.nonzero(Ad)
    A = synth.CSR(n, n, np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64),
                  c.astype(np.int32), Ad[r, c])
    Z, b, dY = synth.dense((n, 4), 1), synth.dense(4, 2), synth.dense((n, 4), 3)
    out = gcn.gcn_prop(A, Z, b, want_grad=dY)
    Dm = np.diag((Ad.sum(1) + 1.0) ** -0.5)
    np.testing.assert_allclose(out["dZ"], Dm @ (Ad + np.eye(n)).T @ Dm @ dY, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(out["dbias"], dY.sum(0), rtol=1e-14)


def test_S_bound():
    """S >= |Y| and the fp64 result agrees with an exact-rational evaluation of the listing
    within a few ulp of S."""
    from fractions import Fraction
    A = graph(10, 0.3, 9, weighted=True)
    Z, b = synth.dense((10, 2), 4), synth.dense(2, 5)
    out = gcn.gcn_prop(A, Z, b)
    assert np.all(out["S"] >= np.abs(out["Y"]) * (1 - 1e-15))
    D = out["D"]
    for i in range(10):
        for c in range(2):
            acc = Fraction(0)
            for p in range(A.indptr[i], A.indptr[i + 1]):
                j = A.indices[p]
                acc += Fraction(A.values[p]) * Fraction(D[j]) * Fraction(Z[j, c])
            acc += Fraction(D[i]) * Fraction(Z[i, c])
            exact = Fraction(D[i]) * acc + Fraction(b[c])
            assert abs(float(Fraction(out["Y"][i, c]) - exact)) <= 16 * 2.0 ** -53 * out["S"][i, c]
