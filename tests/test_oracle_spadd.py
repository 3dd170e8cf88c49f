"""Pins for the Sp+Sp oracle (PAPER 3.1.4 P:466-476, Table 1):
SPEC's worked examples, the paper's Fig. 7 construction of A_N against Eq. mat_1d_fd,
dense brute force, torch autograd for the VJP, exact finite differences and the Euler identity.
CPU only.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import numpy as np
import pytest
import torch

import synth
from test_oracle_pins import PROTOCOL, SPEC
from util import assert_S_close, gather_mask, pattern_dense, to_dense

R64 = 1e-12


def eye_k(n, k=0, scale=1.0):
    """sp.eye(n, k): ones on the k-th diagonal (PAPER Fig. 7)."""
    rows = [i for i in range(n) if 0 <= i + k < n]
    indptr = np.zeros(n + 1, np.int64)
    for i in rows:
        indptr[i + 1] = 1
    indptr = np.cumsum(indptr)
    return synth.CSR(n, n, indptr, np.array([i + k for i in rows], np.int32), np.full(len(rows), scale))


def add(orc, alpha, A, beta, B):
    Cp, Ci = orc.spadd_symbolic(A, B)
    r = orc.spadd_numeric(alpha, A, beta, B, Cp, Ci)
    return synth.CSR(A.nrows, A.ncols, Cp, Ci, r.value), r


def rand_pair(seed, m, n, d):
    A = synth.random_csr(m, n, d, 100 + seed, np.float64, "int")
    B = synth.random_csr(m, n, d, 200 + seed, np.float64, "int")
    return A, B


def test_spadd_spec_examples(orc):
    A = synth.poisson2d(4)
    e = SPEC["spadd_self_cancel"]  # alpha=1, beta=-1, B=A -> zeros, pattern(A) kept
    C, r = add(orc, e["alpha"], A, e["beta"], A)
    assert C.indptr.tolist() == A.indptr.tolist() and C.indices.tolist() == A.indices.tolist()
    assert (C.values == e["value"]).all()
    e = SPEC["spadd_eye_bidiag"]  # 2 I + (-1) I_{k=1} -> upper bidiagonal
    C, _ = add(orc, 2.0, eye_k(3), -1.0, eye_k(3, 1))
    assert C.indptr.tolist() == e["indptr"] and C.indices.tolist() == e["indices"]
    assert C.values.tolist() == e["values"]
    e = SPEC["spadd_vjp_ones"]  # V = ones on the union, alpha = 2 -> gradA = 2
    A, B = rand_pair(3, 8, 8, 0.3)
    Cp, Ci = orc.spadd_symbolic(A, B)
    dA, dB = orc.spadd_bwd(e["alpha"], A, 1.0, B, Cp, Ci, np.ones(len(Ci)))
    assert (dA == e["gradA_value"]).all() and (dB == 1.0).all()


@pytest.mark.parametrize("N", [3, 4, 16, 33])
def test_fig7_construction_is_A_N(orc, N):
    """P:733 builds A_N = sp.eye(N)*2 - sp.eye(N, k=1) - sp.eye(N, k=-1); it must equal
    Eq. mat_1d_fd -- pattern and values."""
    C1, _ = add(orc, 2.0, eye_k(N), -1.0, eye_k(N, 1))
    C2, _ = add(orc, 1.0, C1, -1.0, eye_k(N, -1))
    A = synth.poisson1d(N)
    assert C2.indptr.tolist() == A.indptr.tolist() and C2.indices.tolist() == A.indices.tolist()
    assert C2.values.tolist() == A.values.tolist()


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spadd_dense_bruteforce(orc, seed, m, n, d):
    A = synth.random_csr(m, n, d, 300 + seed, np.float64, "real")
    B = synth.random_csr(m, n, d, 400 + seed, np.float64, "real")
    alpha, beta = 0.75, -1.5
    C, r = add(orc, alpha, A, beta, B)
    np.testing.assert_array_equal(pattern_dense(C), pattern_dense(A) | pattern_dense(B))
    ref = gather_mask(alpha * to_dense(A) + beta * to_dense(B), C.indptr, C.indices)
    assert_S_close(C.values, ref, r.S, R64, "spadd")
    # columns strictly increasing (canonical output, reading A3)
    for i in range(C.nrows):
        assert (np.diff(C.indices[C.indptr[i]:C.indptr[i + 1]]) > 0).all()


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spadd_vjp_dense_autograd(orc, seed, m, n, d):
    A = synth.random_csr(m, n, d, 500 + seed, np.float64, "real")
    B = synth.random_csr(m, n, d, 600 + seed, np.float64, "real")
    alpha, beta = -0.5, 2.25
    Cp, Ci = orc.spadd_symbolic(A, B)
    V = np.random.default_rng(seed).uniform(-1, 1, len(Ci))
    dA, dB = orc.spadd_bwd(alpha, A, beta, B, Cp, Ci, V)
    tA = torch.tensor(to_dense(A), requires_grad=True)
    tB = torch.tensor(to_dense(B), requires_grad=True)
    Vd = np.zeros((m, n))
    Vd[np.repeat(np.arange(m), np.diff(Cp)), Ci] = V
    (torch.tensor(Vd) * (alpha * tA + beta * tB)).sum().backward()
    np.testing.assert_array_equal(dA, gather_mask(tA.grad.numpy(), A.indptr, A.indices))
    np.testing.assert_array_equal(dB, gather_mask(tB.grad.numpy(), B.indptr, B.indices))


def test_spadd_vjp_exact_fd_and_euler(orc):
    """C is linear in A's values: the central difference at h = 1 of L = <V, alpha A + beta B>
    is exact for integer data; Euler: <V, C> = <dA, A> + <dB, B>."""
    A, B = rand_pair(7, 16, 12, 0.3)
    alpha, beta = 3.0, -2.0
    Cp, Ci = orc.spadd_symbolic(A, B)
    V = np.random.default_rng(1).integers(-3, 4, len(Ci)).astype(np.float64)
    dA, dB = orc.spadd_bwd(alpha, A, beta, B, Cp, Ci, V)

    def L(Av, Bv):
        return float(V @ orc.spadd_numeric(alpha, A.with_values(Av), beta, B.with_values(Bv), Cp, Ci).value)

    for q in range(A.nnz):
        e = np.zeros(A.nnz)
        e[q] = 1.0
        assert (L(A.values + e, B.values) - L(A.values - e, B.values)) / 2 == dA[q]
    for q in range(B.nnz):
        e = np.zeros(B.nnz)
        e[q] = 1.0
        assert (L(A.values, B.values + e) - L(A.values, B.values - e)) / 2 == dB[q]
    assert L(A.values, B.values) == dA @ A.values + dB @ B.values


def test_spadd_rejects_foreign_pattern(orc):
    A, B = rand_pair(9, 6, 6, 0.5)
    Cp, Ci = orc.spadd_symbolic(A, A)  # misses B's entries
    if orc.spadd_symbolic(A, B)[1].shape != Ci.shape:
        with pytest.raises(ValueError):
            orc.spadd_numeric(1.0, A, 1.0, B, Cp, Ci)
