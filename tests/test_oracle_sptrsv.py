"""Pins for the SpTRSV oracle (PAPER 3.1.5 P:477-488, Table 1 SpSolve row
P:290-293): SPEC's worked examples, exact solutions by construction (b = T x_int),
the closed form of the 1D Poisson lower bidiagonal solve, dense brute force against
torch.linalg.solve_triangular + autograd (masked gradient), the adjoint identity, central
finite differences, and the error-magnitude S.  CPU only.  P:n = PAPER.md line n, S:n = SPEC.md.
"""
import numpy as np
import pytest
import torch

import synth
from test_oracle_pins import SPEC
from util import assert_S_close, gather_mask, to_dense

R64 = 1e-12
CASES = [(n, d, s) for n in (4, 8, 16, 32) for d in (0.1, 0.3, 1.0) for s in range(2)]  # S:353 protocol


def csr(indptr, indices, values):
    n = len(indptr) - 1
    return synth.CSR(n, n, np.array(indptr, np.int64), np.array(indices, np.int32), np.array(values, np.float64))


def test_spec_identity(orc):
    """I_3, b arbitrary -> x = b."""
    e = SPEC["sptrsv_identity"]
    b = np.array(e["b"])
    I = csr([0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    for upper in (False, True):
        np.testing.assert_array_equal(orc.sptrsv(I, b, upper=upper).value, b)
    np.testing.assert_array_equal(orc.sptrsv(csr([0, 0, 0, 0], [], []), b, unit=True).value, b)


def test_spec_L2_and_flip(orc):
    """S:206 lower example, S:207 the upper one through the flip path."""
    e = SPEC["sptrsv_L2"]
    L = csr(e["indptr"], e["indices"], e["values"])
    np.testing.assert_array_equal(orc.sptrsv(L, np.array(e["b"])).value, e["x"])
    e = SPEC["sptrsv_U2_flip"]
    U = csr(e["indptr"], e["indices"], e["values"])
    np.testing.assert_array_equal(orc.sptrsv(U, np.array(e["b"]), upper=True).value, e["x"])


def test_spec_vjp_identity_and_zero(orc):
    """L = I -> gradb = v, gradL (diagonal) = -v_i x_i.  S:216: v = 0 -> zero gradients."""
    e = SPEC["sptrsv_vjp_identity"]
    v, x = np.array(e["v"]), np.array(e["x"])
    I = csr([0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    dT, db = orc.sptrsv_bwd(I, x, v)
    np.testing.assert_array_equal(db.value, v)
    np.testing.assert_array_equal(dT, -v * x)
    T = synth.tri_random(16, 0.3, 5)
    x = orc.sptrsv(T, synth.dense(16, 6)).value
    dT, db = orc.sptrsv_bwd(T, x, np.zeros(16))
    assert not dT.any() and not db.value.any()


def test_errors(orc):
    """an entry on the wrong side of the diagonal is a shape error, a missing diagonal
    (unit_diag off) is singular."""
    with pytest.raises(orc.TriangularError, match="wrong side"):
        orc.sptrsv(csr([0, 2, 3], [0, 1, 1], [1.0, 1.0, 1.0]), np.ones(2))
    with pytest.raises(orc.TriangularError, match="wrong side"):
        orc.sptrsv(csr([0, 1, 3], [0, 0, 1], [1.0, 1.0, 1.0]), np.ones(2), upper=True)
    with pytest.raises(orc.TriangularError, match="missing diagonal"):
        orc.sptrsv(csr([0, 1, 2], [0, 0], [1.0, 1.0]), np.ones(2))


@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("unit", [False, True])
@pytest.mark.parametrize("n,d,s", CASES[::2])
def test_exact_by_construction(orc, n, d, s, upper, unit):
    """b = T x_int with integer T (diagonal in {+-1, +-2, +-4}, or unit) and integer x_int: every
    numerator is an exact integer, so substitution must return x_int exactly."""
    T = synth.tri_random(n, d, 1000 + s, upper=upper, values="int", unit=unit)
    xi = synth.dense(n, 2000 + s, values="int")
    D = to_dense(T)
    if unit:
        np.fill_diagonal(D, 1.0)
    b = (D.astype(np.int64) @ xi.astype(np.int64)).astype(np.float64)
    np.testing.assert_array_equal(orc.sptrsv(T, b, upper=upper, unit=unit).value, xi)


def test_poisson1d_bidiagonal_closed_form(orc):
    """The lower triangle of A_N (Eq. mat_1d_fd: 2 on the diagonal, -1 below) with b = 1:
    x_i = (1 + x_{i-1}) / 2 from x_0 = 1/2 gives x_i = 1 - 2^-(i+1), exact in binary for i < 53."""
    L = synth.lower_part(synth.poisson1d(50))
    x = orc.sptrsv(L, np.ones(50)).value
    np.testing.assert_array_equal(x, 1.0 - 2.0 ** -(np.arange(50) + 1.0))
    # upper part with the flip: U = L^T, solved from the last row: x_{n-1-i} = 1 - 2^-(i+1)
    U = synth.lower_part(synth.poisson1d(50))
    Ut = orc.csr_transpose(U)
    U = synth.CSR(50, 50, Ut[0], Ut[1], Ut[2])
    np.testing.assert_array_equal(orc.sptrsv(U, np.ones(50), upper=True).value[::-1], x)


@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("n,d,s", CASES)
def test_dense_brute_force(orc, n, d, s, upper):
    """Forward vs torch.linalg.solve_triangular; VJP vs torch autograd of <v, x(T, b)> with the
    gradient gathered at T's stored entries (mask(T))."""
    T = synth.tri_random(n, d, 3000 + s, upper=upper)
    b, v = synth.dense(n, 3100 + s), synth.dense(n, 3200 + s)
    Td = torch.tensor(to_dense(T), requires_grad=True)
    bt = torch.tensor(b, requires_grad=True)
    xt = torch.linalg.solve_triangular(Td, bt[:, None], upper=upper)[:, 0]
    (xt @ torch.tensor(v)).backward()
    r = orc.sptrsv(T, b, upper=upper)
    assert_S_close(r.value, xt.detach().numpy(), r.S, R64, "x")
    dT, db = orc.sptrsv_bwd(T, r.value, v, upper=upper)
    assert_S_close(db.value, bt.grad.numpy(), db.S, R64, "db")
    ref = gather_mask(Td.grad.numpy(), T.indptr, T.indices)
    scale = np.abs(gather_mask(np.outer(db.S, np.abs(r.value) + r.S), T.indptr, T.indices))
    assert_S_close(dT, ref, scale, R64, "dT")
    # no gradient leaks outside the pattern: the dense gradient there is structurally nonzero
    # in general, the sparse VJP simply does not produce it
    assert dT.shape == (T.nnz,)


@pytest.mark.parametrize("n,d,s", CASES[::3])
def test_adjoint_identity(orc, n, d, s):
    """<v, T^{-1} b> = <T^{-T} v, b> (the transpose-solve identity)."""
    T = synth.tri_random(n, d, 4000 + s)
    b, v = synth.dense(n, 4100 + s), synth.dense(n, 4200 + s)
    x = orc.sptrsv(T, b)
    _, w = orc.sptrsv_bwd(T, x.value, v)
    lhs, rhs = float(v @ x.value), float(w.value @ b)
    assert abs(lhs - rhs) <= 1e-12 * (np.abs(v) @ x.S + w.S @ np.abs(b))


def test_finite_differences(orc):
    """Central differences of l = <v, x(T, b)>: exact at h = 1 in b (l is linear in b); in the
    stored values of T (nonlinear) with h = 1e-6, rel 1e-6 (SPEC S:215 tolerance)."""
    n = 24
    T = synth.tri_random(n, 0.3, 77)
    b, v = synth.dense(n, 78), synth.dense(n, 79)
    x = orc.sptrsv(T, b).value
    dT, db = orc.sptrsv_bwd(T, x, v)
    loss = lambda TT, bb: float(v @ orc.sptrsv(TT, bb).value)
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        fd = (loss(T, b + e) - loss(T, b - e)) / 2
        assert abs(fd - db.value[j]) <= 1e-12 * (1 + abs(fd))
    h = 1e-6
    for p in range(T.nnz):
        vp, vm = T.values.copy(), T.values.copy()
        vp[p] += h
        vm[p] -= h
        fd = (loss(T.with_values(vp), b) - loss(T.with_values(vm), b)) / (2 * h)
        assert abs(fd - dT[p]) <= 1e-6 * max(1.0, abs(fd)), p


def test_unit_diagonal_gradient(orc):
    """unit_diag: a stored diagonal is unused by the solve, so its gradient is exactly 0 and the
    solution equals the one with the diagonal entries set to 1."""
    T = synth.tri_random(20, 0.3, 91)
    b, v = synth.dense(20, 92), synth.dense(20, 93)
    rows = np.repeat(np.arange(20), np.diff(T.indptr))
    ones = T.values.copy()
    ones[rows == T.indices] = 1.0
    xu = orc.sptrsv(T, b, unit=True).value
    np.testing.assert_array_equal(xu, orc.sptrsv(T.with_values(ones), b).value)
    dT, _ = orc.sptrsv_bwd(T, xu, v, unit=True)
    assert not dT[rows == T.indices].any()
    dT1, _ = orc.sptrsv_bwd(T.with_values(ones), xu, v)
    np.testing.assert_array_equal(dT[rows != T.indices], dT1[rows != T.indices])


def test_error_magnitude(orc):
    """S = M(T)^{-1}|T||x| dominates |x| and bounds the oracle's own error against the exact
    rational solution (Python fractions over the same binary inputs, forward substitution in
    exact arithmetic): |x - x_exact| <= (max row length + 2) u S."""
    from fractions import Fraction
    n = 14
    T = synth.tri_random(n, 0.4, 55)
    b = synth.dense(n, 56)
    r = orc.sptrsv(T, b)
    assert np.all(r.S >= np.abs(r.value))
    xe = [Fraction(0)] * n
    for i in range(n):
        s, d = Fraction(b[i]), None
        for p in range(T.indptr[i], T.indptr[i + 1]):
            j = int(T.indices[p])
            if j == i:
                d = Fraction(T.values[p])
            else:
                s -= Fraction(T.values[p]) * xe[j]
        xe[i] = s / d
    ell = int(np.diff(T.indptr).max()) + 2
    err = np.array([abs(float(Fraction(r.value[i]) - xe[i])) for i in range(n)])
    assert np.all(err <= ell * 2.0 ** -53 * r.S)
