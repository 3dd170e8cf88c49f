"""Pins for the oracle (CPU only): each check ties oracle/ to something other than
itself -- the paper's / SPEC's printed values (tests/golden), closed forms of the
Poisson stencils, dense torch/numpy brute force on tiny inputs, exact finite
differences of the forward oracle, and the adjoint / Euler identities.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import itertools

import numpy as np
import pytest
import torch

import synth
from util import (assert_S_close, csr_from_pattern, gather_mask, load_fig3, load_json,
                  pattern_dense, to_dense)

R64 = 1e-12  # SURVEY 8(c) c.2 rtol for fp64 (north_star "relative 1e-12")
R32 = 1e-5

SPEC = load_json("spec_examples.json")

# SPEC.md S:353-356 gradcheck protocol: >= 20 seeded instances over n in {4,8,16,32},
# density in {0.1, 0.3, full}, rectangular shapes.
PROTOCOL = [(s, m, n, d) for s, ((m, n), d) in enumerate(itertools.product(
    [(4, 8), (8, 4), (4, 4), (16, 16), (32, 8), (8, 32), (32, 32)], [0.1, 0.3, 1.0]))]
assert len(PROTOCOL) >= 20


def A3():
    e = SPEC["A3_csr"]
    return synth.CSR(3, 3, np.array(e["indptr"], np.int64), np.array(e["indices"], np.int32),
                     np.array(e["values"], np.float64))


def eye(n):
    return synth.CSR(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n))


# ---------------------------------------------------------------- generators
def test_generators_match_paper_definitions():
    # Eq. mat_1d_fd with N=3 equals SPEC's printed CSR
    A = synth.poisson1d(3)
    e = SPEC["A3_csr"]
    assert A.indptr.tolist() == e["indptr"] and A.indices.tolist() == e["indices"]
    assert A.values.tolist() == e["values"]
    # Eq. mat_2d_fd: A_Nx (x) I + I (x) A_Ny via numpy Kronecker products
    for Nx, Ny in [(2, 2), (3, 5), (8, 8)]:
        A1x, A1y = to_dense(synth.poisson1d(Nx)), to_dense(synth.poisson1d(Ny))
        K = np.kron(A1x, np.eye(Ny)) + np.kron(np.eye(Nx), A1y)
        np.testing.assert_array_equal(to_dense(synth.poisson2d(Nx, Ny)), K)
    assert to_dense(synth.poisson2d(2, 2))[0].tolist() == SPEC["poisson2d_2x2_row0"]["row0"]
    assert synth.poisson2d(8, 8).nrows == 64  # P:835 "A in R^{64x64}"
    A1 = to_dense(synth.poisson1d(4))
    I = np.eye(4)
    K3 = np.kron(np.kron(A1, I), I) + np.kron(np.kron(I, A1), I) + np.kron(np.kron(I, I), A1)
    np.testing.assert_array_equal(to_dense(synth.poisson3d(4)), K3)
    for N in range(5, 13):
        assert synth.poisson2d(N).nnz == 5 * N * N - 4 * N
        assert synth.poisson3d(N).nnz == 7 * N ** 3 - 6 * N ** 2


def test_powerlaw_recipe():
    P = synth.powerlaw(1 << 14, seed=7)
    lens = np.diff(P.indptr)
    assert P.nnz == 16 << 14 and lens.min() >= 8
    for i in range(P.nrows):  # canonical: strictly increasing, in range
        seg = P.indices[P.indptr[i]:P.indptr[i + 1]]
        assert (np.diff(seg) > 0).all()
    assert P.indices.min() >= 0 and P.indices.max() < P.ncols


# ---------------------------------------------------------------- spmv fwd
def test_spmv_spec_examples(orc):
    I3 = eye(3)
    assert orc.spmv_fwd(I3, np.array([1., 2, 3])).value.tolist() == SPEC["spmv_identity"]["y"]
    assert orc.spmv_fwd(A3(), np.ones(3)).value.tolist() == SPEC["spmv_A3_ones"]["y"]
    E = synth.CSR(2, 2, np.zeros(3, np.int64), np.zeros(0, np.int32), np.zeros(0))
    r = orc.spmv_fwd(E, np.array([5., 7.]))
    assert r.value.tolist() == [0, 0] and r.S.tolist() == [0, 0]


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spmv_dense_bruteforce(orc, seed, m, n, d):
    A = synth.random_csr(m, n, d, seed)
    D = to_dense(A)
    x, xt = synth.dense(n, seed + 100), synth.dense(m, seed + 200)
    r = orc.spmv_fwd(A, x)
    assert_S_close(r.value, D @ x, r.S, R64, "A x")
    rt = orc.spmv_fwd(A, xt, op=1)
    assert_S_close(rt.value, D.T @ xt, rt.S, R64, "A^T x")


def test_spmv_poisson_eigenvectors(orc):
    """Closed form: v_pq(i,j) = sin(p pi i/(N+1)) sin(q pi j/(N+1)) with
    lambda = 4 - 2cos(p pi/(N+1)) - 2cos(q pi/(N+1))  (2D A_N of P:683-687)."""
    N = 48
    A = synth.poisson2d(N)
    g = np.arange(1, N + 1)
    for p, q in [(1, 1), (3, 7), (N, N - 2)]:
        v = np.outer(np.sin(p * np.pi * g / (N + 1)), np.sin(q * np.pi * g / (N + 1))).ravel()
        lam = 4 - 2 * np.cos(p * np.pi / (N + 1)) - 2 * np.cos(q * np.pi / (N + 1))
        r = orc.spmv_fwd(A, v)
        assert_S_close(r.value, lam * v, r.S, 1e-13 * 8, "eigen")


def test_spmv_rowsum_missing_neighbours(orc):
    """A 1 = number of missing grid neighbours per row (2D Poisson, integers: bit-exact)."""
    N = 37
    A = synth.poisson2d(N)
    ix, iy = np.divmod(np.arange(N * N), N)
    missing = (ix == 0).astype(int) + (ix == N - 1) + (iy == 0) + (iy == N - 1)
    np.testing.assert_array_equal(orc.spmv_fwd(A, np.ones(N * N)).value, missing)
    # and the same in fp32
    A32 = A.with_values(A.values.astype(np.float32))
    y32 = orc.spmv_fwd(A32, np.ones(N * N, np.float32)).value
    assert y32.dtype == np.float32
    np.testing.assert_array_equal(y32, missing)


# ---------------------------------------------------------------- spmv bwd
def test_spmv_vjp_spec_examples(orc):
    e = SPEC["spmv_vjp_I2"]
    dA, dx = orc.spmv_bwd(eye(2), np.array(e["x"], float), np.array(e["v"], float))
    assert dA.tolist() == e["gradA_diag"] and dx.value.tolist() == e["gradx"]
    dA, dx = orc.spmv_bwd(eye(2), np.array(e["x"], float), np.zeros(2))
    assert dA.tolist() == [0, 0] and dx.value.tolist() == [0, 0]
    e = SPEC["spmv_vjp_A3_e1"]
    dA, dx = orc.spmv_bwd(A3(), np.array(e["x"], float), np.array(e["v"], float))
    assert dx.value.tolist() == e["gradx"]
    # gradA on column 0 entries = v_i * 1, zero elsewhere
    assert dA.tolist() == [1, 0, 1, 0, 0, 0, 0]


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spmv_vjp_dense_autograd(orc, seed, m, n, d):
    """Dense torch autograd of L = dy . (A x), then masked (Table 1)."""
    A = synth.random_csr(m, n, d, seed)
    x, dy = synth.dense(n, seed + 1), synth.dense(m, seed + 2)
    Ad = torch.tensor(to_dense(A), requires_grad=True)
    xt = torch.tensor(x, requires_grad=True)
    (torch.tensor(dy) @ (Ad @ xt)).backward()
    dA, dx = orc.spmv_bwd(A, x, dy)
    # dA: one product per stored entry -> bit-exact (reading A18)
    np.testing.assert_array_equal(dA, gather_mask(Ad.grad.numpy(), A.indptr, A.indices))
    assert_S_close(dx.value, xt.grad.numpy(), dx.S, R64, "dx")
    # op = T: y = A^T x (x in R^m)
    x2, dy2 = synth.dense(m, seed + 3), synth.dense(n, seed + 4)
    Ad2 = torch.tensor(to_dense(A), requires_grad=True)
    x2t = torch.tensor(x2, requires_grad=True)
    (torch.tensor(dy2) @ (Ad2.T @ x2t)).backward()
    dA2, dx2 = orc.spmv_bwd(A, x2, dy2, op=1)
    np.testing.assert_array_equal(dA2, gather_mask(Ad2.grad.numpy(), A.indptr, A.indices))
    assert_S_close(dx2.value, x2t.grad.numpy(), dx2.S, R64, "dx op T")


def test_spmv_vjp_exact_fd_and_identities(orc):
    """Integer inputs: L(x) = dy.(Ax) is linear, so central FD with h = 1 is exact; the
    adjoint identity <dy, Ax> = <A^T dy, x> and Euler <dA, A>_F = <dy, Ax> hold exactly."""
    A = synth.random_csr(24, 17, 0.3, 5, values="int")
    x = synth.dense(17, 6, values="int")
    dy = synth.dense(24, 7, values="int")
    dA, dx = orc.spmv_bwd(A, x, dy)
    L = lambda xx: float(dy @ orc.spmv_fwd(A, xx).value)
    fd = np.array([(L(x + e) - L(x - e)) / 2 for e in np.eye(17)])
    np.testing.assert_array_equal(dx.value, fd)
    Lv = lambda vals: float(dy @ orc.spmv_fwd(A.with_values(vals), x).value)
    fdA = np.array([(Lv(A.values + e) - Lv(A.values - e)) / 2 for e in np.eye(A.nnz)])
    np.testing.assert_array_equal(dA, fdA)
    assert float(dy @ orc.spmv_fwd(A, x).value) == float(dx.value @ x) == float(dA @ A.values)


def test_spmv_fp32_rounds_once(orc):
    A = synth.random_csr(40, 30, 0.3, 11, dtype=np.float32)
    x = synth.dense(30, 12, np.float32)
    dy = synth.dense(40, 13, np.float32)
    r = orc.spmv_fwd(A, x)
    assert r.value.dtype == np.float32
    assert_S_close(r.value, to_dense(A) @ x.astype(np.float64), r.S, R32, "fp32 spmv")
    dA, _ = orc.spmv_bwd(A, x, dy)
    rows = np.repeat(np.arange(40), np.diff(A.indptr))
    np.testing.assert_array_equal(dA, dy[rows] * x[A.indices])  # fp32 IEEE multiply


# ---------------------------------------------------------------- spmm
def test_spmm_spec_examples(orc):
    B = np.array(SPEC["spmm_I2"]["B"], float)
    assert orc.spmm_fwd(eye(2), B).value.tolist() == B.tolist()
    dA, dX = orc.spmm_bwd(eye(2), B, B)                                      # gradB = V
    assert dX.value.tolist() == B.tolist()
    assert orc.spmm_fwd(A3(), np.ones((3, 2))).value.tolist() == SPEC["spmm_A3_ones"]["C"]
    dA, _ = orc.spmm_bwd(A3(), np.ones((3, 2)), np.ones((3, 2)))
    assert (dA.value == SPEC["spmm_vjp_A3_ones"]["gradA_value"]).all()


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spmm_dense_autograd(orc, seed, m, n, d):
    k = 5
    A = synth.random_csr(m, n, d, seed)
    X, dY = synth.dense((n, k), seed + 1), synth.dense((m, k), seed + 2)
    Ad = torch.tensor(to_dense(A), requires_grad=True)
    Xt = torch.tensor(X, requires_grad=True)
    Y = Ad @ Xt
    (torch.tensor(dY) * Y).sum().backward()
    r = orc.spmm_fwd(A, X)
    assert_S_close(r.value, Y.detach().numpy(), r.S, R64, "Y")
    dA, dX = orc.spmm_bwd(A, X, dY)
    assert_S_close(dA.value, gather_mask(Ad.grad.numpy(), A.indptr, A.indices), dA.S, R64, "dA")
    assert_S_close(dX.value, Xt.grad.numpy(), dX.S, R64, "dX")


def test_spmm_rank1_reduces_to_spmv(orc):
    """X = x w^T => Y = (A x) w^T; dY = u w^T => dA = (u (X w)^T)(.)mask(A), dX = (A^T u) w^T.
    Integer data so every side is exact."""
    A = synth.poisson2d(9)
    x, w, u = (synth.dense(s, i, values="int") for s, i in [(81, 1), (6, 2), (81, 3)])
    Y = orc.spmm_fwd(A, np.outer(x, w)).value
    np.testing.assert_array_equal(Y, np.outer(orc.spmv_fwd(A, x).value, w))
    X = synth.dense((81, 6), 4, values="int")
    dA, dX = orc.spmm_bwd(A, X, np.outer(u, w))
    dA_ref, dx_ref = orc.spmv_bwd(A, X @ w, u)
    np.testing.assert_array_equal(dA.value, dA_ref)
    dA2, dX2 = orc.spmm_bwd(A, np.outer(x, w), np.outer(u, w))
    np.testing.assert_array_equal(dX2.value, np.outer(dx_ref.value, w))


# ---------------------------------------------------------------- transpose
def test_transpose_spec_examples(orc):
    ATp, ATi, ATv, perm = orc.csr_transpose(eye(3))
    assert ATp.tolist() == [0, 1, 2, 3] and ATi.tolist() == [0, 1, 2]
    ATp, ATi, ATv, perm = orc.csr_transpose(A3())
    assert ATp.tolist() == SPEC["A3_csr"]["indptr"] and ATv.tolist() == SPEC["A3_csr"]["values"]
    e = SPEC["transpose_single"]
    S1 = synth.CSR(2, 3, np.array([0, 1, 1]), np.array([2], np.int32), np.array([5.0]))
    ATp, ATi, ATv, perm = orc.csr_transpose(S1)
    assert ATp.tolist() == [0, 0, 0, 1] and ATi.tolist() == [0] and ATv.tolist() == [5.0]


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_transpose_dense_and_involution(orc, seed, m, n, d):
    A = synth.random_csr(m, n, d, seed, empty_rows=(seed % 2 == 0))
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    AT = synth.CSR(n, m, ATp, ATi, ATv)
    np.testing.assert_array_equal(to_dense(AT), to_dense(A).T)
    np.testing.assert_array_equal(pattern_dense(AT), pattern_dense(A).T)
    for j in range(n):
        assert (np.diff(ATi[ATp[j]:ATp[j + 1]]) > 0).all()
    assert sorted(perm.tolist()) == list(range(A.nnz))
    np.testing.assert_array_equal(A.values[perm], ATv)
    Bp, Bi, Bv, _ = orc.csr_transpose(AT)
    np.testing.assert_array_equal(Bp, A.indptr)
    np.testing.assert_array_equal(Bi, A.indices)
    np.testing.assert_array_equal(Bv, A.values)


def test_transpose_poisson_symmetric(orc):
    A = synth.poisson3d(6)
    ATp, ATi, ATv, perm = orc.csr_transpose(A)
    np.testing.assert_array_equal(ATp, A.indptr)
    np.testing.assert_array_equal(ATi, A.indices)
    np.testing.assert_array_equal(ATv, A.values)


# ---------------------------------------------------------------- spgemm
def _grid_A2_closed_form(N, dim):
    """Entries of A^2 for the dim-D Poisson stencil A = 2dim I - Adj (Appendix A):
    diag (2dim)^2 + deg(i); axis neighbour -4dim; straight distance-2 1; diagonal neighbour 2."""
    n = N ** dim
    coords = np.array(np.unravel_index(np.arange(n), (N,) * dim)).T
    rows, cols, vals = [], [], []
    offsets = {}
    for o in itertools.product(range(-2, 3), repeat=dim):
        o = np.array(o)
        l1 = np.abs(o).sum()
        nz = (o != 0).sum()
        if l1 == 0:
            offsets[tuple(o)] = "diag"
        elif l1 == 1:
            offsets[tuple(o)] = -4 * dim
        elif l1 == 2 and nz == 1:
            offsets[tuple(o)] = 1
        elif l1 == 2 and nz == 2:
            offsets[tuple(o)] = 2
    deg = ((coords > 0).astype(int) + (coords < N - 1)).sum(axis=1)
    for o, v in offsets.items():
        t = coords + np.array(o)
        ok = ((t >= 0) & (t < N)).all(axis=1)
        src = np.flatnonzero(ok)
        dst = np.ravel_multi_index(tuple(t[ok].T), (N,) * dim)
        rows.append(src)
        cols.append(dst)
        vals.append(((2 * dim) ** 2 + deg[src]) if v == "diag" else np.full(src.size, v))
    rows, cols, vals = map(np.concatenate, (rows, cols, vals))
    order = np.lexsort((cols, rows))
    return rows[order], cols[order], vals[order].astype(float)


def _coo(Cp, Ci):
    return np.repeat(np.arange(len(Cp) - 1), np.diff(Cp)), Ci


def test_spgemm_spec_examples(orc):
    C = A3()
    Cp, Ci = orc.spgemm_symbolic(C, C)
    Cv = orc.spgemm_numeric(C, C, Cp, Ci).value
    np.testing.assert_array_equal(to_dense(synth.CSR(3, 3, Cp, Ci, Cv)), SPEC["spgemm_A3_A3"]["dense"])
    e = SPEC["spgemm_cancel"]
    Ar = synth.CSR(1, 2, np.array([0, 2]), np.array([0, 1], np.int32), np.array(e["A_row"], float))
    Bc = synth.CSR(2, 1, np.array([0, 1, 2]), np.array([0, 0], np.int32), np.array(e["B_col"], float))
    Cp, Ci = orc.spgemm_symbolic(Ar, Bc)
    assert Cp[-1] == e["nnz"]
    assert orc.spgemm_numeric(Ar, Bc, Cp, Ci).value.tolist() == [e["value"]]
    A = synth.random_csr(12, 12, 0.3, 3)                                                   # S:134 A I = A
    Cp, Ci = orc.spgemm_symbolic(A, eye(12))
    np.testing.assert_array_equal(Cp, A.indptr)
    np.testing.assert_array_equal(Ci, A.indices)
    np.testing.assert_array_equal(orc.spgemm_numeric(A, eye(12), Cp, Ci).value, A.values)


def test_spgemm_fig3_pattern(orc):
    """PAPER Fig. 3: 9x9 5-point pattern times 9x3 aggregation = printed 9x3 pattern."""
    mats, flows = load_fig3()
    A, B = csr_from_pattern(mats["A"]), csr_from_pattern(mats["B"])
    Cp, Ci = orc.spgemm_symbolic(A, B)
    np.testing.assert_array_equal(pattern_dense(synth.CSR(9, 3, Cp, Ci, np.ones(len(Ci)))), mats["C"])
    # Arrows: a one-hot dC at C(i,j) sends gradient exactly to the drawn A and B entries
    for (ci, cj), a_ent, b_ent in flows:
        rows = np.repeat(np.arange(9), np.diff(Cp))
        dC = ((rows == ci) & (Ci == cj)).astype(float)
        dA, dB = orc.spgemm_bwd(A, B, Cp, Ci, dC)
        Arows = np.repeat(np.arange(9), np.diff(A.indptr))
        Brows = np.repeat(np.arange(9), np.diff(B.indptr))
        got_a = {(int(r), int(c)) for r, c, v in zip(Arows, A.indices, dA.value) if v != 0}
        got_b = {(int(r), int(c)) for r, c, v in zip(Brows, B.indices, dB.value) if v != 0}
        assert got_a == set(a_ent) and got_b == set(b_ent)


@pytest.mark.parametrize("dim,N", [(2, 5), (2, 9), (2, 16), (3, 5), (3, 7)])
def test_spgemm_poisson_closed_forms(orc, dim, N):
    A = synth.poisson2d(N) if dim == 2 else synth.poisson3d(N)
    Cp, Ci = orc.spgemm_symbolic(A, A)
    nnz_closed = 13 * N * N - 20 * N + 4 if dim == 2 else 25 * N ** 3 - 42 * N ** 2 + 12 * N
    assert Cp[-1] == nnz_closed
    r, c, v = _grid_A2_closed_form(N, dim)
    cr, cc = _coo(Cp, Ci)
    np.testing.assert_array_equal(cr, r)
    np.testing.assert_array_equal(cc, c)
    np.testing.assert_array_equal(orc.spgemm_numeric(A, A, Cp, Ci).value, v)


def test_spgemm_config1_sizes(orc):
    """BASELINE config 1: 16x16 2D Poisson; nnz(A^2) = 3012."""
    A = synth.poisson2d(16)
    Cp, Ci = orc.spgemm_symbolic(A, A)
    assert A.nnz == 1216 and Cp[-1] == 3012


@pytest.mark.parametrize("seed,m,n,d", PROTOCOL)
def test_spgemm_dense_autograd(orc, seed, m, n, d):
    p = 7
    A = synth.random_csr(m, n, d, seed)
    B = synth.random_csr(n, p, d, seed + 50)
    Cp, Ci = orc.spgemm_symbolic(A, B)
    # structural pattern vs boolean product of the patterns
    PC = (pattern_dense(A).astype(int) @ pattern_dense(B).astype(int)) > 0
    np.testing.assert_array_equal(pattern_dense(synth.CSR(m, p, Cp, Ci, np.ones(len(Ci)))), PC)
    Ad = torch.tensor(to_dense(A), requires_grad=True)
    Bd = torch.tensor(to_dense(B), requires_grad=True)
    Cd = Ad @ Bd
    r = orc.spgemm_numeric(A, B, Cp, Ci)
    assert_S_close(r.value, gather_mask(Cd.detach().numpy(), Cp, Ci), r.S, R64, "C")
    dC = synth.dense(len(Ci), seed + 9)
    V = np.zeros((m, p))
    V[_coo(Cp, Ci)] = dC
    (torch.tensor(V) * Cd).sum().backward()
    dA, dB = orc.spgemm_bwd(A, B, Cp, Ci, dC)
    assert_S_close(dA.value, gather_mask(Ad.grad.numpy(), A.indptr, A.indices), dA.S, R64, "dA")
    assert_S_close(dB.value, gather_mask(Bd.grad.numpy(), B.indptr, B.indices), dB.S, R64, "dB")


def test_spgemm_vjp_identities(orc):
    """Integer A = B = 2D Poisson-pattern random ints:
    Euler <V, AB> = <dA, A> = <dB, B>; exact central FD (h = 1) of the quadratic
    f(A) = <V, A A> gives dA + dB (reading A13); ones adjoint dA_ik = rowsum(B)_k,
    dB_kj = colsum(A)_k; rank-1 adjoint V = (u w^T)(.)mask(C) => dA = (u (B w)^T)(.)mask(A)."""
    P = synth.poisson2d(6)
    A = P.with_values(synth.dense(P.nnz, 1, values="int"))
    Cp, Ci = orc.spgemm_symbolic(A, A)
    V = synth.dense(len(Ci), 2, values="int")
    C = orc.spgemm_numeric(A, A, Cp, Ci).value
    dA, dB = orc.spgemm_bwd(A, A, Cp, Ci, V)
    assert float(V @ C) == float(dA.value @ A.values) == float(dB.value @ A.values)
    f = lambda vals: float(V @ orc.spgemm_numeric(A.with_values(vals), A.with_values(vals), Cp, Ci).value)
    fd = np.array([(f(A.values + e) - f(A.values - e)) / 2 for e in np.eye(A.nnz)])
    np.testing.assert_array_equal(dA.value + dB.value, fd)
    # ones adjoint
    B = synth.random_csr(36, 36, 0.2, 4, values="int")
    Cp2, Ci2 = orc.spgemm_symbolic(A, B)
    dA1, dB1 = orc.spgemm_bwd(A, B, Cp2, Ci2, np.ones(len(Ci2)))
    rowsumB = orc.spmv_fwd(B, np.ones(36)).value
    colsumA = orc.spmv_fwd(A, np.ones(36), op=1).value
    np.testing.assert_array_equal(dA1.value, rowsumB[A.indices])
    np.testing.assert_array_equal(dB1.value, colsumA[np.repeat(np.arange(36), np.diff(B.indptr))])
    # rank-1 adjoint through SpMV
    u, w = synth.dense(36, 5, values="int"), synth.dense(36, 6, values="int")
    crow, ccol = _coo(Cp2, Ci2)
    dA2, dB2 = orc.spgemm_bwd(A, B, Cp2, Ci2, u[crow] * w[ccol])
    dA_ref, _ = orc.spmv_bwd(A, orc.spmv_fwd(B, w).value, u)
    np.testing.assert_array_equal(dA2.value, dA_ref)
    dB_ref, _ = orc.spmv_bwd(B, w, orc.spmv_fwd(A, u, op=1).value)
    np.testing.assert_array_equal(dB2.value, dB_ref)


def test_spgemm_vjp_spec_examples(orc):
    e = SPEC["spgemm_vjp_diag_full"]
    Ad = synth.CSR(2, 2, np.array([0, 1, 2]), np.array([0, 1], np.int32), np.array(e["a"]))
    Bf = synth.CSR(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1], np.int32), np.array([1., 2, 3, 4]))
    Cp, Ci = orc.spgemm_symbolic(Ad, Bf)
    _, dB = orc.spgemm_bwd(Ad, Bf, Cp, Ci, np.ones(len(Ci)))
    assert dB.value.reshape(2, 2).tolist() == e["gradB"]
    I2 = eye(2)
    Cp, Ci = orc.spgemm_symbolic(I2, I2)
    dA, dB = orc.spgemm_bwd(I2, I2, Cp, Ci, np.ones(2))
    assert dA.value.tolist() == [1, 1] and dB.value.tolist() == [1, 1]
