"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no products, no gradients, no
transposes): it only builds input matrices and dense operands.  Both sides of
every parity check (oracle/ and the CUDA path) receive the same arrays from here.

Matrices:

* ``poisson1d(N)``      A_N = tridiag(-1, 2, -1)           PAPER.md Eq. mat_1d_fd
* ``poisson2d(Nx, Ny)`` A_Nx (x) I + I (x) A_Ny (5-point)   PAPER.md Eq. mat_2d_fd
* ``poisson3d(N)``      three-term Kronecker sum (7-point)  BASELINE.json config 3 (not in the paper)
* ``powerlaw(n)``       power-law row lengths, mean 16/row  BASELINE.json config 4, SURVEY.md 8(d) d.2
* ``random_csr(m, n, density)``  Bernoulli pattern for small tests (SPEC.md S:353-356 protocol)

All index arrays are ``indptr`` int64 and ``indices`` int32; values
are float64 or float32.  Seeds follow SURVEY.md 8(d) d.2: ``1000*cfg + j`` with
j = 1 pattern, 2 values, 3 x/X, 4 dy/dY, 5 dC, 6 L.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "CSR", "poisson1d", "poisson2d", "poisson3d", "powerlaw", "random_csr",
    "dense", "int_values", "real_values", "seed_of",
]


@dataclass
class CSR:
    """Canonical CSR: indptr int64[nrows+1], indices int32[nnz] (strictly increasing per row)."""
    nrows: int
    ncols: int
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray | None

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def with_values(self, values: np.ndarray) -> "CSR":
        assert values.shape == (self.nnz,)
        return CSR(self.nrows, self.ncols, self.indptr, self.indices, values)


def seed_of(cfg: int, j: int) -> int:
    """SURVEY.md 8(d) d.2 seed convention."""
    return 1000 * cfg + j


def _from_candidates(nrows: int, ncols: int, cols: np.ndarray, vals: np.ndarray, valid: np.ndarray, dtype) -> CSR:
    """cols/vals/valid are [nrows, w] candidate tables whose valid columns are already ascending per row."""
    counts = valid.sum(axis=1, dtype=np.int64)
    indptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = cols[valid].astype(np.int32)
    values = vals[valid].astype(dtype)
    return CSR(nrows, ncols, indptr, indices, values)


def poisson1d(N: int, dtype=np.float64) -> CSR:
    """A_N of PAPER.md Eq. mat_1d_fd: 2 on the diagonal, -1 on the first off-diagonals."""
    i = np.arange(N, dtype=np.int64)[:, None]
    off = np.array([-1, 0, 1], dtype=np.int64)[None, :]
    cols = i + off
    valid = (cols >= 0) & (cols < N)
    vals = np.where(off == 0, 2.0, -1.0) * np.ones_like(cols, dtype=np.float64)
    return _from_candidates(N, N, cols, vals, valid, dtype)


def poisson2d(Nx: int, Ny: int | None = None, dtype=np.float64) -> CSR:
    """A_{Nx x Ny} = A_Nx (x) I_Ny + I_Nx (x) A_Ny (PAPER.md Eq. mat_2d_fd), natural ordering
    row = ix*Ny + iy.  Diagonal 4, the four grid neighbours -1."""
    Ny = Nx if Ny is None else Ny
    n = Nx * Ny
    r = np.arange(n, dtype=np.int64)
    ix, iy = r // Ny, r % Ny
    # candidates in ascending column order: (ix-1,iy), (ix,iy-1), diag, (ix,iy+1), (ix+1,iy)
    cols = np.stack([r - Ny, r - 1, r, r + 1, r + Ny], axis=1)
    valid = np.stack([ix > 0, iy > 0, np.ones(n, bool), iy < Ny - 1, ix < Nx - 1], axis=1)
    vals = np.broadcast_to(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), cols.shape)
    return _from_candidates(n, n, cols, vals, valid, dtype)


def poisson3d(N: int, dtype=np.float64) -> CSR:
    """7-point 3D Poisson: A_N(x)I(x)I + I(x)A_N(x)I + I(x)I(x)A_N, row = (ix*N + iy)*N + iz.
    Diagonal 6, the six grid neighbours -1 (BASELINE.json config 3)."""
    n = N * N * N
    r = np.arange(n, dtype=np.int64)
    ix, iy, iz = r // (N * N), (r // N) % N, r % N
    N2 = N * N
    cols = np.stack([r - N2, r - N, r - 1, r, r + 1, r + N, r + N2], axis=1)
    valid = np.stack([ix > 0, iy > 0, iz > 0, np.ones(n, bool), iz < N - 1, iy < N - 1, ix < N - 1], axis=1)
    vals = np.broadcast_to(np.array([-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0]), cols.shape)
    return _from_candidates(n, n, cols, vals, valid, dtype)


def _distinct_sorted_columns(rng: np.random.Generator, lengths: np.ndarray, ncols: int) -> np.ndarray:
    """For every row draw lengths[i] DISTINCT uniform columns in [0, ncols), sorted ascending.
    Returns the flat int32 column array in row order."""
    nrows = lengths.shape[0]
    nnz = int(lengths.sum())
    rows = np.repeat(np.arange(nrows, dtype=np.int64), lengths)
    cols = rng.integers(0, ncols, size=nnz, dtype=np.int64)
    key = rows * ncols + cols
    key.sort()
    del rows, cols
    dup = np.flatnonzero(key[1:] == key[:-1]) + 1
    if dup.size:
        bad_rows = np.unique(key[dup] // ncols)
        starts = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(lengths, out=starts[1:])
        for r in bad_rows:
            s, e = starts[r], starts[r + 1]
            seg = np.unique(key[s:e] - r * ncols)
            while seg.size < e - s:
                extra = rng.integers(0, ncols, size=int(e - s - seg.size), dtype=np.int64)
                seg = np.unique(np.concatenate([seg, extra]))
            key[s:e] = seg + r * ncols
    return (key % ncols).astype(np.int32)


def powerlaw(n: int = 1 << 23, seed: int = seed_of(4, 1), mean: int = 16, dtype=np.float32,
             values: str = "real") -> CSR:
    """BASELINE.json config 4 recipe:
    u_i = (i + 1/2)/n, l_i = min(round(8 u_i^{-1/2}), 65536, n); add +1 to the longest rows
    (stratified order) until sum(l) = mean*n exactly; apply a seeded row permutation; columns
    are l_i distinct uniform draws in [0, n), sorted.  Values: U[-1,1) ('real') or U{-3..3} ('int')."""
    rng = np.random.default_rng(seed)
    u = (np.arange(n, dtype=np.float64) + 0.5) / n
    lengths = np.floor(8.0 * u ** -0.5 + 0.5).astype(np.int64)
    lengths = np.minimum(np.minimum(lengths, 65536), n)
    target = mean * n
    deficit = target - int(lengths.sum())
    if deficit > 0:
        lengths[:deficit] += 1          # rows 0.. are the longest (smallest u)
        lengths = np.minimum(lengths, n)
    elif deficit < 0:
        # only for tiny n where the cap bites from below; trim the shortest rows
        k = -deficit
        lengths[-k:] -= 1
    lengths = lengths[rng.permutation(n)]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=indptr[1:])
    indices = _distinct_sorted_columns(rng, lengths, n)
    vrng = np.random.default_rng(seed + 1)
    vals = real_values(vrng, indptr[-1], dtype) if values == "real" else int_values(vrng, indptr[-1], dtype)
    return CSR(n, n, indptr, indices, vals)


def bidiag_lower(n: int, init: str = "identity", seed: int = seed_of(5, 6)) -> CSR:
    """Lower-bidiagonal L of PAPER 4.3 ("a lower bidiagonal L"), 2n - 1 stored entries.
    init 'identity': L = I with the subdiagonal stored as explicit zeros;
    init 'seeded': diagonal U[0.9, 1.1], subdiagonal U[-0.1, 0.1]."""
    i = np.arange(n, dtype=np.int64)
    cols = np.stack([i - 1, i], axis=1)
    valid = cols >= 0
    if init == "identity":
        vals = np.broadcast_to(np.array([0.0, 1.0]), cols.shape)
    else:
        rng = np.random.default_rng(seed)
        vals = np.stack([rng.uniform(-0.1, 0.1, n), rng.uniform(0.9, 1.1, n)], axis=1)
    return _from_candidates(n, n, cols, vals, valid, np.float64)


def random_csr(m: int, n: int, density: float, seed: int, dtype=np.float64, values: str = "real",
               empty_rows: bool = False) -> CSR:
    """Bernoulli(density) pattern on an m x n grid (density 1.0 = full pattern).  With
    empty_rows=True every third row is emptied (edge case A14)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density if density < 1.0 else np.ones((m, n), bool)
    if empty_rows:
        mask[::3, :] = False
    counts = mask.sum(axis=1, dtype=np.int64)
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.nonzero(mask)[1].astype(np.int32)
    vals = real_values(rng, indptr[-1], dtype) if values == "real" else int_values(rng, indptr[-1], dtype)
    return CSR(m, n, indptr, indices, vals)


def real_values(rng: np.random.Generator, size, dtype=np.float64) -> np.ndarray:
    """U[-1, 1), rounded once to dtype."""
    return rng.uniform(-1.0, 1.0, size=size).astype(dtype)


def int_values(rng: np.random.Generator, size, dtype=np.float64) -> np.ndarray:
    """U{-3, ..., 3}: integer-valued inputs make every op order-independent."""
    return rng.integers(-3, 4, size=size).astype(dtype)


def dense(shape, seed: int, dtype=np.float64, values: str = "real") -> np.ndarray:
    rng = np.random.default_rng(seed)
    return real_values(rng, shape, dtype) if values == "real" else int_values(rng, shape, dtype)


def tri_random(n: int, density: float, seed: int, upper: bool = False, values: str = "real",
               unit: bool = False) -> CSR:
    """Random triangular matrix for the SpTRSV tests (PAPER 3.1.5): a Bernoulli(density)
    pattern strictly below (or above) the diagonal plus the diagonal (omitted when unit).
    'real': off-diagonal U[-1, 1) / (1 + row length), diagonal +-U[1, 2) -- diagonally
    dominant, so substitution is well conditioned.  'int': off-diagonal U{-3..3}, diagonal
    from {+-1, +-2, +-4} (so b = T x_int keeps every step exact in binary floating point)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    mask = np.triu(mask, 1) if upper else np.tril(mask, -1)
    if not unit:
        mask |= np.eye(n, dtype=bool)
    counts = mask.sum(axis=1, dtype=np.int64)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    rows, cols = np.nonzero(mask)
    diag = rows == cols
    if values == "real":
        vals = rng.uniform(-1.0, 1.0, rows.size) / (1.0 + counts[rows])
        vals[diag] = rng.choice([-1.0, 1.0], diag.sum()) * rng.uniform(1.0, 2.0, diag.sum())
    else:
        vals = rng.integers(-3, 4, rows.size).astype(np.float64)
        vals[diag] = rng.choice([-4.0, -2.0, -1.0, 1.0, 2.0, 4.0], diag.sum())
    return CSR(n, n, indptr, cols.astype(np.int32), vals)


def lower_part(A: CSR) -> CSR:
    """The lower triangle (j <= i) of A, entries kept in place -- e.g. the IC(0) pattern of a
    Poisson matrix (SURVEY 8(f) f3 workload)."""
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.indptr))
    keep = A.indices <= rows
    indptr = np.zeros(A.nrows + 1, np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=A.nrows), out=indptr[1:])
    return CSR(A.nrows, A.ncols, indptr, A.indices[keep].copy(),
               None if A.values is None else A.values[keep].copy())


def tri_banded(n: int, per_row: int, band: int, seed: int, upper: bool = False, values: str = "real",
               unit: bool = False) -> CSR:
    """Large random triangular matrix without a dense mask: row i draws per_row candidate
    columns uniformly from the band [i - band, i) (upper: (i, i + band]), duplicates and
    out-of-range candidates dropped, plus the diagonal (omitted when unit).  Values as in
    tri_random (diagonally dominant 'real', or integer with diagonal in {+-1, +-2, +-4})."""
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.int64)[:, None]
    off = rng.integers(1, band + 1, size=(n, per_row))
    cand = i + off if upper else i - off
    cand = np.where((cand >= 0) & (cand < n), cand, -1)
    cand = np.sort(cand, axis=1)
    dup = np.zeros_like(cand, dtype=bool)
    dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
    keep = (cand >= 0) & ~dup
    if not unit:
        cand = np.concatenate([cand, np.broadcast_to(i, (n, 1))], axis=1)
        keep = np.concatenate([keep, np.ones((n, 1), bool)], axis=1)
    order = np.argsort(np.where(keep, cand, np.iinfo(np.int64).max), axis=1, kind="stable")
    cand = np.take_along_axis(cand, order, axis=1)
    keep = np.take_along_axis(keep, order, axis=1)
    counts = keep.sum(axis=1)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    rows = np.repeat(np.arange(n), counts)
    cols = cand[keep]
    diag = rows == cols
    if values == "real":
        vals = rng.uniform(-1.0, 1.0, cols.size) / (1.0 + counts[rows])
        vals[diag] = rng.choice([-1.0, 1.0], diag.sum()) * rng.uniform(1.0, 2.0, diag.sum())
    else:
        vals = rng.integers(-3, 4, cols.size).astype(np.float64)
        vals[diag] = rng.choice([-4.0, -2.0, -1.0, 1.0, 2.0, 4.0], diag.sum())
    return CSR(n, n, indptr, cols.astype(np.int32), vals)


def powerlaw_graph(n: int, mean: float = 5.0, seed: int = 4401, weighted: bool = False,
                   dtype=np.float32) -> CSR:
    """Synthetic graph for the GCN layer (PAPER 4.4 P:951-954: graphs of 1e5 to
    9e5 nodes, "each node has on average 5 incident edges").  Out-degrees l_i =
    round((mean/2) u_i^{-1/2}) (u_i = (i+1/2)/n, power law with exponent 3), adjusted by +-1 on the
    longest / shortest rows to sum exactly to round(mean n), at least 1, seeded row permutation;
    neighbours l_i distinct uniform draws in [0, n), sorted; edge weights 1 (or U[0.5, 2))."""
    rng = np.random.default_rng(seed)
    u = (np.arange(n, dtype=np.float64) + 0.5) / n
    lengths = np.floor(0.5 * mean * u ** -0.5 + 0.5).astype(np.int64)
    lengths = np.clip(lengths, 1, min(65536, n))
    target = int(round(mean * n))
    d = target - int(lengths.sum())
    if d > 0:
        lengths[:d] += 1
    elif d < 0:
        idx = np.nonzero(lengths > 1)[0][::-1][:-d]
        lengths[idx] -= 1
    lengths = lengths[rng.permutation(n)]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=indptr[1:])
    indices = _distinct_sorted_columns(rng, lengths, n)
    vals = (rng.uniform(0.5, 2.0, indptr[-1]) if weighted else np.ones(indptr[-1])).astype(dtype)
    return CSR(n, n, indptr, indices, vals)
