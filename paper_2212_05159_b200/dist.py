"""Row partition + collective layer (BASELINE north_star "Rows of A are
partitioned ... x/B replicated and the dx/dB partial gradients combined by NCCL").

Rows of A are split into contiguous blocks, one per rank.  A rank stores its block with the
columns compacted to the interval [col_lo, col_hi) its rows reference, and holds x / X / the
rows of B over exactly that interval ("replicated where referenced").  Forward products are
row-local (no communication).  The backward partials -- dx = A_r^T dy_r over [col_lo, col_hi),
dX likewise, and dB over the entries of B's rows [col_lo, col_hi) -- are combined by an
INTERVAL REDUCTION: every index has one owner (the rank owning that row), each rank sends the
parts of its partial that other ranks own and adds what it receives (NCCL send/recv, grouped).
For banded / stencil matrices this touches only the neighbours (a halo exchange); for a
matrix whose rows reference every column it moves the same bytes as a reduce-scatter.

The local compute is injected (`local_ops`), so tests/test_dist_cpu.py drives this exact
logic over gloo with the oracle while the GPU path uses the csrk kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import synth


# ---------------------------------------------------------------- partition (host logic)
def balanced_row_splits(indptr: np.ndarray, world: int, work: np.ndarray | None = None) -> np.ndarray:
    """Contiguous row blocks with about equal nonzeros (or equal `work` per row):
    split p starts at the first row whose prefix reaches p*total/world."""
    m = len(indptr) - 1
    pref = indptr.astype(np.int64) if work is None else np.concatenate([[0], np.cumsum(work, dtype=np.int64)])
    total = pref[-1]
    targets = (np.arange(world + 1, dtype=np.float64) * total / world)
    splits = np.searchsorted(pref, targets, side="left").astype(np.int64)
    splits[0], splits[-1] = 0, m
    return np.maximum.accumulate(np.minimum(splits, m))


def row_block(A: synth.CSR, r0: int, r1: int) -> synth.CSR:
    """Rows [r0, r1) of A with global column indices."""
    s, e = A.indptr[r0], A.indptr[r1]
    vals = None if A.values is None else A.values[s:e].copy()
    return synth.CSR(r1 - r0, A.ncols, (A.indptr[r0:r1 + 1] - s).astype(np.int64), A.indices[s:e].copy(), vals)


def compact_columns(A: synth.CSR, lo: int | None = None, hi: int | None = None):
    """Shift the columns of a row block to its referenced interval [lo, hi)."""
    if lo is None:
        lo = int(A.indices.min()) if A.nnz else 0
        hi = int(A.indices.max()) + 1 if A.nnz else 0
    ind = (A.indices.astype(np.int64) - lo).astype(np.int32)
    return synth.CSR(A.nrows, hi - lo, A.indptr, ind, A.values), lo, hi


@dataclass
class Block:
    """One rank's share: A_r (compacted), its column interval, and ownership tables."""
    rank: int
    world: int
    row_splits: np.ndarray   # [world+1] rows owned by each rank (also owns dx / dX indices)
    A: synth.CSR             # local rows, columns compacted to [col_lo, col_hi)
    col_lo: int
    col_hi: int


def make_block(A: synth.CSR, rank: int, world: int, splits: np.ndarray | None = None) -> Block:
    if splits is None:
        splits = balanced_row_splits(A.indptr, world)
    r0, r1 = int(splits[rank]), int(splits[rank + 1])
    Ar, lo, hi = compact_columns(row_block(A, r0, r1))
    return Block(rank, world, splits, Ar, lo, hi)


# ---------------------------------------------------------------- interval reduction
def interval_plan(lo: int, hi: int, all_intervals: list[tuple[int, int]], owner_starts: np.ndarray, rank: int):
    """Which slices go where.  Returns (sends, recvs, own):
    sends[q] = (a, b): global [a, b) of MY partial owned by q;  recvs[q] = (a, b): global [a, b)
    of q's partial that I own;  own = (a, b): the global range I own."""
    world = len(owner_starts) - 1
    own = (int(owner_starts[rank]), int(owner_starts[rank + 1]))
    sends, recvs = {}, {}
    for q in range(world):
        if q == rank:
            continue
        a, b = max(lo, int(owner_starts[q])), min(hi, int(owner_starts[q + 1]))
        if a < b:
            sends[q] = (a, b)
        qlo, qhi = all_intervals[q]
        a, b = max(qlo, own[0]), min(qhi, own[1])
        if a < b:
            recvs[q] = (a, b)
    return sends, recvs, own


def interval_reduce(partial, lo: int, plan, group=None, add=None):
    """Combine per-rank partials over global index intervals (first dim of `partial` covers
    [lo, lo + len)).  Returns this rank's owned slice, summed over all ranks.  torch tensors;
    the exchange is grouped NCCL (or gloo) send/recv."""
    import torch
    import torch.distributed as tdist
    sends, recvs, own = plan
    out = torch.zeros((own[1] - own[0],) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
    a, b = max(own[0], lo), min(own[1], lo + partial.shape[0])
    if a < b:
        out[a - own[0]:b - own[0]] += partial[a - lo:b - lo]
    ops, bufs = [], []
    for q, (sa, sb) in sorted(sends.items()):
        ops.append(tdist.P2POp(tdist.isend, partial[sa - lo:sb - lo].contiguous(), q, group))
    for q, (ra, rb) in sorted(recvs.items()):
        buf = torch.empty((rb - ra,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
        bufs.append((ra, rb, buf))
        ops.append(tdist.P2POp(tdist.irecv, buf, q, group))
    if ops:
        for w in tdist.batch_isend_irecv(ops):
            w.wait()
    for ra, rb, buf in bufs:
        if add is not None:
            add(out[ra - own[0]:rb - own[0]], buf)
        else:
            out[ra - own[0]:rb - own[0]] += buf
    return out


def all_intervals(lo: int, hi: int, world: int, group=None, device="cpu"):
    import torch
    import torch.distributed as tdist
    t = torch.tensor([lo, hi], dtype=torch.int64, device=device)
    got = [torch.empty_like(t) for _ in range(world)]
    tdist.all_gather(got, t, group=group)
    return [(int(g[0]), int(g[1])) for g in got]


# ---------------------------------------------------------------- distributed ops
class DistCSR:
    """Row-block distributed matrix driving injected local kernels.

    local_ops must provide: spmv_fwd(A, x), spmv_bwd(A, x, dy) -> (dA, dx),
    spmm_fwd(A, X), spmm_bwd(A, X, dY) -> (dA, dX), spgemm(A, B) -> (pattern, values),
    spgemm_bwd(A, B, C, dC) -> (dA, dB), to_dev(np) and from_dev(tensor)."""

    def __init__(self, block: Block, group=None, device="cpu"):
        self.b = block
        self.group = group
        self.device = device
        self.intervals = all_intervals(block.col_lo, block.col_hi, block.world, group, device)
        self.vec_plan = interval_plan(block.col_lo, block.col_hi, self.intervals, block.row_splits, block.rank)

    # y_r = A_r x[col_lo:col_hi]   (no communication)
    def spmv_fwd(self, ops, A_dev, x_local):
        return ops.spmv_fwd(A_dev, x_local)

    # dA_r on A_r's pattern (row-local) and dx owned slice (interval reduction of A_r^T dy_r)
    def spmv_bwd(self, ops, A_dev, x_local, dy_r):
        dA, dx_part = ops.spmv_bwd(A_dev, x_local, dy_r)
        return dA, interval_reduce(dx_part, self.b.col_lo, self.vec_plan, self.group)

    def spmm_bwd(self, ops, A_dev, X_local, dY_r):
        dA, dX_part = ops.spmm_bwd(A_dev, X_local, dY_r)
        return dA, interval_reduce(dX_part, self.b.col_lo, self.vec_plan, self.group)


def gemm_blocks(A_global: synth.CSR, block: Block):
    """For C = A A row-sharded: B_r = rows [col_lo, col_hi) of A (the rows A_r references),
    columns compacted to their own interval.  dB partials live on B_r's entries, i.e. on the
    global entry range [indptr[col_lo], indptr[col_hi]) of A; owners by row blocks."""
    Br_rows = row_block(A_global, block.col_lo, block.col_hi)
    Br, blo, bhi = compact_columns(Br_rows)
    e_lo, e_hi = int(A_global.indptr[block.col_lo]), int(A_global.indptr[block.col_hi])
    entry_owner = A_global.indptr[block.row_splits].astype(np.int64)
    return Br, (blo, bhi), (e_lo, e_hi), entry_owner


# ---------------------------------------------------------------- bench support (GPU, NCCL)
def poisson2d_row_block(Nx: int, Ny: int, rank: int, world: int):
    """Rank's row block of the 2D Poisson matrix on an Nx x Ny grid, columns compacted.
    Built from the rows of synth.poisson2d restricted to the block (no global assembly)."""
    assert Nx % world == 0
    nx_r = Nx // world
    # the block's rows reference grid lines [ix0-1, ix1+1); build that sub-grid's rows and keep ours
    ix0, ix1 = rank * nx_r, (rank + 1) * nx_r
    gx0, gx1 = max(ix0 - 1, 0), min(ix1 + 1, Nx)
    # rows of the global matrix on lines [gx0, gx1) equal poisson2d(gx1-gx0, Ny) except for the
    # couplings across the sub-grid boundary, which are exactly the couplings to lines outside
    # [gx0, gx1) -- never referenced by our rows ix0..ix1-1 unless gx0 = ix0 - 1 etc.
    sub = synth.poisson2d(gx1 - gx0, Ny)
    r0, r1 = (ix0 - gx0) * Ny, (ix1 - gx0) * Ny
    Ar = row_block(sub, r0, r1)
    # our rows keep their global couplings: a neighbour line outside the sub-grid would be
    # ix0-2 or ix1+1, which a 5-point row on ix0..ix1-1 never references.
    col_lo = gx0 * Ny
    Ar = synth.CSR(Ar.nrows, (gx1 - gx0) * Ny, Ar.indptr, Ar.indices, Ar.values)
    return Ar, col_lo


def poisson2d_indptr_at(Nx: int, Ny: int, r: int) -> int:
    """Number of stored entries in rows < r of the Nx x Ny 2D Poisson matrix (closed form)."""
    ix, iy = divmod(int(r), Ny)
    full = ix * (Ny + 2 * (Ny - 1)) + Ny * max(ix - 1, 0) + Ny * min(ix, Nx - 1)
    partial = 0
    if ix < Nx:
        partial = iy * (1 + (ix > 0) + (ix < Nx - 1)) + max(iy - 1, 0) + min(iy, Ny - 1)
    return int(full + partial)


class HaloBench:
    """Weak-scaled config-2 step at N > 1 (bench.py): reduces the dx / dX / dB partials."""

    def __init__(self, world, rank):
        self.world, self.rank = world, rank

    def setup(self, W):
        import torch
        Nx, Ny = 2048 * self.world, 2048
        m = Nx * Ny // self.world
        splits = np.arange(self.world + 1, dtype=np.int64) * m
        lo, hi = W.col_lo, W.col_lo + W.n
        ints = all_intervals(lo, hi, self.world, None, W.dev)
        self.vec_plan = interval_plan(lo, hi, ints, splits, self.rank)
        # dB lives on B_r = rows [lo, hi) of the global matrix: entry offsets of the global A
        nnz_row = lambda r: self._global_indptr(Nx, Ny, r)
        e_lo, e_hi = nnz_row(lo), nnz_row(hi)
        e_ints = all_intervals(e_lo, e_hi, self.world, None, W.dev)
        e_own = np.array([nnz_row(int(s)) for s in splits], dtype=np.int64)
        self.e_lo = e_lo
        self.ent_plan = interval_plan(e_lo, e_hi, e_ints, e_own, self.rank)
        self.torch = torch

    @staticmethod
    def _global_indptr(Nx, Ny, r):
        """indptr[r] of the Nx x Ny 2D Poisson matrix in closed form (row r = ix*Ny + iy has
        1 + [ix>0] + [ix<Nx-1] + [iy>0] + [iy<Ny-1] entries)."""
        return poisson2d_indptr_at(Nx, Ny, r)

    def reduce_partials(self, W):
        W.dx_own = interval_reduce(W.dx, 0 + W.col_lo, self.vec_plan)
        W.dX_own = interval_reduce(W.dX, W.col_lo, self.vec_plan)
        W.dB_own = interval_reduce(W.dB_g, self.e_lo, self.ent_plan)


def halo_rows_block(Nx: int, Ny: int, rank: int, world: int):
    """B_r for the bench: rows [col_lo, col_hi) of the global 2D Poisson matrix (the rows A_r
    references), columns compacted to their own interval."""
    nx_r = Nx // world
    ix0, ix1 = rank * nx_r, (rank + 1) * nx_r
    gx0, gx1 = max(ix0 - 1, 0), min(ix1 + 1, Nx)     # lines of B_r's rows
    hx0, hx1 = max(gx0 - 1, 0), min(gx1 + 1, Nx)     # lines B_r's rows reference
    sub = synth.poisson2d(hx1 - hx0, Ny)
    Br = row_block(sub, (gx0 - hx0) * Ny, (gx1 - hx0) * Ny)
    return synth.CSR(Br.nrows, (hx1 - hx0) * Ny, Br.indptr, Br.indices, Br.values)
