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


def _host_staged(group, t) -> bool:
    """gloo exchanges host tensors: a CUDA partial is staged through the host (tests that run
    several ranks on one GPU); NCCL exchanges device memory directly."""
    import torch.distributed as tdist
    return t.is_cuda and tdist.get_backend(group) == "gloo"


def interval_reduce(partial, lo: int, plan, group=None, add=None):
    """Combine per-rank partials over global index intervals (first dim of `partial` covers
    [lo, lo + len)).  Returns this rank's owned slice, summed over all ranks.  torch tensors;
    the exchange is grouped NCCL (or gloo) send/recv."""
    if _host_staged(group, partial):
        return interval_reduce(partial.cpu(), lo, plan, group, add).to(partial.device)
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


def reduce_scatter_owned(partial, lo: int, owner_starts, rank: int, group=None):
    """The dense combine (right when every rank's partial covers most of the index
    space, config 4): the partial, placed in a zero buffer of world x chunk rows (owner q's range
    at q * chunk, chunk = the largest owned range), is reduced and scattered with ONE
    reduce_scatter_tensor (NCCL: ring / NVLS in-switch reduction).  Returns the owned slice."""
    if _host_staged(group, partial):
        return reduce_scatter_owned(partial.cpu(), lo, owner_starts, rank, group).to(partial.device)
    import torch
    import torch.distributed as tdist
    world = len(owner_starts) - 1
    starts = [int(v) for v in owner_starts]
    chunk = max(starts[q + 1] - starts[q] for q in range(world))
    tail = tuple(partial.shape[1:])
    full = torch.zeros((world * chunk,) + tail, dtype=partial.dtype, device=partial.device)
    hi = lo + partial.shape[0]
    for q in range(world):
        a, b = max(lo, starts[q]), min(hi, starts[q + 1])
        if a < b:
            off = q * chunk + (a - starts[q])
            full[off:off + (b - a)] = partial[a - lo:b - lo]
    out = torch.empty((chunk,) + tail, dtype=partial.dtype, device=partial.device)
    tdist.reduce_scatter_tensor(out, full, group=group)
    return out[:starts[rank + 1] - starts[rank]]


class Combiner:
    """Owner combine of per-rank partials over [lo, hi) (dx, dX, dB):
    'interval' = grouped send/recv of only the overlapping slices (halo for stencils),
    'rs' = the dense reduce-scatter.  mode 'auto' picks 'rs' when the interval exchange would move
    more than half the elements of the dense one (every rank referencing most indices)."""

    def __init__(self, lo: int, hi: int, owner_starts, rank: int, group=None, device="cpu", mode="auto"):
        world = len(owner_starts) - 1
        self.lo, self.rank, self.group, self.owner_starts = lo, rank, group, np.asarray(owner_starts, np.int64)
        ints = all_intervals(lo, hi, world, group, device)
        self.plan = interval_plan(lo, hi, ints, self.owner_starts, rank)
        if mode == "auto":
            sent = [sum(b - a for a, b in interval_plan(l, h, ints, self.owner_starts, q)[0].values())
                    for q, (l, h) in enumerate(ints)]
            total = int(self.owner_starts[-1] - self.owner_starts[0])
            mode = "rs" if world > 1 and max(sent) > 0.5 * total * (world - 1) / world else "interval"
        self.mode = mode

    def __call__(self, partial):
        if self.mode == "rs":
            return reduce_scatter_owned(partial, self.lo, self.owner_starts, self.rank, self.group)
        return interval_reduce(partial, self.lo, self.plan, self.group)


def all_intervals(lo: int, hi: int, world: int, group=None, device="cpu"):
    import torch
    import torch.distributed as tdist
    if tdist.get_backend(group) == "gloo":
        device = "cpu"
    t = torch.tensor([lo, hi], dtype=torch.int64, device=device)
    got = [torch.empty_like(t) for _ in range(world)]
    tdist.all_gather(got, t, group=group)
    return [(int(g[0]), int(g[1])) for g in got]


# ---------------------------------------------------------------- distributed ops
class DistCSR:
    """Row-block distributed matrix driving injected local kernels.

    local_ops must provide: spmv_fwd(A, x), spmv_bwd(A, x, dy) -> (dA, dx),
    spmm_fwd(A, X), spmm_bwd(A, X, dY) -> (dA, dX) on the rank's block (columns compacted to
    [col_lo, col_hi)); partials come back as torch tensors.  `combine` picks the owner combine of
    the dx / dX partials ('auto', 'interval' or 'rs', see Combiner)."""

    def __init__(self, block: Block, group=None, device="cpu", combine="auto"):
        self.b = block
        self.group = group
        self.device = device
        self.vec = Combiner(block.col_lo, block.col_hi, block.row_splits, block.rank, group, device, combine)
        self.intervals = all_intervals(block.col_lo, block.col_hi, block.world, group, device)
        self.vec_plan = self.vec.plan

    # y_r = A_r x[col_lo:col_hi]   (no communication)
    def spmv_fwd(self, ops, A_dev, x_local):
        return ops.spmv_fwd(A_dev, x_local)

    # dA_r on A_r's pattern (row-local) and dx owned slice (combine of A_r^T dy_r)
    def spmv_bwd(self, ops, A_dev, x_local, dy_r):
        dA, dx_part = ops.spmv_bwd(A_dev, x_local, dy_r)
        return dA, self.vec(dx_part)

    def spmm_bwd(self, ops, A_dev, X_local, dY_r):
        dA, dX_part = ops.spmm_bwd(A_dev, X_local, dY_r)
        return dA, self.vec(dX_part)


class DistGemm:
    """C = A A row-sharded: rank r computes C_r = A_r B_r with B_r = the rows of A
    its block references (gemm_blocks), no communication forward; the dB partial lives on B_r's
    entries = the global entry range [indptr[col_lo], indptr[col_hi)) of A and is combined onto
    the entry owners (the rank owning the row).  For A A the owner then adds dA_left + dB."""

    def __init__(self, A_global: synth.CSR, block: Block, group=None, device="cpu", combine="auto"):
        self.B, self.b_cols, (self.e_lo, self.e_hi), self.ent_owner = gemm_blocks(A_global, block)
        self.ent = Combiner(self.e_lo, self.e_hi, self.ent_owner, block.rank, group, device, combine)

    def combine_dB(self, dB_part):
        return self.ent(dB_part)


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


# ---------------------------------------------------------------- config 5 row-sharded
class PcgShard:
    """One rank's share of the row-sharded config-5 step (csrk_pcg_loss_grad_dist): contiguous row
    blocks balanced by nonzeros, A_r and L_r with columns compacted to the rank's EXTENDED interval
    [lo, hi) (its rows plus every column its rows of A or L reference: for the 2D Poisson matrix
    the grid line below and above, for the bidiagonal L one entry), b_r, and the halo description
    of csrk_halo.  Every rank derives every rank's interval from the global matrices, so the plan
    needs no communication."""

    def __init__(self, A: synth.CSR, L: synth.CSR, b: np.ndarray, rank: int, world: int, splits=None):
        self.rank, self.world = rank, world
        self.splits = balanced_row_splits(A.indptr, world) if splits is None else np.asarray(splits, np.int64)
        ext = [self.extended(A, L, self.splits, q) for q in range(world)]
        r0, r1 = int(self.splits[rank]), int(self.splits[rank + 1])
        lo, hi = ext[rank]
        self.r0, self.r1, self.lo, self.hi = r0, r1, lo, hi
        self.own_off = r0 - lo
        self.A, _, _ = compact_columns(row_block(A, r0, r1), lo, hi)
        self.L, _, _ = compact_columns(row_block(L, r0, r1), lo, hi)
        self.b = np.ascontiguousarray(b[r0:r1])
        h = {"peer": [], "own_off": [], "own_len": [], "ghost_off": [], "ghost_len": []}
        for q in range(world):
            if q == rank:
                continue
            q0, q1 = int(self.splits[q]), int(self.splits[q + 1])
            qlo, qhi = ext[q]
            g0, g1 = max(lo, q0), min(hi, q1)        # my ghost entries owned by q
            o0, o1 = max(qlo, r0), min(qhi, r1)      # my owned entries q holds as ghosts
            if g1 > g0 or o1 > o0:
                h["peer"].append(q)
                h["own_off"].append(o0 - lo if o1 > o0 else 0)
                h["own_len"].append(max(0, o1 - o0))
                h["ghost_off"].append(g0 - lo if g1 > g0 else 0)
                h["ghost_len"].append(max(0, g1 - g0))
        self.halo = h

    @staticmethod
    def extended(A, L, splits, q):
        q0, q1 = int(splits[q]), int(splits[q + 1])
        lo, hi = q0, q1
        for M in (A, L):
            s, e = int(M.indptr[q0]), int(M.indptr[q1])
            if e > s:
                lo, hi = min(lo, int(M.indices[s:e].min())), max(hi, int(M.indices[s:e].max()) + 1)
        return lo, hi


class StagedComm:
    """The csrk_comm semantics over torch.distributed with host-staged tensors (gloo): used by the
    CPU tests of the halo plan and, through ctypes callbacks (csrk_comm()), to run the CUDA
    sharded step with several ranks on ONE GPU in tests (NCCL refuses two ranks per GPU).  The
    product path uses csrk_comm_nccl_create (comm.cu) instead."""

    def __init__(self, halo: dict, group=None):
        self.h, self.group = halo, group

    def allreduce(self, t):
        import torch.distributed as tdist
        tdist.all_reduce(t, group=self.group)
        return t

    def halo_exchange(self, v, mode: int):
        """v: host tensor (extended vector), modified in place.  mode 0 gather, 1 reduce."""
        import torch
        import torch.distributed as tdist
        h, ops, recv = self.h, [], []
        for q, oo, ol, go, gl in zip(h["peer"], h["own_off"], h["own_len"], h["ghost_off"], h["ghost_len"]):
            if mode == 0:
                if ol:
                    ops.append(tdist.P2POp(tdist.isend, v[oo:oo + ol].clone(), q, self.group))
                if gl:
                    buf = torch.empty(gl, dtype=v.dtype)
                    recv.append((go, buf, False))
                    ops.append(tdist.P2POp(tdist.irecv, buf, q, self.group))
            else:
                if gl:
                    ops.append(tdist.P2POp(tdist.isend, v[go:go + gl].clone(), q, self.group))
                if ol:
                    buf = torch.empty(ol, dtype=v.dtype)
                    recv.append((oo, buf, True))
                    ops.append(tdist.P2POp(tdist.irecv, buf, q, self.group))
        if ops:
            for w in tdist.batch_isend_irecv(ops):
                w.wait()
        for off, buf, add in recv:
            if add:
                v[off:off + buf.numel()] += buf
            else:
                v[off:off + buf.numel()] = buf
        return v

    def csrk_comm(self):
        """A ctypes csrk_comm whose callbacks stage device vectors through the host (not capturable)."""
        import torch
        from paper_2212_05159_b200 import csrk as ck

        class _CAI:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": "<f8",
                                                 "version": 3}

        def dev_view(ptr, n):
            return torch.as_tensor(_CAI(ptr, n), device="cuda")

        n_ext = [0]

        def _allreduce(ctx, buf, count, stream):
            try:
                d = dev_view(buf, count)
                torch.cuda.current_stream().synchronize()
                d.copy_(self.allreduce(d.cpu()))
                return 0
            except Exception:
                return -6

        def _halo(ctx, vec, mode, stream):
            try:
                d = dev_view(vec, n_ext[0])
                torch.cuda.current_stream().synchronize()
                d.copy_(self.halo_exchange(d.cpu(), int(mode)))
                return 0
            except Exception:
                return -6

        self._cb = (ck.AllreduceFn(_allreduce), ck.HaloFn(_halo))   # keep the callbacks alive
        self._n_ext = n_ext
        return ck.Comm(None, self._cb[0], self._cb[1], 0)

    def set_extended_length(self, n):
        self._n_ext[0] = int(n)
