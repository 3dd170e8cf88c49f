"""Multi-process CPU test (gloo, world_size 2) of the row-partition + interval-reduction layer
(paper_2212_05159_b200/dist.py).  Local compute is the oracle (injected), so this checks the
partition and exchange logic exactly: with integer-valued inputs the distributed dA / dx /
dX / dB equal the single-process oracle bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_dir, mode="auto"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2212_05159_b200 import dist as D

    oracle.build()
    if case == "poisson":
        A = synth.poisson2d(12, 10)
        A = A.with_values(synth.int_values(np.random.default_rng(1), A.nnz, np.float64))
    else:
        A = synth.random_csr(90, 90, 0.06, 4, values="int")
    n = A.ncols
    x = synth.dense(n, 2, values="int")
    dy = synth.dense(A.nrows, 3, values="int")
    X = synth.dense((n, 3), 4, values="int")
    dY = synth.dense((A.nrows, 3), 5, values="int")
    blk = D.make_block(A, rank, world)
    r0, r1 = int(blk.row_splits[rank]), int(blk.row_splits[rank + 1])
    dm = D.DistCSR(blk, combine=mode)
    xl = x[blk.col_lo:blk.col_hi]
    Xl = X[blk.col_lo:blk.col_hi]

    class Ops:
        @staticmethod
        def spmv_bwd(Ar, xv, g):
            dA, dx = oracle.spmv_bwd(Ar, xv, g)
            return torch.from_numpy(dA), torch.from_numpy(dx.value)

        @staticmethod
        def spmm_bwd(Ar, Xv, G):
            dA, dX = oracle.spmm_bwd(Ar, Xv, G)
            return torch.from_numpy(dA.value), torch.from_numpy(dX.value)

        @staticmethod
        def spmv_fwd(Ar, xv):
            return torch.from_numpy(oracle.spmv_fwd(Ar, xv).value)

    y_r = dm.spmv_fwd(Ops, blk.A, xl)
    dA_r, dx_own = dm.spmv_bwd(Ops, blk.A, xl, dy[r0:r1])
    dAm_r, dX_own = dm.spmm_bwd(Ops, blk.A, Xl, dY[r0:r1])

    # C = A A row-sharded: dB partials over B_r's entries, reduced to the owners of those rows
    dg = D.DistGemm(A, blk, combine=mode)
    Br, (blo, bhi) = dg.B, dg.b_cols
    Ar_for_B = synth.CSR(blk.A.nrows, blk.A.ncols, blk.A.indptr, blk.A.indices, blk.A.values)
    Cp, Ci = oracle.spgemm_symbolic(Ar_for_B, Br)
    dC = synth.dense(len(Ci), 6 + rank, values="int")
    dAg_r, dBg_part = oracle.spgemm_bwd(Ar_for_B, Br, Cp, Ci, dC)
    dB_own = dg.combine_dB(torch.from_numpy(dBg_part.value))
    if mode != "auto":
        assert dm.vec.mode == mode and dg.ent.mode == mode
    # global C row values of this block, for the single-process reference
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), y=y_r.numpy(), dA=dA_r.numpy(), dx=dx_own.numpy(),
             dAm=dAm_r.numpy(), dX=dX_own.numpy(), dAg=dAg_r.value, dB=dB_own.numpy(), dC=dC,
             Cp=Cp, Ci=Ci, splits=blk.row_splits, col_lo=blk.col_lo, b_lo=blo, vec_mode=dm.vec.mode,
             ent_mode=dg.ent.mode)
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("case,mode", [("poisson", "auto"), ("random", "auto"), ("poisson", "rs"),
                                       ("random", "interval")])
def test_dist_two_ranks_match_single_process(tmp_path, orc, case, mode):
    """auto picks the halo (interval) exchange for the stencil and the dense reduce-scatter for the
    random matrix; both combines are also forced on the other case."""
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path), mode), nprocs=world, join=True)
    if case == "poisson":
        A = synth.poisson2d(12, 10)
        A = A.with_values(synth.int_values(np.random.default_rng(1), A.nnz, np.float64))
    else:
        A = synth.random_csr(90, 90, 0.06, 4, values="int")
    n = A.ncols
    x = synth.dense(n, 2, values="int")
    dy = synth.dense(A.nrows, 3, values="int")
    X = synth.dense((n, 3), 4, values="int")
    dY = synth.dense((A.nrows, 3), 5, values="int")
    R = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    if mode == "auto":
        want = "interval" if case == "poisson" else "rs"
        assert all(str(r["vec_mode"]) == want and str(r["ent_mode"]) == want for r in R)
    cat = lambda k: np.concatenate([r[k] for r in R])
    np.testing.assert_array_equal(cat("y"), orc.spmv_fwd(A, x).value)
    dA, dx = orc.spmv_bwd(A, x, dy)
    np.testing.assert_array_equal(cat("dA"), dA)
    np.testing.assert_array_equal(cat("dx"), dx.value)
    dAm, dX = orc.spmm_bwd(A, X, dY)
    np.testing.assert_array_equal(cat("dAm"), dAm.value)
    np.testing.assert_array_equal(cat("dX"), dX.value)
    # SpGEMM: the row-sharded C (= A A) with the per-rank dC values concatenated
    Cp, Ci = orc.spgemm_symbolic(A, A)
    dC = cat("dC")
    assert dC.shape[0] == len(Ci)
    # per-rank C column indices are relative to B_r's column interval: shift and compare
    cols = np.concatenate([R[r]["Ci"] + int(R[r]["b_lo"]) for r in range(world)])
    np.testing.assert_array_equal(cols, Ci)
    dAg, dB = orc.spgemm_bwd(A, A, Cp, Ci, dC)
    np.testing.assert_array_equal(cat("dAg"), dAg.value)
    np.testing.assert_array_equal(cat("dB"), dB.value)


def test_balanced_splits_and_closed_form_indptr():
    import synth
    from paper_2212_05159_b200 import dist as D
    P = synth.powerlaw(1 << 12, seed=3)
    s = D.balanced_row_splits(P.indptr, 4)
    assert s[0] == 0 and s[-1] == P.nrows and (np.diff(s) >= 0).all()
    per = np.diff(P.indptr[s])
    assert per.max() - per.min() <= np.diff(P.indptr).max() + 1
    for Nx, Ny in [(2, 2), (5, 3), (9, 7)]:
        A = synth.poisson2d(Nx, Ny)
        assert [D.poisson2d_indptr_at(Nx, Ny, r) for r in range(Nx * Ny + 1)] == A.indptr.tolist()
    # row blocks of the bench reproduce the global matrix rows
    for w in (1, 2, 4):
        A = synth.poisson2d(8, 5)
        m = A.nrows // w
        for r in range(w):
            Ar, lo = D.poisson2d_row_block(8, 5, r, w)
            ref, _, _ = D.compact_columns(D.row_block(A, r * m, (r + 1) * m), lo, lo + Ar.ncols)
            np.testing.assert_array_equal(Ar.indices, ref.indices)
            np.testing.assert_array_equal(Ar.values, ref.values)


# ---------------------------------------------------------------- config-5 row sharding (the halo plan)
def _pcg_plan_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2212_05159_b200 import dist as D

    oracle.build()
    A = synth.poisson2d(9, 7)
    L = synth.bidiag_lower(A.nrows, "seeded")
    L = L.with_values(synth.int_values(np.random.default_rng(5), L.nnz, np.float64))
    b = synth.dense(A.nrows, 1, values="int")
    sh = D.PcgShard(A, L, b, rank, world)
    comm = D.StagedComm(sh.halo)
    v = synth.dense(A.nrows, 8, values="int")
    out = {}
    for name, M in (("A", sh.A), ("L", sh.L)):
        # op N: gather the extended input, multiply the local rows
        ext = torch.zeros(sh.hi - sh.lo, dtype=torch.float64)
        ext[sh.own_off:sh.own_off + (sh.r1 - sh.r0)] = torch.from_numpy(v[sh.r0:sh.r1])
        comm.halo_exchange(ext, 0)
        out[f"{name}_ext"] = ext.numpy().copy()
        out[f"{name}_N"] = oracle.spmv_fwd(M, ext.numpy()).value
        # op T: the local rows' partial over the extended interval, reduced onto the owners
        part = torch.from_numpy(oracle.spmv_fwd(M, v[sh.r0:sh.r1], op=1).value.copy())
        comm.halo_exchange(part, 1)
        out[f"{name}_T"] = part[sh.own_off:sh.own_off + (sh.r1 - sh.r0)].numpy().copy()
    dot = torch.tensor([float(v[sh.r0:sh.r1] @ v[sh.r0:sh.r1])])
    out["dot"] = comm.allreduce(dot).numpy()
    np.savez(os.path.join(out_dir, f"p{rank}.npz"), lo=sh.lo, r0=sh.r0, r1=sh.r1, **out)
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pcg_shard_halo_plan_reproduces_global_products(tmp_path, orc, world):
    """The config-5 row sharding (dist.PcgShard + the csrk_comm semantics of dist.StagedComm over
    gloo): gathered extended inputs hold the global values; local op-N products equal the global
    A v / L v rows; halo-reduced op-T partials equal the global A^T v / L^T v rows; the allreduced
    dot is the global one -- exact on integer data (the same plan drives csrk_pcg_loss_grad_dist)."""
    import synth
    mp.spawn(_pcg_plan_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    A = synth.poisson2d(9, 7)
    L = synth.bidiag_lower(A.nrows, "seeded")
    L = L.with_values(synth.int_values(np.random.default_rng(5), L.nnz, np.float64))
    v = synth.dense(A.nrows, 8, values="int")
    R = [np.load(tmp_path / f"p{r}.npz") for r in range(world)]
    assert [int(r["r0"]) for r in R] == sorted(int(r["r0"]) for r in R) and int(R[-1]["r1"]) == A.nrows
    for name, M in (("A", A), ("L", L)):
        for r in R:
            lo = int(r["lo"])
            np.testing.assert_array_equal(r[f"{name}_ext"], v[lo:lo + len(r[f"{name}_ext"])])
        np.testing.assert_array_equal(np.concatenate([r[f"{name}_N"] for r in R]), orc.spmv_fwd(M, v).value)
        np.testing.assert_array_equal(np.concatenate([r[f"{name}_T"] for r in R]), orc.spmv_fwd(M, v, op=1).value)
    assert all(float(r["dot"][0]) == float(v @ v) for r in R)
