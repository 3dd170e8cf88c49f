#!/usr/bin/env python
"""bench.py -- one "step" = one pass of the whole hot path over
BASELINE.json config 2: the 2D Poisson 5-point matrix on a 2048 x 2048 grid (4,194,304 rows,
20,963,328 nonzeros, fp64), dense width k = 32:

    a7  csr_transpose (plan: pattern + perm)          a1  spmv_fwd        a2+a3 spmv_bwd
    a4  spmm_fwd                                      a5+a6 spmm_bwd
    a8+a9 spgemm_symbolic (C = A A, one host sync)    a10 spgemm_numeric  a11+a12 spgemm_bwd
    a13 (N > 1) row-block partition + halo reduction of the dx / dX / dB partials over NCCL

Per-op times for the ops report and the roofline come from a second pass with events around
every op (the timed steps carry no per-op events).  Running the SpGEMM half on a second stream
was measured: no gain (3.45 vs 3.37 ms), the SpMM grids occupy every SM.

Metric (BASELINE.json): algorithmic GB/s of the step (SURVEY.md 8(d) d.4 bytes; one read of
every operand, one write of every result) -- plus GFLOP/s and the roofline fraction of the
dominant kernel against the measured HBM copy bandwidth (MEASURED_PEAKS.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): weak scaling -- rank r owns rows [r m, (r+1) m) of the 2D Poisson matrix on a
(2048 N) x 2048 grid; x / X / dC are replicated over each rank's column interval and the
partial gradients are combined by the halo reduction in paper_2212_05159_b200.dist.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

GRID = 2048
K = 32
S = 8  # bytes per fp64 value


# ---------------------------------------------------------------- algorithmic bytes / flops
def pat_bytes(m, nnz):
    return 8 * (m + 1) + 4 * nnz


def op_costs(m, n, nnz, nnzC, prod, k=K, s=S):
    A = pat_bytes(m, nnz) + s * nnz
    return {
        "csr_transpose": (pat_bytes(m, nnz) + pat_bytes(n, nnz) + 8 * nnz, 0),
        "spmv_fwd": (A + s * n + s * m, 2 * nnz),
        "spmv_bwd": (A + s * m + s * n + s * n + s * nnz, 3 * nnz),
        "spmm_fwd": (A + s * k * n + s * k * m, 2 * nnz * k),
        "spmm_bwd": (A + s * k * (m + 2 * n) + s * nnz, 4 * nnz * k),
        # B aliases A (C = A A): the aliased operand is counted once
        "spgemm_symbolic": (pat_bytes(m, nnz) + pat_bytes(m, nnzC), 0),
        "spgemm_numeric": (A + 8 * (m + 1) + s * nnzC, 2 * prod),
        "spgemm_bwd": (A + pat_bytes(m, nnzC) + s * nnzC + 2 * s * nnz, 4 * prod),
    }


OPS = ["csr_transpose", "spmv_fwd", "spmv_bwd", "spmm_fwd", "spmm_bwd", "spgemm_symbolic", "spgemm_numeric",
       "spgemm_bwd"]


def pcg_costs(n, nnzA, nnzL, N, s=S):
    """Bytes / flops of one config-5 training step (csrk_pcg_loss_grad) AS IMPLEMENTED, op by op:
    SpMV = pattern + values + in + out; VJP of SpMV adds dy, dx, dA; dot 2n reads; a linear
    combination of k vectors k reads + 1 write (the dL += dAt accumulations are separate passes,
    u and z are recomputed in the reverse pass).  Reported as `unfused_bytes`."""
    spa = 8 * (n + 1) + (4 + s) * nnzA + 2 * s * n
    spl = 8 * (n + 1) + (4 + s) * nnzL + 2 * s * n
    splb = 8 * (n + 1) + (4 + s) * nnzL + 3 * s * n + s * nnzL
    spl_dA = 8 * (n + 1) + 4 * nnzL + 2 * s * n + s * nnzL
    dot, lin = 2 * s * n, lambda k, m=n: (k + 1) * s * m
    fwd = dot + lin(1) + 2 * spl + dot
    fwd += N * (spa + dot + lin(2)) + (N - 1) * (2 * spl + dot + lin(2))
    bwd = lin(2)
    bwd += (N - 1) * (dot + 2 * spl + lin(2) + lin(3) + 2 * splb + 2 * lin(2, nnzL) + lin(2))
    bwd += N * (dot + lin(2) + spa + lin(3))
    bwd += lin(2) + spl + splb + lin(2, nnzL) + spl_dA + lin(2, nnzL)
    flops = N * 2 * (2 * nnzA + 4 * nnzL) * 2 + N * 20 * n
    return fwd + bwd, flops


def pcg_costs_fused(n, nnzA, nnzL, N, s=S):
    """SURVEY 8(d) d.4 fused minimum of one config-5 step (the roofline's bytes; DESIGN "Config-5
    bytes").  Passes are cut only where a global scalar (alpha, beta, rho and their adjoints)
    forces a grid-wide reduction; within a pass every operand is read once and every result
    written once, dot products ride on the pass that produces an operand, the masked outer
    products dL += g v^T ride on the VJP pass that reads L (dL read + written), and u = L^T r,
    z = L u are kept from the forward (written there anyway) instead of recomputed.
      forward, per iteration   q = A p (+p.q) | r -= a q (+r.r) | u = L^T r | z = L u (+r.z) |
                               p = z + b p
      reverse, per iteration   pbar.p | zbar = pbar + rb r, rbar += c r + rb z |
                               VJP z = L u (ubar = L^T zbar, dL += zbar u^T) |
                               VJP u = L^T r (rbar += L ubar, dL += r ubar^T) | rbar.q |
                               qbar = -a rbar + sb p | pbar = b pbar + sb q + A^T qbar"""
    v = s * n
    A = 8 * (n + 1) + (4 + s) * nnzA
    L = 8 * (n + 1) + (4 + s) * nnzL
    dL = 2 * s * nnzL                                       # read + write of the accumulated gradient
    fwd_it = (A + 2 * v) + 3 * v + (L + 2 * v) + (L + 3 * v) + 3 * v
    bwd_it = 2 * v + 6 * v + (L + 3 * v + dL) + (L + 4 * v + dL) + 2 * v + 3 * v + (A + 5 * v)
    setup = 2 * v + (L + 2 * v) + (L + 3 * v)              # b.b, z0 = L (L^T b) (+b.z0)
    tail = (L + 3 * v + dL) + (L + 3 * v + dL)             # adjoint of z0 = M b
    return setup + N * fwd_it + N * bwd_it + tail


def run_cfg5(args, torch, ck):
    """BASELINE config 5: one training step = 50 PCG iterations on the 2D
    Poisson 4096^2 matrix with M = L L^T (lower-bidiagonal L), loss and d loss / d L.values.
    N > 1: the same problem row-sharded over N GPUs (strong scaling; dist.PcgShard + the NCCL
    csrk_comm: halo send/recv of the ghost grid lines, allreduced dot products), the whole step
    one CUDA graph per rank."""
    A = synth.poisson2d(4096)
    L = synth.bidiag_lower(A.nrows, "seeded")
    b = np.full(A.nrows, 1.0 / np.sqrt(A.nrows))
    N = 50
    pc = args.precond
    world, rank, local = init_dist(torch) if int(os.environ.get("WORLD_SIZE", "1")) > 1 else (1, 0, 0)
    comm = None
    if world > 1:
        if pc != "mult":
            raise SystemExit("bench.py: --precond solve has no sharded path (the triangular solves are sequential)")
        from paper_2212_05159_b200 import dist as D
        sh = D.PcgShard(A, L, b, rank, world)
        if os.environ.get("CSRK_BENCH_ONE_GPU") == "1":
            sc = D.StagedComm(sh.halo)
            comm = sc.csrk_comm()
            sc.set_extended_length(sh.hi - sh.lo)
        else:
            comm = ck.comm_nccl(rank, world, sh.halo)
        Ad, Ld = ck.CSR.from_host(sh.A), ck.CSR.from_host(sh.L)
        bt = torch.from_numpy(sh.b).cuda()

        def call():
            return ck.pcg_loss_grad_dist(comm, sh.own_off, Ad, Ld, bt, N, 0.6, dL=dL, ws=ws_buf)
    else:
        Ad, Ld = ck.CSR.from_host(A), ck.CSR.from_host(L)
        bt = torch.from_numpy(b).cuda()

        def call():
            return ck.pcg_loss_grad(Ad, Ld, bt, N, 0.6, dL=dL, precond=pc)
    dL = torch.empty_like(Ld.values)
    ws_buf = None
    if world > 1:
        import ctypes
        pa, pl = Ad.pattern(), Ld.pattern()
        nb = ctypes.c_size_t(0)
        ck.lib().csrk_workspace_size(ck.WS["pcg_dist"], ck.F64, ctypes.byref(pa), ctypes.byref(pl), N, 0,
                                     ctypes.byref(nb))
        ws_buf = torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device=bt.device)
    for _ in range(args.warmup):
        call()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    l0 = ck.launch_count()
    ts = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            if world > 1:
                import torch.distributed as tdist
                tdist.barrier()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            loss, res, _ = call()
            e.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e))
    unfused, flops = pcg_costs(A.nrows, A.nnz, L.nnz, N)
    byts = pcg_costs_fused(A.nrows, A.nnz, L.nnz, N)
    ms = float(np.mean(ts))
    if world > 1:
        import torch.distributed as tdist
        ms = float(allreduce_max(torch, torch.tensor([ms], dtype=torch.float64, device=bt.device)).item())
        tdist.barrier()
        if os.environ.get("CSRK_BENCH_ONE_GPU") != "1":
            ck.comm_destroy(comm)
        tdist.destroy_process_group()
        if rank != 0:
            return 0
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = {"metric": "PCG training-step algorithmic GB/s (config 5)", "value": round(byts / (ms * 1e-3) / 1e9, 2),
           "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "config5: 2D Poisson 4096^2 (16,777,216 rows, 83,869,696 nnz), lower-bidiagonal "
                                  f"L (33,554,431 nnz), 50 PCG iterations fwd + reverse, gamma 0.6, {world} GPU(s)",
                      "parallelism": f"rowblock{world}" if world > 1 else "single",
                      "cuda_graph": os.environ.get("CSRK_PCG_GRAPH", "1") != "0",
                      "preconditioner": "M = L L^T (P:836-839)" if pc == "mult" else
                      "M = (L L^T)^-1 by two SpTRSV (SURVEY 8(f) f3); bytes counted as for M = L L^T"},
           "step_bytes": byts, "step_bytes_def": "SURVEY 8(d) d.4 fused minimum (bench.pcg_costs_fused)",
           "unfused_bytes": unfused, "unfused_GB/s": round(unfused / (ms * 1e-3) / 1e9, 1),
           "gflops": round(flops / (ms * 1e-3) / 1e9, 2), "loss": loss,
           "roofline": {"bound": "hbm", "kernel": "whole step", "achieved": round(byts / (ms * 1e-3) / 1e9, 1),
                        "peak": peak * world, "unit": "GB/s",
                        "frac": round(byts / (ms * 1e-3) / 1e9 / (peak * world), 4)},
           "gpu_launches": int((ck.launch_count() - l0) / max(args.steps, 1)), "clocks": clk.summary()}
    traffic, tsrc = _traffic("cfg5" if pc == "mult" else "cfg5_solve", "pcg_loss_grad") if world == 1 else (None, None)
    out["roofline"]["traffic"], out["roofline"]["traffic_source"] = traffic, tsrc
    if args.ops_trace and world == 1:
        write_ops_trace(args.ops_trace, ck, [("pcg_loss_grad", call)])
    print(json.dumps(out))
    return 0


def run_ops_workload(args, torch, ck, cfg):
    """BASELINE configs 3 and 4 at N = 1, op by op: each op timed with CUDA
    events on the launching stream, L2 flushed (512 MiB write) before every timed op.
      cfg3: 3D 7-point Poisson 160^3, fp64, C = A A: symbolic (count + host sync + fill), numeric
            on the reused pattern, backward (dA and dB, summed by the caller per reading A13).
      cfg4: power-law n = 2^23, 16 nnz/row, fp32: spmv fwd, spmv bwd (atomic dx), transpose,
            spmv bwd with the plan, then C = A A symbolic / numeric / backward (nnz(C) ~ 2.1e9)."""
    dev = torch.device("cuda", 0)
    if cfg == 3:
        A = synth.poisson3d(160)
        s, dt_np, dt = 8, np.float64, torch.float64
    else:
        A = synth.powerlaw()
        s, dt_np, dt = 4, np.float32, torch.float32
    m, n, nnz = A.nrows, A.ncols, A.nnz
    Ad = ck.CSR.from_host(A)
    lens = np.diff(A.indptr)
    prod = int(lens[A.indices].sum())
    del A
    x = torch.from_numpy(synth.dense(n, synth.seed_of(cfg, 3), dt_np)).to(dev)
    dy = torch.from_numpy(synth.dense(m, synth.seed_of(cfg, 4), dt_np)).to(dev)
    y, dA_v, dx = torch.empty(m, dtype=dt, device=dev), torch.empty(nnz, dtype=dt, device=dev), \
        torch.empty(n, dtype=dt, device=dev)
    plan = ck.csr_transpose(Ad, with_values=False)
    C = ck.spgemm_symbolic(Ad, Ad)
    nnzC = C.nnz
    q = torch.arange(nnzC, device=dev, dtype=torch.int64)  # counter-based dC (too large for the host at cfg4)
    dC = (((q * 2654435761 + 12345) % 1000003).to(torch.float64) / 500001.5 - 1.0).to(dt)
    del q
    Cv = torch.empty(nnzC, dtype=dt, device=dev)
    dA_g, dB_g = torch.empty(nnz, dtype=dt, device=dev), torch.empty(nnz, dtype=dt, device=dev)
    c = op_costs(m, n, nnz, nnzC, prod, k=1, s=s)
    ops = {}
    if cfg == 4:
        ops["spmv_fwd"] = (lambda: ck.spmv_fwd(Ad, x, out=y), c["spmv_fwd"])
        ops["spmv_bwd"] = (lambda: ck.spmv_bwd(Ad, x, dy, dA=dA_v, dx=dx), c["spmv_bwd"])
        ops["csr_transpose"] = (lambda: ck.csr_transpose(Ad, with_values=False, out=plan), c["csr_transpose"])
        ops["spmv_bwd_plan"] = (lambda: ck.spmv_bwd(Ad, x, dy, plan=plan, dA=dA_v, dx=dx), c["spmv_bwd"])
    ops["spgemm_symbolic"] = (lambda: ck.spgemm_symbolic(Ad, Ad), c["spgemm_symbolic"])
    ops["spgemm_numeric"] = (lambda: ck.spgemm_numeric(Ad, Ad, C, out=Cv), c["spgemm_numeric"])
    ops["spgemm_bwd"] = (lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA_g, dB=dB_g), c["spgemm_bwd"])
    # deterministic dB (column gather through the transpose plan): reported, not in the total
    ops["spgemm_bwd_plan"] = (lambda: ck.spgemm_bwd(Ad, Ad, C, dC, dA=dA_g, dB=dB_g, plan=plan), c["spgemm_bwd"])
    wl = ("config3: 3D Poisson 7-point 160^3 (4,096,000 rows, 28,518,400 nnz), fp64, C = A A "
          f"(nnz(C) {nnzC:,}, prod {prod:,}): symbolic + numeric + bwd" if cfg == 3 else
          "config4: power-law n = 2^23, 2^27 nnz, rows 8..32,769, fp32: spmv fwd/bwd, transpose, C = A A "
          f"(nnz(C) {nnzC:,}, prod {prod:,}) symbolic + numeric + bwd")
    return _time_ops(args, torch, ck, ops, f"SpMV/SpGEMM fwd+bwd algorithmic GB/s (config {cfg})",
                     "f64" if cfg == 3 else "f32", wl, f"cfg{cfg}", exclude=("spmv_bwd_plan", "spgemm_bwd_plan"))


def run_ops_sharded(args, torch, ck, cfg, world, rank, local):
    """BASELINE configs 3 and 4 row-sharded over N GPUs (strong scaling: the global matrix is
    split).  Rank r owns a contiguous row block balanced by SpGEMM work w_i (columns
    compacted to its interval), x over its column interval, and B_r = the rows of A its block
    references.  Forward ops are rank-local; the dx partial (spmv_bwd) and the dB partial
    (spgemm_bwd) are combined onto their owners by dist.Combiner -- the halo send/recv for the 3D
    stencil, one NCCL reduce_scatter for the power-law matrix (every block references ~86 % of
    the columns).  Each op: barrier, CUDA events on the launching stream, L2 flushed; the op time
    is the max over ranks; bytes are the global algorithmic bytes of the 1-GPU line."""
    import torch.distributed as tdist
    from paper_2212_05159_b200 import dist as D
    dev = torch.device("cuda", local)
    if cfg == 3:
        A = synth.poisson3d(160)
        s, dt_np, dt = 8, np.float64, torch.float64
    else:
        A = synth.powerlaw()
        s, dt_np, dt = 4, np.float32, torch.float32
    m, n, nnz = A.nrows, A.ncols, A.nnz
    lens = np.diff(A.indptr)
    prod = int(lens[A.indices].sum())
    work = np.zeros(m, np.int64)
    np.add.at(work, np.repeat(np.arange(m), lens), lens[A.indices])
    splits = D.balanced_row_splits(A.indptr, world, work=work)
    blk = D.make_block(A, rank, world, splits)
    dg = D.DistGemm(A, blk, device=dev)
    r0, r1 = int(splits[rank]), int(splits[rank + 1])
    x = synth.dense(n, synth.seed_of(cfg, 3), dt_np)[blk.col_lo:blk.col_hi]
    dy = synth.dense(m, synth.seed_of(cfg, 4), dt_np)[r0:r1]
    del A
    Ad, Bd = ck.CSR.from_host(blk.A), ck.CSR.from_host(dg.B)
    dm = D.DistCSR(blk, device=dev)
    x, dy = torch.from_numpy(np.ascontiguousarray(x)).to(dev), torch.from_numpy(np.ascontiguousarray(dy)).to(dev)
    plan = ck.csr_transpose(Ad, with_values=False)
    C = ck.spgemm_symbolic(Ad, Bd)
    q = torch.arange(C.nnz, device=dev, dtype=torch.int64) + 7919 * rank
    dC = (((q * 2654435761 + 12345) % 1000003).to(torch.float64) / 500001.5 - 1.0).to(dt)
    del q
    Cv = torch.empty(C.nnz, dtype=dt, device=dev)
    y = torch.empty(Ad.nrows, dtype=dt, device=dev)
    dA_v = torch.empty(Ad.nnz, dtype=dt, device=dev)
    dA_g, dB_g = torch.empty(Ad.nnz, dtype=dt, device=dev), torch.empty(Bd.nnz, dtype=dt, device=dev)
    nnzC = allreduce_sum(torch, torch.tensor([C.nnz], dtype=torch.int64, device=dev))
    c = op_costs(m, n, nnz, int(nnzC.item()), prod, k=1, s=s)

    def spmv_bwd():
        _, dx_part = ck.spmv_bwd(Ad, x, dy, dA=dA_v)
        return dm.vec(dx_part)

    def spgemm_bwd():
        ck.spgemm_bwd(Ad, Bd, C, dC, dA=dA_g, dB=dB_g)
        return dg.combine_dB(dB_g)

    ops = {}
    if cfg == 4:
        ops["spmv_fwd"] = (lambda: ck.spmv_fwd(Ad, x, out=y), c["spmv_fwd"])
        ops["spmv_bwd"] = (spmv_bwd, c["spmv_bwd"])
        ops["csr_transpose"] = (lambda: ck.csr_transpose(Ad, with_values=False, out=plan), c["csr_transpose"])
    ops["spgemm_symbolic"] = (lambda: ck.spgemm_symbolic(Ad, Bd), c["spgemm_symbolic"])
    ops["spgemm_numeric"] = (lambda: ck.spgemm_numeric(Ad, Bd, C, out=Cv), c["spgemm_numeric"])
    ops["spgemm_bwd"] = (spgemm_bwd, c["spgemm_bwd"])
    l2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for f, _c in ops.values():
            f()
    torch.cuda.synchronize()
    times = {k: [] for k in ops}
    l0 = ck.launch_count()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            for k, (f, _c) in ops.items():
                l2.zero_()
                tdist.barrier()
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                f()
                e.record(st)
                times[k].append((a, e))
        torch.cuda.synchronize()
    launches = ck.launch_count() - l0
    med = torch.tensor([float(np.median([a.elapsed_time(e) for a, e in times[k]])) for k in ops],
                       dtype=torch.float64, device=dev)
    allreduce_max(torch, med)
    peak = _peak()
    rep, tot_b, tot_f, tot_ms = {}, 0, 0, 0.0
    for (k, (_f, (b, fl))), ms in zip(ops.items(), med.tolist()):
        rep[k] = {"ms": round(ms, 4), "GB/s": round(b / ms / 1e6, 1), "GFLOP/s": round(fl / ms / 1e6, 1),
                  "frac_of_N_peaks": round(b / ms / 1e6 / (peak * world), 3), "bytes": b}
        tot_b, tot_f, tot_ms = tot_b + b, tot_f + fl, tot_ms + ms
    dom = max(rep, key=lambda k: rep[k]["ms"])
    if rank == 0:
        wl = (f"config3: 3D Poisson 7-point 160^3, fp64, C = A A, row-sharded over {world} GPUs" if cfg == 3 else
              f"config4: power-law n = 2^23, 2^27 nnz, fp32, spmv + C = A A, row-sharded over {world} GPUs")
        out = {"metric": f"SpMV/SpGEMM fwd+bwd algorithmic GB/s (config {cfg})",
               "value": round(tot_b / tot_ms / 1e6, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(tot_ms, 4), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64" if cfg == 3 else "f32", "data": "synthetic",
               "config": {"workload": wl, "l2": "flushed (512 MiB write) before every timed op",
                          "parallelism": f"rowblock{world}", "combine": {"dx": dm.vec.mode, "dB": dg.ent.mode},
                          "row_splits": [int(v) for v in splits]},
               "gflops": round(tot_f / tot_ms / 1e6, 2),
               "roofline": {"bound": "hbm", "kernel": dom, "achieved": rep[dom]["GB/s"], "peak": peak * world,
                            "peak_def": f"{world} x measured HBM copy GB/s", "unit": "GB/s",
                            "frac": rep[dom]["frac_of_N_peaks"], "traffic": None},
               "ops": rep, "gpu_launches": int(launches / max(args.steps, 1)), "clocks": clk.summary()}
        print(json.dumps(out))
    return 0


def run_trsv_workload(args, torch, ck):
    """SpTRSV (PAPER 3.1.5) at N = 1, op by op (CUDA events, L2 flushed before
    every op): the config-5 lower-bidiagonal L (4096^2 = 16,777,216 rows; the chain pass) and
    the IC(0) pattern of the 2D Poisson 2048^2 matrix (its lower triangle; wavefront, the
    sync-free pass), forward x = T^{-1} b and backward (db = T^{-T} v, dT) with a cached plan.
    Algorithmic bytes: fwd = pattern + values + b + x; bwd = pattern + values + v + x + db + dT."""
    dev = torch.device("cuda", 0)
    s = 8
    mats = {"chain": synth.bidiag_lower(4096 * 4096, "seeded"),
            "ic0": synth.lower_part(synth.poisson2d(2048))}
    ops = {}
    keep = []
    for nm, T in mats.items():
        n, nnz = T.nrows, T.nnz
        Td = ck.CSR.from_host(T)
        b = torch.from_numpy(synth.dense(n, synth.seed_of(5, 3))).to(dev)
        v = torch.from_numpy(synth.dense(n, synth.seed_of(5, 4))).to(dev)
        x = ck.sptrsv_fwd(Td, b)
        plan = ck.csr_transpose(Td, with_values=False)
        dT, db = torch.empty_like(Td.values), torch.empty_like(b)
        keep += [Td, b, v, x, plan, dT, db]
        pat = 8 * (n + 1) + 4 * nnz
        ops[f"sptrsv_fwd_{nm}"] = ((lambda Td=Td, b=b, x=x: ck.sptrsv_fwd(Td, b, out=x)),
                                   (pat + s * nnz + 2 * s * n, 2 * nnz))
        ops[f"sptrsv_bwd_{nm}"] = ((lambda Td=Td, x=x, v=v, plan=plan, dT=dT, db=db:
                                    ck.sptrsv_bwd(Td, x, v, plan=plan, dT=dT, db=db)),
                                   (pat + s * nnz + 4 * s * n + s * nnz, 3 * nnz))
    return _time_ops(args, torch, ck, ops, "SpTRSV fwd+bwd algorithmic GB/s", "f64",
                     "SpTRSV: config-5 bidiagonal L (16,777,216 rows, chain pass) and the lower triangle of 2D "
                     "Poisson 2048^2 (4,194,304 rows, wavefront, sync-free pass), fwd + bwd with a cached transpose "
                     "plan", "trsv", keep=keep)


def run_gcn_workload(args, torch, ck):
    """GCN layer (PAPER 4.4 Fig. 12) at N = 1: one training step of one layer on a
    synthetic power-law graph of 2^20 nodes with 5 edges per node on average (the size of the
    paper's largest SuiteSparse graphs), fp32, C = F = 16 (the paper's hidden width):
    forward XTheta = X Theta + fused propagation, backward dZ (transposed propagation with a cached
    plan), dTheta = X^T dZ, dX = dZ Theta^T, dbias.  L2 flushed before every step.
    Algorithmic bytes per op: every operand read once, every result written once."""
    dev = torch.device("cuda", 0)
    s, C, F = 4, 16, 16
    G = synth.powerlaw_graph(1 << 20, 5.0, 4401, dtype=np.float32)
    n, nnz = G.nrows, G.nnz
    Gd = ck.CSR.from_host(G)
    X = torch.from_numpy(synth.dense((n, C), 1, np.float32)).to(dev)
    W = torch.from_numpy(synth.dense((C, F), 2, np.float32)).to(dev)
    b = torch.from_numpy(synth.dense(F, 3, np.float32)).to(dev)
    dY = torch.from_numpy(synth.dense((n, F), 4, np.float32)).to(dev)
    plan = ck.csr_transpose(Gd, with_values=False)
    Z, Y, dZ, dX = (torch.empty((n, F), device=dev), torch.empty((n, F), device=dev),
                    torch.empty((n, F), device=dev), torch.empty((n, C), device=dev))
    dW, db = torch.empty((C, F), device=dev), torch.empty(F, device=dev)
    D = torch.empty(n, dtype=torch.float64, device=dev)
    pat = 8 * (n + 1) + 4 * nnz
    ops = {
        "xtheta": (lambda: ck.dense_gemm_nn(X, W, out=Z), (s * n * (C + F), 2 * n * C * F)),
        "gcn_fwd": (lambda: ck.gcn_fwd(Gd, Z, b, out=Y, D=D), (pat + s * nnz + 2 * s * n * F + 8 * n, 2 * nnz * F)),
        "gcn_bwd": (lambda: ck.gcn_bwd(Gd, D, dY, plan=plan, dZ=dZ, dbias=db),
                    (pat + s * nnz + 2 * s * n * F + 8 * n, 2 * nnz * F + n * F)),
        "dtheta": (lambda: ck.dense_gemm_tn(X, dZ, out=dW), (s * n * (C + F), 2 * n * C * F)),
        "dx": (lambda: ck.dense_gemm_nn(dZ, W, transW=True, out=dX), (s * n * (C + F), 2 * n * C * F)),
    }
    return _time_ops(args, torch, ck, ops, "GCN layer fwd+bwd algorithmic GB/s", "f32", wkey="gcn", workload=
                     "GCN layer (Fig. 12): power-law graph 1,048,576 nodes, 5,242,880 edges (max degree "
                     f"{int(np.diff(G.indptr).max())}), fp32, C = F = 16, fwd + bwd with a cached transpose plan")


def run_f12_workload(args, torch, ck):
    """Sp + Sp (PAPER 3.1.4) and the SPAI loss + gradient (f2, PAPER 4.6) at N = 1:
    C = 2A - 3L on config 2's 2D Poisson 2048^2 and its lower-bidiagonal L (union pattern), forward
    and VJP; ||I - M A||_F^2 and d/dM.values for A = 2D Poisson 1024^2 with pattern(M) = pattern(A)
    (M = mask(A) all ones).  Algorithmic bytes of the SPAI call = those of its constituent
    ops (M A numeric, I - C, sum of squares, the Sp+Sp VJP, the left SpGEMM VJP)."""
    dev = torch.device("cuda", 0)
    s8 = 8
    pat = lambda m, nnz: 8 * (m + 1) + 4 * nnz
    A = synth.poisson2d(GRID)
    L = synth.bidiag_lower(A.nrows, "seeded")
    Ad, Ld = ck.CSR.from_host(A), ck.CSR.from_host(L)
    C = ck.spadd_symbolic(Ad, Ld)
    Cv = torch.empty(C.nnz, dtype=torch.float64, device=dev)
    dC = torch.from_numpy(synth.dense(C.nnz, 12)).to(dev)
    dA, dL = torch.empty_like(Ad.values), torch.empty_like(Ld.values)
    m, na, nl, nc = A.nrows, A.nnz, L.nnz, C.nnz
    A2 = synth.poisson2d(1024)
    A2d = ck.CSR.from_host(A2)
    M = ck.CSR(A2d.nrows, A2d.ncols, A2d.indptr, A2d.indices, torch.ones_like(A2d.values))
    plan = ck.spai_plan(M, A2d)
    dM = torch.empty_like(M.values)
    n2, nz2, nC2, nR2 = A2.nrows, A2.nnz, plan.C.nnz, plan.R.nnz
    prod2 = int(np.diff(A2.indptr)[A2.indices].sum())
    spai_bytes = ((pat(n2, nz2) + s8 * nz2) * 2 + 8 * (n2 + 1) + s8 * nC2          # C = M A
                  + pat(n2, nC2) + s8 * nC2 + pat(n2, nR2) + s8 * nR2               # R = I - C
                  + s8 * nR2                                                        # sum R^2
                  + pat(n2, nR2) + s8 * nR2 + s8 * nC2                              # dC from dR
                  + (pat(n2, nz2) + s8 * nz2) * 2 + pat(n2, nC2) + s8 * nC2 + s8 * nz2)  # dM
    ops = {
        "spadd_symbolic": (lambda: ck.spadd_symbolic(Ad, Ld), (pat(m, na) + pat(m, nl) + pat(m, nc), 0)),
        "spadd_numeric": (lambda: ck.spadd_numeric(2.0, Ad, -3.0, Ld, C, out=Cv),
                          (pat(m, na) + pat(m, nl) + pat(m, nc) + s8 * (na + nl + nc), 2 * nc)),
        "spadd_bwd": (lambda: ck.spadd_bwd(2.0, Ad, -3.0, Ld, C, dC, dA=dA, dB=dL),
                      (pat(m, na) + pat(m, nl) + pat(m, nc) + s8 * (nc + na + nl), na + nl)),
        "spai_loss_grad": (lambda: ck.spai_loss_grad(plan, M, A2d, dM=dM), (spai_bytes, 6 * prod2)),
    }
    return _time_ops(args, torch, ck, ops, "Sp+Sp and SPAI fwd+bwd algorithmic GB/s", "f64", wkey="f12", workload=
                     "Sp+Sp: 2 A - 3 L, A = 2D Poisson 2048^2, L lower bidiagonal (fwd + VJP); SPAI: ||I - M A||_F^2 "
                     "+ gradient, A = 2D Poisson 1024^2, pattern(M) = pattern(A)")


def _time_ops(args, torch, ck, ops, metric, dtype, workload, wkey, exclude=(), keep=None):
    """Time a dict name -> (fn, (bytes, flops)) op by op: CUDA events on the current stream,
    L2 flushed (512 MiB write) before every op, median over --steps.  Ops in `exclude` are
    reported but not part of the step total (alternative paths of an op)."""
    dev = torch.device("cuda", 0)
    l2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for f, _c in ops.values():
            f()
    torch.cuda.synchronize()
    times = {k: [] for k in ops}
    l0 = ck.launch_count()
    with Clocks(0) as clk:
        for _ in range(args.steps):
            for k, (f, _c) in ops.items():
                l2.zero_()
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                f()
                e.record(st)
                times[k].append((a, e))
        torch.cuda.synchronize()
    launches = ck.launch_count() - l0
    peak = _peak()
    rep, tot_b, tot_f, tot_ms = {}, 0, 0, 0.0
    for k, ev in times.items():
        ms = float(np.median([a.elapsed_time(e) for a, e in ev]))
        b, fl = ops[k][1]
        all_ms = [a.elapsed_time(e) for a, e in ev]
        rep[k] = {"ms": round(ms, 4), "GB/s": round(b / ms / 1e6, 1), "GFLOP/s": round(fl / ms / 1e6, 1),
                  "frac": round(b / ms / 1e6 / peak, 3), "bytes": b, "ms_min": round(float(np.min(all_ms)), 4),
                  "ms_p90": round(float(np.percentile(all_ms, 90)), 4)}
        if k not in exclude:
            tot_b, tot_f, tot_ms = tot_b + b, tot_f + fl, tot_ms + ms
    dom = max((k for k in rep if k not in exclude), key=lambda k: rep[k]["ms"])
    traffic, tsrc = _traffic(wkey, dom)
    out = {"metric": metric, "value": round(tot_b / tot_ms / 1e6, 2), "unit": "GB/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_ms, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
           "config": {"workload": workload, "l2": "flushed (512 MiB write) before every timed op"},
           "gflops": round(tot_f / tot_ms / 1e6, 2),
           "roofline": {"bound": "hbm", "kernel": dom, "achieved": rep[dom]["GB/s"], "peak": peak, "unit": "GB/s",
                        "frac": rep[dom]["frac"], "traffic": traffic, "traffic_source": tsrc,
                        "algorithmic_bytes": ops[dom][1][0]},
           "ops": rep, "gpu_launches": int(launches / max(args.steps, 1)), "clocks": clk.summary()}
    if args.ops_trace:
        write_ops_trace(args.ops_trace, ck, [(k, f) for k, (f, _c) in ops.items()])
    print(json.dumps(out))
    return 0


def _traffic(workload, op):
    """DRAM bytes (read + write) of one call of `op` in `workload`, from the committed ncu launch
    list attributed by tools/traffic.py (profiles/traffic_<workload>.json); (None, None) if absent."""
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        prof = json.load(open(path))
        return int(prof["ops"][op]["dram_bytes"]), os.path.relpath(path, ROOT) + " <- " + prof.get("source", "?")
    except Exception:
        return None, None


def _peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload
class Workload:
    """Config-2 inputs resident on the device plus preallocated outputs."""

    def __init__(self, torch, ck, rank=0, world=1, dist=None):
        self.torch, self.ck, self.dist = torch, ck, dist
        self.rank, self.world = rank, world
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        # rank's row block of the (GRID*world) x GRID grid: rows [r*m, (r+1)*m)
        from paper_2212_05159_b200 import dist as D
        if world == 1:
            A = synth.poisson2d(GRID)
            self.col_lo = 0
        else:
            A, self.col_lo = D.poisson2d_row_block(GRID * world, GRID, rank, world)
        self.A_host = A
        self.m, self.n, self.nnz = A.nrows, A.ncols, A.nnz
        ck_ = ck
        self.A = ck_.CSR.from_host(A)
        cfg = 2
        self.x = torch.from_numpy(synth.dense(self.n, synth.seed_of(cfg, 3) + 100 * rank)).to(dev)
        self.dy = torch.from_numpy(synth.dense(self.m, synth.seed_of(cfg, 4) + 100 * rank)).to(dev)
        self.X = torch.from_numpy(synth.dense((self.n, K), synth.seed_of(cfg, 3) + 100 * rank + 1)).to(dev)
        self.dY = torch.from_numpy(synth.dense((self.m, K), synth.seed_of(cfg, 4) + 100 * rank + 1)).to(dev)
        # C = A B with B = the rows of A over this rank's column interval (B = A at N = 1)
        self.B = self.A if world == 1 else ck_.CSR.from_host(D.halo_rows_block(GRID * world, GRID, rank, world))
        # outputs / plans (allocated once, reused)
        self.plan = ck_.csr_transpose(self.A, with_values=False)
        self.C = ck_.spgemm_symbolic(self.A, self.B)
        self.nnzC = self.C.nnz
        self.prod = int(np.diff(self.B.indptr.cpu().numpy())[A.indices].sum())
        self.dC = torch.from_numpy(synth.dense(self.nnzC, synth.seed_of(cfg, 5) + 100 * rank)).to(dev)
        e = torch.empty
        f64 = torch.float64
        self.y = e(self.m, dtype=f64, device=dev)
        self.dA_v = e(self.nnz, dtype=f64, device=dev)
        self.dx = e(self.n, dtype=f64, device=dev)
        self.Y = e((self.m, K), dtype=f64, device=dev)
        self.dA_m = e(self.nnz, dtype=f64, device=dev)
        self.dX = e((self.n, K), dtype=f64, device=dev)
        self.Cv = e(self.nnzC, dtype=f64, device=dev)
        self.dA_g = e(self.nnz, dtype=f64, device=dev)
        self.dB_g = e(self.B.nnz, dtype=f64, device=dev)
        self.costs = op_costs(self.m, self.n, self.nnz, self.nnzC, self.prod)

    def op_list(self):
        """The step's ops in order, (name, fn) -- a7, a1, a2+a3, a4, a5+a6, a8+a9, a10, a11+a12 (+ a13)."""
        ck = self.ck

        def symbolic():
            C = ck.spgemm_symbolic(self.A, self.B)
            assert C.nnz == self.nnzC
            self.C = C

        ops = [
            ("csr_transpose", lambda: ck.csr_transpose(self.A, with_values=False, out=self.plan)),
            ("spmv_fwd", lambda: ck.spmv_fwd(self.A, self.x, out=self.y)),
            # atomic scatter for dx: measured faster than the transpose-plan gather here
            ("spmv_bwd", lambda: ck.spmv_bwd(self.A, self.x, self.dy, dA=self.dA_v, dx=self.dx)),
            ("spmm_fwd", lambda: ck.spmm_fwd(self.A, self.X, out=self.Y)),
            ("spmm_bwd", lambda: ck.spmm_bwd(self.A, self.X, self.dY, plan=self.plan, dA=self.dA_m, dX=self.dX)),
            ("spgemm_symbolic", symbolic),
            ("spgemm_numeric", lambda: ck.spgemm_numeric(self.A, self.B, self.C, out=self.Cv)),
            ("spgemm_bwd", lambda: ck.spgemm_bwd(self.A, self.B, self.C, self.dC, dA=self.dA_g, dB=self.dB_g)),
        ]
        if self.dist is not None:
            ops.append(("halo_reduce", lambda: self.dist.reduce_partials(self)))
        return ops

    def step(self, ev=None):
        """One pass of the hot path; `ev` (dict op -> (start, end) events) brackets each op."""
        st = self.torch.cuda.current_stream()
        for name, fn in self.op_list():
            if ev is not None:
                ev[name][0].record(st)
            fn()
            if ev is not None:
                ev[name][1].record(st)


NOMINAL_HBM_GBS = 8000.0  # north_star "~8 TB/s" (SURVEY 8(d) d.1 gates on it)


def gate_report(costs, op_ms, peak):
    """SURVEY 8(d) d.1 gate: (bytes_fwd + bytes_bwd) / (t_fwd + t_bwd) for SpMV and SpMM on config 2,
    as a fraction of the measured copy peak and of the nominal 8 TB/s (target >= 0.60)."""
    out = {}
    for nm in ("spmv", "spmm"):
        b = costs[f"{nm}_fwd"][0] + costs[f"{nm}_bwd"][0]
        t = (op_ms[f"{nm}_fwd"] + op_ms[f"{nm}_bwd"]) * 1e-3
        gbs = b / t / 1e9
        out[f"{nm}_fwd_bwd"] = {"GB/s": round(gbs, 1), "frac_measured": round(gbs / peak, 3),
                                "frac_nominal": round(gbs / NOMINAL_HBM_GBS, 3)}
    return out


def flush_l2(torch, buf):
    buf.zero_()


def host_cpu_info():
    """CPU model, logical CPUs available to this process and SMT state."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    smt = None
    try:
        smt = open("/sys/devices/system/cpu/smt/active").read().strip() == "1"
    except OSError:
        pass
    return {"model": model, "affinity_cpus": len(os.sched_getaffinity(0)), "smt_active": smt}


def run_cpu_baseline(threads=None, rows_sample=1 << 22):
    """The oracle, as it stands, on a bounded sample of the same workload: the 2D Poisson
    5-point stencil on a (rows_sample/2048) x 2048 grid, the same step (all ops), fp64."""
    import oracle
    nthreads = threads or len(os.sched_getaffinity(0))
    oracle.set_threads(nthreads)
    A = synth.poisson2d(rows_sample // GRID, GRID)
    m = A.nrows
    x, dy = synth.dense(m, 1), synth.dense(m, 2)
    X, dY = synth.dense((m, K), 3), synth.dense((m, K), 4)
    t0 = time.perf_counter()
    oracle.csr_transpose(A)
    oracle.spmv_fwd(A, x)
    oracle.spmv_bwd(A, x, dy)
    oracle.spmm_fwd(A, X)
    oracle.spmm_bwd(A, X, dY)
    Cp, Ci = oracle.spgemm_symbolic(A, A)
    oracle.spgemm_numeric(A, A, Cp, Ci)
    dC = synth.dense(len(Ci), 5)
    t1 = time.perf_counter()
    oracle.spgemm_bwd(A, A, Cp, Ci, dC)
    t2 = time.perf_counter()
    prod = int(np.diff(A.indptr)[A.indices].sum())
    costs = op_costs(m, m, A.nnz, len(Ci), prod)
    tot_bytes = sum(b for b, _ in costs.values())
    secs = t2 - t0 - 0.0 * (t2 - t1)
    return {"value": tot_bytes / secs / 1e9, "unit": "GB/s", "cores": nthreads, "kind": "oracle",
            "sample": f"2D Poisson {m // GRID}x{GRID} ({m} rows, nnz {A.nnz}), whole step, fp64, "
                      f"{secs:.2f} s wall", "seconds": secs}


def run_reference(args):
    """--impl reference: the oracle (the only reference this paper-only tier has) on bounded
    samples of the config-2 workload, timed on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        run_cpu_baseline(rows_sample=1 << 15)
    vals, secs = [], []
    for _ in range(args.steps):
        r = run_cpu_baseline(rows_sample=1 << 16)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = float(np.median(vals))
    out = {"impl": "reference", "metric": "SpMV/SpMM/SpGEMM fwd+bwd step algorithmic GB/s (config 2 workload)",
           "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": float(np.median(secs)) * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "config2-sample: 2D Poisson 32x2048 grid, whole hot-path step (oracle)"},
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": r["cores"], "kind": "oracle", "sample": r["sample"],
                            "host": host_cpu_info()},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def spawn_ranks(args):
    """One process per GPU (the driver's contract).  Under a launcher (WORLD_SIZE set) the world
    size must equal --gpus.  Without one, --gpus N > 1 starts N ranks itself through
    torch.distributed.run on 127.0.0.1; it fails (exit 2, nothing printed on stdout) when fewer
    than N GPUs are visible.  Returns an exit code, or None to run this process as the rank."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
            return 2
        return None
    if args.gpus == 1:
        return None
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}\n")
        return 2
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_dist(torch):
    """torch.distributed for N > 1: NCCL, one GPU per rank (LOCAL_RANK).  CSRK_BENCH_ONE_GPU=1 runs
    every rank on cuda:0 over gloo instead -- a functional check of the sharded paths on a 1-GPU box
    (its numbers are not bench values).  Returns (world, rank, local device index)."""
    import torch.distributed as tdist
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    one = os.environ.get("CSRK_BENCH_ONE_GPU") == "1"
    local = 0 if one else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        if one:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(torch, t):
    """Max over ranks of a device tensor (staged through the host on gloo)."""
    import torch.distributed as tdist
    if tdist.get_backend() == "gloo":
        h = t.cpu()
        tdist.all_reduce(h, op=tdist.ReduceOp.MAX)
        t.copy_(h)
    else:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return t


def allreduce_sum(torch, t):
    import torch.distributed as tdist
    if tdist.get_backend() == "gloo":
        h = t.cpu()
        tdist.all_reduce(h)
        t.copy_(h)
    else:
        tdist.all_reduce(t)
    return t


def write_ops_trace(path, ck, ops_in_order):
    """Run each (name, fn) once and record the csrk launches it made, in launch order."""
    import torch
    torch.cuda.synchronize()
    out = []
    for name, fn in ops_in_order:
        l0 = ck.launch_count()
        fn()
        out.append([name, int(ck.launch_count() - l0)])
    torch.cuda.synchronize()
    with open(path, "w") as f:
        json.dump({"ops": out}, f)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5", "trsv", "gcn", "f12"])
    ap.add_argument("--precond", default="mult", choices=["mult", "solve"], help="cfg5: M = L L^T or (L L^T)^-1")
    ap.add_argument("--ops-trace", default=None,
                    help="after the timed region, run one more pass and write its op -> csrk launch counts "
                         "(tools/traffic.py attributes an ncu launch list of this run to ops with it)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    rc = spawn_ranks(args)
    if rc is not None:
        return rc

    import torch
    import torch.distributed as tdist
    from paper_2212_05159_b200 import csrk as ck

    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.workload in ("cfg3", "cfg4"):
        world, rank, local = init_dist(torch)
        try:
            return run_ops_sharded(args, torch, ck, int(args.workload[-1]), world, rank, local)
        finally:
            tdist.destroy_process_group()
    if args.workload not in ("cfg2", "cfg3", "cfg4", "cfg5") and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        sys.stderr.write(f"bench.py: --workload {args.workload} has no sharded (N > 1) path\n")
        return 2
    if args.workload == "cfg5":
        return run_cfg5(args, torch, ck)
    if args.workload == "trsv":
        return run_trsv_workload(args, torch, ck)
    if args.workload == "gcn":
        return run_gcn_workload(args, torch, ck)
    if args.workload == "f12":
        return run_f12_workload(args, torch, ck)
    if args.workload in ("cfg3", "cfg4"):
        return run_ops_workload(args, torch, ck, int(args.workload[-1]))

    world, rank, local = init_dist(torch)
    dist = None
    if world > 1:
        from paper_2212_05159_b200 import dist as dist_mod
        dist = dist_mod.HaloBench(world, rank)
    W = Workload(torch, ck, rank, world, dist)
    if dist is not None:
        dist.setup(W)
    l2_flush = torch.empty(512 << 20, dtype=torch.uint8, device=W.dev)  # > 126 MB L2

    stepper = W.step
    for _ in range(args.warmup):
        W.step()
    torch.cuda.synchronize()

    names = OPS + (["halo_reduce"] if dist is not None else [])
    evs = [{nm: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for nm in names}
           for _ in range(args.steps)]
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    launches0 = ck.launch_count()
    st = torch.cuda.current_stream()
    with Clocks(local) as clk:
        # the timed steps (headline): the whole pass, L2 flushed before each
        for i in range(args.steps):
            flush_l2(torch, l2_flush)
            step_ev[i][0].record(st)
            stepper()
            step_ev[i][1].record(st)
        torch.cuda.synchronize()
    launches = ck.launch_count() - launches0
    # per-op times (ops report, roofline): the same pass serialised, each op bracketed by events
    for i in range(args.steps):
        flush_l2(torch, l2_flush)
        W.step(evs[i])
    torch.cuda.synchronize()
    # warm-L2 per-op times (SURVEY 8(d) d.5 "also report warm numbers"): no flush between passes
    evs_warm = [{nm: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for nm in names}
                for _ in range(max(2, min(args.steps, 5)))]
    for e in evs_warm:
        W.step(e)
    torch.cuda.synchronize()
    op_ms_warm = {nm: float(np.median([e[nm][0].elapsed_time(e[nm][1]) for e in evs_warm])) for nm in names}
    if world > 1:
        tdist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    tot_ms = float(sum(step_ms))
    op_ms = {nm: float(np.mean([e[nm][0].elapsed_time(e[nm][1]) for e in evs])) for nm in names}
    if world > 1:
        tot_ms = float(allreduce_max(torch, torch.tensor([tot_ms], dtype=torch.float64, device=W.dev)).item())
    ms_per_step = tot_ms / args.steps
    step_bytes = sum(b for b, _ in W.costs.values())
    step_flops = sum(f for _, f in W.costs.values())
    value = step_bytes * world / (ms_per_step * 1e-3) / 1e9

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # dominant kernel: the op with the largest share of the step
    dom = max(OPS, key=lambda nm: op_ms[nm])
    dom_bytes = W.costs[dom][0]
    achieved = dom_bytes / (op_ms[dom] * 1e-3) / 1e9
    # DRAM traffic of that op per call, from the committed ncu launch list (tools/traffic.py)
    traffic, traffic_src = _traffic("cfg2" if world == 1 else f"cfg2_n{world}", dom)
    ops_report = {nm: {"ms": round(op_ms[nm], 4),
                       "GB/s": round(W.costs[nm][0] / (op_ms[nm] * 1e-3) / 1e9, 1) if nm in W.costs else None,
                       "GFLOP/s": round(W.costs[nm][1] / (op_ms[nm] * 1e-3) / 1e9, 1) if nm in W.costs else None,
                       "frac": round(W.costs[nm][0] / (op_ms[nm] * 1e-3) / 1e9 / peak, 3) if nm in W.costs else None}
                  for nm in names}

    out = None
    if rank == 0:
        out = {"metric": "SpMV/SpMM/SpGEMM fwd+bwd step algorithmic GB/s (config 2 workload)",
               "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": "config2: 2D Poisson 5-point 2048x2048 per GPU (4,194,304 rows, "
                                      "20,963,328 nnz), fp64, SpMM k=32, C=A*A; all 8(a) rows per step",
                          "rows_per_gpu": W.m, "nnz_per_gpu": W.nnz, "nnzC_per_gpu": W.nnzC, "k": K,
                          "l2": "flushed (512 MiB write) between timed steps",
                          "parallelism": f"rowblock{world}"},
               "step_ms_stats": {"median": round(float(np.median(step_ms)), 4), "min": round(float(np.min(step_ms)), 4),
                                 "p90": round(float(np.percentile(step_ms, 90)), 4)},
               "gflops": round(step_flops * world / (ms_per_step * 1e-3) / 1e9, 2),
               "step_bytes_per_gpu": step_bytes,
               "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                            "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                            "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes": dom_bytes},
               "ops": ops_report, "ops_warm_ms": {nm: round(v, 4) for nm, v in op_ms_warm.items()},
               "gate": gate_report(W.costs, op_ms, peak), "gpu_launches": int(launches),
               "clocks": clk.summary()}
    # ---------------- e2e: same metric through the public API with pinned host buffers
    if not args.no_e2e:
        e2e = run_e2e(torch, ck, W, args, world)
        if out is not None:
            out["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = run_cpu_baseline()
        cb.pop("seconds", None)
        # also single-threaded (the paper's CPU methodology), on a
        # 1/16 sample of the rows
        st1 = run_cpu_baseline(threads=1, rows_sample=1 << 18)
        cb["single_thread"] = {"value": st1["value"], "unit": "GB/s", "cores": 1, "sample": st1["sample"]}
        cb["host"] = host_cpu_info()
        out["cpu_baseline"] = cb
    if args.ops_trace and rank == 0:
        write_ops_trace(args.ops_trace, ck, W.op_list())
    if out is not None:
        print(json.dumps(out))
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def run_e2e(torch, ck, W, args, world):
    """End to end through the public API: per step the H2D copy of every input (A, x, dy, X, dY,
    dC) from pinned host memory, the step, and the D2H copy of every result (y, dA, dx, Y, dA, dX,
    C, dA, dB) -- all inside the timed region.  Steps are software-pipelined over two device buffer
    sets and three streams: the inputs of step i + 1 are copied in (copy stream 1) while step i
    computes and the results of step i - 1 are copied out (copy stream 2); the host link is full
    duplex, so the two directions overlap each other and the kernels."""
    pin = lambda t: t.cpu().pin_memory()
    Ws = [W, Workload(torch, ck, W.rank, W.world, W.dist)]  # second buffer set, built untimed
    hA = [pin(W.A.indptr), pin(W.A.indices), pin(W.A.values)]
    hin = [pin(W.x), pin(W.dy), pin(W.X), pin(W.dY), pin(W.dC)]
    dev_in = lambda w: [w.A.indptr, w.A.indices, w.A.values, w.x, w.dy, w.X, w.dY, w.dC]
    dev_out = lambda w: [w.y, w.dA_v, w.dx, w.Y, w.dA_m, w.dX, w.Cv, w.dA_g, w.dB_g, w.C.indptr, w.C.indices]
    hout = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in dev_out(W)]
    h2d = sum(t.numel() * t.element_size() for t in hA + hin)
    d2h = sum(t.numel() * t.element_size() for t in hout)
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    Ev = torch.cuda.Event
    steps = max(2, min(args.steps, 20))   # pipeline fill and drain amortised over up to 20 steps
    for w in Ws:  # warm the second buffer set (plans, workspaces)
        w.step()
    torch.cuda.synchronize()
    done_comp = [None, None]   # step i's compute finished: its inputs may be overwritten
    done_out = [None, None]    # step i's results copied out: its outputs may be overwritten
    in_ready = [None, None]

    def copy_in(i):
        b = i % 2
        with torch.cuda.stream(s_in):
            if done_comp[b] is not None:
                s_in.wait_event(done_comp[b])
            for d, h in zip(dev_in(Ws[b]), hA + hin):
                d.copy_(h, non_blocking=True)
            in_ready[b] = Ev()
            in_ready[b].record(s_in)

    ev0, ev1 = Ev(enable_timing=True), Ev(enable_timing=True)
    ev0.record(comp)
    s_in.wait_event(ev0)
    s_out.wait_event(ev0)
    copy_in(0)
    for i in range(steps):
        b = i % 2
        if i + 1 < steps:
            copy_in(i + 1)
        comp.wait_event(in_ready[b])
        if done_out[b] is not None:
            comp.wait_event(done_out[b])
        Ws[b].step()
        done_comp[b] = Ev()
        done_comp[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(done_comp[b])
            for h, d in zip(hout, dev_out(Ws[b])):
                h.copy_(d, non_blocking=True)
            done_out[b] = Ev()
            done_out[b].record(s_out)
    comp.wait_event(done_out[(steps - 1) % 2])
    comp.wait_stream(s_in)
    ev1.record(comp)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    if world > 1:
        import torch.distributed as tdist
        ms = float(allreduce_max(torch, torch.tensor([ms], dtype=torch.float64, device=W.dev)).item())
    step_bytes = sum(b for b, _ in W.costs.values())
    return {"value": round(step_bytes * world / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "pipelined": "2 buffer sets, copy-in / compute / copy-out streams"}


if __name__ == "__main__":
    sys.exit(main())
