"""Thin Python binding of the C-ABI in include/csrk.h (argument marshalling only).

Every function here forwards device pointers of torch CUDA tensors to libcsrk.so on the
current torch stream; all arithmetic runs in the sm_100a kernels.  There is no CPU or
PyTorch fallback: if libcsrk.so is missing or a call fails, an exception is raised.

Names follow the ABI (and the paper's operations, Table 1):
spmv_fwd / spmv_bwd (SpMV), spmm_fwd / spmm_bwd (SpDMM), csr_transpose,
spgemm_symbolic / spgemm_numeric / spgemm_bwd (SpSpMM), spadd_symbolic / spadd_numeric /
spadd_bwd (Sp + Sp), sptrsv_fwd / sptrsv_bwd (SpTRSV), gcn_fwd / gcn_bwd / dense_gemm_nn /
dense_gemm_tn (GCN layer, PAPER 4.4).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcsrk.so")

F32, F64 = 0, 1
OP_N, OP_T = 0, 1
WS = dict(spmv_fwd=0, spmv_bwd=1, spmm_fwd=2, spmm_bwd=3, csr_transpose=4, spgemm_symbolic=5,
          spgemm_numeric=6, spgemm_bwd=7, pcg=8, spadd_symbolic=9, spai=10, sptrsv_fwd=11,
          sptrsv_bwd=12, gcn_fwd=13, gcn_bwd=14, dense_gemm_tn=15, pcg_dist=16)

# Every symbol declared in include/csrk.h (checked by tests/test_abi_cpu.py).
ABI_SYMBOLS = ("csrk_spmv_fwd", "csrk_spmv_bwd", "csrk_spmm_fwd", "csrk_spmm_bwd", "csrk_csr_transpose",
               "csrk_spgemm_symbolic", "csrk_spgemm_numeric", "csrk_spgemm_bwd", "csrk_spgemm_bwd_plan",
               "csrk_workspace_size",
               "csrk_status_string", "csrk_launch_count", "csrk_version", "csrk_pcg_loss_grad",
               "csrk_spadd_symbolic", "csrk_spadd_numeric", "csrk_spadd_bwd", "csrk_spai_loss_grad",
               "csrk_sptrsv_fwd", "csrk_sptrsv_bwd", "csrk_gcn_fwd", "csrk_gcn_bwd", "csrk_dense_gemm_nn",
               "csrk_dense_gemm_tn", "csrk_pcg_loss_grad_dist", "csrk_comm_nccl_unique_id", "csrk_comm_nccl_create",
               "csrk_comm_nccl_destroy")


class Pattern(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p)]


AllreduceFn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
HaloFn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


class Comm(ctypes.Structure):
    """csrk_comm (include/csrk.h): the exchanges of a row-sharded step."""
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce_sum", AllreduceFn), ("halo", HaloFn),
                ("capturable", ctypes.c_int)]


class Halo(ctypes.Structure):
    _fields_ = [("npeers", ctypes.c_int), ("peer", ctypes.POINTER(ctypes.c_int)),
                ("own_off", ctypes.POINTER(ctypes.c_int64)), ("own_len", ctypes.POINTER(ctypes.c_int64)),
                ("ghost_off", ctypes.POINTER(ctypes.c_int64)), ("ghost_len", ctypes.POINTER(ctypes.c_int64))]


class CsrkError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcsrk.so; raises if the CUDA extension has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcsrk.so not found at {LIB_PATH}: run `python -m paper_2212_05159_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, SZ, Pat = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, Pattern
    PatP = ctypes.POINTER(Pattern)
    I = ctypes.c_int
    L.csrk_spmv_fwd.argtypes = [I, I, Pat, P, PatP, P, P, P, P, SZ, P]
    L.csrk_spmv_bwd.argtypes = [I, I, Pat, P, PatP, P, P, P, P, P, P, SZ, P]
    L.csrk_spmm_fwd.argtypes = [I, Pat, P, I64, P, I64, P, I64, P, SZ, P]
    L.csrk_spmm_bwd.argtypes = [I, Pat, P, PatP, P, I64, P, I64, P, I64, P, P, I64, P, SZ, P]
    L.csrk_csr_transpose.argtypes = [I, Pat, P, P, P, P, P, P, SZ, P]
    L.csrk_spgemm_symbolic.argtypes = [Pat, Pat, P, P, ctypes.POINTER(I64), P, SZ, P]
    L.csrk_spgemm_numeric.argtypes = [I, Pat, P, Pat, P, Pat, P, P, SZ, P]
    L.csrk_spgemm_bwd.argtypes = [I, Pat, P, Pat, P, Pat, P, P, P, P, SZ, P]
    L.csrk_spgemm_bwd_plan.argtypes = [I, Pat, P, PatP, P, Pat, P, Pat, P, P, P, P, SZ, P]
    L.csrk_workspace_size.argtypes = [I, I, PatP, PatP, I64, I, ctypes.POINTER(SZ)]
    D = ctypes.c_double
    L.csrk_pcg_loss_grad.argtypes = [Pat, P, Pat, P, P, I, D, I, ctypes.POINTER(D), ctypes.POINTER(D), P, P, SZ, P]
    L.csrk_spadd_symbolic.argtypes = [Pat, Pat, P, P, ctypes.POINTER(I64), P, SZ, P]
    L.csrk_spadd_numeric.argtypes = [I, D, Pat, P, D, Pat, P, Pat, P, P, SZ, P]
    L.csrk_spadd_bwd.argtypes = [I, D, Pat, D, Pat, Pat, P, P, P, P, SZ, P]
    L.csrk_spai_loss_grad.argtypes = [Pat, P, Pat, P, Pat, Pat, Pat, ctypes.POINTER(D), P, P, SZ, P]
    L.csrk_sptrsv_fwd.argtypes = [I, Pat, P, I, I, P, P, P, SZ, P]
    L.csrk_sptrsv_bwd.argtypes = [I, Pat, P, PatP, P, I, I, P, P, P, P, P, SZ, P]
    L.csrk_gcn_fwd.argtypes = [I, Pat, P, I64, P, I64, P, P, I64, P, P, SZ, P]
    L.csrk_gcn_bwd.argtypes = [I, Pat, P, PatP, P, I64, P, P, I64, P, I64, P, P, SZ, P]
    L.csrk_dense_gemm_nn.argtypes = [I, I64, I64, I64, P, I64, P, I, P, I64, P]
    L.csrk_dense_gemm_tn.argtypes = [I, I64, I64, I64, P, I64, P, I64, P, P, SZ, P]
    L.csrk_pcg_loss_grad_dist.argtypes = [ctypes.POINTER(Comm), I64, Pat, P, Pat, P, P, I, D, ctypes.POINTER(D),
                                          ctypes.POINTER(D), P, P, SZ, P]
    L.csrk_comm_nccl_unique_id.argtypes = [P]
    L.csrk_comm_nccl_create.argtypes = [P, I, I, ctypes.POINTER(Halo), ctypes.POINTER(Comm)]
    L.csrk_comm_nccl_destroy.argtypes = [ctypes.POINTER(Comm)]
    L.csrk_status_string.restype = ctypes.c_char_p
    L.csrk_status_string.argtypes = [I]
    L.csrk_launch_count.restype = ctypes.c_uint64
    L.csrk_version.restype = ctypes.c_char_p
    for name in ABI_SYMBOLS:
        if name not in ("csrk_status_string", "csrk_launch_count", "csrk_version"):
            getattr(L, name).restype = I
    _lib = L
    return L


def launch_count() -> int:
    return int(lib().csrk_launch_count())


def _check(st: int, what: str):
    if st != 0:
        raise CsrkError(f"{what}: {lib().csrk_status_string(st).decode()} ({st})")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


@dataclass
class CSR:
    """Device CSR: indptr int64[nrows+1], indices int32[nnz], values float32/64[nnz] or None."""
    nrows: int
    ncols: int
    indptr: torch.Tensor
    indices: torch.Tensor
    values: torch.Tensor | None = None

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    def pattern(self) -> Pattern:
        return Pattern(self.nrows, self.ncols, self.nnz, self.indptr.data_ptr(), self.indices.data_ptr())

    @staticmethod
    def from_host(A, device="cuda", dtype=None) -> "CSR":
        """Upload a synth.CSR (numpy) to the device."""
        vals = None if A.values is None else torch.from_numpy(A.values).to(device)
        if vals is not None and dtype is not None:
            vals = vals.to(dtype)
        return CSR(A.nrows, A.ncols, torch.from_numpy(A.indptr).to(device), torch.from_numpy(A.indices).to(device), vals)


@dataclass
class TransposePlan:
    """Cached A^T: pattern (n x m) plus perm[q] = position in A of A^T's q-th entry."""
    AT: CSR
    perm: torch.Tensor

    def args(self):
        p = self.AT.pattern()
        return ctypes.byref(p), _ptr(self.perm), p  # keep p alive


_ws_cache: dict = {}


def _workspace(op: str, dtype: int, A: CSR, B: CSR | None = None, k: int = 0, have_plan: bool = False):
    pa = A.pattern()
    pb = B.pattern() if B is not None else None
    n = ctypes.c_size_t(0)
    _check(lib().csrk_workspace_size(WS[op], dtype, ctypes.byref(pa), ctypes.byref(pb) if pb else None, k,
                                     int(have_plan), ctypes.byref(n)), f"workspace_size({op})")
    nbytes = int(n.value)
    if nbytes == 0:
        return None, 0
    dev = A.indptr.device
    # one cached scratch buffer per (device, stream): ops enqueued on different streams may
    # run concurrently and must not share scratch
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return _ptr(buf), buf.numel()


def spmv_fwd(A: CSR, x: torch.Tensor, op: int = OP_N, plan: TransposePlan | None = None,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """y = A x (op N) or y = A^T x (op T).  PAPER 3.1.1."""
    dt = _dt(A.values)
    y = out if out is not None else torch.empty(A.nrows if op == OP_N else A.ncols, dtype=A.values.dtype,
                                                device=A.values.device)
    pp = plan.args() if plan else (None, None, None)
    ws, wsb = _workspace("spmv_fwd", dt, A, have_plan=plan is not None)
    _check(lib().csrk_spmv_fwd(dt, op, A.pattern(), _ptr(A.values), pp[0], pp[1], _ptr(x), _ptr(y), ws, wsb,
                               _stream()), "spmv_fwd")
    return y


def spmv_bwd(A: CSR, x: torch.Tensor, dy: torch.Tensor, op: int = OP_N, plan: TransposePlan | None = None,
             need_dA: bool = True, need_dx: bool = True, dA: torch.Tensor | None = None,
             dx: torch.Tensor | None = None):
    """VJP of SpMV (Table 1): dA = (dy x^T) (.) mask(A) on A's pattern, dx = A^T dy."""
    dt = _dt(A.values)
    if need_dA and dA is None:
        dA = torch.empty_like(A.values)
    if need_dx and dx is None:
        dx = torch.empty(A.ncols if op == OP_N else A.nrows, dtype=A.values.dtype, device=A.values.device)
    pp = plan.args() if plan else (None, None, None)
    ws, wsb = _workspace("spmv_bwd", dt, A, have_plan=plan is not None)
    _check(lib().csrk_spmv_bwd(dt, op, A.pattern(), _ptr(A.values), pp[0], pp[1], _ptr(x), _ptr(dy),
                               _ptr(dA if need_dA else None), _ptr(dx if need_dx else None), ws, wsb, _stream()),
           "spmv_bwd")
    return (dA if need_dA else None), (dx if need_dx else None)


def spmm_fwd(A: CSR, X: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Y = A X, X row-major n x k."""
    dt = _dt(A.values)
    k = X.shape[1]
    Y = out if out is not None else torch.empty((A.nrows, k), dtype=X.dtype, device=X.device)
    ws, wsb = _workspace("spmm_fwd", dt, A, k=k)
    _check(lib().csrk_spmm_fwd(dt, A.pattern(), _ptr(A.values), k, _ptr(X), X.stride(0), _ptr(Y), Y.stride(0), ws,
                               wsb, _stream()), "spmm_fwd")
    return Y


def spmm_bwd(A: CSR, X: torch.Tensor, dY: torch.Tensor, plan: TransposePlan | None = None, need_dA: bool = True,
             need_dX: bool = True, dA: torch.Tensor | None = None, dX: torch.Tensor | None = None):
    """VJP of SpDMM (Table 1): dA = (dY X^T) (.) mask(A), dX = A^T dY."""
    dt = _dt(A.values)
    k = X.shape[1]
    if need_dA and dA is None:
        dA = torch.empty_like(A.values)
    if need_dX and dX is None:
        dX = torch.empty((A.ncols, k), dtype=X.dtype, device=X.device)
    pp = plan.args() if plan else (None, None, None)
    ws, wsb = _workspace("spmm_bwd", dt, A, k=k, have_plan=plan is not None)
    _check(lib().csrk_spmm_bwd(dt, A.pattern(), _ptr(A.values), pp[0], pp[1], k, _ptr(X), X.stride(0), _ptr(dY),
                               dY.stride(0), _ptr(dA if need_dA else None), _ptr(dX if need_dX else None),
                               dX.stride(0) if need_dX else k, ws, wsb, _stream()), "spmm_bwd")
    return (dA if need_dA else None), (dX if need_dX else None)


def csr_transpose(A: CSR, with_values: bool = True, out: TransposePlan | None = None) -> TransposePlan:
    """A^T in canonical CSR + perm.  Values optional (gathered through perm)."""
    dev = A.indptr.device
    dt = _dt(A.values) if A.values is not None else F64
    if out is None:
        ATv = torch.empty_like(A.values) if (with_values and A.values is not None) else None
        out = TransposePlan(CSR(A.ncols, A.nrows, torch.empty(A.ncols + 1, dtype=torch.int64, device=dev),
                                torch.empty(A.nnz, dtype=torch.int32, device=dev), ATv),
                            torch.empty(A.nnz, dtype=torch.int64, device=dev))
    ws, wsb = _workspace("csr_transpose", dt, A)
    _check(lib().csrk_csr_transpose(dt, A.pattern(), _ptr(A.values), _ptr(out.AT.indptr), _ptr(out.AT.indices),
                                    _ptr(out.AT.values), _ptr(out.perm), ws, wsb, _stream()), "csr_transpose")
    return out


def spgemm_symbolic(A: CSR, B: CSR) -> CSR:
    """Structural pattern of C = A B, columns sorted.  One host sync for nnz(C)."""
    dev = A.indptr.device
    Cp = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
    nnz = ctypes.c_int64(0)
    ws, wsb = _workspace("spgemm_symbolic", F64, A, B)
    _check(lib().csrk_spgemm_symbolic(A.pattern(), B.pattern(), _ptr(Cp), None, ctypes.byref(nnz), ws, wsb,
                                      _stream()), "spgemm_symbolic(count)")
    Ci = torch.empty(int(nnz.value), dtype=torch.int32, device=dev)
    if Ci.numel() == 0:
        return CSR(A.nrows, B.ncols, Cp, Ci, None)
    _check(lib().csrk_spgemm_symbolic(A.pattern(), B.pattern(), _ptr(Cp), _ptr(Ci), None, ws, wsb, _stream()),
           "spgemm_symbolic(fill)")
    return CSR(A.nrows, B.ncols, Cp, Ci, None)


def spgemm_numeric(A: CSR, B: CSR, C: CSR, out: torch.Tensor | None = None) -> torch.Tensor:
    """C_ij = sum_k A_ik B_kj over the symbolic pattern."""
    dt = _dt(A.values)
    Cv = out if out is not None else torch.empty(C.nnz, dtype=A.values.dtype, device=A.values.device)
    ws, wsb = _workspace("spgemm_numeric", dt, A, B)
    _check(lib().csrk_spgemm_numeric(dt, A.pattern(), _ptr(A.values), B.pattern(), _ptr(B.values), C.pattern(),
                                     _ptr(Cv), ws, wsb, _stream()), "spgemm_numeric")
    return Cv


def spgemm_bwd(A: CSR, B: CSR, C: CSR, dC: torch.Tensor, need_dA: bool = True, need_dB: bool = True,
               dA: torch.Tensor | None = None, dB: torch.Tensor | None = None, plan: TransposePlan | None = None):
    """VJP of SpGEMM (Table 1): dA = (dC B^T) (.) mask(A), dB = (A^T dC) (.) mask(B).
    plan = A's transpose plan: dB by the deterministic column gather instead of atomics."""
    dt = _dt(A.values)
    if need_dA and dA is None:
        dA = torch.empty_like(A.values)
    if need_dB and dB is None:
        dB = torch.empty_like(B.values)
    ws, wsb = _workspace("spgemm_bwd", dt, A, B, have_plan=plan is not None)
    if plan is None:
        _check(lib().csrk_spgemm_bwd(dt, A.pattern(), _ptr(A.values), B.pattern(), _ptr(B.values), C.pattern(),
                                     _ptr(dC), _ptr(dA if need_dA else None), _ptr(dB if need_dB else None), ws,
                                     wsb, _stream()), "spgemm_bwd")
    else:
        pp = plan.args()
        _check(lib().csrk_spgemm_bwd_plan(dt, A.pattern(), _ptr(A.values), pp[0], pp[1], B.pattern(),
                                          _ptr(B.values), C.pattern(), _ptr(dC), _ptr(dA if need_dA else None),
                                          _ptr(dB if need_dB else None), ws, wsb, _stream()), "spgemm_bwd_plan")
    return (dA if need_dA else None), (dB if need_dB else None)


def spadd_symbolic(A: CSR, B: CSR) -> CSR:
    """pattern(alpha A + beta B) = pattern(A) U pattern(B), columns sorted.  One
    host sync for nnz(C)."""
    dev = A.indptr.device
    Cp = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
    nnz = ctypes.c_int64(0)
    ws, wsb = _workspace("spadd_symbolic", F64, A, B)
    _check(lib().csrk_spadd_symbolic(A.pattern(), B.pattern(), _ptr(Cp), None, ctypes.byref(nnz), ws, wsb,
                                     _stream()), "spadd_symbolic(count)")
    Ci = torch.empty(int(nnz.value), dtype=torch.int32, device=dev)
    if Ci.numel() > 0:
        _check(lib().csrk_spadd_symbolic(A.pattern(), B.pattern(), _ptr(Cp), _ptr(Ci), None, ws, wsb, _stream()),
               "spadd_symbolic(fill)")
    return CSR(A.nrows, A.ncols, Cp, Ci, None)


def spadd_numeric(alpha: float, A: CSR, beta: float, B: CSR, C: CSR, out: torch.Tensor | None = None):
    """C = alpha A + beta B on C = spadd_symbolic(A, B)."""
    dt = _dt(A.values)
    Cv = out if out is not None else torch.empty(C.nnz, dtype=A.values.dtype, device=A.values.device)
    _check(lib().csrk_spadd_numeric(dt, float(alpha), A.pattern(), _ptr(A.values), float(beta), B.pattern(),
                                    _ptr(B.values), C.pattern(), _ptr(Cv), None, 0, _stream()), "spadd_numeric")
    return Cv


def spadd_bwd(alpha: float, A: CSR, beta: float, B: CSR, C: CSR, dC: torch.Tensor, need_dA: bool = True,
              need_dB: bool = True, dA: torch.Tensor | None = None, dB: torch.Tensor | None = None):
    """VJP of Sp+Sp (Table 1): dA = alpha dC (.) mask(A), dB = beta dC (.) mask(B)."""
    dt = _dt(dC)
    if need_dA and dA is None:
        dA = torch.empty(A.nnz, dtype=dC.dtype, device=dC.device)
    if need_dB and dB is None:
        dB = torch.empty(B.nnz, dtype=dC.dtype, device=dC.device)
    _check(lib().csrk_spadd_bwd(dt, float(alpha), A.pattern(), float(beta), B.pattern(), C.pattern(), _ptr(dC),
                                _ptr(dA if need_dA else None), _ptr(dB if need_dB else None), None, 0, _stream()),
           "spadd_bwd")
    return (dA if need_dA else None), (dB if need_dB else None)


@dataclass
class SpaiPlan:
    """Cached patterns of the SPAI workload: C = pattern(M A), the identity
    pattern I and R = pattern(I) U C.  Value-independent: built once per pattern(M), pattern(A)."""
    C: CSR
    I: CSR
    R: CSR


def spai_plan(M: CSR, A: CSR) -> SpaiPlan:
    n = A.nrows
    dev = A.indptr.device
    I = CSR(n, n, torch.arange(n + 1, dtype=torch.int64, device=dev), torch.arange(n, dtype=torch.int32, device=dev))
    C = spgemm_symbolic(M, A)
    return SpaiPlan(C, I, spadd_symbolic(I, C))


def spai_loss_grad(plan: SpaiPlan, M: CSR, A: CSR, dM: torch.Tensor | None = None):
    """loss = ||I - M A||_F^2 and d loss / d M.values (PAPER 4.6).  fp64."""
    if dM is None:
        dM = torch.empty_like(M.values)
    pc, pr = plan.C.pattern(), plan.R.pattern()
    nbytes = ctypes.c_size_t(0)
    _check(lib().csrk_workspace_size(WS["spai"], F64, ctypes.byref(pc), ctypes.byref(pr), A.nrows, 0,
                                     ctypes.byref(nbytes)), "workspace_size(spai)")
    dev = A.indptr.device
    buf = _ws_cache.get(dev)
    if buf is None or buf.numel() < int(nbytes.value):
        buf = torch.empty(max(int(nbytes.value), 1 << 20), dtype=torch.uint8, device=dev)
        _ws_cache[dev] = buf
    loss = ctypes.c_double(0.0)
    _check(lib().csrk_spai_loss_grad(A.pattern(), _ptr(A.values), M.pattern(), _ptr(M.values), pc, pr,
                                     plan.I.pattern(), ctypes.byref(loss), _ptr(dM), _ptr(buf), buf.numel(),
                                     _stream()), "spai_loss_grad")
    return float(loss.value), dM


def sptrsv_fwd(T: CSR, b: torch.Tensor, upper: bool = False, unit: bool = False,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """x = T^{-1} b, T triangular (PAPER 3.1.5)."""
    dt = _dt(T.values)
    x = out if out is not None else torch.empty(T.nrows, dtype=T.values.dtype, device=T.values.device)
    ws, wsb = _workspace("sptrsv_fwd", dt, T)
    _check(lib().csrk_sptrsv_fwd(dt, T.pattern(), _ptr(T.values), int(upper), int(unit), _ptr(b), _ptr(x), ws, wsb,
                                 _stream()), "sptrsv_fwd")
    return x


def sptrsv_bwd(T: CSR, x: torch.Tensor, v: torch.Tensor, upper: bool = False, unit: bool = False,
               plan: TransposePlan | None = None, need_dT: bool = True, need_db: bool = True,
               dT: torch.Tensor | None = None, db: torch.Tensor | None = None):
    """VJP of x = T^{-1} b: db = T^{-T} v, dT = -db x^T (.) mask(T)."""
    dt = _dt(T.values)
    if need_dT and dT is None:
        dT = torch.empty_like(T.values)
    if need_db and db is None:
        db = torch.empty(T.nrows, dtype=T.values.dtype, device=T.values.device)
    pp = plan.args() if plan else (None, None, None)
    ws, wsb = _workspace("sptrsv_bwd", dt, T, have_plan=plan is not None)
    _check(lib().csrk_sptrsv_bwd(dt, T.pattern(), _ptr(T.values), pp[0], pp[1], int(upper), int(unit), _ptr(x),
                                 _ptr(v), _ptr(dT if need_dT else None), _ptr(db if need_db else None), ws, wsb,
                                 _stream()), "sptrsv_bwd")
    return (dT if need_dT else None), (db if need_db else None)


def gcn_fwd(A: CSR, Z: torch.Tensor, bias: torch.Tensor | None = None, out: torch.Tensor | None = None,
            D: torch.Tensor | None = None):
    """Y = D (A (D Z) + D Z) + bias, D = (row_sum(A) + 1)^-1/2 (PAPER 4.4 Fig. 12).  Returns (Y, D)."""
    dt = _dt(Z)
    n, F = Z.shape
    Y = out if out is not None else torch.empty((n, F), dtype=Z.dtype, device=Z.device)
    D = D if D is not None else torch.empty(n, dtype=torch.float64, device=Z.device)
    ws, wsb = _workspace("gcn_fwd", dt, A, k=F)
    _check(lib().csrk_gcn_fwd(dt, A.pattern(), _ptr(A.values), F, _ptr(Z), Z.stride(0), _ptr(bias), _ptr(Y),
                              Y.stride(0), _ptr(D), ws, wsb, _stream()), "gcn_fwd")
    return Y, D


def gcn_bwd(A: CSR, D: torch.Tensor, dY: torch.Tensor, plan: TransposePlan | None = None, need_dZ: bool = True,
            need_dbias: bool = True, dZ: torch.Tensor | None = None, dbias: torch.Tensor | None = None):
    """VJP of gcn_fwd (graph constant): dZ = D (A^T (D dY) + D dY), dbias = column sums of dY."""
    dt = _dt(dY)
    n, F = dY.shape
    if need_dZ and dZ is None:
        dZ = torch.empty_like(dY)
    if need_dbias and dbias is None:
        dbias = torch.empty(F, dtype=dY.dtype, device=dY.device)
    pp = plan.args() if plan else (None, None, None)
    ws, wsb = _workspace("gcn_bwd", dt, A, k=F, have_plan=plan is not None)
    _check(lib().csrk_gcn_bwd(dt, A.pattern(), _ptr(A.values), pp[0], pp[1], F, _ptr(D), _ptr(dY), dY.stride(0),
                              _ptr(dZ if need_dZ else None), dZ.stride(0) if need_dZ else F,
                              _ptr(dbias if need_dbias else None), ws, wsb, _stream()), "gcn_bwd")
    return (dZ if need_dZ else None), (dbias if need_dbias else None)


def dense_gemm_nn(X: torch.Tensor, W: torch.Tensor, transW: bool = False, out: torch.Tensor | None = None):
    """Z = X W (W: C x F) or X W^T (W: F x C) -- the XTheta / dX products of the GCN layer."""
    n, C = X.shape
    F = W.shape[0] if transW else W.shape[1]
    Z = out if out is not None else torch.empty((n, F), dtype=X.dtype, device=X.device)
    _check(lib().csrk_dense_gemm_nn(_dt(X), n, C, F, _ptr(X), X.stride(0), _ptr(W.contiguous()), int(transW), _ptr(Z),
                                    Z.stride(0), _stream()), "dense_gemm_nn")
    return Z


def dense_gemm_tn(X: torch.Tensor, dZ: torch.Tensor, out: torch.Tensor | None = None):
    """dW = X^T dZ (C x F) -- dTheta of the GCN layer."""
    n, C = X.shape
    F = dZ.shape[1]
    dW = out if out is not None else torch.empty((C, F), dtype=X.dtype, device=X.device)
    dims = CSR(n, C, X.new_zeros(1, dtype=torch.int64), X.new_zeros(0, dtype=torch.int32))  # sizes only
    ws, wsb = _workspace("dense_gemm_tn", _dt(X), dims, k=F)
    _check(lib().csrk_dense_gemm_tn(_dt(X), n, C, F, _ptr(X), X.stride(0), _ptr(dZ), dZ.stride(0), _ptr(dW), ws, wsb,
                                    _stream()), "dense_gemm_tn")
    return dW


def gcn_layer_fwd(A: CSR, X: torch.Tensor, Theta: torch.Tensor, bias: torch.Tensor):
    """The GCN layer of Fig. 12: XTheta = X Theta, then the fused propagation.  Returns (Y, D)."""
    return gcn_fwd(A, dense_gemm_nn(X, Theta), bias)


def gcn_layer_bwd(A: CSR, D: torch.Tensor, X: torch.Tensor, Theta: torch.Tensor, dY: torch.Tensor,
                  plan: TransposePlan | None = None):
    """VJP of the layer: (dX, dTheta, dbias) with dZ from gcn_bwd, dTheta = X^T dZ, dX = dZ Theta^T."""
    dZ, dbias = gcn_bwd(A, D, dY, plan=plan)
    return dense_gemm_nn(dZ, Theta, transW=True), dense_gemm_tn(X, dZ), dbias


def pcg_loss_grad(A: CSR, L: CSR, b: torch.Tensor, n_it: int = 50, gamma: float = 0.6,
                  dL: torch.Tensor | None = None, precond: str = "mult"):
    """Config-5 composition (PAPER 4.3): n_it PCG iterations with M = L L^T, the
    weighted residual loss and its gradient w.r.t. L.values.  fp64.
    precond="solve": M = (L L^T)^{-1} applied by two triangular solves.
    Returns (loss, residual norms ||r^(1..n_it)||, dL on L's pattern)."""
    pc = {"mult": 0, "solve": 1}[precond]
    if dL is None:
        dL = torch.empty_like(L.values)
    pa, pl = A.pattern(), L.pattern()
    nbytes = ctypes.c_size_t(0)
    _check(lib().csrk_workspace_size(WS["pcg"], F64, ctypes.byref(pa), ctypes.byref(pl), n_it, pc,
                                     ctypes.byref(nbytes)), "workspace_size(pcg)")
    ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=b.device)
    loss = ctypes.c_double(0.0)
    resid = (ctypes.c_double * n_it)()
    _check(lib().csrk_pcg_loss_grad(pa, _ptr(A.values), pl, _ptr(L.values), _ptr(b), int(n_it), float(gamma), pc,
                                    ctypes.byref(loss), resid, _ptr(dL), _ptr(ws), ws.numel(), _stream()),
           "pcg_loss_grad")
    return float(loss.value), list(resid), dL


# ---------------------------------------------------------------- row-sharded multi-GPU
def halo_struct(spec):
    """ctypes csrk_halo from a dict of equal-length lists: peer, own_off, own_len, ghost_off, ghost_len."""
    n = len(spec["peer"])
    arr = lambda t, v: (t * max(n, 1))(*v)
    h = Halo(n, arr(ctypes.c_int, spec["peer"]), arr(ctypes.c_int64, spec["own_off"]),
             arr(ctypes.c_int64, spec["own_len"]), arr(ctypes.c_int64, spec["ghost_off"]),
             arr(ctypes.c_int64, spec["ghost_len"]))
    return h


def comm_nccl(rank: int, world: int, halo_spec, group=None) -> Comm:
    """csrk_comm over NCCL (comm.cu): rank 0 draws the NCCL unique id, torch.distributed broadcasts
    it, every rank creates its communicator (collective).  Destroy with comm_destroy."""
    import torch.distributed as tdist
    buf = (ctypes.c_char * 128)()
    if rank == 0:
        _check(lib().csrk_comm_nccl_unique_id(buf), "comm_nccl_unique_id")
    obj = [bytes(buf)]
    tdist.broadcast_object_list(obj, src=0, group=group)
    ctypes.memmove(buf, obj[0], 128)
    c = Comm()
    h = halo_struct(halo_spec)
    _check(lib().csrk_comm_nccl_create(buf, rank, world, ctypes.byref(h), ctypes.byref(c)), "comm_nccl_create")
    return c


def comm_destroy(c: Comm):
    _check(lib().csrk_comm_nccl_destroy(ctypes.byref(c)), "comm_nccl_destroy")


def pcg_loss_grad_dist(comm: Comm | None, own_off: int, A: CSR, L: CSR, b: torch.Tensor, n_it: int = 50,
                       gamma: float = 0.6, dL: torch.Tensor | None = None, ws: torch.Tensor | None = None):
    """One rank's share of the row-sharded config-5 step (csrk_pcg_loss_grad_dist): A, L = the
    rank's rows (columns in extended coordinates), b its owned entries.  Returns (loss, residual
    norms, dL on L's rows) -- loss and residuals are global.  `ws` may be passed to reuse a
    workspace across calls (the CUDA-graph cache is keyed by it)."""
    if dL is None:
        dL = torch.empty_like(L.values)
    pa, pl = A.pattern(), L.pattern()
    nbytes = ctypes.c_size_t(0)
    _check(lib().csrk_workspace_size(WS["pcg_dist"], F64, ctypes.byref(pa), ctypes.byref(pl), n_it, 0,
                                     ctypes.byref(nbytes)), "workspace_size(pcg_dist)")
    if ws is None or ws.numel() < int(nbytes.value):
        ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=b.device)
    loss = ctypes.c_double(0.0)
    resid = (ctypes.c_double * n_it)()
    _check(lib().csrk_pcg_loss_grad_dist(ctypes.byref(comm) if comm is not None else None, int(own_off), pa,
                                         _ptr(A.values), pl, _ptr(L.values), _ptr(b), int(n_it), float(gamma),
                                         ctypes.byref(loss), resid, _ptr(dL), _ptr(ws), ws.numel(), _stream()),
           "pcg_loss_grad_dist")
    return float(loss.value), list(resid), dL
