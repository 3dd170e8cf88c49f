"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain CPU implementation of the hot path of Nytko et al. (arXiv 2212.05159),
written from the paper (see csr_oracle.c for the per-function citations).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` and
``--impl reference``) may import this package.  It shares no code with the CUDA
path and never imports ``paper_2212_05159_b200``.

Every reduced output comes with ``S`` = sum of |terms| (SURVEY.md 8(c) c.2,
DESIGN.md reading A6) so callers can apply |gpu - orc| <= rtol * S.

fp32 inputs are widened exactly to float64, reduced in long double, and the
result is rounded ONCE to float32 here.  Parity status: every function below is
pinned by tests/test_oracle_pins.py (closed forms, paper/SPEC worked examples,
dense brute force, finite differences, adjoint/Euler identities).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile csr_oracle.c with gcc (no -ffast-math: IEEE semantics are the point)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-ffp-contract=off",
                               "-shared", "-fPIC", "-std=c11", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.orc_spmv.argtypes = [ctypes.c_int, _I64, _I64, _P, _P, _P, _P, _P, _P]
        L.orc_spmv_bwd.argtypes = [ctypes.c_int, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P]
        L.orc_spmm.argtypes = [_I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _I64, _P]
        L.orc_spmm_bwd.argtypes = [_I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _I64, _P]
        L.orc_csr_transpose.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P, _P]
        L.orc_spgemm_symbolic.argtypes = [_I64, _I64, _I64, _P, _P, _P, _P, _P, _P]
        L.orc_spgemm_symbolic.restype = _I64
        L.orc_spgemm_numeric.argtypes = [_I64, _I64, _I64] + [_P] * 10
        L.orc_spgemm_numeric.restype = ctypes.c_int
        L.orc_spgemm_bwd.argtypes = [_I64, _I64, _I64] + [_P] * 13
        L.orc_spgemm_bwd.restype = ctypes.c_int
        L.orc_spadd_symbolic.argtypes = [_I64, _P, _P, _P, _P, _P, _P]
        L.orc_spadd_symbolic.restype = _I64
        L.orc_spadd_numeric.argtypes = [_I64, ctypes.c_double, ctypes.c_double] + [_P] * 10
        L.orc_spadd_numeric.restype = ctypes.c_int
        L.orc_spadd_bwd.argtypes = [_I64, ctypes.c_double, ctypes.c_double] + [_P] * 9
        L.orc_spadd_bwd.restype = ctypes.c_int
        L.orc_sptrsv.argtypes = [ctypes.c_int, ctypes.c_int, _I64] + [_P] * 6
        L.orc_sptrsv.restype = ctypes.c_int
        L.orc_sptrsv_bwd.argtypes = [ctypes.c_int, ctypes.c_int, _I64] + [_P] * 8
        L.orc_sptrsv_bwd.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_get_threads.restype = ctypes.c_int
    return _lib


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def get_threads() -> int:
    return lib().orc_get_threads()


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _pat(A):
    return (np.ascontiguousarray(A.indptr, dtype=np.int64), np.ascontiguousarray(A.indices, dtype=np.int32))


def _out(a, dtype):
    """Round the double result once to the data type."""
    return a if dtype == np.float64 else a.astype(dtype)


@dataclass
class Result:
    value: np.ndarray
    S: np.ndarray | None = None


def spmv_fwd(A, x, op: int = 0) -> Result:
    """op 0: y = A x.  op 1: y = A^T x."""
    ip, ix = _pat(A)
    dt = A.values.dtype
    out_len = A.nrows if op == 0 else A.ncols
    assert x.shape == ((A.ncols if op == 0 else A.nrows),)
    y = np.empty(out_len, np.float64)
    S = np.empty(out_len, np.float64)
    v, xx = _f64(A.values), _f64(x)
    lib().orc_spmv(op, A.nrows, A.ncols, _p(ip), _p(ix), _p(v), _p(xx), _p(y), _p(S))
    return Result(_out(y, dt), S)


def spmv_bwd(A, x, dy, op: int = 0, want_dA: bool = True, want_dx: bool = True):
    """VJP of SpMV (Table 1).  Returns (dA on A's pattern, Result(dx, S))."""
    ip, ix = _pat(A)
    dt = A.values.dtype
    v, xx, g = _f64(A.values), _f64(x), _f64(dy)
    dA = np.empty(A.nnz, np.float64) if want_dA else None
    dx_len = A.ncols if op == 0 else A.nrows
    dx = np.empty(dx_len, np.float64) if want_dx else None
    S = np.empty(dx_len, np.float64) if want_dx else None
    lib().orc_spmv_bwd(op, A.nrows, A.ncols, _p(ip), _p(ix), _p(v), _p(xx), _p(g), _p(dA), _p(dx), _p(S))
    return (None if dA is None else _out(dA, dt)), (None if dx is None else Result(_out(dx, dt), S))


def spmm_fwd(A, X) -> Result:
    """Y = A X, X row-major n x k."""
    ip, ix = _pat(A)
    dt = A.values.dtype
    X64 = _f64(X)
    k = X64.shape[1]
    Y = np.empty((A.nrows, k), np.float64)
    S = np.empty((A.nrows, k), np.float64)
    lib().orc_spmm(A.nrows, A.ncols, k, _p(ip), _p(ix), _p(_f64(A.values)), _p(X64), k, _p(Y), k, _p(S))
    return Result(_out(Y, dt), S)


def spmm_bwd(A, X, dY, want_dA: bool = True, want_dX: bool = True):
    """VJP of SpDMM (Table 1).  Returns (Result(dA,S), Result(dX,S))."""
    ip, ix = _pat(A)
    dt = A.values.dtype
    X64, G = _f64(X), _f64(dY)
    k = X64.shape[1]
    dA = np.empty(A.nnz, np.float64) if want_dA else None
    SA = np.empty(A.nnz, np.float64) if want_dA else None
    dX = np.empty((A.ncols, k), np.float64) if want_dX else None
    SX = np.empty((A.ncols, k), np.float64) if want_dX else None
    lib().orc_spmm_bwd(A.nrows, A.ncols, k, _p(ip), _p(ix), _p(_f64(A.values)), _p(X64), k, _p(G), k,
                       _p(dA), _p(SA), _p(dX), k, _p(SX))
    return (None if dA is None else Result(_out(dA, dt), SA)), (None if dX is None else Result(_out(dX, dt), SX))


def csr_transpose(A):
    """A^T in canonical CSR plus perm.  Returns (AT_indptr, AT_indices, AT_values|None, perm)."""
    ip, ix = _pat(A)
    ATp = np.empty(A.ncols + 1, np.int64)
    ATi = np.empty(A.nnz, np.int32)
    perm = np.empty(A.nnz, np.int64)
    ATv = None
    if A.values is not None:
        ATv = np.empty(A.nnz, np.float64)
        lib().orc_csr_transpose(A.nrows, A.ncols, _p(ip), _p(ix), _p(_f64(A.values)), _p(ATp), _p(ATi), _p(ATv), _p(perm))
        ATv = ATv.astype(A.values.dtype)
    else:
        lib().orc_csr_transpose(A.nrows, A.ncols, _p(ip), _p(ix), None, _p(ATp), _p(ATi), None, _p(perm))
    return ATp, ATi, ATv, perm


def spgemm_symbolic(A, B):
    """Structural pattern of C = A B.  Returns (C_indptr, C_indices)."""
    assert A.ncols == B.nrows
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    Cp = np.empty(A.nrows + 1, np.int64)
    nnz = lib().orc_spgemm_symbolic(A.nrows, A.ncols, B.ncols, _p(ap), _p(ai), _p(bp), _p(bi), _p(Cp), None)
    Ci = np.empty(nnz, np.int32)
    lib().orc_spgemm_symbolic(A.nrows, A.ncols, B.ncols, _p(ap), _p(ai), _p(bp), _p(bi), _p(Cp), _p(Ci))
    return Cp, Ci


def spgemm_numeric(A, B, Cp, Ci) -> Result:
    """C_ij = sum_k A_ik B_kj over the symbolic pattern."""
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    dt = A.values.dtype
    Cv = np.empty(Ci.shape[0], np.float64)
    S = np.empty(Ci.shape[0], np.float64)
    rc = lib().orc_spgemm_numeric(A.nrows, A.ncols, B.ncols, _p(ap), _p(ai), _p(_f64(A.values)),
                                  _p(bp), _p(bi), _p(_f64(B.values)), _p(Cp), _p(Ci), _p(Cv), _p(S))
    if rc != 0:
        raise ValueError("spgemm_numeric: a product falls outside C's pattern")
    return Result(_out(Cv, dt), S)


def spgemm_bwd(A, B, Cp, Ci, dC, want_dA: bool = True, want_dB: bool = True):
    """VJP of SpGEMM (Table 1).  Returns (Result(dA,S), Result(dB,S))."""
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    dt = A.values.dtype
    g = _f64(dC)
    dA = np.empty(A.nnz, np.float64) if want_dA else None
    SA = np.empty(A.nnz, np.float64) if want_dA else None
    dB = np.empty(B.nnz, np.float64) if want_dB else None
    SB = np.empty(B.nnz, np.float64) if want_dB else None
    rc = lib().orc_spgemm_bwd(A.nrows, A.ncols, B.ncols, _p(ap), _p(ai), _p(_f64(A.values)),
                              _p(bp), _p(bi), _p(_f64(B.values)), _p(Cp), _p(Ci), _p(g),
                              _p(dA), _p(SA), _p(dB), _p(SB))
    if rc != 0:
        raise ValueError("spgemm_bwd: dC's pattern does not cover the products")
    return (None if dA is None else Result(_out(dA, dt), SA)), (None if dB is None else Result(_out(dB, dt), SB))


def spadd_symbolic(A, B):
    """pattern(alpha A + beta B) = pattern(A) U pattern(B), row by row."""
    assert (A.nrows, A.ncols) == (B.nrows, B.ncols), "Sp+Sp: shape mismatch"
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    Cp = np.empty(A.nrows + 1, np.int64)
    nnz = lib().orc_spadd_symbolic(A.nrows, _p(ap), _p(ai), _p(bp), _p(bi), _p(Cp), None)
    Ci = np.empty(nnz, np.int32)
    lib().orc_spadd_symbolic(A.nrows, _p(ap), _p(ai), _p(bp), _p(bi), _p(Cp), _p(Ci))
    return Cp, Ci


def spadd_numeric(alpha, A, beta, B, Cp, Ci) -> Result:
    """C = alpha A + beta B on the union pattern."""
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    dt = A.values.dtype
    Cv = np.empty(Ci.shape[0], np.float64)
    S = np.empty(Ci.shape[0], np.float64)
    rc = lib().orc_spadd_numeric(A.nrows, float(alpha), float(beta), _p(ap), _p(ai), _p(_f64(A.values)),
                                 _p(bp), _p(bi), _p(_f64(B.values)), _p(Cp), _p(Ci), _p(Cv), _p(S))
    if rc != 0:
        raise ValueError("spadd_numeric: an entry of A or B is missing from C's pattern")
    return Result(_out(Cv, dt), S)


def spadd_bwd(alpha, A, beta, B, Cp, Ci, dC, want_dA: bool = True, want_dB: bool = True):
    """VJP of Sp+Sp (Table 1): (alpha V (.) mask(A), beta V (.) mask(B))."""
    ap, ai = _pat(A)
    bp, bi = _pat(B)
    dt = dC.dtype
    g = _f64(dC)
    dA = np.empty(A.nnz, np.float64) if want_dA else None
    dB = np.empty(B.nnz, np.float64) if want_dB else None
    rc = lib().orc_spadd_bwd(A.nrows, float(alpha), float(beta), _p(ap), _p(ai), _p(bp), _p(bi), _p(Cp), _p(Ci),
                             _p(g), _p(dA), _p(dB))
    if rc != 0:
        raise ValueError("spadd_bwd: V's pattern misses an entry of A or B")
    return (None if dA is None else _out(dA, dt)), (None if dB is None else _out(dB, dt))


class TriangularError(ValueError):
    pass


def _trsv_rc(rc, what):
    if rc == -2:
        raise TriangularError(f"{what}: stored entry on the wrong side of the diagonal (S:203 shape error)")
    if rc == -3:
        raise TriangularError(f"{what}: missing diagonal with unit_diag = False (S:203 singular)")


def sptrsv(T, b, upper: bool = False, unit: bool = False) -> Result:
    """x = T^{-1} b by forward (lower) or backward (upper) substitution.
    S = M(T)^{-1} |T| |x| (the componentwise error magnitude, DESIGN reading R-TRSV)."""
    assert T.nrows == T.ncols and b.shape == (T.nrows,)
    ip, ix = _pat(T)
    dt = T.values.dtype
    x = np.empty(T.nrows, np.float64)
    S = np.empty(T.nrows, np.float64)
    _trsv_rc(lib().orc_sptrsv(int(upper), int(unit), T.nrows, _p(ip), _p(ix), _p(_f64(T.values)), _p(_f64(b)),
                          _p(x), _p(S)), "sptrsv")
    return Result(_out(x, dt), S)


def sptrsv_bwd(T, x, v, upper: bool = False, unit: bool = False, want_dT: bool = True, want_db: bool = True):
    """VJP of x = T^{-1} b (Table 1): db = T^{-T} v, dT = -db x^T (.) mask(T).
    Returns (dT on T's pattern, Result(db, S))."""
    ip, ix = _pat(T)
    dt = T.values.dtype
    dT = np.empty(T.nnz, np.float64) if want_dT else None
    db = np.empty(T.nrows, np.float64)
    S = np.empty(T.nrows, np.float64)
    _trsv_rc(lib().orc_sptrsv_bwd(int(upper), int(unit), T.nrows, _p(ip), _p(ix), _p(_f64(T.values)), _p(_f64(x)),
                                  _p(_f64(v)), _p(dT), _p(db), _p(S)), "sptrsv_bwd")
    return (None if dT is None else _out(dT, dt)), (Result(_out(db, dt), S) if want_db else None)

