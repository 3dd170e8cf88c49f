"""CPU-only checks of the C-ABI boundary: libcsrk.so builds for sm_100a, loads, exports every
function include/csrk.h declares, and rejects bad arguments on the host (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "csrk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(csrk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for op in ["spmv_fwd", "spmv_bwd", "spmm_fwd", "spmm_bwd", "spgemm_symbolic", "spgemm_numeric",
               "spgemm_bwd", "csr_transpose"]:
        assert f"csrk_{op}" in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2212_05159_b200 import csrk
    names = declared_functions()
    assert set(names) == set(csrk.ABI_SYMBOLS)
    for n in names:
        assert hasattr(lib, n), n


def test_sass_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2212_05159_b200", "libcsrk.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_argument_checks(lib):
    from paper_2212_05159_b200 import csrk
    P = csrk.Pattern
    assert lib.csrk_version().decode().startswith("csrk")
    assert b"WORKSPACE" in lib.csrk_status_string(-4)
    bad = P(-1, 3, 0, 8, 0)
    assert lib.csrk_spmv_fwd(1, 0, bad, None, None, None, None, None, None, 0, None) == -1
    assert lib.csrk_spmv_fwd(7, 0, P(2, 2, 0, 8, 0), None, None, None, None, None, None, 0, None) == -1
    assert lib.csrk_spmv_fwd(1, 5, P(2, 2, 0, 8, 0), None, None, None, None, None, None, 0, None) == -1
    huge = P(1 << 32, 4, 0, 8, 0)
    assert lib.csrk_spmv_fwd(1, 0, huge, None, None, None, None, None, None, 0, None) == -5
    A, B = P(3, 4, 0, 8, 0), P(5, 2, 0, 8, 0)
    nnz = ctypes.c_int64(0)
    assert lib.csrk_spgemm_symbolic(A, B, 8, None, ctypes.byref(nnz), None, 0, None) == -2
    # transpose plan with the wrong shape
    T = P(3, 3, 0, 8, 0)
    assert lib.csrk_spmv_fwd(1, 1, P(3, 4, 0, 8, 0), None, ctypes.byref(T), 8, None, 8, None, 0, None) == -2
    # workspace sizing is host-only
    n = ctypes.c_size_t(0)
    A = P(1000, 1000, 5000, 8, 8)
    assert lib.csrk_workspace_size(4, 1, ctypes.byref(A), None, 0, 0, ctypes.byref(n)) == 0 and n.value > 0
    assert lib.csrk_workspace_size(0, 1, ctypes.byref(A), None, 0, 0, ctypes.byref(n)) == 0 and n.value > 0
    # a too-small workspace is rejected on the host before any launch
    assert lib.csrk_spmv_fwd(1, 0, A, 8, None, None, 8, 8, None, 0, None) == -4
    assert lib.csrk_workspace_size(5, 1, ctypes.byref(A), ctypes.byref(A), 0, 0, ctypes.byref(n)) == 0 and n.value > 0
    # SpGEMM backward with a transpose plan: the plan must be A^T's shape, plan and perm together;
    # the plan path needs no dB scratch (its workspace is not larger than the atomic path's)
    S = P(4, 4, 6, 8, 8)
    bad_T = P(4, 5, 6, 8, 8)
    assert lib.csrk_spgemm_bwd_plan(1, S, 8, ctypes.byref(bad_T), 8, S, 8, S, 8, 8, 8, None, 0, None) == -2
    good_T = P(4, 4, 6, 8, 8)
    assert lib.csrk_spgemm_bwd_plan(1, S, 8, ctypes.byref(good_T), None, S, 8, S, 8, 8, 8, None, 0, None) == -1
    assert lib.csrk_spgemm_bwd_plan(1, S, 8, None, None, P(5, 4, 6, 8, 8), 8, S, 8, 8, 8, None, 0, None) == -2
    n_plain, n_plan = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.csrk_workspace_size(7, 0, ctypes.byref(A), ctypes.byref(A), 0, 0, ctypes.byref(n_plain)) == 0
    assert lib.csrk_workspace_size(7, 0, ctypes.byref(A), ctypes.byref(A), 0, 1, ctypes.byref(n_plan)) == 0
    assert 0 < n_plan.value <= n_plain.value + (1 << 20)
    assert lib.csrk_launch_count() == 0


def test_host_side_argument_checks_f_rows(lib):
    """Sp+Sp / SpTRSV / GCN entry points reject bad shapes and arguments on the host."""
    from paper_2212_05159_b200 import csrk
    P = csrk.Pattern
    nnz = ctypes.c_int64(0)
    # Sp + Sp: shapes must match
    assert lib.csrk_spadd_symbolic(P(3, 4, 0, 8, 0), P(3, 5, 0, 8, 0), 8, None, ctypes.byref(nnz), None, 0,
                                   None) == -2
    # SpTRSV: square only, b / x required
    assert lib.csrk_sptrsv_fwd(1, P(3, 4, 0, 8, 0), None, 0, 0, 8, 8, None, 0, None) == -2
    assert lib.csrk_sptrsv_fwd(1, P(3, 3, 3, 8, 8), 8, 0, 0, None, 8, None, 0, None) == -1
    # SpTRSV backward: nothing requested -> no-op
    assert lib.csrk_sptrsv_bwd(1, P(3, 3, 3, 8, 8), 8, None, None, 0, 0, 8, 8, None, None, None, 0, None) == 0
    # GCN: width 1..128, ld >= F
    assert lib.csrk_gcn_fwd(1, P(3, 3, 0, 8, 0), None, 0, 8, 0, None, 8, 0, 8, None, 0, None) == -1
    assert lib.csrk_gcn_fwd(1, P(3, 3, 0, 8, 0), None, 129, 8, 129, None, 8, 129, 8, None, 0, None) == -1
    assert lib.csrk_gcn_fwd(1, P(3, 3, 0, 8, 0), None, 16, 8, 8, None, 8, 16, 8, None, 0, None) == -1
    assert lib.csrk_gcn_fwd(1, P(3, 4, 0, 8, 0), None, 16, 8, 16, None, 8, 16, 8, None, 0, None) == -2
    # dense products: leading dimensions, shared-memory limits
    assert lib.csrk_dense_gemm_nn(1, 10, 4, 8, 8, 3, 8, 0, 8, 8, None) == -1
    assert lib.csrk_dense_gemm_tn(1, 10, 300, 16, 8, 300, 8, 16, 8, None, 0, None) == -1
    # workspace sizing of the f-row ops is host-only and positive
    n = ctypes.c_size_t(0)
    A = P(1000, 1000, 5000, 8, 8)
    for op, k, plan in ((11, 0, 0), (12, 0, 0), (12, 0, 1), (13, 16, 0), (14, 16, 0), (14, 16, 1)):
        assert lib.csrk_workspace_size(op, 1, ctypes.byref(A), None, k, plan, ctypes.byref(n)) == 0, op
        assert n.value > 0, op
    assert lib.csrk_launch_count() == 0


def build_abi_demo(lib, out="/tmp/csrk_abi_demo"):
    """Compile tests/abi_demo.c as plain C99 against include/csrk.h and link libcsrk.so + cudart."""
    import subprocess
    libdir = os.path.join(ROOT, "paper_2212_05159_b200")
    cuda = "/usr/local/cuda"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O1", os.path.join(ROOT, "tests", "abi_demo.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           "-L", libdir, "-lcsrk", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_header_is_plain_c_and_links(lib):
    """include/csrk.h is a C header: a C99 program (tests/abi_demo.c) compiles with -Wall -Werror
    and links against libcsrk.so (run on the GPU by tests/test_gpu_validate.py)."""
    assert os.path.exists(build_abi_demo(lib))
