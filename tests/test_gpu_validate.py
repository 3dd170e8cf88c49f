"""CSRK_VALIDATE=1 (the opt-in structural checks of include/csrk.h): non-canonical CSR is
rejected with CSRK_ERR_PATTERN before any launch, and the triangular solve rejects entries on
the wrong side of the diagonal and missing diagonals; canonical inputs pass.  The
flag is read once per process, so the checks run in a subprocess."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import synth
from paper_2212_05159_b200 import csrk as ck

def expect_pattern_error(fn):
    try:
        fn()
    except ck.CsrkError as e:
        assert "PATTERN" in str(e), e
        return
    raise AssertionError("expected CSRK_ERR_PATTERN")

# unsorted column indices in a row
bad = synth.CSR(2, 3, np.array([0, 2, 3], np.int64), np.array([2, 0, 1], np.int32), np.ones(3))
expect_pattern_error(lambda: ck.spmv_fwd(ck.CSR.from_host(bad), torch.ones(3, dtype=torch.float64, device="cuda")))
# column out of range
bad = synth.CSR(2, 3, np.array([0, 1, 2], np.int64), np.array([0, 3], np.int32), np.ones(2))
expect_pattern_error(lambda: ck.spmv_fwd(ck.CSR.from_host(bad), torch.ones(3, dtype=torch.float64, device="cuda")))
b = torch.ones(3, dtype=torch.float64, device="cuda")
# wrong side of the diagonal (lower solve with an upper entry)
up = synth.CSR(3, 3, np.array([0, 2, 3, 4], np.int64), np.array([0, 2, 1, 2], np.int32), np.ones(4))
expect_pattern_error(lambda: ck.sptrsv_fwd(ck.CSR.from_host(up), b))
# missing diagonal without unit_diag; accepted with unit_diag
nod = synth.CSR(3, 3, np.array([0, 1, 2, 3], np.int64), np.array([0, 0, 2], np.int32), np.ones(3))
expect_pattern_error(lambda: ck.sptrsv_fwd(ck.CSR.from_host(nod), b))
ck.sptrsv_fwd(ck.CSR.from_host(nod), b, unit=True)
# canonical inputs pass
A = synth.poisson2d(8)
ck.spmv_fwd(ck.CSR.from_host(A), torch.ones(64, dtype=torch.float64, device="cuda"))
ck.sptrsv_fwd(ck.CSR.from_host(synth.lower_part(A)), torch.ones(64, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("validate OK")
'''


def test_validate_mode():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CSRK_VALIDATE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "validate OK" in r.stdout


def test_abi_demo_plain_c_program():
    """tests/abi_demo.c -- a C99 program that uses only include/csrk.h and the CUDA runtime (no
    Python on the compute path) -- runs SpMV and the two-call SpGEMM on the GPU and checks the
    closed forms of PAPER Eq. mat_1d_fd (A 1 = e_0 + e_{N-1}; A^2 = tridiag^2 stencil)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_abi_cpu import build_abi_demo
    from paper_2212_05159_b200 import build, csrk
    build.build()
    exe = build_abi_demo(csrk.lib(), out=os.path.join("/tmp", f"csrk_abi_demo_{os.getpid()}"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "abi_demo OK" in r.stdout, (r.stdout, r.stderr)
