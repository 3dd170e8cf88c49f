"""fp32 data accumulates in fp64 (DESIGN reading A5; include/csrk.h "Values").

Adversarial fp32 cases, one per atomic accumulation site of the library, each summing
m = 2^24 + 2^22 terms equal to 1 into ONE output: the exact sum m = 20,971,520 is representable
in fp32, but an fp32 accumulator stalls at 2^24 (2^24 + 1 rounds back to 2^24), so an fp32
atomic sum would be off by 4,194,304 = 0.2 m -- far outside 1e-5 S (S = m).  Sites:
  * spmv_bwd dx = A^T dy without a plan (fp64 atomic scatter; rows.cuh / tile.cuh),
  * spmv_fwd op T without a plan (the same scatter),
  * spgemm_bwd dB over the short-row path (k_gemm_S),
  * spgemm_numeric C of a big row (one row of m entries: k_gemm_big_win, one window),
  * spgemm_bwd dA of a big row spanning m / 4096 windows (fp64 target + single rounding).
The oracle (long double) gives m exactly; the S-rule of reading A6 is asserted."""
import numpy as np
import pytest
import torch

import synth
from util import assert_S_close

pytestmark = pytest.mark.gpu

M = (1 << 24) + (1 << 22)
RTOL32 = 1e-5


@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def column_of_ones(m):
    """m x 1, every row one entry (column 0) of value 1."""
    return synth.CSR(m, 1, np.arange(m + 1, dtype=np.int64), np.zeros(m, np.int32), np.ones(m, np.float32))


def row_of_ones(m):
    """1 x m, one row with all m columns, value 1."""
    return synth.CSR(1, m, np.array([0, m], np.int64), np.arange(m, dtype=np.int32), np.ones(m, np.float32))


def test_spmv_scatter_fp32_accumulates_in_fp64(ck, orc):
    A = column_of_ones(M)
    Ad = ck.CSR.from_host(A)
    dy = np.ones(M, np.float32)
    x = np.ones(1, np.float32)
    _, dx = ck.spmv_bwd(Ad, torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda())
    _, ref = orc.spmv_bwd(A, x, dy)
    assert ref.value[0] == M
    assert_S_close(dx.cpu().numpy(), ref.value, ref.S, RTOL32, "spmv_bwd dx (atomic)")
    y = ck.spmv_fwd(Ad, torch.from_numpy(dy).cuda(), op=ck.OP_T)
    r = orc.spmv_fwd(A, dy, op=1)
    assert_S_close(y.cpu().numpy(), r.value, r.S, RTOL32, "spmv_fwd op T (atomic)")
    # the deterministic plan path (fp64 register sum over the 2^24 + 2^22-entry row of A^T)
    _, dxp = ck.spmv_bwd(Ad, torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda(), plan=ck.csr_transpose(Ad))
    assert_S_close(dxp.cpu().numpy(), ref.value, ref.S, RTOL32, "spmv_bwd dx (plan)")


def test_spgemm_dB_fp32_accumulates_in_fp64(ck, orc):
    """C = A B, A = m x 1 ones, B = [1]: dB_00 = sum_i A_i0 dC_i0 = m (short rows, k_gemm_S)."""
    A = column_of_ones(M)
    B = synth.CSR(1, 1, np.array([0, 1], np.int64), np.zeros(1, np.int32), np.ones(1, np.float32))
    Ad, Bd = ck.CSR.from_host(A), ck.CSR.from_host(B)
    C = ck.spgemm_symbolic(Ad, Bd)
    Cp, Ci = orc.spgemm_symbolic(A, B)
    assert np.array_equal(C.indptr.cpu().numpy(), Cp) and np.array_equal(C.indices.cpu().numpy(), Ci)
    dC = np.ones(len(Ci), np.float32)
    dA, dB = ck.spgemm_bwd(Ad, Bd, C, torch.from_numpy(dC).cuda())
    rA, rB = orc.spgemm_bwd(A, B, Cp, Ci, dC)
    assert rB.value[0] == M
    assert_S_close(dB.cpu().numpy(), rB.value, rB.S, RTOL32, "spgemm dB")
    assert_S_close(dA.cpu().numpy(), rA.value, rA.S, RTOL32, "spgemm dA")


def test_spgemm_big_row_numeric_fp32_accumulates_in_fp64(ck, orc):
    """C = A B, A = 1 x m ones, B = m x 1 ones: C_00 = m (one big row, k_gemm_big_win)."""
    A, B = row_of_ones(M), column_of_ones(M)
    Ad, Bd = ck.CSR.from_host(A), ck.CSR.from_host(B)
    C = ck.spgemm_symbolic(Ad, Bd)
    Cp, Ci = orc.spgemm_symbolic(A, B)
    assert np.array_equal(C.indices.cpu().numpy(), Ci)
    Cv = ck.spgemm_numeric(Ad, Bd, C)
    r = orc.spgemm_numeric(A, B, Cp, Ci)
    assert r.value[0] == M
    assert_S_close(Cv.cpu().numpy(), r.value, r.S, RTOL32, "spgemm C (big row)")


def test_spgemm_big_row_multiwindow_dA_fp32_accumulates_in_fp64(ck, orc):
    """C = A B, A = [1] (1 x 1), B = 1 x m ones, dC = ones: dA_00 = sum_j dC_0j B_0j = m, the row
    of C spans m / 4096 windows (fp64 dA target, one rounding)."""
    A = synth.CSR(1, 1, np.array([0, 1], np.int64), np.zeros(1, np.int32), np.ones(1, np.float32))
    B = row_of_ones(M)
    Ad, Bd = ck.CSR.from_host(A), ck.CSR.from_host(B)
    C = ck.spgemm_symbolic(Ad, Bd)
    Cp, Ci = orc.spgemm_symbolic(A, B)
    assert np.array_equal(C.indptr.cpu().numpy(), Cp)
    dC = np.ones(len(Ci), np.float32)
    dA, dB = ck.spgemm_bwd(Ad, Bd, C, torch.from_numpy(dC).cuda())
    rA, rB = orc.spgemm_bwd(A, B, Cp, Ci, dC)
    assert rA.value[0] == M
    assert_S_close(dA.cpu().numpy(), rA.value, rA.S, RTOL32, "spgemm dA (multi-window)")
    assert_S_close(dB.cpu().numpy(), rB.value, rB.S, RTOL32, "spgemm dB")
