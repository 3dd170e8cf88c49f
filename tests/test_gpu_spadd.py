"""GPU parity for Sp + Sp (PAPER 3.1.4 P:466-476, Table 1)
through the C-ABI against the oracle: union pattern bit-exact, values within the S-scaled
tolerance (bit-exact for integer data), VJP bit-exact (one multiply per entry)."""
import numpy as np
import pytest
import torch

import synth
from test_gpu_parity import RTOL, empty_matrix, skew
from util import assert_S_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def shifted(A, seed, values):
    """Same shape as A, a different random pattern of similar density."""
    d = max(A.nnz / max(A.nrows * A.ncols, 1), 1e-3)
    return synth.random_csr(A.nrows, A.ncols, min(d, 1.0), seed, A.values.dtype, values)


def pairs(dt, values):
    P = synth.poisson2d(40, dtype=dt)
    if values == "int":
        P = P.with_values(synth.int_values(np.random.default_rng(3), P.nnz, dt))
    R1 = synth.random_csr(3001, 2003, 0.004, 11, dt, values, empty_rows=True)
    R2 = synth.random_csr(3001, 2003, 0.003, 12, dt, values)
    S1 = skew(3000, 2500, 5, dt, values)  # long rows: unstaged tiles
    S2 = skew(3000, 900, 6, dt, values)
    PL = synth.powerlaw(1 << 13, seed=41, dtype=dt, values=values)
    return {
        "poisson_self": (P, P),
        "poisson_vs_random": (P, shifted(P, 1, values)),
        "rect_empty_rows": (R1, R2),
        "skew_long_rows": (S1, S2),
        "powerlaw_vs_random": (PL, synth.random_csr(PL.nrows, PL.ncols, 4e-4, 9, dt, values)),
        "one_empty": (R1, empty_matrix(R1.nrows, R1.ncols, dt)),
        "both_empty": (empty_matrix(50, 70, dt), empty_matrix(50, 70, dt)),
    }


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("values", ["real", "int"])
@pytest.mark.parametrize("case", ["poisson_self", "poisson_vs_random", "rect_empty_rows", "skew_long_rows",
                                  "powerlaw_vs_random", "one_empty", "both_empty"])
def test_spadd_parity(ck, orc, case, dt, values):
    A, B = pairs(dt, values)[case]
    alpha, beta = (2.0, -3.0) if values == "int" else (0.625, -1.375)
    Ad, Bd = ck.CSR.from_host(A), ck.CSR.from_host(B)
    Cp, Ci = orc.spadd_symbolic(A, B)
    C = ck.spadd_symbolic(Ad, Bd)
    np.testing.assert_array_equal(C.indptr.cpu().numpy(), Cp)
    np.testing.assert_array_equal(C.indices.cpu().numpy(), Ci)
    r = orc.spadd_numeric(alpha, A, beta, B, Cp, Ci)
    Cv = ck.spadd_numeric(alpha, Ad, beta, Bd, C).cpu().numpy()
    if values == "int":
        np.testing.assert_array_equal(Cv, r.value)
    else:
        assert_S_close(Cv, r.value, r.S, RTOL[dt], "C values")
    dC = synth.dense(len(Ci), 5, dt, values)
    dA_ref, dB_ref = orc.spadd_bwd(alpha, A, beta, B, Cp, Ci, dC)
    dA, dB = ck.spadd_bwd(alpha, Ad, beta, Bd, C, torch.from_numpy(dC).cuda())
    np.testing.assert_array_equal(dA.cpu().numpy(), dA_ref)   # one multiply: bit-exact
    np.testing.assert_array_equal(dB.cpu().numpy(), dB_ref)
    dA_only, _ = ck.spadd_bwd(alpha, Ad, beta, Bd, C, torch.from_numpy(dC).cuda(), need_dB=False)
    np.testing.assert_array_equal(dA_only.cpu().numpy(), dA_ref)


def test_spadd_fig7_A_N(ck):
    """PAPER Fig. 7: sp.eye(N)*2 - sp.eye(N, k=1) - sp.eye(N, k=-1) = A_N (Eq. mat_1d_fd)."""
    from test_oracle_spadd import eye_k
    N = 1000
    I, U, Lo = (ck.CSR.from_host(eye_k(N, k)) for k in (0, 1, -1))
    C1 = ck.spadd_symbolic(I, U)
    C1.values = ck.spadd_numeric(2.0, I, -1.0, U, C1)
    C2 = ck.spadd_symbolic(C1, Lo)
    C2.values = ck.spadd_numeric(1.0, C1, -1.0, Lo, C2)
    A = synth.poisson1d(N)
    np.testing.assert_array_equal(C2.indptr.cpu().numpy(), A.indptr)
    np.testing.assert_array_equal(C2.indices.cpu().numpy(), A.indices)
    np.testing.assert_array_equal(C2.values.cpu().numpy(), A.values)


def test_spadd_rejects_bad_args(ck):
    A = ck.CSR.from_host(synth.poisson2d(8))
    B = ck.CSR.from_host(synth.poisson2d(9))
    with pytest.raises(ck.CsrkError):
        ck.spadd_symbolic(A, B)
