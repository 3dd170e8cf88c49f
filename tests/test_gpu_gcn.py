"""GPU parity for the GCN layer (PAPER 4.4 Eq. gcn_update, Fig. 12
P:905-925) through the C-ABI against the oracle (oracle/gcn.py, the Fig. 12 listing in CPU torch
float64 + autograd): the fused propagation Y = D (A (D Z) + D Z) + bias and D within the S-scaled
tolerance, its VJP dZ = D (A^T (D dY) + D dY) and dbias with and without a transpose plan, the
small dense products, and the whole layer (Y, dX, dTheta, dbias) -- random and power-law graphs
with hubs (> 64 neighbours), widths F in {7, 16, 64, 128}, fp64 and fp32."""
import numpy as np
import pytest
import torch

import synth
from oracle import gcn as ogcn
from util import assert_S_close

pytestmark = pytest.mark.gpu
RTOL = {np.float64: 1e-12, np.float32: 1e-5}


@pytest.fixture(scope="module")
def ck():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05159_b200 import build
    build.build()
    from paper_2212_05159_b200 import csrk
    return csrk


def graphs(dt):
    R = synth.random_csr(300, 300, 0.02, 5, dt)
    R = R.with_values(np.abs(R.values) + dt(0.25))
    return {"random": R,
            "powerlaw": synth.powerlaw_graph(20000, 5.0, 77, weighted=False, dtype=dt),
            "powerlaw_w": synth.powerlaw_graph(6000, 8.0, 78, weighted=True, dtype=dt),
            "empty": synth.CSR(50, 50, np.zeros(51, np.int64), np.zeros(0, np.int32), np.zeros(0, dt))}


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("F", [7, 16, 64, 128])
@pytest.mark.parametrize("case", ["random", "powerlaw", "powerlaw_w", "empty"])
def test_gcn_prop_parity(ck, case, F, dt):
    A = graphs(dt)[case]
    n = A.nrows
    Z = synth.dense((n, F), 11, dt)
    b = synth.dense(F, 12, dt)
    dY = synth.dense((n, F), 13, dt)
    Ad = ck.CSR.from_host(A)
    Y, D = ck.gcn_fwd(Ad, torch.from_numpy(Z).cuda(), torch.from_numpy(b).cuda())
    ref = ogcn.gcn_prop(A, Z, b, want_grad=dY)
    np.testing.assert_allclose(D.cpu().numpy(), ref["D"], rtol=1e-15, atol=0)
    assert_S_close(Y.cpu().numpy(), ref["Y"], ref["S"], RTOL[dt], f"{case} Y")
    for plan in (None, ck.csr_transpose(Ad, with_values=False)):
        dZ, dbias = ck.gcn_bwd(Ad, D, torch.from_numpy(dY).cuda(), plan=plan)
        assert_S_close(dZ.cpu().numpy(), ref["dZ"], ref["S_dZ"], RTOL[dt], f"{case} dZ")
        assert_S_close(dbias.cpu().numpy(), ref["dbias"], ref["S_dbias"], RTOL[dt], f"{case} dbias")


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_dense_gemms(ck, dt):
    n, C, F = 5000, 24, 40
    X, W, dZ = synth.dense((n, C), 1, dt), synth.dense((C, F), 2, dt), synth.dense((n, F), 3, dt)
    t = lambda a: torch.from_numpy(a).cuda()
    X64, W64, dZ64 = X.astype(np.float64), W.astype(np.float64), dZ.astype(np.float64)
    Z = ck.dense_gemm_nn(t(X), t(W)).cpu().numpy()
    assert_S_close(Z, X64 @ W64, np.abs(X64) @ np.abs(W64), RTOL[dt], "X W")
    dX = ck.dense_gemm_nn(t(dZ), t(W), transW=True).cpu().numpy()
    assert_S_close(dX, dZ64 @ W64.T, np.abs(dZ64) @ np.abs(W64.T), RTOL[dt], "dZ W^T")
    dW = ck.dense_gemm_tn(t(X), t(dZ)).cpu().numpy()
    assert_S_close(dW, X64.T @ dZ64, np.abs(X64.T) @ np.abs(dZ64), RTOL[dt], "X^T dZ")


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_gcn_layer(ck, dt):
    """The whole Fig. 12 layer forward + backward against the oracle's autograd of the listing."""
    A = synth.powerlaw_graph(8000, 5.0, 91, dtype=dt)
    n, C, F = A.nrows, 32, 16
    X, W, b, dY = (synth.dense((n, C), 1, dt), synth.dense((C, F), 2, dt), synth.dense(F, 3, dt),
                   synth.dense((n, F), 4, dt))
    t = lambda a: torch.from_numpy(a).cuda()
    Ad = ck.CSR.from_host(A)
    Y, D = ck.gcn_layer_fwd(Ad, t(X), t(W), t(b))
    dX, dW, db = ck.gcn_layer_bwd(Ad, D, t(X), t(W), t(dY))
    ref = ogcn.gcn_layer(A, X, W, b, want_grad=dY)
    # composite S (reading R-GCN): the propagation's magnitude over |X||W| bounds every stage's
    # terms (the GEMM, the rounding of Z = X W to dtype, the propagation); rtol >> u covers the sum
    # of the stages' first-order errors
    P = ogcn.gcn_prop(A, np.abs(X.astype(np.float64)) @ np.abs(W.astype(np.float64)), np.abs(b), want_grad=np.abs(dY))
    assert_S_close(Y.cpu().numpy(), ref["Y"], P["S"], RTOL[dt], "layer Y")
    SdZ = P["S_dZ"]
    assert_S_close(dX.cpu().numpy(), ref["dX"], SdZ @ np.abs(W.astype(np.float64)).T, RTOL[dt], "layer dX")
    assert_S_close(dW.cpu().numpy(), ref["dTheta"], np.abs(X.astype(np.float64)).T @ SdZ, RTOL[dt], "layer dTheta")
    assert_S_close(db.cpu().numpy(), ref["dbias"], P["S_dbias"], RTOL[dt], "layer dbias")


def test_gcn_bench_size(ck):
    """The bench configuration (2^20 nodes, 5 edges per node, hubs up to ~3600, F = 16, fp32):
    forward and backward propagation against the oracle on every node."""
    A = synth.powerlaw_graph(1 << 20, 5.0, 4401, dtype=np.float32)
    n, F = A.nrows, 16
    Z = synth.dense((n, F), 2, np.float32)
    b = synth.dense(F, 3, np.float32)
    dY = synth.dense((n, F), 4, np.float32)
    Ad = ck.CSR.from_host(A)
    Y, D = ck.gcn_fwd(Ad, torch.from_numpy(Z).cuda(), torch.from_numpy(b).cuda())
    dZ, db = ck.gcn_bwd(Ad, D, torch.from_numpy(dY).cuda(), plan=ck.csr_transpose(Ad, with_values=False))
    ref = ogcn.gcn_prop(A, Z, b, want_grad=dY)
    assert_S_close(Y.cpu().numpy(), ref["Y"], ref["S"], RTOL[np.float32], "Y")
    assert_S_close(dZ.cpu().numpy(), ref["dZ"], ref["S_dZ"], RTOL[np.float32], "dZ")
    assert_S_close(db.cpu().numpy(), ref["dbias"], ref["S_dbias"], RTOL[np.float32], "dbias")
