"""GPU parity of the radix-sort transpose (radix.cu) on small and ragged inputs: the path is
chosen by size (scattered columns, config 4), so a subprocess forces it with
CSRK_TRANSPOSE_RADIX=1 and checks AT_indptr / AT_indices / perm bit-exactly against the oracle's
stable counting sort, values through perm."""
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
import synth, oracle
from paper_2212_05159_b200 import csrk as ck
cases = [synth.random_csr(1, 1, 1.0, 1), synth.random_csr(300, 70000, 0.01, 2), synth.random_csr(5000, 300, 0.05, 3,
         empty_rows=True), synth.powerlaw(1 << 16, seed=5), synth.poisson2d(64), synth.random_csr(40, 1 << 20, 0.001, 6),
         synth.CSR(7, 9, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0))]
for A in cases:
    Ad = ck.CSR.from_host(A)
    plan = ck.csr_transpose(Ad)
    p, i, v, perm = oracle.csr_transpose(A)
    assert np.array_equal(plan.AT.indptr.cpu().numpy(), p), "indptr"
    assert np.array_equal(plan.AT.indices.cpu().numpy(), i), "indices"
    assert np.array_equal(plan.perm.cpu().numpy(), perm), "perm"
    if A.nnz:
        assert np.array_equal(plan.AT.values.cpu().numpy(), v), "values"
print("radix OK", len(cases))
'''


def test_radix_transpose_parity():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CSRK_TRANSPOSE_RADIX="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "radix OK" in r.stdout
