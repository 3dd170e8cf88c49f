import sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2212_05159_b200 import csrk as ck
A = ck.CSR.from_host(synth.poisson2d(2048))
for _ in range(3):
    p = ck.csr_transpose(A, with_values=False)
torch.cuda.synchronize()
