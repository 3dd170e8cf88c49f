import os, sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2212_05159_b200 import csrk as ck
A = synth.poisson2d(2048)
Ad = ck.CSR.from_host(A)
for _ in range(3):
    C = ck.spgemm_symbolic(Ad, Ad)
torch.cuda.synchronize()
print("nnzC", C.nnz)
