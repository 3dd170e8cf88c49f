"""paper_2212_05159_b200 -- B200 (sm_100a) implementation of the hot path of Nytko et al.,
"Optimized Sparse Matrix Operations for Reverse Mode Automatic Differentiation"
(arXiv 2212.05159): CSR SpMV / SpMM / SpGEMM forward + VJP and csr_transpose, plus Sp + Sp,
SpTRSV, the GCN layer and the PCG / SPAI compositions.

The compute lives in libcsrk.so (csrc/*.cu, C-ABI in include/csrk.h); ``csrk`` is the
ctypes binding, ``dist`` the row-partition + NCCL layer.
"""
from .csrk import (CSR, TransposePlan, CsrkError, csr_transpose, launch_count, lib, spgemm_bwd,  # noqa: F401
                   spgemm_numeric, spgemm_symbolic, spmm_bwd, spmm_fwd, spmv_bwd, spmv_fwd, OP_N, OP_T,
                   spadd_symbolic, spadd_numeric, spadd_bwd, sptrsv_fwd, sptrsv_bwd, gcn_fwd, gcn_bwd,
                   dense_gemm_nn, dense_gemm_tn, gcn_layer_fwd, gcn_layer_bwd, pcg_loss_grad, spai_plan,
                   spai_loss_grad)
