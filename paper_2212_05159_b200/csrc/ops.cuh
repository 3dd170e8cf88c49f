// ops.cuh -- internal entry points behind the C-ABI (abi.cu does validation + dispatch).
#pragma once

#include "csrk_internal.cuh"

namespace csrk {

// A dot product fused into an SpMV (internal): *out = sum_i y_i w_i over the product's rows, from
// per-CTA partials in part[cdiv(nrows, 256)], summed in a fixed order.
struct FusedDot {
    const void *w;
    double *part;
    double *out;
};
// accumulate_y (internal, fp64, not in the ABI): y += op(A) x instead of y = (PCG adjoint sums);
// dot (internal, fp64 op N): the fused dot product of y with dot->w
int spmv_fwd(csrk_dtype dt, csrk_op op, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT,
             const int64_t *perm, const void *x, void *y, Bump &ws, cudaStream_t s, int accumulate_y = 0,
             const FusedDot *dot = nullptr);
// accumulate_dA / accumulate_dx (internal, not in the ABI): dA += the masked gradient, dx += op(A)^T dy
// (fp64 only) instead of overwriting (the PCG's dL and rbar)
int spmv_bwd(csrk_dtype dt, csrk_op op, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT,
             const int64_t *perm, const void *x, const void *dy, void *dA, void *dx, Bump &ws, cudaStream_t s,
             int accumulate_dA = 0, int accumulate_dx = 0);
int spmm_fwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t k, const void *X, int64_t ldx,
             void *Y, int64_t ldy, Bump &ws, cudaStream_t s);
int spmm_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
             int64_t k, const void *X, int64_t ldx, const void *dY, int64_t lddy, void *dA, void *dX, int64_t lddx,
             Bump &ws, cudaStream_t s);
int csr_transpose(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t *AT_indptr, int32_t *AT_indices,
                  void *AT_val, int64_t *perm, Bump &ws, cudaStream_t s);
int spgemm_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *C_indptr, int32_t *C_indices,
                    int64_t *nnzC_host, Bump &ws, cudaStream_t s);
// forget symbolic FILL caches whose workspace lies in [ws, ws + bytes) (another op may overwrite it)
void gemm_fill_cache_invalidate(const void *ws, size_t bytes);
int spgemm_numeric(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern &B,
                   const void *B_val, const csrk_pattern &C, void *C_val, Bump &ws, cudaStream_t s);
// AT/perm (A's transpose plan, nullable): dB by the deterministic gather over A's columns
int spgemm_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
               const csrk_pattern &B, const void *B_val, const csrk_pattern &C, const void *dC, void *dA, void *dB,
               Bump &ws, cudaStream_t s);

int spadd_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *C_indptr, int32_t *C_indices,
                   int64_t *nnzC_host, Bump &ws, cudaStream_t s);
int spadd_numeric(csrk_dtype dt, double alpha, double beta, const csrk_pattern &A, const void *A_val,
                  const csrk_pattern &B, const void *B_val, const csrk_pattern &C, void *C_val, Bump &ws,
                  cudaStream_t s);
int spadd_bwd(csrk_dtype dt, double alpha, double beta, const csrk_pattern &A, const csrk_pattern &B,
              const csrk_pattern &C, const void *dC, void *dA, void *dB, Bump &ws, cudaStream_t s);

int spai_loss_grad(const csrk_pattern &A, const double *Av, const csrk_pattern &M, const double *Mv,
                   const csrk_pattern &C, const csrk_pattern &R, const csrk_pattern &I, double *loss_host,
                   double *dM, Bump &ws, cudaStream_t s);

int sptrsv_fwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int upper, int unit, const void *b, void *x,
               Bump &ws, cudaStream_t s);
int sptrsv_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
               int upper, int unit, const void *x, const void *v, void *dA, void *db, Bump &ws, cudaStream_t s);

int gcn_fwd(csrk_dtype dt, const csrk_pattern &A, const void *Av, int64_t F, const void *Z, int64_t ldz,
            const void *bias, void *Y, int64_t ldy, double *D, Bump &ws, cudaStream_t s);
int gcn_bwd(csrk_dtype dt, const csrk_pattern &A, const void *Av, const csrk_pattern *AT, const int64_t *perm,
            int64_t F, const double *D, const void *dY, int64_t lddy, void *dZ, int64_t lddz, void *dbias, Bump &ws,
            cudaStream_t s);
int dense_gemm_nn(csrk_dtype dt, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *W,
                  int transW, void *Z, int64_t ldz, cudaStream_t s);
int dense_gemm_tn(csrk_dtype dt, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *dZ,
                  int64_t lddz, void *dW, Bump &ws, cudaStream_t s);

// dA[p] = -(w_i x_j) at the stored (i, j) of A (fp64; the masked outer product of the SpTRSV VJP)
int trsv_outer(const csrk_pattern &A, const double *w, const double *x, double *dA, cudaStream_t s);

// comm == nullptr, off == 0: one GPU; else the rank's rows of a row-sharded step (extended vectors)
int pcg_loss_grad(const csrk_comm *comm, int64_t off, const csrk_pattern &A, const double *Av, const csrk_pattern &L,
                  const double *Lv, const double *b, int N, double gamma, int precond, double *loss_host,
                  double *resid_host, double *dL, Bump &ws, cudaStream_t s);

}  // namespace csrk
