// spai.cu -- SPAI workload (PAPER 4.6): loss and gradient of
//
//     l = || I - M A ||_F^2         over the stored entries of M, pattern(M) fixed
//
// composed from the library's own kernels, in the paper's terms:
//   C  = M A                       spgemm_numeric on the cached pattern C = pattern(M A)
//   R  = 1 I + (-1) C              spadd_numeric on the cached union pattern R = pattern(I) U C
//   l  = sum R_ij^2,  dR = 2 R     k_sumsq_scale + k_sum_final (fixed grid, fixed order)
//   dC = (-1) dR (.) mask(C)       spadd_bwd (Table 1)
//   dM = (dC A^T) (.) mask(M)      spgemm_bwd, left operand only (Table 1)
// fp64 only; deterministic (no atomics on this path: spgemm_bwd without dB is a gather).
#include "ops.cuh"

namespace csrk {

constexpr int kSqTPB = 256;
constexpr int kSqGrid = kNumSMs * 4;

__device__ __forceinline__ double sq_block_sum(double v)
{
    __shared__ double s[kSqTPB / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kSqTPB / 32; ++i) t += s[i];
    return t;
}

__global__ __launch_bounds__(kSqTPB) void k_ones(int64_t n, double *x)
{
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)kSqTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSqTPB) x[i] = 1.0;
}

// part[blk] = sum r_i^2 over the block's grid-stride share;  d_i = 2 r_i
__global__ __launch_bounds__(kSqTPB) void k_sumsq_scale(int64_t n, const double *r, double *d, double *part)
{
    pdl_wait();
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kSqTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSqTPB) {
        const double v = r[i];
        acc = fma(v, v, acc);
        d[i] = 2.0 * v;
    }
    const double t = sq_block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ __launch_bounds__(kSqTPB) void k_sum_final(const double *part, int nb, double *dst)
{
    pdl_wait();
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += kSqTPB) acc += part[i];
    const double t = sq_block_sum(acc);
    if (threadIdx.x == 0) *dst = t;
}

int spai_loss_grad(const csrk_pattern &A, const double *Av, const csrk_pattern &M, const double *Mv,
                   const csrk_pattern &C, const csrk_pattern &R, const csrk_pattern &I, double *loss_host,
                   double *dM, Bump &ws, cudaStream_t s)
{
    const int64_t n = A.nrows;
    double *Iv = ws.take<double>(n > 0 ? n : 1);
    double *Cv = ws.take<double>(C.nnz > 0 ? C.nnz : 1);
    double *Rv = ws.take<double>(R.nnz > 0 ? R.nnz : 1);
    double *dR = ws.take<double>(R.nnz > 0 ? R.nnz : 1);
    double *dC = ws.take<double>(C.nnz > 0 ? C.nnz : 1);
    double *part = ws.take<double>(kSqGrid + 1);
    if (ws.sizing()) {   // the sub-operations carve the rest, in the same order as below
        CSRK_TRY(spgemm_numeric(CSRK_F64, M, Mv, A, Av, C, Cv, ws, s));
        CSRK_TRY(spadd_numeric(CSRK_F64, 1.0, -1.0, I, Iv, C, Cv, R, Rv, ws, s));
        CSRK_TRY(spadd_bwd(CSRK_F64, 1.0, -1.0, I, C, R, dR, nullptr, dC, ws, s));
        return spgemm_bwd(CSRK_F64, M, Mv, nullptr, nullptr, A, Av, C, dC, dM, nullptr, ws, s);
    }
    if (n > 0) CSRK_LAUNCH(k_ones, (unsigned)(cdiv(n, kSqTPB) < kSqGrid ? cdiv(n, kSqTPB) : kSqGrid), kSqTPB, 0, s, n, Iv);
    CSRK_TRY(spgemm_numeric(CSRK_F64, M, Mv, A, Av, C, Cv, ws, s));
    CSRK_TRY(spadd_numeric(CSRK_F64, 1.0, -1.0, I, Iv, C, Cv, R, Rv, ws, s));
    CSRK_LAUNCH(k_sumsq_scale, kSqGrid, kSqTPB, 0, s, R.nnz, Rv, dR, part);
    CSRK_LAUNCH(k_sum_final, 1, kSqTPB, 0, s, part, kSqGrid, part + kSqGrid);
    CSRK_TRY(spadd_bwd(CSRK_F64, 1.0, -1.0, I, C, R, dR, nullptr, dC, ws, s));
    if (M.nnz > 0) CSRK_TRY(spgemm_bwd(CSRK_F64, M, Mv, nullptr, nullptr, A, Av, C, dC, dM, nullptr, ws, s));
    CSRK_CUDA(cudaMemcpyAsync(loss_host, part + kSqGrid, sizeof(double), cudaMemcpyDeviceToHost, s));
    CSRK_CUDA(cudaStreamSynchronize(s));
    return CSRK_OK;
}

}  // namespace csrk
