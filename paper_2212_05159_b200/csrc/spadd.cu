// spadd.cu -- Sp + Sp: C = alpha A + beta B and its VJP (PAPER 3.1.4, P:466-476;
// Table 1).
//
// mask(C) = mask(A) U mask(B) -- "the computation of C is viewed as a union over the rows of
// A and B ... implemented in parallel over each row".  The backward pass is "the
// row-wise reduction from V to the sparsity mask of A or B": walking the same
// union, every stored entry of A (B) picks V at its position in C and scales it by alpha
// (beta) -- one multiply, no accumulation.
//
// Kernel: a CTA owns kATile consecutive rows, one thread per row.  The tile's segments of A,
// B (and C for the value phases) are contiguous in memory, so they are staged in shared
// memory with coalesced loads; each thread merges its two sorted column lists from shared
// memory; outputs are staged and written back coalesced.  Tiles whose segments exceed the
// staging capacity run the same merge directly on global memory.
#include "ops.cuh"

namespace csrk {

constexpr int kATile = 128;   // rows (= threads) per CTA
constexpr int kACapAB = 1024; // staged entries of A and of B per tile
constexpr int kACapC = 2048;  // staged entries of C per tile

enum { AD_COUNT = 0, AD_FILL = 1, AD_NUM = 2, AD_BWD = 3 };

template <typename T>
struct AddArgs {
    int64_t m;
    double alpha, beta;
    const int64_t *Ap; const int32_t *Ai; const T *Av;
    const int64_t *Bp; const int32_t *Bi; const T *Bv;
    int64_t *Cp; int32_t *Ci; T *Cv; const T *dC;
    T *dA; T *dB;
};

// Merge of row lists a[0..la) and b[0..lb) (sorted, unique) in union order.  Pointers are
// generic (shared or global).  Returns the union length.
template <typename T, int PH>
__device__ __forceinline__ int add_merge(const AddArgs<T> &g, const int32_t *ai, int la, const int32_t *bi, int lb,
                                         const T *av, const T *bv, int32_t *ci, T *cv, const T *dc, T *da, T *db)
{
    int a = 0, b = 0, c = 0;
    while (a < la || b < lb) {
        const int32_t ja = a < la ? ai[a] : INT32_MAX, jb = b < lb ? bi[b] : INT32_MAX;
        const bool ta = ja <= jb, tb = jb <= ja;
        if (PH == AD_FILL) ci[c] = ta ? ja : jb;
        if (PH == AD_NUM) {
            const double x = ta ? (double)av[a] : 0.0, y = tb ? (double)bv[b] : 0.0;
            cv[c] = (T)fma(g.alpha, x, g.beta * y);
        }
        if (PH == AD_BWD) {
            const double v = (double)dc[c];
            if (ta && da) da[a] = (T)(g.alpha * v);
            if (tb && db) db[b] = (T)(g.beta * v);
        }
        a += ta;
        b += tb;
        ++c;
    }
    return c;
}

template <typename T, int PH>
__global__ __launch_bounds__(kATile) void k_spadd(AddArgs<T> g)
{
    pdl_wait();
    __shared__ int64_t s_ap[kATile + 1], s_bp[kATile + 1], s_cp[kATile + 1];
    __shared__ int32_t s_ai[kACapAB], s_bi[kACapAB];
    constexpr bool VAL = PH == AD_NUM || PH == AD_BWD;
    // NUM: A / B values in, C values out.  BWD: dC in, dA / dB out (same buffers).
    __shared__ T s_av[VAL ? kACapAB : 1], s_bv[VAL ? kACapAB : 1];
    __shared__ T s_cv[VAL ? kACapC : 1];
    __shared__ int32_t s_ci[PH == AD_FILL ? kACapC : 1];

    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kATile;
    const int nr = (int)(g.m - r0 < kATile ? g.m - r0 : kATile);
    for (int i = tid; i <= nr; i += kATile) {
        s_ap[i] = g.Ap[r0 + i];
        s_bp[i] = g.Bp[r0 + i];
        if (PH != AD_COUNT) s_cp[i] = g.Cp[r0 + i];
    }
    __syncthreads();
    const int64_t a0 = s_ap[0], b0 = s_bp[0], c0 = PH != AD_COUNT ? s_cp[0] : 0;
    const int64_t tA = s_ap[nr] - a0, tB = s_bp[nr] - b0, tC = PH != AD_COUNT ? s_cp[nr] - c0 : 0;
    const bool staged = tA <= kACapAB && tB <= kACapAB && tC <= kACapC;   // tile-uniform
    if (staged) {
        for (int e = tid; e < (int)tA; e += kATile) {
            s_ai[e] = g.Ai[a0 + e];
            if (PH == AD_NUM) s_av[e] = g.Av[a0 + e];
        }
        for (int e = tid; e < (int)tB; e += kATile) {
            s_bi[e] = g.Bi[b0 + e];
            if (PH == AD_NUM) s_bv[e] = g.Bv[b0 + e];
        }
        if (PH == AD_BWD)
            for (int e = tid; e < (int)tC; e += kATile) s_cv[e] = g.dC[c0 + e];
        __syncthreads();
    }
    if (tid < nr) {
        const int64_t pa = s_ap[tid], pb = s_bp[tid];
        const int la = (int)(s_ap[tid + 1] - pa), lb = (int)(s_bp[tid + 1] - pb);
        const int64_t pc = PH != AD_COUNT ? s_cp[tid] : 0;
        int cnt;
        if (staged) {
            const int oa = (int)(pa - a0), ob = (int)(pb - b0), oc = (int)(pc - c0);
            cnt = add_merge<T, PH>(g, s_ai + oa, la, s_bi + ob, lb, s_av + oa, s_bv + ob, s_ci + oc, s_cv + oc,
                                   s_cv + oc, s_av + oa, s_bv + ob);
        } else {
            cnt = add_merge<T, PH>(g, g.Ai + pa, la, g.Bi + pb, lb, g.Av ? g.Av + pa : nullptr,
                                   g.Bv ? g.Bv + pb : nullptr, g.Ci ? g.Ci + pc : nullptr, g.Cv ? g.Cv + pc : nullptr,
                                   g.dC ? g.dC + pc : nullptr, g.dA ? g.dA + pa : nullptr, g.dB ? g.dB + pb : nullptr);
        }
        if (PH == AD_COUNT) g.Cp[r0 + tid + 1] = cnt;
    }
    if (staged && PH != AD_COUNT) {
        __syncthreads();
        if (PH == AD_FILL)
            for (int e = tid; e < (int)tC; e += kATile) g.Ci[c0 + e] = s_ci[e];
        if (PH == AD_NUM)
            for (int e = tid; e < (int)tC; e += kATile) g.Cv[c0 + e] = s_cv[e];
        if (PH == AD_BWD) {
            if (g.dA)
                for (int e = tid; e < (int)tA; e += kATile) g.dA[a0 + e] = s_av[e];
            if (g.dB)
                for (int e = tid; e < (int)tB; e += kATile) g.dB[b0 + e] = s_bv[e];
        }
    }
}

template <typename T, int PH>
static int launch_spadd(const AddArgs<T> &g, cudaStream_t s)
{
    if (g.m <= 0) return CSRK_OK;
    CSRK_LAUNCH((k_spadd<T, PH>), (unsigned)cdiv(g.m, kATile), kATile, 0, s, g);
    return CSRK_OK;
}

int spadd_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *Cp, int32_t *Ci, int64_t *nnzC_host,
                   Bump &ws, cudaStream_t s)
{
    if (ws.sizing()) return scan_counts_i64(nullptr, A.nrows, ws, s);
    AddArgs<double> g{};
    g.m = A.nrows;
    g.Ap = A.indptr; g.Ai = A.indices; g.Bp = B.indptr; g.Bi = B.indices;
    g.Cp = Cp; g.Ci = Ci;
    if (!Ci) {
        CSRK_CUDA(cudaMemsetAsync(Cp, 0, sizeof(int64_t), s));
        CSRK_TRY((launch_spadd<double, AD_COUNT>(g, s)));
        CSRK_TRY(scan_counts_i64(Cp, A.nrows, ws, s));
        CSRK_CUDA(cudaMemcpyAsync(nnzC_host, Cp + A.nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSRK_CUDA(cudaStreamSynchronize(s));
        return CSRK_OK;
    }
    return launch_spadd<double, AD_FILL>(g, s);
}

template <typename T>
static int spadd_values_t(int PH, double alpha, double beta, const csrk_pattern &A, const T *Av,
                          const csrk_pattern &B, const T *Bv, const csrk_pattern &C, T *Cv, const T *dC, T *dA, T *dB,
                          cudaStream_t s)
{
    AddArgs<T> g{};
    g.m = A.nrows; g.alpha = alpha; g.beta = beta;
    g.Ap = A.indptr; g.Ai = A.indices; g.Av = Av;
    g.Bp = B.indptr; g.Bi = B.indices; g.Bv = Bv;
    g.Cp = const_cast<int64_t *>(C.indptr); g.Ci = const_cast<int32_t *>(C.indices); g.Cv = Cv; g.dC = dC;
    g.dA = dA; g.dB = dB;
    if (PH == AD_NUM) return launch_spadd<T, AD_NUM>(g, s);
    return launch_spadd<T, AD_BWD>(g, s);
}

int spadd_numeric(csrk_dtype dt, double alpha, double beta, const csrk_pattern &A, const void *Av,
                  const csrk_pattern &B, const void *Bv, const csrk_pattern &C, void *Cv, Bump &ws, cudaStream_t s)
{
    if (ws.sizing()) return CSRK_OK;
    if (dt == CSRK_F64)
        return spadd_values_t<double>(AD_NUM, alpha, beta, A, (const double *)Av, B, (const double *)Bv, C,
                                      (double *)Cv, nullptr, nullptr, nullptr, s);
    return spadd_values_t<float>(AD_NUM, alpha, beta, A, (const float *)Av, B, (const float *)Bv, C, (float *)Cv,
                                 nullptr, nullptr, nullptr, s);
}

int spadd_bwd(csrk_dtype dt, double alpha, double beta, const csrk_pattern &A, const csrk_pattern &B,
              const csrk_pattern &C, const void *dC, void *dA, void *dB, Bump &ws, cudaStream_t s)
{
    if (ws.sizing()) return CSRK_OK;
    if (dt == CSRK_F64)
        return spadd_values_t<double>(AD_BWD, alpha, beta, A, nullptr, B, nullptr, C, nullptr, (const double *)dC,
                                      (double *)dA, (double *)dB, s);
    return spadd_values_t<float>(AD_BWD, alpha, beta, A, nullptr, B, nullptr, C, nullptr, (const float *)dC,
                                 (float *)dA, (float *)dB, s);
}

}  // namespace csrk
