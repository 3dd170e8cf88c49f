// spgemm.cu -- SpGEMM C = A B: symbolic, numeric and backward
// (PAPER 3.1.2; Table 1; Fig. 3).
//
// Rows of A are binned by l_i = row length and w_i = sum_{k in row i} len_B(k) (the
// product count, "estimated work"):
//   S  (l_i <= 8, w_i <= 512): one THREAD per row runs an l_i-way merge of the sorted
//      B rows.  The merge emits C's columns in ascending order, so symbolic needs no
//      sort, numeric sums each C_ij over k ascending (deterministic, the oracle's order)
//      and the backward pass meets dC_ij in C's storage order without any search.
//   M  (w_i <= 8192): one CTA per row; products gathered to shared memory.  Symbolic:
//      bitonic sort + unique.  Numeric/backward: binary search of each product's column
//      in the C row (shared memory) -- numeric accumulates with shared-memory atomics.
//   L  (w_i > 8192): one CTA per row; symbolic uses shared-memory bitmap windows over the
//      column range (sorted output for free); numeric/backward search the C row in global
//      memory and accumulate with global atomics.
// Rows with w_i = 0 ("E") produce empty C rows and zero dA.
// The backward pass computes dA_ik = sum_j dC_ij B_kj per A entry (deterministic) and
// scatters dB_kj += A_ik dC_ij with global atomic adds (reading A9).
#include "ops.cuh"

namespace csrk {

constexpr int kSMaxL = 8;
constexpr int64_t kSMaxW = 512;
constexpr int kMMaxW = 8192;
constexpr int kGemmTPB = 256;
constexpr int kBitmapWords = 24576;  // 96 KB -> windows of 786,432 columns

enum : uint8_t { BIN_E = 0, BIN_S = 1, BIN_M = 2, BIN_L = 3 };
enum { PH_COUNT = 0, PH_FILL = 1, PH_NUM = 2, PH_BWD = 3 };

struct Bins {
    uint8_t *bin;
    int32_t *listM, *listL;
    int *cnt;  // [2]
};

// ---------------------------------------------------------------- binning (8 lanes per row)
__global__ __launch_bounds__(256) void k_gemm_bin(int64_t m, const int64_t *__restrict__ Ap,
                                                  const int32_t *__restrict__ Ai, const int64_t *__restrict__ Bp,
                                                  Bins b)
{
    constexpr int G = 8;
    const int lane = threadIdx.x & (G - 1);
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    if (i >= m) return;
    const unsigned gmask = 0xffu << ((threadIdx.x & 31) & ~(G - 1));
    const int64_t s = Ap[i], e = Ap[i + 1];
    int64_t w = 0;
    for (int64_t p = s + lane; p < e; p += G) {
        const int32_t k = Ai[p];
        w += Bp[k + 1] - Bp[k];
    }
    for (int o = G >> 1; o > 0; o >>= 1) w += __shfl_xor_sync(gmask, w, o, G);
    if (lane == 0) {
        const int64_t l = e - s;
        uint8_t bin = w == 0 ? BIN_E : ((l <= kSMaxL && w <= kSMaxW) ? BIN_S : (w <= kMMaxW ? BIN_M : BIN_L));
        b.bin[i] = bin;
        if (bin == BIN_M) b.listM[atomicAdd(&b.cnt[0], 1)] = (int32_t)i;
        if (bin == BIN_L) b.listL[atomicAdd(&b.cnt[1], 1)] = (int32_t)i;
    }
}

// ---------------------------------------------------------------- S rows: thread-per-row merge
template <typename T, int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_S(int64_t m, const uint8_t *__restrict__ bin,
                                                     const int64_t *__restrict__ Ap, const int32_t *__restrict__ Ai,
                                                     const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                                     const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                     int64_t *__restrict__ Cp, int32_t *__restrict__ Ci,
                                                     T *__restrict__ Cv, const T *__restrict__ dC, T *__restrict__ dA,
                                                     T *__restrict__ dB)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint8_t bn = bin[i];
    const int64_t as = Ap[i];
    if (bn == BIN_E) {
        if (PH == PH_COUNT) Cp[i + 1] = 0;
        if (PH == PH_BWD && dA)
            for (int64_t p = as; p < Ap[i + 1]; ++p) dA[p] = (T)0;
        return;
    }
    if (bn != BIN_S) return;
    const int l = (int)(Ap[i + 1] - as);
    int64_t cur[kSMaxL], end[kSMaxL];
    int32_t head[kSMaxL];
    double av[kSMaxL], dacc[kSMaxL];
#pragma unroll
    for (int t = 0; t < kSMaxL; ++t) {
        head[t] = INT32_MAX;
        cur[t] = end[t] = 0;
        av[t] = dacc[t] = 0.0;
        if (t < l) {
            const int32_t k = Ai[as + t];
            cur[t] = Bp[k];
            end[t] = Bp[k + 1];
            if (cur[t] < end[t]) head[t] = Bi[cur[t]];
            if (PH == PH_NUM || PH == PH_BWD) av[t] = (double)Av[as + t];
        }
    }
    int64_t c = PH == PH_COUNT ? 0 : Cp[i];
    while (true) {
        int32_t v = INT32_MAX;
#pragma unroll
        for (int t = 0; t < kSMaxL; ++t) v = head[t] < v ? head[t] : v;
        if (v == INT32_MAX) break;
        double acc = 0.0;
        const double g = PH == PH_BWD ? (double)dC[c] : 0.0;
#pragma unroll
        for (int t = 0; t < kSMaxL; ++t) {
            if (head[t] == v) {
                if (PH == PH_NUM) acc = fma(av[t], (double)Bv[cur[t]], acc);
                if (PH == PH_BWD) {
                    dacc[t] = fma(g, (double)Bv[cur[t]], dacc[t]);
                    if (dB) red_add(&dB[cur[t]], (T)(av[t] * g));
                }
                ++cur[t];
                head[t] = cur[t] < end[t] ? Bi[cur[t]] : INT32_MAX;
            }
        }
        if (PH == PH_FILL) Ci[c] = v;
        if (PH == PH_NUM) Cv[c] = (T)acc;
        ++c;
    }
    if (PH == PH_COUNT) Cp[i + 1] = c;
    if (PH == PH_BWD && dA) {
#pragma unroll
        for (int t = 0; t < kSMaxL; ++t)
            if (t < l) dA[as + t] = (T)dacc[t];
    }
}

// ---------------------------------------------------------------- block helpers
__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t *s_red)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    int64_t t = 0;
    for (int i = 0; i < kGemmTPB / 32; ++i) t += s_red[i];
    __syncthreads();
    return t;
}

// exclusive scan over the block (kGemmTPB threads); returns prefix, total via ref
__device__ __forceinline__ int64_t block_excl_scan_i64(int64_t v, int64_t *s_red, int64_t &total)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    __syncthreads();
    if (lane == 31) s_red[w] = x;
    __syncthreads();
    int64_t off = 0;
    total = 0;
    for (int i = 0; i < kGemmTPB / 32; ++i) {
        if (i < w) off += s_red[i];
        total += s_red[i];
    }
    __syncthreads();
    return off + x - v;
}

__device__ __forceinline__ int pow2ceil_i(int x)
{
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

__device__ __forceinline__ void bitonic_keys(int32_t *key, int P)
{
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += kGemmTPB) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool asc = (i & k) == 0;
                    const int32_t a = key[i], b = key[ixj];
                    if ((a > b) == asc) { key[i] = b; key[ixj] = a; }
                }
            }
            __syncthreads();
        }
}

// lower_bound of v in sorted c[0..n)
__device__ __forceinline__ int64_t lbound(const int32_t *c, int64_t n, int32_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (c[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- M rows: symbolic
template <int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_M_sym(const int32_t *__restrict__ list, const int *__restrict__ cnt,
                                                         const int64_t *__restrict__ Ap, const int32_t *__restrict__ Ai,
                                                         const int64_t *__restrict__ Bp, const int32_t *__restrict__ Bi,
                                                         int64_t *__restrict__ Cp, int32_t *__restrict__ Ci)
{
    __shared__ int32_t s_key[kMMaxW];
    __shared__ int s_cnt;
    __shared__ int64_t s_red[kGemmTPB / 32];
    const int nrows = *cnt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = blockIdx.x; it < nrows; it += gridDim.x) {
        const int64_t i = list[it];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int64_t a = as + warp; a < ae; a += kGemmTPB / 32) {
            const int32_t k = Ai[a];
            const int64_t bs = Bp[k];
            const int bl = (int)(Bp[k + 1] - bs);
            int base = 0;
            if (lane == 0 && bl > 0) base = atomicAdd(&s_cnt, bl);
            base = __shfl_sync(0xffffffffu, base, 0);
            for (int j = lane; j < bl; j += 32) s_key[base + j] = Bi[bs + j];
        }
        __syncthreads();
        const int w = s_cnt;
        const int P = pow2ceil_i(w);
        for (int e = w + threadIdx.x; e < P; e += kGemmTPB) s_key[e] = INT32_MAX;
        __syncthreads();
        bitonic_keys(s_key, P);
        // thread-contiguous chunks of the sorted keys
        const int per = (P + kGemmTPB - 1) / kGemmTPB;
        const int e0 = threadIdx.x * per;
        int64_t mine = 0;
        for (int e = e0; e < e0 + per && e < w; ++e) mine += (e == 0 || s_key[e] != s_key[e - 1]);
        if (PH == PH_COUNT) {
            const int64_t tot = block_sum_i64(mine, s_red);
            if (threadIdx.x == 0) Cp[i + 1] = tot;
        } else {
            int64_t tot;
            int64_t r = Cp[i] + block_excl_scan_i64(mine, s_red, tot);
            for (int e = e0; e < e0 + per && e < w; ++e)
                if (e == 0 || s_key[e] != s_key[e - 1]) Ci[r++] = s_key[e];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- L rows: symbolic (bitmap windows)
template <int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_L_sym(const int32_t *__restrict__ list, const int *__restrict__ cnt,
                                                         int64_t ncolsB, const int64_t *__restrict__ Ap,
                                                         const int32_t *__restrict__ Ai, const int64_t *__restrict__ Bp,
                                                         const int32_t *__restrict__ Bi, int64_t *__restrict__ Cp,
                                                         int32_t *__restrict__ Ci)
{
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bm = reinterpret_cast<uint32_t *>(smem);
    __shared__ int64_t s_red[kGemmTPB / 32];
    const int nrows = *cnt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t W = (int64_t)kBitmapWords * 32;
    for (int it = blockIdx.x; it < nrows; it += gridDim.x) {
        const int64_t i = list[it];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        int64_t done = 0;
        for (int64_t w0 = 0; w0 < ncolsB; w0 += W) {
            for (int e = threadIdx.x; e < kBitmapWords; e += kGemmTPB) bm[e] = 0u;
            __syncthreads();
            for (int64_t a = as + warp; a < ae; a += kGemmTPB / 32) {
                const int32_t k = Ai[a];
                const int64_t bs = Bp[k], be = Bp[k + 1];
                for (int64_t b = bs + lane; b < be; b += 32) {
                    const int64_t j = Bi[b];
                    if (j >= w0 && j < w0 + W) atomicOr(&bm[(j - w0) >> 5], 1u << (j & 31));
                }
            }
            __syncthreads();
            constexpr int per = kBitmapWords / kGemmTPB;
            const int e0 = threadIdx.x * per;
            int64_t mine = 0;
            for (int e = e0; e < e0 + per; ++e) mine += __popc(bm[e]);
            int64_t tot;
            const int64_t off = block_excl_scan_i64(mine, s_red, tot);
            if (PH == PH_FILL) {
                int64_t r = Cp[i] + done + off;
                for (int e = e0; e < e0 + per; ++e) {
                    uint32_t bits = bm[e];
                    while (bits) {
                        const int bpos = __ffs(bits) - 1;
                        bits &= bits - 1;
                        Ci[r++] = (int32_t)(w0 + (int64_t)e * 32 + bpos);
                    }
                }
            }
            done += tot;
            __syncthreads();
        }
        if (PH == PH_COUNT && threadIdx.x == 0) Cp[i + 1] = done;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- M/L rows: numeric + backward
// C row in shared memory when it fits (nnz(C_i) <= kMMaxW), else searched in global memory.
template <typename T, int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_ML_val(const int32_t *__restrict__ list, const int *__restrict__ cnt,
                                                          const int64_t *__restrict__ Ap, const int32_t *__restrict__ Ai,
                                                          const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                                          const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                          const int64_t *__restrict__ Cp, const int32_t *__restrict__ Ci,
                                                          T *__restrict__ Cv, const T *__restrict__ dC,
                                                          T *__restrict__ dA, T *__restrict__ dB)
{
    extern __shared__ __align__(16) unsigned char smem[];
    double *s_val = reinterpret_cast<double *>(smem);                             // acc (NUM) or dC (BWD)
    int32_t *s_col = reinterpret_cast<int32_t *>(smem + sizeof(double) * kMMaxW);
    const int nrows = *cnt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = blockIdx.x; it < nrows; it += gridDim.x) {
        const int64_t i = list[it];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        const int64_t cs = Cp[i], nc = Cp[i + 1] - cs;
        const bool in_smem = nc <= kMMaxW;
        if (in_smem) {
            for (int64_t e = threadIdx.x; e < nc; e += kGemmTPB) {
                s_col[e] = Ci[cs + e];
                s_val[e] = PH == PH_NUM ? 0.0 : (double)dC[cs + e];
            }
        } else if (PH == PH_NUM) {
            for (int64_t e = threadIdx.x; e < nc; e += kGemmTPB) Cv[cs + e] = (T)0;
        }
        __syncthreads();
        const int32_t *ccol = in_smem ? s_col : Ci + cs;
        for (int64_t a = as + warp; a < ae; a += kGemmTPB / 32) {
            const int32_t k = Ai[a];
            const double av = (double)Av[a];
            const int64_t bs = Bp[k], be = Bp[k + 1];
            double t = 0.0;
            for (int64_t b = bs + lane; b < be; b += 32) {
                const int64_t pos = lbound(ccol, nc, Bi[b]);
                const double bv = (double)Bv[b];
                if (PH == PH_NUM) {
                    if (in_smem) atomicAdd(&s_val[pos], av * bv);
                    else red_add(&Cv[cs + pos], (T)(av * bv));
                } else {
                    const double g = in_smem ? s_val[pos] : (double)dC[cs + pos];
                    t = fma(g, bv, t);
                    if (dB) red_add(&dB[b], (T)(av * g));
                }
            }
            if (PH == PH_BWD) {
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (lane == 0 && dA) dA[a] = (T)t;
            }
        }
        __syncthreads();
        if (PH == PH_NUM && in_smem)
            for (int64_t e = threadIdx.x; e < nc; e += kGemmTPB) Cv[cs + e] = (T)s_val[e];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host side
static int carve_bins(const csrk_pattern &A, Bins &b, Bump &ws)
{
    const int64_t m = A.nrows > 0 ? A.nrows : 1;
    b.bin = ws.take<uint8_t>(m);
    b.listM = ws.take<int32_t>(m);
    b.listL = ws.take<int32_t>(m);
    b.cnt = ws.take<int>(2);
    return CSRK_OK;
}

static int run_bins(const csrk_pattern &A, const csrk_pattern &B, Bins &b, cudaStream_t s)
{
    CSRK_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(int) * 2, s));
    CSRK_LAUNCH(k_gemm_bin, (unsigned)cdiv(A.nrows * 8, 256), 256, 0, s, A.nrows, A.indptr, A.indices, B.indptr, b);
    return CSRK_OK;
}

static unsigned ml_grid() { return (unsigned)(kNumSMs * 4); }

static int set_smem_attrs()
{
    static bool done = false;
    if (done) return CSRK_OK;
    const int bm = (int)(sizeof(uint32_t) * kBitmapWords);
    const int mv = (int)((sizeof(double) + sizeof(int32_t)) * kMMaxW);
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_L_sym<PH_COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bm));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_L_sym<PH_FILL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bm));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_ML_val<double, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, mv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_ML_val<double, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, mv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_ML_val<float, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, mv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_ML_val<float, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, mv));
    done = true;
    return CSRK_OK;
}

int spgemm_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *Cp, int32_t *Ci, int64_t *nnzC_host,
                    Bump &ws, cudaStream_t s)
{
    Bins b{};
    carve_bins(A, b, ws);
    if (ws.sizing()) return scan_counts_i64(nullptr, A.nrows, ws, s);
    const int64_t m = A.nrows;
    CSRK_TRY(set_smem_attrs());
    if (!Ci) {
        CSRK_CUDA(cudaMemsetAsync(Cp, 0, sizeof(int64_t), s));
        if (m > 0) {
            CSRK_TRY(run_bins(A, B, b, s));
            CSRK_LAUNCH((k_gemm_S<double, PH_COUNT>), (unsigned)cdiv(m, kGemmTPB), kGemmTPB, 0, s, m,
                        (const uint8_t *)b.bin, A.indptr, A.indices, (const double *)nullptr, B.indptr, B.indices,
                        (const double *)nullptr, Cp, (int32_t *)nullptr, (double *)nullptr, (const double *)nullptr,
                        (double *)nullptr, (double *)nullptr);
            CSRK_LAUNCH(k_gemm_M_sym<PH_COUNT>, ml_grid(), kGemmTPB, 0, s, (const int32_t *)b.listM,
                        (const int *)b.cnt, A.indptr, A.indices, B.indptr, B.indices, Cp, (int32_t *)nullptr);
            CSRK_LAUNCH(k_gemm_L_sym<PH_COUNT>, (unsigned)kNumSMs, kGemmTPB, sizeof(uint32_t) * kBitmapWords, s,
                        (const int32_t *)b.listL, (const int *)(b.cnt + 1), B.ncols, A.indptr, A.indices, B.indptr,
                        B.indices, Cp, (int32_t *)nullptr);
            CSRK_TRY(scan_counts_i64(Cp, m, ws, s));
        }
        CSRK_CUDA(cudaMemcpyAsync(nnzC_host, Cp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSRK_CUDA(cudaStreamSynchronize(s));
        return CSRK_OK;
    }
    if (m == 0) return CSRK_OK;
    CSRK_TRY(run_bins(A, B, b, s));
    CSRK_LAUNCH((k_gemm_S<double, PH_FILL>), (unsigned)cdiv(m, kGemmTPB), kGemmTPB, 0, s, m, (const uint8_t *)b.bin,
                A.indptr, A.indices, (const double *)nullptr, B.indptr, B.indices, (const double *)nullptr, Cp, Ci,
                (double *)nullptr, (const double *)nullptr, (double *)nullptr, (double *)nullptr);
    CSRK_LAUNCH(k_gemm_M_sym<PH_FILL>, ml_grid(), kGemmTPB, 0, s, (const int32_t *)b.listM, (const int *)b.cnt,
                A.indptr, A.indices, B.indptr, B.indices, Cp, Ci);
    CSRK_LAUNCH(k_gemm_L_sym<PH_FILL>, (unsigned)kNumSMs, kGemmTPB, sizeof(uint32_t) * kBitmapWords, s,
                (const int32_t *)b.listL, (const int *)(b.cnt + 1), B.ncols, A.indptr, A.indices, B.indptr, B.indices,
                Cp, Ci);
    return CSRK_OK;
}

template <typename T>
static int spgemm_values_t(int PH, const csrk_pattern &A, const T *Av, const csrk_pattern &B, const T *Bv,
                           const csrk_pattern &C, T *Cv, const T *dC, T *dA, T *dB, Bump &ws, cudaStream_t s)
{
    Bins b{};
    carve_bins(A, b, ws);
    if (ws.sizing()) return CSRK_OK;
    CSRK_TRY(set_smem_attrs());
    if (PH == PH_BWD && dB) CSRK_CUDA(cudaMemsetAsync(dB, 0, sizeof(T) * (size_t)B.nnz, s));
    const int64_t m = A.nrows;
    if (m == 0) return CSRK_OK;
    CSRK_TRY(run_bins(A, B, b, s));
    const size_t mv = (sizeof(double) + sizeof(int32_t)) * kMMaxW;
    if (PH == PH_NUM) {
        CSRK_LAUNCH((k_gemm_S<T, PH_NUM>), (unsigned)cdiv(m, kGemmTPB), kGemmTPB, 0, s, m, (const uint8_t *)b.bin,
                    A.indptr, A.indices, Av, B.indptr, B.indices, Bv, (int64_t *)C.indptr, (int32_t *)nullptr, Cv,
                    (const T *)nullptr, (T *)nullptr, (T *)nullptr);
        CSRK_LAUNCH((k_gemm_ML_val<T, PH_NUM>), ml_grid(), kGemmTPB, mv, s, (const int32_t *)b.listM,
                    (const int *)b.cnt, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, C.indptr, C.indices, Cv,
                    (const T *)nullptr, (T *)nullptr, (T *)nullptr);
        CSRK_LAUNCH((k_gemm_ML_val<T, PH_NUM>), ml_grid(), kGemmTPB, mv, s, (const int32_t *)b.listL,
                    (const int *)(b.cnt + 1), A.indptr, A.indices, Av, B.indptr, B.indices, Bv, C.indptr, C.indices,
                    Cv, (const T *)nullptr, (T *)nullptr, (T *)nullptr);
    } else {
        CSRK_LAUNCH((k_gemm_S<T, PH_BWD>), (unsigned)cdiv(m, kGemmTPB), kGemmTPB, 0, s, m, (const uint8_t *)b.bin,
                    A.indptr, A.indices, Av, B.indptr, B.indices, Bv, (int64_t *)C.indptr, (int32_t *)nullptr,
                    (T *)nullptr, dC, dA, dB);
        CSRK_LAUNCH((k_gemm_ML_val<T, PH_BWD>), ml_grid(), kGemmTPB, mv, s, (const int32_t *)b.listM,
                    (const int *)b.cnt, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, C.indptr, C.indices,
                    (T *)nullptr, dC, dA, dB);
        CSRK_LAUNCH((k_gemm_ML_val<T, PH_BWD>), ml_grid(), kGemmTPB, mv, s, (const int32_t *)b.listL,
                    (const int *)(b.cnt + 1), A.indptr, A.indices, Av, B.indptr, B.indices, Bv, C.indptr, C.indices,
                    (T *)nullptr, dC, dA, dB);
    }
    return CSRK_OK;
}

int spgemm_numeric(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern &B, const void *B_val,
                   const csrk_pattern &C, void *C_val, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return spgemm_values_t<double>(PH_NUM, A, (const double *)A_val, B, (const double *)B_val, C, (double *)C_val,
                                       nullptr, nullptr, nullptr, ws, s);
    return spgemm_values_t<float>(PH_NUM, A, (const float *)A_val, B, (const float *)B_val, C, (float *)C_val,
                                  nullptr, nullptr, nullptr, ws, s);
}

int spgemm_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern &B, const void *B_val,
               const csrk_pattern &C, const void *dC, void *dA, void *dB, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return spgemm_values_t<double>(PH_BWD, A, (const double *)A_val, B, (const double *)B_val, C, nullptr,
                                       (const double *)dC, (double *)dA, (double *)dB, ws, s);
    return spgemm_values_t<float>(PH_BWD, A, (const float *)A_val, B, (const float *)B_val, C, nullptr,
                                  (const float *)dC, (float *)dA, (float *)dB, ws, s);
}

}  // namespace csrk
