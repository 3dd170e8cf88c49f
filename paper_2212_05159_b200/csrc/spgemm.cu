// spgemm.cu -- SpGEMM C = A B: symbolic, numeric and backward
// (PAPER 3.1.2; Table 1; Fig. 3).
//
// Every phase (COUNT, FILL of the symbolic pattern; NUM; BWD) runs two kernels:
//
//   k_gemm_S   one THREAD per row of A.  A row with l_i <= 8 entries whose product count
//              w_i = sum_k len_B(k) is <= 512 ("short") runs an l_i-way merge of its sorted B
//              rows.  The merge emits C's columns in ascending order, so the symbolic phase
//              needs no sort, the numeric phase sums each C_ij over k ascending (the
//              oracle's order, deterministic) and the backward pass meets dC_ij in C's
//              storage order with no search.  The merge is specialised on the warp's
//              largest l_i, and when all 32 rows of a warp are short their C (and dA)
//              ranges are contiguous, so outputs are staged in shared memory and written
//              (and dC read) coalesced.  Every other row is queued (warp-aggregated atomic).
//   k_gemm_big one CTA per queued row.  w_i <= 8192: products gathered to shared memory;
//              symbolic = bitonic sort + unique; numeric/backward binary-search each
//              product's column in the C row (shared memory) -- numeric accumulates with
//              shared-memory atomics.  w_i > 8192: symbolic uses shared-memory bitmap
//              windows over the column range (sorted output for free); numeric/backward
//              search the C row in global memory and accumulate with global atomics.
//
// The backward pass computes dA_ik = sum_j dC_ij B_kj per A entry (deterministic) and
// scatters dB_kj += A_ik dC_ij with global atomic adds (reading A9).
#include "ops.cuh"

namespace csrk {

constexpr int kSMaxL = 8;
constexpr int64_t kSMaxW = 512;
constexpr int kMMaxW = 8192;
constexpr int kSTPB = 128;           // k_gemm_S: 4 warps
constexpr int kSWarps = kSTPB / 32;
constexpr int kSBuf = 832;           // staged C entries per warp (3D 7-point A^2: 32 x 25 = 800)
constexpr int kSBufA = 32 * kSMaxL;  // staged dA entries per warp
constexpr int kGemmTPB = 256;        // k_gemm_big
constexpr int kBitmapWords = 24576;  // 96 KB -> windows of 786,432 columns

enum { PH_COUNT = 0, PH_FILL = 1, PH_NUM = 2, PH_BWD = 3 };

struct BigList {
    int32_t *rows;
    int *count;
};

// ---------------------------------------------------------------- short rows: thread-per-row merge
// Predicated loads (no branch): the merge step updates every list with selects so the warp
// never diverges per list.
__device__ __forceinline__ void ld_pred(int32_t &v, const int32_t *p, bool pred)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.b32 %0, [%1]; }"
                 : "+r"(v) : "l"(p), "r"((int)pred));
}
__device__ __forceinline__ void ld_pred(double &v, const double *p, bool pred)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.f64 %0, [%1]; }"
                 : "+d"(v) : "l"(p), "r"((int)pred));
}
__device__ __forceinline__ void ld_pred(double &v, const float *p, bool pred)
{
    float f = 0.f;
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.f32 %0, [%1]; }"
                 : "+f"(f) : "l"(p), "r"((int)pred));
    if (pred) v = (double)f;
}

// Branchy merge: only the lists whose head matched advance (a divergent branch per list).
// Measured best for the symbolic phases and the backward pass (fewer registers).
template <typename T, int PH, int L>
__device__ __forceinline__ int64_t s_merge_br(int64_t as, int l, const int32_t *__restrict__ Ai,
                                              const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                              const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                              int32_t *outI, T *outV, const T *dCrow, T *dArow,
                                              T *__restrict__ dB)
{
    int64_t cur[L];
    int rem[L];
    int32_t head[L];
    double av[L], dacc[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
        rem[t] = 0;
        head[t] = INT32_MAX;
        cur[t] = 0;
        av[t] = dacc[t] = 0.0;
        if (t < l) {
            const int32_t k = Ai[as + t];
            cur[t] = Bp[k];
            rem[t] = (int)(Bp[k + 1] - cur[t]);
            if (PH == PH_NUM || PH == PH_BWD) av[t] = (double)Av[as + t];
            if (rem[t] > 0) head[t] = Bi[cur[t]];
        }
    }
    int64_t c = 0;
    while (true) {
        int32_t v = head[0];
#pragma unroll
        for (int t = 1; t < L; ++t) v = head[t] < v ? head[t] : v;
        if (v == INT32_MAX) break;
        double acc = 0.0;
        const double g = PH == PH_BWD ? (double)dCrow[c] : 0.0;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            if (head[t] == v) {
                if (PH == PH_NUM) acc = fma(av[t], (double)Bv[cur[t]], acc);
                if (PH == PH_BWD) {
                    dacc[t] = fma(g, (double)Bv[cur[t]], dacc[t]);
                    if (dB) red_add(&dB[cur[t]], (T)(av[t] * g));
                }
                ++cur[t];
                head[t] = --rem[t] > 0 ? Bi[cur[t]] : INT32_MAX;
            }
        }
        if (PH == PH_FILL) outI[c] = v;
        if (PH == PH_NUM) outV[c] = (T)acc;
        ++c;
    }
    if (PH == PH_BWD && dArow) {
#pragma unroll
        for (int t = 0; t < L; ++t)
            if (t < l) dArow[t] = (T)dacc[t];
    }
    return c;
}

// Branch-free merge: every list is updated with selects and predicated loads each step, the
// head's value cached in a register.  Measured best for the numeric phase.
template <typename T, int PH, int L>
__device__ __forceinline__ int64_t s_merge_bl(int64_t as, int l, const int32_t *__restrict__ Ai,
                                              const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                              const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                              int32_t *outI, T *outV, const T *dCrow, T *dArow,
                                              T *__restrict__ dB)
{
    constexpr bool VAL = PH == PH_NUM || PH == PH_BWD;
    int64_t cur[L];   // position in B of list t's head
    int rem[L];       // entries left in list t including the head
    int32_t head[L];  // column at the head (INT32_MAX when exhausted)
    double hv[L];     // value at the head (VAL)
    double av[L], dacc[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
        rem[t] = 0;
        head[t] = INT32_MAX;
        cur[t] = 0;
        hv[t] = av[t] = dacc[t] = 0.0;
        if (t < l) {
            const int32_t k = Ai[as + t];
            cur[t] = Bp[k];
            rem[t] = (int)(Bp[k + 1] - cur[t]);
            if (VAL) av[t] = (double)Av[as + t];
            if (rem[t] > 0) {
                head[t] = Bi[cur[t]];
                if (VAL) hv[t] = (double)Bv[cur[t]];
            }
        }
    }
    int64_t c = 0;
    while (true) {
        int32_t v = head[0];
#pragma unroll
        for (int t = 1; t < L; ++t) v = min(v, head[t]);
        if (v == INT32_MAX) break;
        double acc = 0.0;
        const double g = PH == PH_BWD ? (double)dCrow[c] : 0.0;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            const bool mt = head[t] == v;
            if (PH == PH_NUM) acc = fma(av[t], mt ? hv[t] : 0.0, acc);
            if (PH == PH_BWD) {
                dacc[t] = fma(g, mt ? hv[t] : 0.0, dacc[t]);
                if (dB && mt) red_add(&dB[cur[t]], (T)(av[t] * g));
            }
            cur[t] += mt;
            rem[t] -= mt;
            const bool more = mt && rem[t] > 0;
            ld_pred(head[t], Bi + cur[t], more);
            if (VAL) ld_pred(hv[t], Bv + cur[t], more);
            head[t] = (mt && !more) ? INT32_MAX : head[t];
        }
        if (PH == PH_FILL) outI[c] = v;
        if (PH == PH_NUM) outV[c] = (T)acc;
        ++c;
    }
    if (PH == PH_BWD && dArow) {
#pragma unroll
        for (int t = 0; t < L; ++t)
            if (t < l) dArow[t] = (T)dacc[t];
    }
    return c;
}

template <typename T, int PH, int L>
__device__ __forceinline__ int64_t s_merge(int64_t as, int l, const int32_t *__restrict__ Ai,
                                           const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                           const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                           int32_t *outI, T *outV, const T *dCrow, T *dArow, T *__restrict__ dB)
{
    if constexpr (PH == PH_NUM)
        return s_merge_bl<T, PH, L>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB);
    else
        return s_merge_br<T, PH, L>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB);
}

template <typename T, int PH>
__global__ __launch_bounds__(kSTPB) void k_gemm_S(int64_t m, const int64_t *__restrict__ Ap,
                                                  const int32_t *__restrict__ Ai, const T *__restrict__ Av,
                                                  const int64_t *__restrict__ Bp, const int32_t *__restrict__ Bi,
                                                  const T *__restrict__ Bv, int64_t *__restrict__ Cp,
                                                  int32_t *__restrict__ Ci, T *__restrict__ Cv,
                                                  const T *__restrict__ dC, T *__restrict__ dA, T *__restrict__ dB,
                                                  BigList big, int use_stage)
{
    // per-warp staging buffers in dynamic shared memory (none when use_stage == 0, which
    // leaves the whole carve-out to L1 for the merge's list reads)
    constexpr int BUFB = (PH == PH_FILL) ? (int)sizeof(int32_t) * kSBuf : (int)sizeof(T) * kSBuf;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *s_buf_w = s_dyn + (size_t)warp * BUFB;
    T *s_dA_w = reinterpret_cast<T *>(s_dyn + (size_t)kSWarps * BUFB) + warp * kSBufA;
    const int64_t i0 = (int64_t)blockIdx.x * kSTPB + warp * 32;   // first row of this warp
    const int64_t i = i0 + lane;
    const bool valid = i < m;
    int64_t as = 0;
    int l = 0;
    int64_t w = 0;
    if (valid) {
        as = Ap[i];
        const int64_t ll = Ap[i + 1] - as;
        l = ll > kSMaxL ? kSMaxL + 1 : (int)ll;
        if (l <= kSMaxL)
            for (int t = 0; t < l; ++t) {
                const int32_t k = Ai[as + t];
                w += Bp[k + 1] - Bp[k];
            }
    }
    const bool isS = valid && l <= kSMaxL && w <= kSMaxW;
    // queue the other rows (warp-aggregated)
    const unsigned bigmask = __ballot_sync(0xffffffffu, valid && !isS);
    if (bigmask) {
        int base = 0;
        if (lane == 0) base = atomicAdd(big.count, __popc(bigmask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (valid && !isS) big.rows[base + __popc(bigmask & ((1u << lane) - 1))] = (int32_t)i;
    }
    const int Lw = (int)__reduce_max_sync(0xffffffffu, isS ? (unsigned)l : 0u);
    // staging: all rows of the warp short, C range of the warp small enough
    const int64_t iend = i0 + 32 < m ? i0 + 32 : m;
    bool stage = false;
    int64_t c_lo = 0, a_lo = 0;
    if (PH != PH_COUNT) {
        stage = use_stage && __all_sync(0xffffffffu, !valid || isS) && i0 < m;
        if (stage) {
            c_lo = Cp[i0];
            stage = Cp[iend] - c_lo <= kSBuf;
            a_lo = Ap[i0];
        }
    }
    const int64_t c_hi = stage ? Cp[iend] : 0;
    T *sv = reinterpret_cast<T *>(s_buf_w);
    int32_t *si = reinterpret_cast<int32_t *>(s_buf_w);
    if (PH == PH_BWD && stage) {
        for (int64_t e = c_lo + lane; e < c_hi; e += 32) sv[e - c_lo] = dC[e];
        __syncwarp();
    }
    if (isS) {
        const int64_t cs = PH == PH_COUNT ? 0 : Cp[i];
        int32_t *outI = PH == PH_FILL ? (stage ? si + (cs - c_lo) : Ci + cs) : nullptr;
        T *outV = PH == PH_NUM ? (stage ? sv + (cs - c_lo) : Cv + cs) : nullptr;
        const T *dCrow = PH == PH_BWD ? (stage ? sv + (cs - c_lo) : dC + cs) : nullptr;
        T *dArow = (PH == PH_BWD && dA) ? (stage ? s_dA_w + (as - a_lo) : dA + as) : nullptr;
        int64_t cnt = 0;
        switch (Lw) {
        case 1: cnt = s_merge<T, PH, 1>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 2: cnt = s_merge<T, PH, 2>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 3: cnt = s_merge<T, PH, 3>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 4: cnt = s_merge<T, PH, 4>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 5: cnt = s_merge<T, PH, 5>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 6: cnt = s_merge<T, PH, 6>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 7: cnt = s_merge<T, PH, 7>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        case 8: cnt = s_merge<T, PH, 8>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB); break;
        default: break;  // l == 0: empty row
        }
        if (PH == PH_COUNT) Cp[i + 1] = cnt;
    }
    if (stage) {
        __syncwarp();
        if (PH == PH_FILL)
            for (int64_t e = c_lo + lane; e < c_hi; e += 32) Ci[e] = si[e - c_lo];
        if (PH == PH_NUM)
            for (int64_t e = c_lo + lane; e < c_hi; e += 32) Cv[e] = sv[e - c_lo];
        if (PH == PH_BWD && dA) {
            const int64_t a_hi = Ap[iend];
            for (int64_t e = a_lo + lane; e < a_hi; e += 32) dA[e] = s_dA_w[e - a_lo];
        }
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

// w_i = sum_k len_B(k) over row i (block reduction)
__device__ __forceinline__ int64_t row_work(int64_t as, int64_t ae, const int32_t *__restrict__ Ai,
                                            const int64_t *__restrict__ Bp, int64_t *s_red)
{
    int64_t w = 0;
    for (int64_t a = as + threadIdx.x; a < ae; a += kGemmTPB) {
        const int32_t k = Ai[a];
        w += Bp[k + 1] - Bp[k];
    }
    return block_sum_i64(w, s_red);
}

// ---------------------------------------------------------------- big rows: symbolic
template <int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_big_sym(BigList big, int64_t ncolsB,
                                                           const int64_t *__restrict__ Ap,
                                                           const int32_t *__restrict__ Ai,
                                                           const int64_t *__restrict__ Bp,
                                                           const int32_t *__restrict__ Bi, int64_t *__restrict__ Cp,
                                                           int32_t *__restrict__ Ci)
{
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *s_key = reinterpret_cast<int32_t *>(smem);   // kMMaxW keys (M path)
    uint32_t *bm = reinterpret_cast<uint32_t *>(smem);    // kBitmapWords (L path)
    __shared__ int s_cnt;
    __shared__ int64_t s_red[kGemmTPB / 32];
    const int nrows = *(volatile int *)big.count;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = blockIdx.x; it < nrows; it += gridDim.x) {
        const int64_t i = big.rows[it];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        const int64_t w = row_work(as, ae, Ai, Bp, s_red);
        if (w <= kMMaxW) {
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
            const int wn = s_cnt;
            const int P = pow2ceil_i(wn > 0 ? wn : 1);
            for (int e = wn + threadIdx.x; e < P; e += kGemmTPB) s_key[e] = INT32_MAX;
            __syncthreads();
            bitonic_keys(s_key, P);
            const int per = (P + kGemmTPB - 1) / kGemmTPB;
            const int e0 = threadIdx.x * per;
            int64_t mine = 0;
            for (int e = e0; e < e0 + per && e < wn; ++e) mine += (e == 0 || s_key[e] != s_key[e - 1]);
            if (PH == PH_COUNT) {
                const int64_t tot = block_sum_i64(mine, s_red);
                if (threadIdx.x == 0) Cp[i + 1] = tot;
            } else {
                int64_t tot;
                int64_t r = Cp[i] + block_excl_scan_i64(mine, s_red, tot);
                for (int e = e0; e < e0 + per && e < wn; ++e)
                    if (e == 0 || s_key[e] != s_key[e - 1]) Ci[r++] = s_key[e];
            }
            __syncthreads();
            continue;
        }
        // bitmap windows over [0, ncolsB)
        const int64_t W = (int64_t)kBitmapWords * 32;
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

// ---------------------------------------------------------------- big rows: numeric + backward
// C row in shared memory when it fits (nnz(C_i) <= kMMaxW), else searched in global memory.
template <typename T, int PH>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_big_val(BigList big, const int64_t *__restrict__ Ap,
                                                           const int32_t *__restrict__ Ai, const T *__restrict__ Av,
                                                           const int64_t *__restrict__ Bp,
                                                           const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                           const int64_t *__restrict__ Cp,
                                                           const int32_t *__restrict__ Ci, T *__restrict__ Cv,
                                                           const T *__restrict__ dC, T *__restrict__ dA,
                                                           T *__restrict__ dB)
{
    extern __shared__ __align__(16) unsigned char smem[];
    double *s_val = reinterpret_cast<double *>(smem);                             // acc (NUM) or dC (BWD)
    int32_t *s_col = reinterpret_cast<int32_t *>(smem + sizeof(double) * kMMaxW);
    const int nrows = *(volatile int *)big.count;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = blockIdx.x; it < nrows; it += gridDim.x) {
        const int64_t i = big.rows[it];
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
static unsigned big_grid() { return (unsigned)(kNumSMs * 2); }

static size_t big_sym_smem() { return sizeof(uint32_t) * kBitmapWords; }
static size_t big_val_smem() { return (sizeof(double) + sizeof(int32_t)) * kMMaxW; }

static int set_smem_attrs()
{
    static bool done = false;
    if (done) return CSRK_OK;
    const int bs = (int)big_sym_smem(), bv = (int)big_val_smem();
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_FILL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_val<double, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_val<double, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, bv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_val<float, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bv));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_val<float, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, bv));
    done = true;
    return CSRK_OK;
}

// Dynamic shared memory of k_gemm_S: the per-warp output staging (knob GEMM_STAGE, default on).
template <typename T>
static size_t s_smem(int PH, int use)
{
    if (!use || PH == PH_COUNT) return 0;
    size_t b = (size_t)kSWarps * kSBuf * (PH == PH_FILL ? sizeof(int32_t) : sizeof(T));
    if (PH == PH_BWD) b += (size_t)kSWarps * kSBufA * sizeof(T);
    return b;
}

// Staging pays for the symbolic fill (4-byte scattered stores); for numeric / backward the
// shared memory is worth more as L1 for the merge's list reads (measured: 388 vs 436 us and
// 677 vs 802 us on config 2).
static int stage_fill() { static int v = knob("GEMM_STAGE_FILL", 1); return v; }
static int stage_vals() { static int v = knob("GEMM_STAGE_VALS", 0); return v; }

static void carve_big(const csrk_pattern &A, BigList &b, Bump &ws)
{
    b.rows = ws.take<int32_t>(A.nrows > 0 ? A.nrows : 1);
    b.count = ws.take<int>(1);
}

int spgemm_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *Cp, int32_t *Ci, int64_t *nnzC_host,
                    Bump &ws, cudaStream_t s)
{
    BigList b{};
    carve_big(A, b, ws);
    if (ws.sizing()) return scan_counts_i64(nullptr, A.nrows, ws, s);
    const int64_t m = A.nrows;
    CSRK_TRY(set_smem_attrs());
    const unsigned gS = (unsigned)cdiv(m, kSTPB);
    if (!Ci) {
        CSRK_CUDA(cudaMemsetAsync(Cp, 0, sizeof(int64_t), s));
        if (m > 0) {
            CSRK_CUDA(cudaMemsetAsync(b.count, 0, sizeof(int), s));
            CSRK_LAUNCH((k_gemm_S<double, PH_COUNT>), gS, kSTPB, 0, s, m, A.indptr, A.indices,
                        (const double *)nullptr, B.indptr, B.indices, (const double *)nullptr, Cp, (int32_t *)nullptr,
                        (double *)nullptr, (const double *)nullptr, (double *)nullptr, (double *)nullptr, b, 0);
            CSRK_LAUNCH(k_gemm_big_sym<PH_COUNT>, big_grid(), kGemmTPB, big_sym_smem(), s, b, B.ncols, A.indptr,
                        A.indices, B.indptr, B.indices, Cp, (int32_t *)nullptr);
            CSRK_TRY(scan_counts_i64(Cp, m, ws, s));
        }
        CSRK_CUDA(cudaMemcpyAsync(nnzC_host, Cp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSRK_CUDA(cudaStreamSynchronize(s));
        return CSRK_OK;
    }
    if (m == 0) return CSRK_OK;
    CSRK_CUDA(cudaMemsetAsync(b.count, 0, sizeof(int), s));
    CSRK_LAUNCH((k_gemm_S<double, PH_FILL>), gS, kSTPB, s_smem<double>(PH_FILL, stage_fill()), s, m, A.indptr,
                A.indices, (const double *)nullptr, B.indptr, B.indices, (const double *)nullptr, Cp, Ci,
                (double *)nullptr, (const double *)nullptr, (double *)nullptr, (double *)nullptr, b, stage_fill());
    CSRK_LAUNCH(k_gemm_big_sym<PH_FILL>, big_grid(), kGemmTPB, big_sym_smem(), s, b, B.ncols, A.indptr, A.indices,
                B.indptr, B.indices, Cp, Ci);
    return CSRK_OK;
}

template <typename T>
static int spgemm_values_t(int PH, const csrk_pattern &A, const T *Av, const csrk_pattern &B, const T *Bv,
                           const csrk_pattern &C, T *Cv, const T *dC, T *dA, T *dB, Bump &ws, cudaStream_t s)
{
    BigList b{};
    carve_big(A, b, ws);
    if (ws.sizing()) return CSRK_OK;
    CSRK_TRY(set_smem_attrs());
    if (PH == PH_BWD && dB) CSRK_CUDA(cudaMemsetAsync(dB, 0, sizeof(T) * (size_t)B.nnz, s));
    const int64_t m = A.nrows;
    if (m == 0) return CSRK_OK;
    CSRK_CUDA(cudaMemsetAsync(b.count, 0, sizeof(int), s));
    const unsigned gS = (unsigned)cdiv(m, kSTPB);
    int64_t *Cp = const_cast<int64_t *>(C.indptr);
    if (PH == PH_NUM) {
        CSRK_LAUNCH((k_gemm_S<T, PH_NUM>), gS, kSTPB, s_smem<T>(PH_NUM, stage_vals()), s, m, A.indptr, A.indices,
                    Av, B.indptr, B.indices, Bv, Cp, (int32_t *)nullptr, Cv, (const T *)nullptr, (T *)nullptr,
                    (T *)nullptr, b, stage_vals());
        CSRK_LAUNCH((k_gemm_big_val<T, PH_NUM>), big_grid(), kGemmTPB, big_val_smem(), s, b, A.indptr, A.indices, Av,
                    B.indptr, B.indices, Bv, C.indptr, C.indices, Cv, (const T *)nullptr, (T *)nullptr, (T *)nullptr);
    } else {
        CSRK_LAUNCH((k_gemm_S<T, PH_BWD>), gS, kSTPB, s_smem<T>(PH_BWD, stage_vals()), s, m, A.indptr, A.indices,
                    Av, B.indptr, B.indices, Bv, Cp, (int32_t *)nullptr, (T *)nullptr, dC, dA, dB, b, stage_vals());
        CSRK_LAUNCH((k_gemm_big_val<T, PH_BWD>), big_grid(), kGemmTPB, big_val_smem(), s, b, A.indptr, A.indices, Av,
                    B.indptr, B.indices, Bv, C.indptr, C.indices, (T *)nullptr, dC, dA, dB);
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
