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
//   k_gemm_W   one WARP per queued row with l_i <= kWL and w_i <= kWW (power-law "medium" rows,
//              SURVEY 8(d) config 4): the row's products are enumerated flat (list offsets in
//              shared memory); COUNT inserts the columns into a shared-memory hash table, FILL
//              sorts them (warp bitonic network) and compacts the unique ones, NUM / BWD
//              binary-search each product's column in the C row staged in shared memory
//              (NUM: shared atomics into the row accumulator; BWD: dA by a segmented warp
//              reduction per A entry, dB by global atomics).  Rows with w_i > kWW are passed on.
//   k_gemm_big one CTA per remaining row.  w_i <= 8192: products gathered to shared memory;
//              symbolic = bitonic sort + unique; numeric/backward binary-search each
//              product's column in the C row (shared memory) -- numeric accumulates with
//              shared-memory atomics.  w_i > 8192: symbolic uses shared-memory bitmap
//              windows over the column range (sorted output for free); numeric/backward
//              search the C row in global memory and accumulate with global atomics.
//
// The backward pass computes dA_ik = sum_j dC_ij B_kj per A entry (deterministic) and
// scatters dB_kj += A_ik dC_ij with global atomic adds (reading A9).
#include <cooperative_groups.h>
#include <mutex>
#include <vector>

#include "ops.cuh"

namespace csrk {

#ifndef CSRK_S_MAXL
#define CSRK_S_MAXL 8
#endif
constexpr int kSMaxL = CSRK_S_MAXL;  // A/B via CSRK_NVCC_EXTRA
#ifndef CSRK_S_MAXW
#define CSRK_S_MAXW 64  // stencil rows (w <= 49) merge per thread; heavier short rows (power-law, random B rows:
                        // the per-thread merge becomes a chain of dependent gathers) go to the warp path
#endif
constexpr int64_t kSMaxW = CSRK_S_MAXW;
constexpr int kMMaxW = 8192;
constexpr int kSTPB = 128;           // k_gemm_S: 4 warps
constexpr int kSWarps = kSTPB / 32;
#ifndef CSRK_S_MINB
#define CSRK_S_MINB 6  // measured: numeric 421 -> 355 us, bwd dA 452 -> 410 us on config 2 (1 and 4: no change)
#endif
constexpr int kSMinBlocks = CSRK_S_MINB;
#ifndef CSRK_S_BWD_BL
#define CSRK_S_BWD_BL 0
#endif  // k_gemm_S occupancy hint (A/B via CSRK_NVCC_EXTRA)
constexpr int kSBuf = 832;           // staged C entries per warp (3D 7-point A^2: 32 x 25 = 800)
constexpr int kSBufA = 32 * kSMaxL;  // staged dA entries per warp
constexpr int kSCache = 32;          // symbolic: C columns of a short row kept from COUNT for FILL
constexpr int kGemmTPB = 512;        // k_gemm_big*
constexpr int kBitmapWords = 51200;  // 200 KB -> windows of 1,638,400 columns (config 4: 6 windows)
constexpr int kWL = 64;              // k_gemm_W: max entries of the A row
constexpr int kWW = 512;             // k_gemm_W: max products w_i
constexpr int kWTPB = 128;           // k_gemm_W: 4 warps
constexpr int kWWarps = kWTPB / 32;

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
template <typename T, int PH, int L, typename IX = int64_t>
__device__ __forceinline__ int64_t s_merge_br(int64_t as, int l, const int32_t *__restrict__ Ai,
                                              const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                              const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                              int32_t *outI, T *outV, const T *dCrow, T *dArow,
                                              double *__restrict__ dB, int64_t cstride = 0)
{
    IX cur[L], end[L];
    int32_t head[L];
    double av[L], dacc[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
        head[t] = INT32_MAX;
        cur[t] = end[t] = 0;
        av[t] = dacc[t] = 0.0;
        if (t < l) {
            const int32_t k = Ai[as + t];
            cur[t] = (IX)Bp[k];
            end[t] = (IX)Bp[k + 1];
            if (PH == PH_NUM || PH == PH_BWD) av[t] = (double)Av[as + t];
            if (cur[t] < end[t]) head[t] = Bi[cur[t]];
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
                    if (dB) atomicAdd(&dB[cur[t]], av[t] * g);
                }
                ++cur[t];
                head[t] = cur[t] < end[t] ? Bi[cur[t]] : INT32_MAX;
            }
        }
        if (PH == PH_FILL) outI[c] = v;
        if (PH == PH_COUNT && outI && c < kSCache) outI[c * cstride] = v;  // FILL's copy (k_gemm_S `cache`)
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
template <typename T, int PH, int L, typename IX = int64_t>
__device__ __forceinline__ int64_t s_merge_bl(int64_t as, int l, const int32_t *__restrict__ Ai,
                                              const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                              const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                              int32_t *outI, T *outV, const T *dCrow, T *dArow,
                                              double *__restrict__ dB)
{
    constexpr bool VAL = PH == PH_NUM || PH == PH_BWD;
    IX cur[L];        // position in B of list t's head
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
            cur[t] = (IX)Bp[k];
            rem[t] = (int)(Bp[k + 1] - Bp[k]);
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
                if (dB && mt) atomicAdd(&dB[cur[t]], av[t] * g);
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

template <typename T, int PH, int L, typename IX>
__device__ __forceinline__ int64_t s_merge(int64_t as, int l, const int32_t *__restrict__ Ai,
                                           const T *__restrict__ Av, const int64_t *__restrict__ Bp,
                                           const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                           int32_t *outI, T *outV, const T *dCrow, T *dArow, double *__restrict__ dB,
                                           int64_t cstride)
{
    if constexpr (PH == PH_NUM || (PH == PH_BWD && CSRK_S_BWD_BL))
        return s_merge_bl<T, PH, L, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB);
    else
        return s_merge_br<T, PH, L, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, cstride);
}

template <typename T, int PH, typename IX = int64_t>
__global__ __launch_bounds__(kSTPB, kSMinBlocks) void k_gemm_S(int64_t m, const int64_t *__restrict__ Ap,
                                                  const int32_t *__restrict__ Ai, const T *__restrict__ Av,
                                                  const int64_t *__restrict__ Bp, const int32_t *__restrict__ Bi,
                                                  const T *__restrict__ Bv, int64_t *__restrict__ Cp,
                                                  int32_t *__restrict__ Ci, T *__restrict__ Cv,
                                                  const T *__restrict__ dC, T *__restrict__ dA, double *__restrict__ dB,
                                                  BigList wl, BigList big, int use_stage,
                                                  int32_t *__restrict__ cache)
{
    pdl_wait();
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
    int64_t ll = 0;
    // rows whose columns COUNT kept (flag byte after the cache slots): FILL needs no
    // classification (no A-row / B-row-length reads), the row is short by construction
    uint8_t *cflag = cache ? reinterpret_cast<uint8_t *>(cache + m * kSCache) : nullptr;
    const bool pre = PH == PH_FILL && cflag && valid && cflag[i];
    if (valid) {
        as = Ap[i];
        ll = Ap[i + 1] - as;
        l = ll > kSMaxL ? kSMaxL + 1 : (int)ll;
        if (l <= kSMaxL && !pre)
            for (int t = 0; t < l; ++t) {
                const int32_t k = Ai[as + t];
                w += Bp[k + 1] - Bp[k];
            }
    }
    const bool isS = valid && (pre || (l <= kSMaxL && w <= kSMaxW));
    // queue the other rows (warp-aggregated): l_i <= kWL to the warp path, longer to the CTA path
    const bool toW = valid && !isS && ll <= kWL;
    const unsigned wmask = __ballot_sync(0xffffffffu, toW);
    if (wmask) {
        int base = 0;
        if (lane == 0) base = atomicAdd(wl.count, __popc(wmask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (toW) wl.rows[base + __popc(wmask & ((1u << lane) - 1))] = (int32_t)i;
    }
    const unsigned bigmask = __ballot_sync(0xffffffffu, valid && !isS && !toW);
    if (bigmask) {
        int base = 0;
        if (lane == 0) base = atomicAdd(big.count, __popc(bigmask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (valid && !isS && !toW) big.rows[base + __popc(bigmask & ((1u << lane) - 1))] = (int32_t)i;
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
    bool unc = false;
    if (isS) {
        const int64_t cs = PH == PH_COUNT ? 0 : Cp[i];
        int32_t *outI = PH == PH_FILL ? (stage ? si + (cs - c_lo) : Ci + cs)
                                      : (PH == PH_COUNT && cache ? cache + i : nullptr);
        T *outV = PH == PH_NUM ? (stage ? sv + (cs - c_lo) : Cv + cs) : nullptr;
        const T *dCrow = PH == PH_BWD ? (stage ? sv + (cs - c_lo) : dC + cs) : nullptr;
        T *dArow = (PH == PH_BWD && dA) ? (stage ? s_dA_w + (as - a_lo) : dA + as) : nullptr;
        int64_t cnt = 0;
        // FILL of a row whose columns COUNT kept (<= kSCache of them): a copy, no second merge
        const int nfill = PH == PH_FILL && cache ? (int)(Cp[i + 1] - cs) : kSCache + 1;
        if (PH == PH_FILL && nfill <= kSCache) {
            // slot c of every row is contiguous (cache[c m + i]): the warp's loads coalesce; a batch
            // of 8 loads is issued before its stores (independent DRAM round trips in flight)
            for (int c0 = 0; c0 < nfill; c0 += 8) {
                int32_t q[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    q[u] = c0 + u < nfill ? __ldcs(cache + (int64_t)(c0 + u) * m + i) : 0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (c0 + u < nfill) outI[c0 + u] = q[u];
            }
        } else
        switch (Lw) {
        case 1: cnt = s_merge<T, PH, 1, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 2: cnt = s_merge<T, PH, 2, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 3: cnt = s_merge<T, PH, 3, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 4: cnt = s_merge<T, PH, 4, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 5: cnt = s_merge<T, PH, 5, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 6: cnt = s_merge<T, PH, 6, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 7: cnt = s_merge<T, PH, 7, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        case 8: cnt = s_merge<T, PH, 8, IX>(as, l, Ai, Av, Bp, Bi, Bv, outI, outV, dCrow, dArow, dB, m); break;
        default: break;  // l == 0: empty row
        }
        if (PH == PH_COUNT) Cp[i + 1] = cnt;
        if (PH == PH_COUNT && cflag) cflag[i] = cnt <= kSCache ? 1 : 0;
        unc = PH == PH_COUNT && cflag && cnt > kSCache;
    } else if (PH == PH_COUNT && cflag && valid) {
        cflag[i] = 0;
    }
    if (PH == PH_COUNT && cflag) {   // short rows whose columns the cache could not keep (wl.count[3])
        const unsigned um = __ballot_sync(0xffffffffu, unc);
        if (um && lane == 0) atomicAdd(wl.count + 3, __popc(um));
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

// Position index of a sorted C row (columns key[0..nc), distinct) held in shared memory: the
// column range [key[0], key[nc-1]] is cut into NB buckets by a monotone map (the identity when
// the range has at most NB columns, else a 32-bit fixed-point scale), and bst[b] = first position
// whose column maps to a bucket >= b (bst[NB] = nc).  A column j of the row then lies in
// [bst[b(j)], bst[b(j)+1]) -- a binary search over ~nc / NB entries instead of log2(nc) steps
// (config 4's C rows have uniformly spread columns: ~1-2 entries per bucket).  Exact for any
// column distribution: a clustered row only makes its buckets longer.
struct PosIdx {
    int32_t mn;
    uint32_t scale;   // 0: identity map
};
__device__ __forceinline__ int pos_bucket(const PosIdx &x, int32_t j)
{
    const uint32_t d = (uint32_t)(j - x.mn);
    return (int)(x.scale ? __umulhi(d, x.scale) : d);
}
template <int NB>
__device__ __forceinline__ PosIdx pos_index_params(const int32_t *key, int nc)
{
    PosIdx x;
    x.mn = nc > 0 ? key[0] : 0;
    const uint64_t span = nc > 0 ? (uint64_t)(key[nc - 1] - x.mn) + 1 : 1;
    x.scale = span <= (uint64_t)NB ? 0u : (uint32_t)(((uint64_t)NB << 32) / span);
    return x;
}
// build bst[0..NB] with threads t = 0..nt-1 (the caller synchronises before and after)
template <int NB>
__device__ __forceinline__ void pos_index_build(const int32_t *key, int nc, const PosIdx &x, uint16_t *bst, int t,
                                                int nt)
{
    for (int q = t; q < nc; q += nt) {
        const int bq = pos_bucket(x, key[q]);
        const int bp = q > 0 ? pos_bucket(x, key[q - 1]) : -1;
        for (int b = bp + 1; b <= bq; ++b) bst[b] = (uint16_t)q;
    }
    const int blast = nc > 0 ? pos_bucket(x, key[nc - 1]) : -1;
    for (int b = blast + 1 + t; b <= NB; b += nt) bst[b] = (uint16_t)nc;
}
// position of column j (present in the row)
__device__ __forceinline__ int pos_find(const int32_t *key, const uint16_t *bst, const PosIdx &x, int32_t j)
{
    const int b = pos_bucket(x, j);
    int lo = bst[b], hi = bst[b + 1];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key[mid] < j) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- medium rows: warp per row
// per-phase layout (shared memory decides how many warps an SM holds): COUNT keeps a hash table
// of 2 WW columns, FILL the WW gathered columns, NUM / BWD the C row (columns + fp64 values) and
// the row's A values / dA
template <int WW, int WL, int PH>
struct WSmemT {
    static constexpr bool VAL = PH == PH_NUM || PH == PH_BWD;
    double val[PH == PH_FILL ? 1 : WW];  // NUM: row accumulator; BWD: dC row; COUNT: hash table (2 WW int32)
    double dA[VAL ? WL : 1];             // BWD: dA of the row's A entries
    double av[VAL ? WL : 1];             // NUM / BWD: A values of the row
    int64_t bs[WL];                      // start in B of list t
    int32_t key[PH == PH_COUNT ? 1 : WW];// FILL: product columns (sorted); NUM / BWD: C row columns
    int32_t off[WL + 1];                 // flat offset of list t (off[l] = w)
    int32_t tmp[PH == PH_FILL ? WW : 1]; // FILL: the bucket-sorted columns
    int32_t cnt[PH == PH_FILL ? WW / 2 : 1];  // FILL: bucket counts / offsets
    uint16_t bst[VAL ? WW / 2 + 1 : 1];       // NUM / BWD: position index of the C row (PosIdx)
    uint8_t lst[PH == PH_NUM ? WW : 1];       // NUM: flat product -> its list (A entry) of the row
};
// symbolic-only warp class for 512 < w <= kW2W (config-4 rows the CTA path sorted slowly)
constexpr int kW2W = 1024;

// last t in [0, l) with off[t] <= e (the list holding flat product e; empty lists skipped)
__device__ __forceinline__ int w_list_of(const int32_t *off, int l, int e)
{
    int lo = 0, hi = l - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint32_t w_hash(int32_t j) { return (uint32_t)j * 0x9E3779B1u; }


// Bitonic sort of P = 32 R keys held in registers, element r * 32 + lane in v[r] (ascending):
// partners within a lane are register compare-exchanges, partners across lanes shuffles.
template <int R>
__device__ __forceinline__ void warp_bitonic(int32_t (&v)[R], int lane)
{
    constexpr int P = 32 * R;
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int pr = r ^ jr;
                    if (pr > r) {
                        const bool asc = (((r << 5) + lane) & k) == 0;
                        const int32_t a = v[r], b = v[pr];
                        const bool sw = (a > b) == asc;
                        v[r] = sw ? b : a;
                        v[pr] = sw ? a : b;
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool asc = (((r << 5) + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    v[r] = (lower == asc) ? min(v[r], o) : max(v[r], o);
                }
            }
        }
    }
}

// FILL of a warp-path row: sort the w gathered columns, write the distinct ones in order
template <int R>
__device__ __forceinline__ void w_sort_fill(const int32_t *key, int w, int32_t *out, int lane)
{
    int32_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = (r << 5) + lane < w ? key[(r << 5) + lane] : INT32_MAX;
    warp_bitonic<R>(v, lane);
    int base = 0;
    int32_t carry = 0;  // last key of the previous register row (lane 31)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = (r << 5) + lane;
        int32_t prev = __shfl_up_sync(0xffffffffu, v[r], 1);
        if (lane == 0) prev = carry;
        const bool f = e < w && (e == 0 || v[r] != prev);
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) out[base + __popc(m & ((1u << lane) - 1))] = v[r];
        base += __popc(m);
        carry = __shfl_sync(0xffffffffu, v[r], 31);
    }
}

// FILL fallback of a warp-path row with w > 64 whose columns overflow a bucket (clustered or
// repeated columns): bitonic sort of the P = pow2ceil(w) <= WW keys in shared memory (no register
// arrays: keeps the kernel's register count, hence its occupancy, at the bucket path's), then the
// distinct ones written in order
__device__ __noinline__ void w_smem_sort_fill(int32_t *key, int w, int32_t *out, int lane)
{
    const unsigned FULL = 0xffffffffu;
    int P = 32;
    while (P < w) P <<= 1;
    for (int e = w + lane; e < P; e += 32) key[e] = INT32_MAX;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool asc = (i & k) == 0;
                    const int32_t a = key[i], b = key[ixj];
                    if ((a > b) == asc) { key[i] = b; key[ixj] = a; }
                }
            }
            __syncwarp();
        }
    int base = 0;
    for (int e0 = 0; e0 < w; e0 += 32) {
        const int e = e0 + lane;
        const int32_t v = e < w ? key[e] : 0;
        const bool f = e < w && (e == 0 || v != key[e - 1]);
        const unsigned m = __ballot_sync(FULL, f);
        if (f) out[base + __popc(m & ((1u << lane) - 1))] = v;
        base += __popc(m);
    }
    __syncwarp();
}

// FILL of a warp-path row by a bucket sort (no compare network): the w columns are counted into
// WW/2 buckets of equal width over [min, max] (shared-memory atomics), the counts scanned, the
// columns scattered to their buckets, each lane insertion-sorts its WW/64 consecutive buckets, and
// the distinct columns are written in order.  Linear in w for spread columns (config 4: uniform
// columns, ~2 per bucket); returns false without writing when a bucket holds more than kBucketMax
// columns (clustered or repeated columns) -- the caller then runs the bitonic network.
constexpr int kBucketMax = 16;
template <int WW>
__device__ __forceinline__ bool w_bucket_fill(const int32_t *key, int32_t *tmp, int32_t *cnt, int w, int32_t *out,
                                              int lane)
{
    constexpr int NB = WW / 2, PER = NB / 32;
    const unsigned FULL = 0xffffffffu;
    __syncwarp();   // the gathered columns of every lane are in key[]
    int32_t mn = INT32_MAX, mx = 0;
    for (int e = lane; e < w; e += 32) {
        const int32_t k = key[e];
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    mn = (int32_t)__reduce_min_sync(FULL, (unsigned)mn);
    mx = (int32_t)__reduce_max_sync(FULL, (unsigned)mx);
    const uint64_t span = (uint64_t)(mx - mn) + 1;
    // monotone bucket map without a per-key 64-bit division: identity when the span has at most
    // NB columns, else floor((k - mn) * floor(2^32 NB / span) / 2^32) < NB
    const uint32_t scale = span <= (uint64_t)NB ? 0u : (uint32_t)(((uint64_t)NB << 32) / span);
    auto bucket = [&](int32_t k) {
        const uint32_t d = (uint32_t)(k - mn);
        return (int)(scale ? __umulhi(d, scale) : d);
    };
    for (int b = lane; b < NB; b += 32) cnt[b] = 0;
    __syncwarp();
    for (int e = lane; e < w; e += 32) atomicAdd(&cnt[bucket(key[e])], 1);
    __syncwarp();
    int loc[PER], sum = 0, mxc = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        loc[q] = cnt[lane * PER + q];
        sum += loc[q];
        mxc = loc[q] > mxc ? loc[q] : mxc;
    }
    if (__reduce_max_sync(FULL, (unsigned)mxc) > (unsigned)kBucketMax) return false;
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    const int s0 = x - sum, s1 = x;   // this lane's region of tmp
    int run = s0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        cnt[lane * PER + q] = run;
        run += loc[q];
    }
    __syncwarp();
    for (int e = lane; e < w; e += 32) {
        const int32_t k = key[e];
        tmp[atomicAdd(&cnt[bucket(k)], 1)] = k;
    }
    __syncwarp();
    for (int i = s0 + 1; i < s1; ++i) {   // buckets are ordered: an element only moves inside its bucket
        const int32_t v = tmp[i];
        int j = i - 1;
        while (j >= s0 && tmp[j] > v) {
            tmp[j + 1] = tmp[j];
            --j;
        }
        tmp[j + 1] = v;
    }
    __syncwarp();
    int base = 0;
    for (int e0 = 0; e0 < w; e0 += 32) {
        const int e = e0 + lane;
        const int32_t v = e < w ? tmp[e] : 0;
        const bool f = e < w && (e == 0 || v != tmp[e - 1]);
        const unsigned m = __ballot_sync(FULL, f);
        if (f) out[base + __popc(m & ((1u << lane) - 1))] = v;
        base += __popc(m);
    }
    return true;
}

#ifndef CSRK_W_MINB
#define CSRK_W_MINB 1
#endif
#ifndef CSRK_W_LMAP
#define CSRK_W_LMAP 1
#endif
#ifndef CSRK_W_BUCKET
#define CSRK_W_BUCKET 1
#endif
template <typename T, int PH, bool W2 = false>
__global__ __launch_bounds__(kWTPB, CSRK_W_MINB) void k_gemm_W(BigList wl, BigList big, BigList w2l, const int64_t *__restrict__ Ap,
                                                  const int32_t *__restrict__ Ai, const T *__restrict__ Av,
                                                  const int64_t *__restrict__ Bp, const int32_t *__restrict__ Bi,
                                                  const T *__restrict__ Bv, int64_t *__restrict__ Cp,
                                                  int32_t *__restrict__ Ci, T *__restrict__ Cv,
                                                  const T *__restrict__ dC, T *__restrict__ dA, double *__restrict__ dB)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int WW = W2 ? kW2W : kWW;
    using SM = WSmemT<WW, kWL, PH>;
    SM &S = reinterpret_cast<SM *>(s_dyn)[warp];
    const unsigned FULL = 0xffffffffu;
    const int nrows = *(volatile int *)wl.count;
    constexpr bool knob_bucket = CSRK_W_BUCKET != 0;
    for (int it = blockIdx.x * kWWarps + warp; it < nrows; it += gridDim.x * kWWarps) {
        __syncwarp();  // the previous row's shared-memory reads complete before this row's writes
        const int64_t i = wl.rows[it];
        const int64_t as = Ap[i];
        const int l = (int)(Ap[i + 1] - as);
        // flat offsets of the l lists (warp scan of the B row lengths)
        int64_t run = 0;
        for (int t0 = 0; t0 < l; t0 += 32) {
            const int t = t0 + lane;
            int64_t len = 0, bs = 0;
            if (t < l) {
                const int32_t k = Ai[as + t];
                bs = Bp[k];
                len = Bp[k + 1] - bs;
            }
            int64_t x = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            const int64_t excl = run + x - len;
            if (t < l) {
                S.off[t] = excl > WW ? WW + 1 : (int32_t)excl;
                S.bs[t] = bs;
                if (PH == PH_NUM || PH == PH_BWD) S.av[t] = (double)Av[as + t];
            }
            run += __shfl_sync(FULL, x, 31);
        }
        if (run > WW) {  // too many products for the warp: the symbolic W2 class or the CTA path
            if (lane == 0) {
                if (!W2 && w2l.rows && run <= kW2W)
                    w2l.rows[atomicAdd(w2l.count, 1)] = (int32_t)i;
                else
                    big.rows[atomicAdd(big.count, 1)] = (int32_t)i;
            }
            continue;
        }
        const int w = (int)run;
        if (lane == 0) S.off[l] = w;
        __syncwarp();
        const int64_t cs = PH == PH_COUNT ? 0 : Cp[i];
        const int nc = PH == PH_COUNT ? 0 : (int)(Cp[i + 1] - cs);
        int32_t *tab = reinterpret_cast<int32_t *>(S.val);
        int H = 64;
        if (PH == PH_COUNT) {
            while (H < 2 * w) H <<= 1;
            for (int e = lane; e < H; e += 32) tab[e] = -1;
        } else if (PH == PH_NUM || PH == PH_BWD) {
            for (int c = lane; c < nc; c += 32) {
                S.key[c] = Ci[cs + c];
                S.val[c] = PH == PH_NUM ? 0.0 : (double)dC[cs + c];
            }
            if (PH == PH_BWD)
                for (int t = lane; t < l; t += 32) S.dA[t] = 0.0;
        }
        __syncwarp();
        PosIdx px{};
        if (PH == PH_NUM || PH == PH_BWD) {
            px = pos_index_params<WW / 2>(S.key, nc);
            pos_index_build<WW / 2>(S.key, nc, px, S.bst, lane, 32);
            __syncwarp();
        }
        int cnt = 0;
        int t = w > 0 ? w_list_of(S.off, l, lane < w ? lane : 0) : 0;
        constexpr bool LMAP = CSRK_W_LMAP && PH == PH_NUM;   // (measured: numeric -6 %, symbolic / backward slower)
        if (LMAP) {   // product -> list map: one shared load per product instead of a walk
            for (int tq = lane; tq < l; tq += 32)
                for (int e = S.off[tq]; e < S.off[tq + 1]; ++e) S.lst[e] = (uint8_t)tq;
            __syncwarp();
        }
#ifndef CSRK_W_U
#define CSRK_W_U 8
#endif
        constexpr int U = CSRK_W_U;  // products gathered per lane before use: U loads in flight
        for (int e00 = 0; e00 < w; e00 += 32 * U) {
            int32_t jv[U];
            double bv[U];
            int64_t bb[U];
            int tv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e00 + u * 32 + lane;
                const bool ok = e < w;
                if (LMAP) t = ok ? S.lst[e] : t;
                else
                    while (ok && t + 1 < l && S.off[t + 1] <= e) ++t;
                tv[u] = ok ? t : -1;
                bb[u] = ok ? S.bs[t] + (e - S.off[t]) : 0;
                jv[u] = ok ? Bi[bb[u]] : 0;
                bv[u] = (PH == PH_NUM || PH == PH_BWD) && ok ? (double)Bv[bb[u]] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e00 + u * 32 + lane;
                const bool ok = e < w;
                const int32_t j = jv[u];
                if (PH == PH_COUNT && ok) {
                    uint32_t h = w_hash(j) & (uint32_t)(H - 1);
                    while (true) {
                        const int32_t old = atomicCAS(&tab[h], -1, j);
                        if (old == -1) { ++cnt; break; }
                        if (old == j) break;
                        h = (h + 1) & (uint32_t)(H - 1);
                    }
                }
                if (PH == PH_FILL && ok) S.key[e] = j;
                if (PH == PH_NUM && ok) {  // (a match_any merge instead of the atomic: 75 vs 72 ms, config 4)
                    const int pos = pos_find(S.key, S.bst, px, j);
                    atomicAdd(&S.val[pos], S.av[tv[u]] * bv[u]);
                }
                if (PH == PH_BWD && e00 + u * 32 < w) {
                    double g = 0.0, v = 0.0;
                    if (ok) {
                        const int pos = pos_find(S.key, S.bst, px, j);
                        g = S.val[pos];
                        v = g * bv[u];
                        if (dB) atomicAdd(&dB[bb[u]], S.av[tv[u]] * g);
                    }
                    // segmented sum of v over lanes with equal list (nondecreasing in the lane)
                    const int tt = tv[u];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double y = __shfl_up_sync(FULL, v, o);
                        const int ty = __shfl_up_sync(FULL, tt, o);
                        if (lane >= o && ty == tt) v += y;
                    }
                    const int tn = __shfl_down_sync(FULL, tt, 1);
                    if (ok && (lane == 31 || tn != tt)) S.dA[tt] += v;  // one tail per list per step
                    __syncwarp();
                }
            }
        }
        if (PH == PH_COUNT) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
            if (lane == 0) Cp[i + 1] = cnt;
        }
        if (PH == PH_FILL && w > 64 && knob_bucket && w_bucket_fill<WW>(S.key, S.tmp, S.cnt, w, Ci + cs, lane)) {
            // sorted by buckets
        } else if (PH == PH_FILL) {
            __syncwarp();
            if (w <= 32) w_sort_fill<1>(S.key, w, Ci + cs, lane);
            else if (w <= 64) w_sort_fill<2>(S.key, w, Ci + cs, lane);
            else w_smem_sort_fill(S.key, w, Ci + cs, lane);   // rare: a bucket overflowed
        }
        __syncwarp();
        if (PH == PH_NUM)
            for (int c = lane; c < nc; c += 32) Cv[cs + c] = (T)S.val[c];
        if (PH == PH_BWD && dA)
            for (int tq = lane; tq < l; tq += 32) dA[as + tq] = (T)S.dA[tq];
        __syncwarp();
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


// CTA-wide FILL of a big row (the CTA analogue of w_bucket_fill): the w gathered columns in key[]
// are counted into NB = kMMaxW / 2 buckets of equal width over [min, max], scanned, scattered into
// tmp, every thread insertion-sorts its NB / kGemmTPB consecutive buckets, and writes the distinct
// columns of its region at their place (a block scan of the per-thread unique counts).  Returns
// false without writing when a bucket holds more than kBucketMax columns.
__device__ __forceinline__ int64_t block_max_i64(int64_t v, int64_t *s_red)
{
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y > v ? y : v;
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    int64_t t = s_red[0];
    for (int i = 1; i < kGemmTPB / 32; ++i) t = s_red[i] > t ? s_red[i] : t;
    __syncthreads();
    return t;
}

__device__ bool cta_bucket_fill(const int32_t *key, int32_t *tmp, int32_t *cnt, int w, int32_t *out, int64_t *s_red)
{
    constexpr int NB = kMMaxW / 2, PER = NB / kGemmTPB;
    int32_t mn = INT32_MAX, mx = 0;
    for (int e = threadIdx.x; e < w; e += kGemmTPB) {
        const int32_t k = key[e];
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    mn = (int32_t)-block_max_i64(-(int64_t)mn, s_red);
    mx = (int32_t)block_max_i64(mx, s_red);
    const uint64_t span = (uint64_t)(mx - mn) + 1;
    const uint32_t scale = span <= (uint64_t)NB ? 0u : (uint32_t)(((uint64_t)NB << 32) / span);  // as w_bucket_fill
    auto bucket = [&](int32_t k) {
        const uint32_t d = (uint32_t)(k - mn);
        return (int)(scale ? __umulhi(d, scale) : d);
    };
    for (int b = threadIdx.x; b < NB; b += kGemmTPB) cnt[b] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < w; e += kGemmTPB) atomicAdd(&cnt[bucket(key[e])], 1);
    __syncthreads();
    int loc[PER], sum = 0, mxc = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        loc[q] = cnt[threadIdx.x * PER + q];
        sum += loc[q];
        mxc = loc[q] > mxc ? loc[q] : mxc;
    }
    if (block_max_i64(mxc, s_red) > kBucketMax) return false;
    int64_t tot;
    const int s0 = (int)block_excl_scan_i64(sum, s_red, tot), s1 = s0 + sum;
    int run = s0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        cnt[threadIdx.x * PER + q] = run;
        run += loc[q];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < w; e += kGemmTPB) {
        const int32_t k = key[e];
        tmp[atomicAdd(&cnt[bucket(k)], 1)] = k;
    }
    __syncthreads();
    for (int i = s0 + 1; i < s1; ++i) {
        const int32_t v = tmp[i];
        int j = i - 1;
        while (j >= s0 && tmp[j] > v) {
            tmp[j + 1] = tmp[j];
            --j;
        }
        tmp[j + 1] = v;
    }
    __syncthreads();
    int64_t mine = 0;
    for (int e = s0; e < s1; ++e) mine += (e == 0 || tmp[e] != tmp[e - 1]);
    int64_t o = block_excl_scan_i64(mine, s_red, tot);
    for (int e = s0; e < s1; ++e)
        if (e == 0 || tmp[e] != tmp[e - 1]) out[o++] = tmp[e];
    __syncthreads();
    return true;
}

// ---------------------------------------------------------------- big rows
// Rows the S and W paths pass on (l_i > kWL or w_i > kWW: power-law heads).  Their products are
// enumerated flat: k_big_prep stores, at every A position a of a big row, loff[a] = the flat
// offset of list a's first product within the row, and w_r.  Each thread then walks a
// CONTIGUOUS run of products (one binary search in loff, then linear), so long B rows are
// spread over many threads and the loads of a thread are sequential.
//   symbolic  one CTA per row: w <= kMMaxW -> products gathered to shared memory, bitonic sort,
//             unique; else bitmap windows over the column range (sorted for free).
//   numeric / backward  work items = windows of kValSm entries of the C row (k_big_items:
//             single-CTA scan of the per-row window counts), many CTAs per long row; see
//             k_gemm_big_win.
constexpr int kValSm = 4096;

struct BigRows {
    const int32_t *rows;
    const int *count;
    int64_t *loff;   // [nnz(A)]
    int64_t *w;      // [m]  products of the r-th big row
    int32_t *items;  // [m + 1] item offsets
    int32_t *huge;   // symbolic (nullable): big-row ordinals r with w > kMMaxW, appended by k_big_prep
    int *nhuge;
};

// last a in [lo, hi) with loff[a] <= e (the list holding product e; empty lists skipped)
__device__ __forceinline__ int64_t big_list_of(const int64_t *loff, int64_t lo, int64_t hi, int64_t e)
{
    hi -= 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (loff[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ __launch_bounds__(kGemmTPB) void k_big_prep(BigRows br, const int64_t *__restrict__ Ap,
                                                       const int32_t *__restrict__ Ai, const int64_t *__restrict__ Bp)
{
    // one warp per big row (most have 33..512 A entries: a CTA per row left most threads idle
    // behind three block barriers per 512 entries); lanes over the row's entries, warp scans
    pdl_wait();
    const int n = *(volatile const int *)br.count;
    const int lane = threadIdx.x & 31;
    const int warps = (int)(gridDim.x * (kGemmTPB / 32));
    for (int r = blockIdx.x * (kGemmTPB / 32) + (threadIdx.x >> 5); r < n; r += warps) {
        const int64_t i = br.rows[r];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        int64_t run = 0;
        for (int64_t a0 = as; a0 < ae; a0 += 32) {
            const int64_t a = a0 + lane;
            int64_t len = 0;
            if (a < ae) {
                const int32_t k = Ai[a];
                len = Bp[k + 1] - Bp[k];
            }
            int64_t x = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (a < ae) br.loff[a] = run + x - len;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
            br.w[r] = run;
            if (br.huge && run > kMMaxW) br.huge[atomicAdd(br.nhuge, 1)] = r;
        }
    }
}

constexpr int kItemsTPB = 1024;

// walk products [e_lo, e_hi) of the row: f(e, a, b) with a = A position, b = B position
template <typename F>
__device__ __forceinline__ void big_walk(const int64_t *__restrict__ loff, const int32_t *__restrict__ Ai,
                                         const int64_t *__restrict__ Bp, int64_t as, int64_t ae, int64_t e_lo,
                                         int64_t e_hi, F &&f)
{
    if (e_lo >= e_hi) return;
    int64_t a = big_list_of(loff, as, ae, e_lo);
    int64_t lo = loff[a], bs = Bp[Ai[a]];
    int64_t nx = a + 1 < ae ? loff[a + 1] : INT64_MAX;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        while (e >= nx) {
            ++a;
            lo = nx;
            nx = a + 1 < ae ? loff[a + 1] : INT64_MAX;
            bs = Bp[Ai[a]];
        }
        f(e, a, bs + (e - lo));
    }
}

// ---------------------------------------------------------------- big rows: symbolic
#ifndef CSRK_BIG_HASH
#define CSRK_BIG_HASH 1   // big-row symbolic: hash-set COUNT + bucket-sort FILL (0: bitonic sort for both)
#endif
constexpr bool kBigHash = CSRK_BIG_HASH != 0;
template <int PH, bool HUGE>
__global__ __launch_bounds__(kGemmTPB) void k_gemm_big_sym(BigRows br, int64_t ncolsB,
                                                           const int64_t *__restrict__ Ap,
                                                           const int32_t *__restrict__ Ai,
                                                           const int64_t *__restrict__ Bp,
                                                           const int32_t *__restrict__ Bi, int64_t *__restrict__ Cp,
                                                           int32_t *__restrict__ Ci)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *s_key = reinterpret_cast<int32_t *>(smem);   // kMMaxW keys (sort path)
    uint32_t *bm = reinterpret_cast<uint32_t *>(smem);    // kBitmapWords (bitmap path)
    __shared__ int64_t s_red[kGemmTPB / 32];
    const int nrows = *(volatile const int *)br.count;
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int64_t i = br.rows[r];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        const int64_t w = br.w[r];
        if (HUGE != (w > kMMaxW)) continue;  // the other kernel takes this row
        if (!HUGE) {
            const int64_t per = (w + kGemmTPB - 1) / kGemmTPB;
            const int64_t e_lo = threadIdx.x * per, e_hi = e_lo + per < w ? e_lo + per : w;
            if (PH == PH_COUNT && kBigHash) {
                // distinct columns by a shared-memory hash set (no sort needed to count)
                int32_t *tab = s_key;
                const int H = pow2ceil_i((int)(2 * w > 64 ? 2 * w : 64));
                for (int e = threadIdx.x; e < H; e += kGemmTPB) tab[e] = -1;
                __syncthreads();
                int64_t mine = 0;
                big_walk(br.loff, Ai, Bp, as, ae, e_lo, e_hi, [&](int64_t, int64_t, int64_t b) {
                    const int32_t j = __ldg(Bi + b);
                    uint32_t h = w_hash(j) & (uint32_t)(H - 1);
                    while (true) {
                        const int32_t old = atomicCAS(&tab[h], -1, j);
                        if (old == -1) { ++mine; break; }
                        if (old == j) break;
                        h = (h + 1) & (uint32_t)(H - 1);
                    }
                });
                const int64_t tot = block_sum_i64(mine, s_red);
                if (threadIdx.x == 0) Cp[i + 1] = tot;
                __syncthreads();
                continue;
            }
            big_walk(br.loff, Ai, Bp, as, ae, e_lo, e_hi, [&](int64_t e, int64_t, int64_t b) { s_key[e] = Bi[b]; });
            const int wn = (int)w;
            if (PH == PH_FILL && kBigHash) {
                __syncthreads();
                if (cta_bucket_fill(s_key, s_key + kMMaxW, s_key + 2 * kMMaxW, wn, Ci + Cp[i], s_red)) continue;
            }
            const int P = pow2ceil_i(wn > 0 ? wn : 1);
            for (int e = wn + threadIdx.x; e < P; e += kGemmTPB) s_key[e] = INT32_MAX;
            __syncthreads();
            bitonic_keys(s_key, P);
            const int pe = (P + kGemmTPB - 1) / kGemmTPB;
            const int e0 = threadIdx.x * pe;
            int64_t mine = 0;
            for (int e = e0; e < e0 + pe && e < wn; ++e) mine += (e == 0 || s_key[e] != s_key[e - 1]);
            if (PH == PH_COUNT) {
                const int64_t tot = block_sum_i64(mine, s_red);
                if (threadIdx.x == 0) Cp[i + 1] = tot;
            } else {
                int64_t tot;
                int64_t o = Cp[i] + block_excl_scan_i64(mine, s_red, tot);
                for (int e = e0; e < e0 + pe && e < wn; ++e)
                    if (e == 0 || s_key[e] != s_key[e - 1]) Ci[o++] = s_key[e];
            }
            __syncthreads();
            continue;
        }
        // bitmap windows over [0, ncolsB)
        const int64_t W = (int64_t)kBitmapWords * 32;
        const int64_t per = (w + kGemmTPB - 1) / kGemmTPB;
        const int64_t e_lo = threadIdx.x * per, e_hi = e_lo + per < w ? e_lo + per : w;
        int64_t done = 0;
        for (int64_t w0 = 0; w0 < ncolsB; w0 += W) {
            for (int e = threadIdx.x; e < kBitmapWords; e += kGemmTPB) bm[e] = 0u;
            __syncthreads();
            big_walk(br.loff, Ai, Bp, as, ae, e_lo, e_hi, [&](int64_t, int64_t, int64_t b) {
                const int64_t j = Bi[b];
                if (j >= w0 && j < w0 + W) atomicOr(&bm[(j - w0) >> 5], 1u << (j & 31));
            });
            __syncthreads();
            constexpr int pw = kBitmapWords / kGemmTPB;
            const int q0 = threadIdx.x * pw;
            int64_t mine = 0;
            for (int q = q0; q < q0 + pw; ++q) mine += __popc(bm[q]);
            int64_t tot;
            const int64_t off = block_excl_scan_i64(mine, s_red, tot);
            if (PH == PH_FILL) {
                int64_t o = Cp[i] + done + off;
                for (int q = q0; q < q0 + pw; ++q) {
                    uint32_t bits = bm[q];
                    while (bits) {
                        const int bpos = __ffs(bits) - 1;
                        bits &= bits - 1;
                        Ci[o++] = (int32_t)(w0 + (int64_t)q * 32 + bpos);
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

// Huge rows (w > kMMaxW), symbolic: one 8-CTA thread-block CLUSTER per row.  CTA c of the cluster
// owns the bitmap of columns [s0 + c W, s0 + (c + 1) W) (W = 1.6M columns, 200 KB of shared memory),
// so a super-window of 8 W = 13.1M columns (all of config 4's 8.4M) is covered in ONE pass over the
// row's products: the 4096 threads of the cluster split the products into equal contiguous runs and
// set each column's bit in the owning CTA's bitmap through distributed shared memory (remote
// atomicOr).  Each CTA then counts its window (block scan of the per-thread popcounts), the window
// counts are exchanged over DSMEM for the offsets, and FILL writes the set bits in ascending order.
// (The one-CTA-per-row form walked every product once per 1.6M-column window, and the largest rows
// -- 500K products -- set the kernel's critical path.)
constexpr int kHugeCl = 8;
template <int PH>
__global__ void __cluster_dims__(kHugeCl, 1, 1) __launch_bounds__(kGemmTPB)
    k_gemm_huge_sym(BigRows br, int64_t ncolsB, const int64_t *__restrict__ Ap, const int32_t *__restrict__ Ai,
                    const int64_t *__restrict__ Bp, const int32_t *__restrict__ Bi, int64_t *__restrict__ Cp,
                    int32_t *__restrict__ Ci)
{
    namespace cg = cooperative_groups;
    pdl_wait();
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bm = reinterpret_cast<uint32_t *>(smem);
    __shared__ int64_t s_red[kGemmTPB / 32];
    __shared__ int64_t s_cnt;
    const int rank = (int)cl.block_rank();
    const int ncl = (int)(gridDim.x / kHugeCl), cid = (int)(blockIdx.x / kHugeCl);
    const int nh = *(volatile const int *)br.nhuge;
    constexpr int64_t W = (int64_t)kBitmapWords * 32;
    constexpr int64_t SW = W * kHugeCl;
    constexpr int pw = kBitmapWords / kGemmTPB;
    for (int h = cid; h < nh; h += ncl) {
        const int r = br.huge[h];
        const int64_t i = br.rows[r];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        const int64_t w = br.w[r];
        const int64_t per = (w + kHugeCl * kGemmTPB - 1) / (kHugeCl * kGemmTPB);
        const int64_t e_lo = ((int64_t)rank * kGemmTPB + threadIdx.x) * per;
        const int64_t e_hi = e_lo + per < w ? e_lo + per : w;
        int64_t done = 0;
        for (int64_t s0 = 0; s0 < ncolsB; s0 += SW) {
            for (int e = threadIdx.x; e < kBitmapWords; e += kGemmTPB) bm[e] = 0u;
            cl.sync();
            big_walk(br.loff, Ai, Bp, as, ae, e_lo, e_hi, [&](int64_t, int64_t, int64_t b) {
                const int64_t d = (int64_t)__ldg(Bi + b) - s0;
                if (d >= 0 && d < SW) {
                    const int c = (int)(d / W);
                    const int64_t q = d - c * W;
                    atomicOr(cl.map_shared_rank(bm, c) + (q >> 5), 1u << (q & 31));
                }
            });
            cl.sync();
            const int q0 = threadIdx.x * pw;
            int64_t mine = 0;
            for (int q = q0; q < q0 + pw; ++q) mine += __popc(bm[q]);
            int64_t tot;
            const int64_t off = block_excl_scan_i64(mine, s_red, tot);
            if (threadIdx.x == 0) s_cnt = tot;
            cl.sync();
            int64_t before = 0, all = 0;
            for (int c = 0; c < kHugeCl; ++c) {
                const int64_t v = *cl.map_shared_rank(&s_cnt, c);
                before += c < rank ? v : 0;
                all += v;
            }
            if (PH == PH_FILL) {
                int64_t o = Cp[i] + done + before + off;
                const int64_t c0 = s0 + (int64_t)rank * W;
                for (int q = q0; q < q0 + pw; ++q) {
                    uint32_t bits = bm[q];
                    while (bits) {
                        const int bpos = __ffs(bits) - 1;
                        bits &= bits - 1;
                        Ci[o++] = (int32_t)(c0 + (int64_t)q * 32 + bpos);
                    }
                }
            }
            done += all;
            cl.sync();   // remote reads of s_cnt done before it and the bitmaps are reused
        }
        if (PH == PH_COUNT && rank == 0 && threadIdx.x == 0) Cp[i + 1] = done;
    }
}

// ---------------------------------------------------------------- big rows: numeric + backward
// Work item = (big row i, window q): C entries [Cp[i] + q kValSm, +kValSm) of the row -- their
// columns (and dC for the backward) staged in shared memory, C values accumulated in fp64 shared
// memory and written ONCE (no global atomics, no zeroing pass).  Every A entry (i, k) of the row
// contributes the part of B row k whose columns fall in the window's column range [c_lo, c_hi]
// (binary searches in B row k when the row has several windows; the whole B row otherwise): a
// thread per A entry walks short parts, parts longer than 32 products are queued and walked by a
// warp.  Backward: dA_ik = sum_j dC_ij B_kj is a register (fp64) sum per A entry and window --
// stored directly when the row has one window, else added (fp64 atomic) into dA64, the fp64
// target zeroed by k_big_zero; dB_kj += A_ik dC_ij into the fp64 dB target (reading A9).
constexpr int kWinQ = 128;   // queued long parts per item (static shared memory: 3 CTAs per SM)

__device__ __forceinline__ int64_t lbound64(const int32_t *c, int64_t n, int32_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(c + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// single CTA: items[r] = sum_{r' < r} nwin(r'), items[n] = total;  nwin = max(1, ceil(nnz(C_i) / kValSm))
__global__ __launch_bounds__(kItemsTPB) void k_big_items(BigRows br, const int64_t *__restrict__ Cp)
{
    pdl_wait();
    __shared__ int64_t s_w[kItemsTPB / 32];
    const int n = *(volatile const int *)br.count;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t run = 0;
    for (int r0 = 0; r0 < n; r0 += kItemsTPB) {
        const int r = r0 + threadIdx.x;
        int64_t c = 0;
        if (r < n) {
            const int64_t i = br.rows[r];
            const int64_t nc = Cp[i + 1] - Cp[i];
            c = nc > kValSm ? (nc + kValSm - 1) / kValSm : 1;
        }
        int64_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        int64_t off = 0, tot = 0;
        for (int q = 0; q < kItemsTPB / 32; ++q) {
            if (q < warp) off += s_w[q];
            tot += s_w[q];
        }
        if (r < n) br.items[r] = (int32_t)(run + off + x - c);
        run += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) br.items[n] = (int32_t)run;
}

// backward: a big row sums its dA in shared memory when it has one window and at most kDACap A
// entries; otherwise into the fp64 dA target (zeroed first)
constexpr int kDACap = 2048;
__device__ __forceinline__ bool big_dA_global(int64_t nc, int64_t l) { return nc > kValSm || l > kDACap; }

// backward, rows summing dA in the fp64 target: zero their entries first
__global__ __launch_bounds__(kGemmTPB) void k_big_zero(BigRows br, const int64_t *__restrict__ Ap,
                                                       const int64_t *__restrict__ Cp, double *__restrict__ dA64)
{
    pdl_wait();
    const int n = *(volatile const int *)br.count;
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t i = br.rows[r];
        if (!big_dA_global(Cp[i + 1] - Cp[i], Ap[i + 1] - Ap[i])) continue;
        for (int64_t e = Ap[i] + threadIdx.x; e < Ap[i + 1]; e += kGemmTPB) dA64[e] = 0.0;
    }
}

// backward, fp32 data: round the fp64 dA of multi-window rows once
__global__ __launch_bounds__(kGemmTPB) void k_big_cvt(BigRows br, const int64_t *__restrict__ Ap,
                                                      const int64_t *__restrict__ Cp, const double *__restrict__ dA64,
                                                      float *__restrict__ dA)
{
    pdl_wait();
    const int n = *(volatile const int *)br.count;
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t i = br.rows[r];
        if (!big_dA_global(Cp[i + 1] - Cp[i], Ap[i + 1] - Ap[i])) continue;
        for (int64_t e = Ap[i] + threadIdx.x; e < Ap[i + 1]; e += kGemmTPB) dA[e] = (float)dA64[e];
    }
}

#ifndef CSRK_BIG_FLAT
#define CSRK_BIG_FLAT 1   // one-window rows: equal flat product runs per thread (0: a thread per A entry)
#endif
#ifndef CSRK_BIG_WIN_MINB
#define CSRK_BIG_WIN_MINB 2   // measured (config 4): 2 CTAs x batch 8: numeric 57.1 -> 53.1 ms, backward 67.1 -> 61.7 ms
#endif
#ifndef CSRK_BIG_BATCH
#define CSRK_BIG_BATCH 8
#endif
template <typename T, int PH>
__global__ __launch_bounds__(kGemmTPB, CSRK_BIG_WIN_MINB) void k_gemm_big_win(BigRows br, const int64_t *__restrict__ Ap,
                                                           const int32_t *__restrict__ Ai, const T *__restrict__ Av,
                                                           const int64_t *__restrict__ Bp,
                                                           const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                           const int64_t *__restrict__ Cp,
                                                           const int32_t *__restrict__ Ci, T *__restrict__ Cv,
                                                           const T *__restrict__ dC, T *__restrict__ dA,
                                                           double *__restrict__ dA64, double *__restrict__ dB)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char s_dyn[];
    double *s_val = reinterpret_cast<double *>(s_dyn);                  // NUM: accumulators; BWD: dC
    double *s_dA = s_val + kValSm;                                      // BWD: dA of a one-window row
    int32_t *s_col = reinterpret_cast<int32_t *>(s_dA + kDACap);        // the window's C columns
    uint16_t *s_bst = reinterpret_cast<uint16_t *>(s_col + kValSm);     // position index of the window
    __shared__ int64_t s_qa[kWinQ], s_qlo[kWinQ], s_qhi[kWinQ];
    __shared__ int s_nq, s_r;
    __shared__ int32_t s_alist[kGemmTPB];   // one-window rows: the A entry holding each thread's first product
    const int n = *(volatile const int *)br.count;
    const int total = n > 0 ? br.items[n] : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int it = blockIdx.x; it < total; it += gridDim.x) {
        if (threadIdx.x == 0) {
            int lo = 0, hi = n - 1;   // the row r holding item it: last r with items[r] <= it
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (br.items[mid] <= it) lo = mid; else hi = mid - 1;
            }
            s_r = lo;
        }
        __syncthreads();
        const int r = s_r;
        const int64_t i = br.rows[r];
        const int64_t as = Ap[i], ae = Ap[i + 1];
        const int64_t row_nc = Cp[i + 1] - Cp[i];
        const bool single = row_nc <= kValSm;
        const int64_t cs = Cp[i] + (int64_t)(it - br.items[r]) * kValSm;
        const int nc = (int)(Cp[i + 1] - cs < kValSm ? Cp[i + 1] - cs : kValSm);
        for (int q = threadIdx.x; q < nc; q += kGemmTPB) {
            s_col[q] = Ci[cs + q];
            s_val[q] = PH == PH_NUM ? 0.0 : (double)dC[cs + q];
        }
        if (threadIdx.x == 0) s_nq = 0;
        const int64_t l = ae - as;
        const bool dA_sm = PH == PH_BWD && dA && !big_dA_global(row_nc, l);
        if (dA_sm)
            for (int64_t t = threadIdx.x; t < l; t += kGemmTPB) s_dA[t] = 0.0;
        __syncthreads();
        const PosIdx px = pos_index_params<kValSm / 2>(s_col, nc);
        pos_index_build<kValSm / 2>(s_col, nc, px, s_bst, threadIdx.x, kGemmTPB);
        __syncthreads();
        if (single && CSRK_BIG_FLAT) {
            // one window: the row's w products split into equal contiguous runs of the flat order
            // of k_big_prep, whatever the B row lengths.  The A entry holding each run's first
            // product is scattered into s_alist by the lists themselves (list a covers the runs
            // starting in [loff[a], loff[a+1])): no per-thread binary search over loff in global
            // memory.  A run is walked in batches of CSRK_BIG_BATCH products, loads first.
            const int64_t w = br.w[r];
            const int64_t per = (w + kGemmTPB - 1) / kGemmTPB;
            for (int64_t a = as + threadIdx.x; a < ae; a += kGemmTPB) {
                const int64_t lo = br.loff[a], hi = a + 1 < ae ? br.loff[a + 1] : w;
                int64_t t0 = (lo + per - 1) / per, t1 = (hi + per - 1) / per;
                t1 = t1 < kGemmTPB ? t1 : kGemmTPB;
                for (int64_t t = t0; t < t1; ++t) s_alist[t] = (int32_t)(a - as);
            }
            __syncthreads();
            const int64_t p_lo = threadIdx.x * per, p_hi = p_lo + per < w ? p_lo + per : w;
            int64_t cur_a = -1;
            double av = 0.0, dacc = 0.0;
            auto flush = [&]() {
                if (PH != PH_BWD || !dA || cur_a < 0) return;
                if (dA_sm) atomicAdd(&s_dA[cur_a - as], dacc);
                else atomicAdd(&dA64[cur_a], dacc);
            };
            if (p_lo < p_hi) {
                int64_t a = as + s_alist[threadIdx.x];
                int64_t lo = br.loff[a], bs = Bp[Ai[a]];
                int64_t nx = a + 1 < ae ? br.loff[a + 1] : INT64_MAX;
                constexpr int UB = CSRK_BIG_BATCH;
                for (int64_t e0 = p_lo; e0 < p_hi; e0 += UB) {
                    int32_t jv[UB];
                    double bv[UB];
                    int64_t bb[UB], aa[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int64_t e = e0 + u;
                        if (e < p_hi) {
                            while (e >= nx) {
                                ++a;
                                lo = nx;
                                nx = a + 1 < ae ? br.loff[a + 1] : INT64_MAX;
                                bs = Bp[Ai[a]];
                            }
                            bb[u] = bs + (e - lo);
                            aa[u] = a;
                            jv[u] = __ldg(Bi + bb[u]);
                            bv[u] = (double)__ldg(Bv + bb[u]);
                        } else {
                            aa[u] = -1;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        if (aa[u] < 0) break;
                        if (aa[u] != cur_a) {
                            flush();
                            cur_a = aa[u];
                            av = (double)Av[cur_a];
                            dacc = 0.0;
                        }
                        const int pos = pos_find(s_col, s_bst, px, jv[u]);
                        if (PH == PH_NUM) {
                            atomicAdd(&s_val[pos], av * bv[u]);
                        } else {
                            const double g = s_val[pos];
                            dacc = fma(g, bv[u], dacc);
                            if (dB) atomicAdd(&dB[bb[u]], av * g);
                        }
                    }
                }
            }
            flush();
            __syncthreads();
            if (PH == PH_NUM)
                for (int q = threadIdx.x; q < nc; q += kGemmTPB) Cv[cs + q] = (T)s_val[q];
            if (dA_sm)
                for (int64_t t = threadIdx.x; t < l; t += kGemmTPB) dA[as + t] = (T)s_dA[t];
            __syncthreads();
            continue;
        }
        const int32_t c_lo = nc > 0 ? s_col[0] : 0, c_hi = nc > 0 ? s_col[nc - 1] : -1;
        // one product b of A entry a (value av): NUM adds av B_kj into C_ij; BWD returns dC_ij B_kj
        auto prod = [&](double av, int64_t b, double &dacc) {
            const int32_t j = __ldg(Bi + b);
            const double bv = (double)__ldg(Bv + b);
            const int pos = pos_find(s_col, s_bst, px, j);
            if (PH == PH_NUM) {
                atomicAdd(&s_val[pos], av * bv);
            } else {
                const double g = s_val[pos];
                dacc = fma(g, bv, dacc);
                if (dB) atomicAdd(&dB[b], av * g);
            }
        };
        auto put_dA = [&](int64_t a, double dacc, bool any) {
            if (PH != PH_BWD || !dA || !any) return;
            if (dA_sm) atomicAdd(&s_dA[a - as], dacc);
            else atomicAdd(&dA64[a], dacc);
        };
        for (int64_t a = as + threadIdx.x; a < ae; a += kGemmTPB) {
            const int32_t k = Ai[a];
            const double av = (double)Av[a];
            int64_t b0 = Bp[k], b1 = Bp[k + 1];
            if (!single && b1 > b0) {   // the part of B row k inside [c_lo, c_hi]
                const int64_t l0 = b0 + lbound64(Bi + b0, b1 - b0, c_lo);
                b1 = l0 + lbound64(Bi + l0, b1 - l0, c_hi + 1);
                b0 = l0;
            }
            if (b1 - b0 > 32) {
                const int slot = atomicAdd(&s_nq, 1);
                if (slot < kWinQ) {
                    s_qa[slot] = a;
                    s_qlo[slot] = b0;
                    s_qhi[slot] = b1;
                    continue;
                }
            }
            double dacc = 0.0;
            for (int64_t b = b0; b < b1; ++b) prod(av, b, dacc);
            put_dA(a, dacc, b1 > b0);
        }
        __syncthreads();
        const int nq = s_nq < kWinQ ? s_nq : kWinQ;
        for (int e = warp; e < nq; e += kGemmTPB / 32) {   // long parts: a warp each, fixed lane order
            const int64_t a = s_qa[e];
            const double av = (double)Av[a];
            double dacc = 0.0;
            for (int64_t b = s_qlo[e] + lane; b < s_qhi[e]; b += 32) prod(av, b, dacc);
            if (PH == PH_BWD) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
                if (lane == 0) put_dA(a, dacc, true);
            }
        }
        __syncthreads();
        if (PH == PH_NUM)
            for (int q = threadIdx.x; q < nc; q += kGemmTPB) Cv[cs + q] = (T)s_val[q];
        if (dA_sm)
            for (int64_t t = threadIdx.x; t < l; t += kGemmTPB) dA[as + t] = (T)s_dA[t];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host side
static unsigned big_grid() { return (unsigned)(kNumSMs * 2); }

static size_t big_sym_smem() { return sizeof(uint32_t) * kBitmapWords; }
static size_t big_win_smem()
{
    return (sizeof(double) + sizeof(int32_t)) * kValSm + sizeof(double) * kDACap + sizeof(uint16_t) * (kValSm / 2 + 1);
}
static size_t big_sort_smem() { return sizeof(int32_t) * (2 * kMMaxW + kMMaxW / 2); }
static unsigned sort_grid() { return (unsigned)(kNumSMs * 4); }
static unsigned val_grid() { return (unsigned)(kNumSMs * 4); }
template <int WW, int PH> static size_t wsm() { return sizeof(WSmemT<WW, kWL, PH>) * kWWarps; }
// enough CTAs to fill every SM at the occupancy the phase's shared memory allows
static unsigned wgrid(size_t smem)
{
    size_t per = smem > 0 ? (size_t)(227 * 1024) / (smem + 1024) : 16;
    per = per < 1 ? 1 : per > 16 ? 16 : per;
    return (unsigned)(kNumSMs * per);
}

static int set_smem_attrs()
{
    static DevOnce once;
    if (!once.need()) return CSRK_OK;
    const int bs = (int)big_sym_smem();
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_COUNT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_FILL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_huge_sym<PH_COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_huge_sym<PH_FILL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_COUNT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)big_sort_smem()));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_sym<PH_FILL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)big_sort_smem()));
    const int ww = (int)wsm<kWW, PH_NUM>();
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)wsm<kWW, PH_COUNT>()));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_COUNT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)wsm<kW2W, PH_COUNT>()));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_FILL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)wsm<kW2W, PH_FILL>()));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_FILL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)wsm<kWW, PH_FILL>()));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, ww));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ww));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<float, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, ww));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<float, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ww));
    const int w2n = (int)wsm<kW2W, PH_NUM>(), w2b = (int)wsm<kW2W, PH_BWD>();
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_NUM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2n));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<double, PH_BWD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2b));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<float, PH_NUM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2n));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_W<float, PH_BWD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2b));
    const int bw = (int)big_win_smem();
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_win<double, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_win<double, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_win<float, PH_NUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw));
    CSRK_CUDA(cudaFuncSetAttribute(k_gemm_big_win<float, PH_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw));
    once.done();
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
// numeric phase: stage C's values in shared memory when rows of C are long on average (3D
// stencils: 25 per row, measured 832 -> 796 us on config 3; 2D: 13 per row, staging is slower)
static int stage_num(const csrk_pattern &A, const csrk_pattern &C)
{
    static int v = knob("GEMM_STAGE_NUM", -1);
    if (v >= 0) return v;
    if (stage_vals()) return 1;
    return C.nnz > 20 * (A.nrows > 0 ? A.nrows : 1) ? 1 : 0;
}

// both queue counters live in one 8-byte word so one memset clears them
static bool huge_cluster() { static int v = knob("GEMM_HUGE_CLUSTER", 1); return v != 0; }
static void carve_lists(const csrk_pattern &A, BigList &wl, BigList &big, BigRows &br, Bump &ws,
                        BigList *w2 = nullptr)
{
    const int64_t m = A.nrows > 0 ? A.nrows : 1;
    wl.rows = ws.take<int32_t>(m);
    big.rows = ws.take<int32_t>(m);
    int32_t *w2rows = ws.take<int32_t>(m);
    int *cnt = ws.take<int>(5);
    wl.count = cnt;
    big.count = cnt ? cnt + 1 : nullptr;
    if (w2) {
        w2->rows = w2rows;
        w2->count = cnt ? cnt + 2 : nullptr;
    }
    br.rows = big.rows;
    br.count = big.count;
    br.loff = ws.take<int64_t>(A.nnz > 0 ? A.nnz : 1);
    br.w = ws.take<int64_t>(m);
    br.items = ws.take<int32_t>(m + 1);
    if (w2 && huge_cluster()) {   // symbolic: the huge-row list reuses the W2 list (consumed before k_big_prep)
        br.huge = w2rows;
        br.nhuge = cnt ? cnt + 4 : nullptr;
    }
}

// k_gemm_S with 32-bit B positions when B has fewer than 2^31 entries (cheaper merge steps)
template <typename T, int PH, typename... Args>
static int launch_S(bool small, unsigned grid, size_t smem, cudaStream_t s, Args... args)
{
    if (small) CSRK_LAUNCH((k_gemm_S<T, PH, int32_t>), grid, kSTPB, smem, s, args...);
    else CSRK_LAUNCH((k_gemm_S<T, PH, int64_t>), grid, kSTPB, smem, s, args...);
    return CSRK_OK;
}

// The COUNT call keeps each short row's columns (<= kSCache) in the workspace; the FILL call
// copies them instead of merging again when it receives the same workspace for the same A, B
// right after that COUNT (checked here on the host; anything else merges again).
struct CountStamp {
    const void *ws;
    const int64_t *Ap, *Bp;
    const int32_t *Ai, *Bi;
    int64_t m, nnzA, nnzB;
    int ncls[4];   // rows COUNT queued to the W / big / W2 paths, short rows not cached (not identity)
    bool operator==(const CountStamp &o) const
    {
        return ws == o.ws && Ap == o.Ap && Bp == o.Bp && Ai == o.Ai && Bi == o.Bi && m == o.m && nnzA == o.nnzA &&
               nnzB == o.nnzB;
    }
};
static std::mutex g_stamp_mu;
static std::vector<CountStamp> g_stamps;  // one per workspace in use (a handful)
static int use_fill_cache() { static int v = knob("GEMM_FILL_CACHE", 1); return v; }

void gemm_fill_cache_invalidate(const void *ws, size_t bytes)
{
    const char *lo = static_cast<const char *>(ws), *hi = lo + bytes;
    std::lock_guard<std::mutex> g(g_stamp_mu);
    for (size_t q = 0; q < g_stamps.size(); ++q) {
        const char *w = static_cast<const char *>(g_stamps[q].ws);
        if (w >= lo && w < hi) g_stamps.erase(g_stamps.begin() + (long)q--);
    }
}

// FILL when COUNT kept every row's columns (all rows short, <= kSCache columns each): a warp per
// 32 rows loads slot c of its rows coalesced (cache[c m + i]), kFcBatch slots in flight per
// thread, stages the rows in shared memory in C order and writes the warp's C range coalesced.
#ifndef CSRK_FC_TPB
#define CSRK_FC_TPB 256
#endif
#ifndef CSRK_FC_BATCH
#define CSRK_FC_BATCH 8   // measured (4 / 6 / 8 / 16 / 32): 8 and below ~342 us, 16: 353, 32: 556 (config 2)
#endif
constexpr int kFcTPB = CSRK_FC_TPB;       // A/B via CSRK_NVCC_EXTRA
constexpr int kFcBatch = CSRK_FC_BATCH;
__global__ __launch_bounds__(kFcTPB) void k_fill_copy(int64_t m, const int64_t *__restrict__ Cp,
                                                      const int32_t *__restrict__ cache, int32_t *__restrict__ Ci)
{
    pdl_wait();
    __shared__ int32_t s_c[kFcTPB / 32][32 * kSCache];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * kFcTPB + w * 32;
    if (i0 >= m) return;
    const int64_t i = i0 + lane;
    const int64_t iend = i0 + 32 < m ? i0 + 32 : m;
    const int64_t c0 = Cp[i0], c1 = Cp[iend];
    const int64_t cs = i < m ? Cp[i] : c1;
    const int n = i < m ? (int)(Cp[i + 1] - cs) : 0;
    const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
    int32_t *dst = s_c[w] + (cs - c0);
    for (int b = 0; b < nmax; b += kFcBatch) {
        int32_t q[kFcBatch];
#pragma unroll
        for (int u = 0; u < kFcBatch; ++u) q[u] = b + u < n ? __ldcs(cache + (int64_t)(b + u) * m + i) : 0;
#pragma unroll
        for (int u = 0; u < kFcBatch; ++u)
            if (b + u < n) dst[b + u] = q[u];
    }
    __syncwarp();
    for (int64_t e = c0 + lane; e < c1; e += 32) Ci[e] = s_c[w][e - c0];
}

int spgemm_symbolic(const csrk_pattern &A, const csrk_pattern &B, int64_t *Cp, int32_t *Ci, int64_t *nnzC_host,
                    Bump &ws, cudaStream_t s)
{
    BigList wl{}, b{}, w2{};
    BigRows br{};
    carve_lists(A, wl, b, br, ws, &w2);
    // kSCache column slots per row, then one flag byte per row
    const size_t mr = (size_t)(A.nrows > 0 ? A.nrows : 1);
    int32_t *cache = use_fill_cache() ? ws.take<int32_t>(mr * kSCache + (mr + 3) / 4) : nullptr;
    if (ws.sizing()) return scan_counts_i64(nullptr, A.nrows, ws, s);
    CountStamp stamp{ws.base, A.indptr, B.indptr, A.indices, B.indices, A.nrows, A.nnz, B.nnz, {1, 1, 1, 1}};
    const int64_t m = A.nrows;
    CSRK_TRY(set_smem_attrs());
    const unsigned gS = (unsigned)cdiv(m, kSTPB);
    const int32_t *Bi = B.indices;
    const double *dn = nullptr;
    double *dw = nullptr;
    if (!Ci) {
        CSRK_CUDA(cudaMemsetAsync(Cp, 0, sizeof(int64_t), s));
        if (m > 0) {
            CSRK_CUDA(cudaMemsetAsync(wl.count, 0, 5 * sizeof(int), s));
            {
                std::lock_guard<std::mutex> g(g_stamp_mu);
                for (size_t q = 0; q < g_stamps.size(); ++q)
                    if (g_stamps[q].ws == ws.base) g_stamps.erase(g_stamps.begin() + (long)q--);
            }
            CSRK_TRY((launch_S<double, PH_COUNT>)(B.nnz < INT32_MAX, gS, 0, s, m, A.indptr, A.indices, dn, B.indptr, Bi, dn,
                        Cp, (int32_t *)nullptr, dw, dn, dw, dw, wl, b, 0, cache));
            CSRK_LAUNCH((k_gemm_W<double, PH_COUNT>), wgrid((wsm<kWW, PH_COUNT>())), kWTPB, (wsm<kWW, PH_COUNT>()), s, wl, b, w2, A.indptr, A.indices,
                        dn, B.indptr, Bi, dn, Cp, (int32_t *)nullptr, dw, dn, dw, dw);
            CSRK_LAUNCH((k_gemm_W<double, PH_COUNT, true>), wgrid((wsm<kW2W, PH_COUNT>())), kWTPB,
                        (wsm<kW2W, PH_COUNT>()), s, w2, b, BigList{},
                        A.indptr, A.indices, dn, B.indptr, Bi, dn, Cp, (int32_t *)nullptr, dw, dn, dw, dw);
            CSRK_LAUNCH(k_big_prep, big_grid(), kGemmTPB, 0, s, br, A.indptr, A.indices, B.indptr);
            CSRK_LAUNCH((k_gemm_big_sym<PH_COUNT, false>), sort_grid(), kGemmTPB, big_sort_smem(), s, br, B.ncols,
                        A.indptr, A.indices, B.indptr, Bi, Cp, (int32_t *)nullptr);
            if (br.huge)
                CSRK_LAUNCH(k_gemm_huge_sym<PH_COUNT>, (unsigned)(kNumSMs / kHugeCl * kHugeCl), kGemmTPB,
                            big_sym_smem(), s, br, B.ncols, A.indptr, A.indices, B.indptr, Bi, Cp, (int32_t *)nullptr);
            else
                CSRK_LAUNCH((k_gemm_big_sym<PH_COUNT, true>), big_grid(), kGemmTPB, big_sym_smem(), s, br, B.ncols,
                            A.indptr, A.indices, B.indptr, Bi, Cp, (int32_t *)nullptr);
            CSRK_TRY(scan_counts_i64(Cp, m, ws, s));
        }
        CSRK_CUDA(cudaMemcpyAsync(nnzC_host, Cp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        int cls[4] = {1, 1, 1, 1};
        if (m > 0) CSRK_CUDA(cudaMemcpyAsync(cls, wl.count, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CSRK_CUDA(cudaStreamSynchronize(s));
        if (m > 0) {
            // the class sizes travel with the stamp: FILL on the same arguments skips the launches
            // of the empty classes (the row classes depend on A's and B's patterns only)
            for (int c = 0; c < 4; ++c) stamp.ncls[c] = cls[c];
            std::lock_guard<std::mutex> g(g_stamp_mu);
            g_stamps.push_back(stamp);
        }
        return CSRK_OK;
    }
    if (m == 0) return CSRK_OK;
    bool found = false;
    {
        std::lock_guard<std::mutex> g(g_stamp_mu);
        for (size_t q = 0; q < g_stamps.size(); ++q)
            if (g_stamps[q] == stamp) {
                found = true;
                for (int c = 0; c < 4; ++c) stamp.ncls[c] = g_stamps[q].ncls[c];
                g_stamps.erase(g_stamps.begin() + (long)q);  // one FILL per COUNT
                break;
            }
    }
    const bool cached = found && cache;
    // without the COUNT of these arguments every class is launched (ncls stays {1, 1, 1, 1})
    if (cached && !stamp.ncls[0] && !stamp.ncls[1] && !stamp.ncls[2] && !stamp.ncls[3] && knob("GEMM_FILL_COPY", 1)) {
        // every row is short and kept in the cache: FILL is a copy (k_fill_copy), nothing else
        const unsigned g = (unsigned)cdiv(m, kFcTPB);
        CSRK_LAUNCH(k_fill_copy, g, kFcTPB, 0, s, m, (const int64_t *)Cp, (const int32_t *)cache, Ci);
        return CSRK_OK;
    }
    CSRK_CUDA(cudaMemsetAsync(wl.count, 0, 5 * sizeof(int), s));
    CSRK_TRY((launch_S<double, PH_FILL>)(B.nnz < INT32_MAX, gS, s_smem<double>(PH_FILL, stage_fill()), s, m, A.indptr,
                A.indices, dn, B.indptr, Bi, dn, Cp, Ci, dw, dn, dw, dw, wl, b, stage_fill(),
                cached ? cache : (int32_t *)nullptr));
    // the W kernel also forwards rows to the W2 list: it runs when either class is non-empty
    if (stamp.ncls[0] || stamp.ncls[2])
        CSRK_LAUNCH((k_gemm_W<double, PH_FILL>), wgrid((wsm<kWW, PH_FILL>())), kWTPB, (wsm<kWW, PH_FILL>()), s, wl, b,
                    w2, A.indptr, A.indices, dn, B.indptr, Bi, dn, Cp, Ci, dw, dn, dw, dw);
    if (stamp.ncls[2])
        CSRK_LAUNCH((k_gemm_W<double, PH_FILL, true>), wgrid((wsm<kW2W, PH_FILL>())), kWTPB,
                    (wsm<kW2W, PH_FILL>()), s, w2, b, BigList{}, A.indptr,
                    A.indices, dn, B.indptr, Bi, dn, Cp, Ci, dw, dn, dw, dw);
    if (stamp.ncls[1]) {
        CSRK_LAUNCH(k_big_prep, big_grid(), kGemmTPB, 0, s, br, A.indptr, A.indices, B.indptr);
        CSRK_LAUNCH((k_gemm_big_sym<PH_FILL, false>), sort_grid(), kGemmTPB, big_sort_smem(), s, br, B.ncols,
                    A.indptr, A.indices, B.indptr, Bi, Cp, Ci);
        if (br.huge)
            CSRK_LAUNCH(k_gemm_huge_sym<PH_FILL>, (unsigned)(kNumSMs / kHugeCl * kHugeCl), kGemmTPB, big_sym_smem(),
                        s, br, B.ncols, A.indptr, A.indices, B.indptr, Bi, Cp, Ci);
        else
            CSRK_LAUNCH((k_gemm_big_sym<PH_FILL, true>), big_grid(), kGemmTPB, big_sym_smem(), s, br, B.ncols,
                    A.indptr, A.indices, B.indptr, Bi, Cp, Ci);
    }
    return CSRK_OK;
}

// fp64 target of an atomic scatter into out[n] (reading A5): out itself for fp64 data, else scratch
template <typename T>
static int round_f64(const double *acc, T *out, int64_t n, cudaStream_t s)
{
    if constexpr (sizeof(T) == sizeof(double)) return CSRK_OK;
    else return f64_to_f32(acc, out, n, s);
}
template <typename T>
static double *f64_target(T *out, int64_t n, Bump &ws)
{
    if constexpr (sizeof(T) == sizeof(double)) return reinterpret_cast<double *>(out);
    else return ws.take<double>(n > 0 ? n : 1);
}

template <typename T>
static int spgemm_values_t(int PH, const csrk_pattern &A, const T *Av, const csrk_pattern &B, const T *Bv,
                           const csrk_pattern &C, T *Cv, const T *dC, T *dA, T *dB, Bump &ws, cudaStream_t s)
{
    BigList wl{}, b{}, w2{};
    BigRows br{};
    carve_lists(A, wl, b, br, ws, &w2);
    br.huge = nullptr;   // (the huge-row list is the symbolic phase's)
    // backward: fp64 targets of the dB scatter and of the multi-window big-row dA (fp32 data:
    // scratch, rounded once at the end)
    double *dB64 = nullptr, *dA64 = nullptr;
    if (PH == PH_BWD) {
        if (dB || ws.sizing()) dB64 = f64_target(dB, B.nnz, ws);
        if (dA || ws.sizing()) dA64 = f64_target(dA, A.nnz, ws);
    }
    if (ws.sizing()) return CSRK_OK;
    CSRK_TRY(set_smem_attrs());
    if (PH == PH_BWD && dB) CSRK_CUDA(cudaMemsetAsync(dB64, 0, sizeof(double) * (size_t)B.nnz, s));
    const int64_t m = A.nrows;
    if (m == 0) return dB ? round_f64(dB64, dB, B.nnz, s) : CSRK_OK;
    CSRK_CUDA(cudaMemsetAsync(wl.count, 0, 5 * sizeof(int), s));
    const unsigned gS = (unsigned)cdiv(m, kSTPB);
    int64_t *Cp = const_cast<int64_t *>(C.indptr);
    T *tn = nullptr;
    const T *ctn = nullptr;
    double *dn = nullptr;
    if (PH == PH_NUM) {
        const int sn = stage_num(A, C);
        CSRK_TRY((launch_S<T, PH_NUM>)(B.nnz < INT32_MAX, gS, s_smem<T>(PH_NUM, sn), s, m, A.indptr, A.indices,
                    Av, B.indptr, B.indices, Bv, Cp, (int32_t *)nullptr, Cv, ctn, tn, dn, wl, b, sn,
                    (int32_t *)nullptr));
        CSRK_LAUNCH((k_gemm_W<T, PH_NUM>), wgrid((wsm<kWW, PH_NUM>())), kWTPB, (wsm<kWW, PH_NUM>()), s, wl, b,
                    w2, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, Cp,
                    const_cast<int32_t *>(C.indices), Cv, ctn, tn, dn);
        CSRK_LAUNCH((k_gemm_W<T, PH_NUM, true>), wgrid((wsm<kW2W, PH_NUM>())), kWTPB, (wsm<kW2W, PH_NUM>()), s, w2,
                    b, BigList{}, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, Cp,
                    const_cast<int32_t *>(C.indices), Cv, ctn, tn, dn);
        CSRK_LAUNCH(k_big_prep, big_grid(), kGemmTPB, 0, s, br, A.indptr, A.indices, B.indptr);
        CSRK_LAUNCH(k_big_items, 1, kItemsTPB, 0, s, br, (const int64_t *)Cp);
        CSRK_LAUNCH((k_gemm_big_win<T, PH_NUM>), val_grid(), kGemmTPB, big_win_smem(), s, br, A.indptr, A.indices, Av,
                    B.indptr, B.indices, Bv, C.indptr, C.indices, Cv, ctn, tn, dn, dn);
        return CSRK_OK;
    }
    CSRK_TRY((launch_S<T, PH_BWD>)(B.nnz < INT32_MAX, gS, s_smem<T>(PH_BWD, stage_vals()), s, m, A.indptr,
                A.indices, Av, B.indptr, B.indices, Bv, Cp, (int32_t *)nullptr, tn, dC, dA, dB ? dB64 : dn, wl, b,
                stage_vals(), (int32_t *)nullptr));
    CSRK_LAUNCH((k_gemm_W<T, PH_BWD>), wgrid((wsm<kWW, PH_BWD>())), kWTPB, (wsm<kWW, PH_BWD>()), s, wl, b,
                w2, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, Cp, const_cast<int32_t *>(C.indices),
                tn, dC, dA, dB ? dB64 : dn);
    CSRK_LAUNCH((k_gemm_W<T, PH_BWD, true>), wgrid((wsm<kW2W, PH_BWD>())), kWTPB, (wsm<kW2W, PH_BWD>()), s, w2, b,
                BigList{}, A.indptr, A.indices, Av, B.indptr, B.indices, Bv, Cp, const_cast<int32_t *>(C.indices),
                tn, dC, dA, dB ? dB64 : dn);
    CSRK_LAUNCH(k_big_prep, big_grid(), kGemmTPB, 0, s, br, A.indptr, A.indices, B.indptr);
    CSRK_LAUNCH(k_big_items, 1, kItemsTPB, 0, s, br, (const int64_t *)Cp);
    if (dA) CSRK_LAUNCH(k_big_zero, big_grid(), kGemmTPB, 0, s, br, A.indptr, C.indptr, dA64);
    CSRK_LAUNCH((k_gemm_big_win<T, PH_BWD>), val_grid(), kGemmTPB, big_win_smem(), s, br, A.indptr, A.indices, Av,
                B.indptr, B.indices, Bv, C.indptr, C.indices, tn, dC, dA, dA ? dA64 : dn, dB ? dB64 : dn);
    if constexpr (sizeof(T) == sizeof(float)) {
        if (dA) CSRK_LAUNCH(k_big_cvt, big_grid(), kGemmTPB, 0, s, br, A.indptr, C.indptr, (const double *)dA64, dA);
    }
    return dB ? round_f64(dB64, dB, B.nnz, s) : CSRK_OK;
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

// ---------------------------------------------------------------- deterministic dB (transpose plan)
// dB_kj = sum_{i : (i,k) in A} A_ik dC_ij, evaluated per stored (k, j) of B as a gather over
// column k of A -- row k of the caller's A^T plan (pattern + perm) -- i.e. the paper's "modified
// version of the SpGEMM algorithm that operates on columns of A".  For each i of A^T
// row k, in ascending order, the columns of B row k are located in C row i (C is the structural
// product, so C_i contains every column of B_k) and acc_j = fma(A_ik, dC_ij, acc_j) in fp64.
// Fixed order, no atomics: bit-identical from run to run, whatever the schedule.
//   k_gemm_dB_rows    one THREAD per row k of B with len(B_k) <= kDbR: the row's columns and
//                     accumulators in registers; per i one forward (galloping) walk over C_i,
//                     since B_k's columns come in ascending order.  Longer rows are queued.
//   k_gemm_dB_long    one WARP per queued row, lanes over B_k's entries, binary search per i.
constexpr int kDbTPB = 256;
constexpr int kDbR = 16;

// queued long rows: slot -> row and its first chunk; ctr = (slots << 32) | chunks
struct DbLong {
    int32_t *rows;
    int64_t *chunk0;
    unsigned long long *ctr;
};

// first position p in [c, c1) with Ci[p] >= v, searching forward from c (galloping)
__device__ __forceinline__ int64_t gallop_lb(const int32_t *__restrict__ Ci, int64_t c, int64_t c1, int32_t v)
{
    if (c >= c1 || __ldg(Ci + c) >= v) return c;
    int64_t lo = c, step = 1;   // Ci[lo] < v
    while (lo + step < c1 && __ldg(Ci + lo + step) < v) {
        lo += step;
        step <<= 1;
    }
    int64_t hi = lo + step < c1 ? lo + step : c1;   // Ci[hi] >= v or hi == c1
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(Ci + mid) < v) lo = mid; else hi = mid;
    }
    return hi;
}

template <typename T>
__global__ __launch_bounds__(kDbTPB) void k_gemm_dB_rows(int64_t mB, const int64_t *__restrict__ Bp,
                                                         const int32_t *__restrict__ Bi,
                                                         const int64_t *__restrict__ ATp,
                                                         const int32_t *__restrict__ ATi,
                                                         const int64_t *__restrict__ perm, const T *__restrict__ Av,
                                                         const int64_t *__restrict__ Cp,
                                                         const int32_t *__restrict__ Ci, const T *__restrict__ dC,
                                                         T *__restrict__ dB, DbLong lng)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * kDbTPB;
    for (int64_t k0 = (int64_t)blockIdx.x * kDbTPB + threadIdx.x - lane; k0 < mB; k0 += stride) {
        const int64_t k = k0 + lane;
        const bool valid = k < mB;
        const int64_t b0 = valid ? __ldg(Bp + k) : 0, b1 = valid ? __ldg(Bp + k + 1) : 0;
        const int lb = (int)(b1 - b0 < kDbR + 1 ? b1 - b0 : kDbR + 1);
        const bool lng_row = valid && lb > kDbR;
        if (lng_row) {
            // one atomic hands out the list slot (high word) and the row's first 32-entry chunk
            // (low word), so chunk offsets ascend with the slot
            const unsigned long long nch = (unsigned long long)((b1 - b0 + 31) >> 5);
            const unsigned long long old = atomicAdd(lng.ctr, (1ull << 32) | nch);
            const int slot = (int)(old >> 32);
            lng.rows[slot] = (int32_t)k;
            lng.chunk0[slot] = (int64_t)(old & 0xffffffffull);
        }
        if (!valid || lng_row || lb == 0) continue;
        int32_t bj[kDbR];
        double acc[kDbR];
#pragma unroll
        for (int p = 0; p < kDbR; ++p) {
            bj[p] = p < lb ? __ldg(Bi + b0 + p) : 0;
            acc[p] = 0.0;
        }
        const int64_t q1 = __ldg(ATp + k + 1);
        for (int64_t q = __ldg(ATp + k); q < q1; ++q) {
            const int32_t i = __ldg(ATi + q);
            const double a = (double)__ldg(Av + __ldg(perm + q));
            int64_t c = __ldg(Cp + i);
            const int64_t c1 = __ldg(Cp + i + 1);
#pragma unroll
            for (int p = 0; p < kDbR; ++p) {
                if (p < lb) {
                    c = gallop_lb(Ci, c, c1, bj[p]);
                    if (c < c1 && __ldg(Ci + c) == bj[p]) acc[p] = fma(a, (double)__ldg(dC + c), acc[p]);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < kDbR; ++p)
            if (p < lb) dB[b0 + p] = (T)acc[p];
    }
}

template <typename T>
__global__ __launch_bounds__(kDbTPB) void k_gemm_dB_long(const int64_t *__restrict__ Bp,
                                                         const int32_t *__restrict__ Bi,
                                                         const int64_t *__restrict__ ATp,
                                                         const int32_t *__restrict__ ATi,
                                                         const int64_t *__restrict__ perm, const T *__restrict__ Av,
                                                         const int64_t *__restrict__ Cp,
                                                         const int32_t *__restrict__ Ci, const T *__restrict__ dC,
                                                         T *__restrict__ dB, DbLong lng)
{
    pdl_wait();
    const unsigned long long ctr = *(volatile const unsigned long long *)lng.ctr;
    const int n = (int)(ctr >> 32);
    const int64_t nchunks = (int64_t)(ctr & 0xffffffffull);
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (kDbTPB / 32);
    // one warp per 32-entry chunk of a long row (many warps per row), lanes over its entries
    for (int64_t ch = (int64_t)blockIdx.x * (kDbTPB / 32) + (threadIdx.x >> 5); ch < nchunks; ch += warps) {
        int lo = 0, hi = n - 1;   // the slot holding chunk ch: last slot with chunk0 <= ch
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (lng.chunk0[mid] <= ch) lo = mid; else hi = mid - 1;
        }
        const int64_t k = lng.rows[lo];
        const int64_t pb = __ldg(Bp + k) + (ch - lng.chunk0[lo]) * 32 + lane;
        if (pb >= __ldg(Bp + k + 1)) continue;
        const int32_t j = __ldg(Bi + pb);
        double acc = 0.0;
        const int64_t q1 = __ldg(ATp + k + 1);
        for (int64_t q = __ldg(ATp + k); q < q1; ++q) {
            const int32_t i = __ldg(ATi + q);
            const double a = (double)__ldg(Av + __ldg(perm + q));
            const int64_t c0 = __ldg(Cp + i), c1 = __ldg(Cp + i + 1);
            int64_t l = c0, h = c1;
            while (l < h) {
                const int64_t mid = (l + h) >> 1;
                if (__ldg(Ci + mid) < j) l = mid + 1; else h = mid;
            }
            if (l < c1 && __ldg(Ci + l) == j) acc = fma(a, (double)__ldg(dC + l), acc);
        }
        dB[pb] = (T)acc;
    }
}

// Fused deterministic backward through A's transpose plan (short rows of B): the thread of B row k
// walks, for every i of A^T row k (ascending), C row i against B row k (B_k is a subset of C_i's
// columns) and reads each dC_ij once for BOTH gradients:
//   dB_kj += A_ik dC_ij           (fp64 register accumulators, i ascending -- k_gemm_dB_rows' order)
//   dA_ik  = sum_j dC_ij B_kj     (j ascending -- the row traversal's order: the same bits)
// C row i is read in chunks of 16 columns loaded together (independent loads) and matched against
// B_k's columns in registers, instead of a galloping search of dependent loads per column.  dA of
// the entries of long B rows is left to k_gemm_dA_long.  No atomics: bit-reproducible.
constexpr int kBwdR = 8;       // B rows of at most 8 entries (stencils: 5 / 7); longer ones are queued
#ifndef CSRK_BWD_CHUNK
#define CSRK_BWD_CHUNK 8
#endif
constexpr int kBwdChunk = CSRK_BWD_CHUNK;   // C-row columns (and dC) loaded together
constexpr int kBwdQ = 8;       // A^T rows of at most 8 entries: metadata preloaded
#ifndef CSRK_BWD_PRELOAD
#define CSRK_BWD_PRELOAD 1
#endif
#ifndef CSRK_BWD_MINB
#define CSRK_BWD_MINB 1
#endif
template <typename T>
__global__ __launch_bounds__(kDbTPB, CSRK_BWD_MINB) void k_gemm_bwd_rows(int64_t mB, const int64_t *__restrict__ Bp,
                                                          const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                          const int64_t *__restrict__ ATp,
                                                          const int32_t *__restrict__ ATi,
                                                          const int64_t *__restrict__ perm, const T *__restrict__ Av,
                                                          const int64_t *__restrict__ Cp,
                                                          const int32_t *__restrict__ Ci, const T *__restrict__ dC,
                                                          T *__restrict__ dA, T *__restrict__ dB, DbLong lng)
{
    pdl_wait();
    // the thread's B row (columns, values) and dB accumulators in shared memory, [entry][thread]:
    // the merge pointer into them is data-dependent (registers would spill)
    __shared__ int32_t s_bj[kBwdR][kDbTPB];
    __shared__ double s_bv[kBwdR][kDbTPB], s_acc[kBwdR][kDbTPB];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t stride = (int64_t)gridDim.x * kDbTPB;
    for (int64_t k0 = (int64_t)blockIdx.x * kDbTPB + tid - lane; k0 < mB; k0 += stride) {
        const int64_t k = k0 + lane;
        const bool valid = k < mB;
        const int64_t b0 = valid ? __ldg(Bp + k) : 0, b1 = valid ? __ldg(Bp + k + 1) : 0;
        const int lb = (int)(b1 - b0 < kBwdR + 1 ? b1 - b0 : kBwdR + 1);
        const bool lng_row = valid && lb > kBwdR;
        if (lng_row) {
            const unsigned long long nch = (unsigned long long)((b1 - b0 + 31) >> 5);
            const unsigned long long old = atomicAdd(lng.ctr, (1ull << 32) | nch);
            const int slot = (int)(old >> 32);
            lng.rows[slot] = (int32_t)k;
            lng.chunk0[slot] = (int64_t)(old & 0xffffffffull);
        }
        if (!valid || lng_row) continue;
        const int64_t q0 = __ldg(ATp + k), q1 = __ldg(ATp + k + 1);
        for (int p = 0; p < lb; ++p) {
            s_bj[p][tid] = __ldg(Bi + b0 + p);
            s_bv[p][tid] = (double)__ldg(Bv + b0 + p);
            s_acc[p][tid] = 0.0;
        }
        // walk C row i against B row k: B_k's columns are a sorted subset of C_i's (two pointers)
        auto walk = [&](int64_t pa, double a, int64_t c0, int64_t c1) {
            double dacc = 0.0;
            int p = 0;
            int32_t cur = lb > 0 ? s_bj[0][tid] : INT32_MAX;
            for (int64_t cb = c0; cb < c1 && p < lb; cb += kBwdChunk) {
                int32_t cc[kBwdChunk];
                double dv[kBwdChunk];
#pragma unroll
                for (int t = 0; t < kBwdChunk; ++t) {
                    const bool in = cb + t < c1;
                    cc[t] = in ? __ldg(Ci + cb + t) : INT32_MIN;
                    dv[t] = in ? (double)__ldg(dC + cb + t) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < kBwdChunk; ++t) {
                    if (cc[t] == cur) {
                        const double g = dv[t];
                        s_acc[p][tid] = fma(a, g, s_acc[p][tid]);
                        dacc = fma(g, s_bv[p][tid], dacc);
                        ++p;
                        cur = p < lb ? s_bj[p][tid] : INT32_MAX;
                    }
                }
            }
            if (p < lb) {
                // the walk stalled on B_k's column p, absent from C_i (a caller's C narrower than
                // the structural product: dC_ij = 0 there, csrk.h); the columns after it are
                // located by binary search, in ascending order (same summation order)
                for (int pp = p + 1; pp < lb; ++pp) {
                    const int32_t j = s_bj[pp][tid];
                    int64_t lo = c0, hi = c1;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (__ldg(Ci + mid) < j) lo = mid + 1; else hi = mid;
                    }
                    if (lo < c1 && __ldg(Ci + lo) == j) {
                        const double g = (double)__ldg(dC + lo);
                        s_acc[pp][tid] = fma(a, g, s_acc[pp][tid]);
                        dacc = fma(g, s_bv[pp][tid], dacc);
                    }
                }
            }
            if (dA) dA[pa] = (T)dacc;
        };
        if (CSRK_BWD_PRELOAD && q1 - q0 <= kBwdQ) {
            // the row's A^T entries, their C-row extents and A values loaded together up front:
            // three levels of dependent loads per B row instead of three per entry
            const int lq = (int)(q1 - q0);
            int32_t iu[kBwdQ];
            int64_t pau[kBwdQ], cs[kBwdQ];
            int32_t cn[kBwdQ];
            double au[kBwdQ];
#pragma unroll
            for (int u = 0; u < kBwdQ; ++u) {
                iu[u] = u < lq ? __ldg(ATi + q0 + u) : 0;
                pau[u] = u < lq ? __ldg(perm + q0 + u) : 0;
            }
#pragma unroll
            for (int u = 0; u < kBwdQ; ++u) {
                cs[u] = u < lq ? __ldg(Cp + iu[u]) : 0;
                cn[u] = u < lq ? (int32_t)(__ldg(Cp + iu[u] + 1) - cs[u]) : 0;
                au[u] = u < lq ? (double)__ldg(Av + pau[u]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kBwdQ; ++u)
                if (u < lq) walk(pau[u], au[u], cs[u], cs[u] + cn[u]);
        } else {
            for (int64_t q = q0; q < q1; ++q) {
                const int32_t i = __ldg(ATi + q);
                const int64_t pa = __ldg(perm + q);
                walk(pa, (double)__ldg(Av + pa), __ldg(Cp + i), __ldg(Cp + i + 1));
            }
        }
        if (dB)
            for (int p = 0; p < lb; ++p) dB[b0 + p] = (T)s_acc[p][tid];
    }
}

// dA of the A entries (i, k) whose B row k is long (queued by k_gemm_bwd_rows): one warp per row,
// lanes over B_k's entries in chunks of 32, binary search of each column in C_i, the chunk's
// partial sums reduced in a fixed lane order and added in chunk order -- deterministic.
template <typename T>
__global__ __launch_bounds__(kDbTPB) void k_gemm_dA_long(const int64_t *__restrict__ Bp,
                                                         const int32_t *__restrict__ Bi, const T *__restrict__ Bv,
                                                         const int64_t *__restrict__ ATp,
                                                         const int32_t *__restrict__ ATi,
                                                         const int64_t *__restrict__ perm,
                                                         const int64_t *__restrict__ Cp,
                                                         const int32_t *__restrict__ Ci, const T *__restrict__ dC,
                                                         T *__restrict__ dA, DbLong lng)
{
    pdl_wait();
    const unsigned long long ctr = *(volatile const unsigned long long *)lng.ctr;
    const int n = (int)(ctr >> 32);
    const int lane = threadIdx.x & 31;
    const int warps = (int)(gridDim.x * (kDbTPB / 32));
    for (int r = blockIdx.x * (kDbTPB / 32) + (threadIdx.x >> 5); r < n; r += warps) {
        const int64_t k = lng.rows[r];
        const int64_t b0 = __ldg(Bp + k), b1 = __ldg(Bp + k + 1);
        const int64_t q1 = __ldg(ATp + k + 1);
        for (int64_t q = __ldg(ATp + k); q < q1; ++q) {
            const int32_t i = __ldg(ATi + q);
            const int64_t c0 = __ldg(Cp + i), c1 = __ldg(Cp + i + 1);
            double tot = 0.0;
            for (int64_t pb0 = b0; pb0 < b1; pb0 += 32) {
                const int64_t pb = pb0 + lane;
                double v = 0.0;
                if (pb < b1) {
                    const int32_t j = __ldg(Bi + pb);
                    int64_t l = c0, h = c1;
                    while (l < h) {
                        const int64_t mid = (l + h) >> 1;
                        if (__ldg(Ci + mid) < j) l = mid + 1; else h = mid;
                    }
                    if (l < c1 && __ldg(Ci + l) == j) v = (double)__ldg(dC + l) * (double)__ldg(Bv + pb);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                tot += v;
            }
            if (lane == 0) dA[__ldg(perm + q)] = (T)tot;
        }
    }
}

// Scattered patterns (config 4: C rows are random, far beyond L2): the thread-per-row walk reads C
// rows sector by sector from DRAM, so every stored entry of B is taken as in k_gemm_dB_long, a warp
// per 32 consecutive entries (binary search per i); the chunk's first row by a binary search over
// B's row starts, each lane's row by a galloping search from there.
template <typename T>
__global__ __launch_bounds__(kDbTPB) void k_gemm_dB_flat(int64_t nnzB, int64_t mB, const int64_t *__restrict__ Bp,
                                                         const int32_t *__restrict__ Bi,
                                                         const int64_t *__restrict__ ATp,
                                                         const int32_t *__restrict__ ATi,
                                                         const int64_t *__restrict__ perm, const T *__restrict__ Av,
                                                         const int64_t *__restrict__ Cp,
                                                         const int32_t *__restrict__ Ci, const T *__restrict__ dC,
                                                         T *__restrict__ dB)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * kDbTPB;
    for (int64_t base = ((int64_t)blockIdx.x * kDbTPB + threadIdx.x) - lane; base < nnzB; base += stride) {
        int64_t k0 = 0;
        if (lane == 0) {
            int64_t lo = 0, hi = mB - 1;   // last row r with Bp[r] <= base
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (__ldg(Bp + mid) <= base) lo = mid; else hi = mid - 1;
            }
            k0 = lo;
        }
        k0 = __shfl_sync(0xffffffffu, k0, 0);
        const int64_t pb = base + lane;
        if (pb >= nnzB) continue;
        int64_t lo = k0, step = 1;   // last r >= k0 with Bp[r] <= pb
        while (lo + step < mB && __ldg(Bp + lo + step) <= pb) {
            lo += step;
            step <<= 1;
        }
        int64_t hi = lo + step < mB ? lo + step : mB;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(Bp + mid) <= pb) lo = mid; else hi = mid;
        }
        const int64_t k = lo;
        const int32_t j = __ldg(Bi + pb);
        double acc = 0.0;
        const int64_t q1 = __ldg(ATp + k + 1);
        for (int64_t q = __ldg(ATp + k); q < q1; ++q) {
            const int32_t i = __ldg(ATi + q);
            const double a = (double)__ldg(Av + __ldg(perm + q));
            const int64_t c0 = __ldg(Cp + i), c1 = __ldg(Cp + i + 1);
            int64_t l = c0, h = c1;
            while (l < h) {
                const int64_t mid = (l + h) >> 1;
                if (__ldg(Ci + mid) < j) l = mid + 1; else h = mid;
            }
            if (l < c1 && __ldg(Ci + l) == j) acc = fma(a, (double)__ldg(dC + l), acc);
        }
        dB[pb] = (T)acc;
    }
}

static bool fused_plan_bwd() { static int v = knob("GEMM_BWD_FUSED", 1); return v != 0; }
static bool dB_flat(const csrk_pattern &B)
{
    static int k = knob("GEMM_DB_FLAT", -1);
    if (k >= 0) return k != 0;
    return B.ncols >= (int64_t(1) << 22) && B.nnz >= 8 * B.ncols;
}

template <typename T>
static int launch_dB_gather(const csrk_pattern &B, const csrk_pattern &AT, const int64_t *perm, const T *Av,
                            const csrk_pattern &C, const T *dC, T *dB, Bump &ws, cudaStream_t s)
{
    if (!ws.sizing() && B.nnz > 0 && dB_flat(B)) {
        const int64_t warps = cdiv(B.nnz, 32);
        const int64_t cap = (int64_t)kNumSMs * 8 * (kDbTPB / 32);
        const int64_t grid = cdiv(warps < cap ? warps : cap, kDbTPB / 32);
        CSRK_LAUNCH(k_gemm_dB_flat<T>, (unsigned)grid, kDbTPB, 0, s, B.nnz, B.nrows, B.indptr, B.indices, AT.indptr,
                    AT.indices, perm, Av, C.indptr, C.indices, dC, dB);
        return CSRK_OK;
    }
    DbLong lng{};
    lng.ctr = ws.take<unsigned long long>(1);
    lng.rows = ws.take<int32_t>(B.nrows > 0 ? B.nrows : 1);
    lng.chunk0 = ws.take<int64_t>(B.nrows > 0 ? B.nrows : 1);
    if (ws.sizing() || B.nnz == 0) return CSRK_OK;
    if (B.nnz / 32 + B.nrows >= (int64_t)UINT32_MAX) return CSRK_ERR_INDEX_OVERFLOW;
    CSRK_CUDA(cudaMemsetAsync(lng.ctr, 0, sizeof(unsigned long long), s));
    const int64_t warps = cdiv(B.nrows, 32);
    const int64_t cap = (int64_t)kNumSMs * 8 * (kDbTPB / 32);
    const int64_t grid = cdiv(warps < cap ? warps : cap, kDbTPB / 32);
    CSRK_LAUNCH(k_gemm_dB_rows<T>, (unsigned)grid, kDbTPB, 0, s, B.nrows, B.indptr, B.indices, AT.indptr, AT.indices,
                perm, Av, C.indptr, C.indices, dC, dB, lng);
    CSRK_LAUNCH(k_gemm_dB_long<T>, (unsigned)(kNumSMs * 8), kDbTPB, 0, s, B.indptr, B.indices, AT.indptr,
                AT.indices, perm, Av, C.indptr, C.indices, dC, dB, lng);
    return CSRK_OK;
}

template <typename T>
static int spgemm_bwd_t(const csrk_pattern &A, const T *Av, const csrk_pattern *AT, const int64_t *perm,
                        const csrk_pattern &B, const T *Bv, const csrk_pattern &C, const T *dC, T *dA, T *dB,
                        Bump &ws, cudaStream_t s)
{
    if (!AT) return spgemm_values_t<T>(PH_BWD, A, Av, B, Bv, C, nullptr, dC, dA, dB, ws, s);
    size_t fused_used = 0;
    if (!dB_flat(B) && fused_plan_bwd() && (ws.sizing() || (dA && dB))) {
        // both gradients in one pass over B's rows (k_gemm_bwd_rows), dB of long B rows by
        // k_gemm_dB_long and their dA by k_gemm_dA_long.  (Sizing: the larger of this and the
        // two-pass path below, which a call without dA or dB takes.)
        Bump wf = ws;
        DbLong lng{};
        lng.ctr = wf.take<unsigned long long>(1);
        lng.rows = wf.take<int32_t>(B.nrows > 0 ? B.nrows : 1);
        lng.chunk0 = wf.take<int64_t>(B.nrows > 0 ? B.nrows : 1);
        if (wf.overflow) return CSRK_ERR_WORKSPACE;
        fused_used = wf.used;
    }
    if (!ws.sizing() && fused_used) {
        DbLong lng{};
        lng.ctr = ws.take<unsigned long long>(1);
        lng.rows = ws.take<int32_t>(B.nrows > 0 ? B.nrows : 1);
        lng.chunk0 = ws.take<int64_t>(B.nrows > 0 ? B.nrows : 1);
        if (A.nnz == 0) return B.nnz > 0 ? (cudaMemsetAsync(dB, 0, sizeof(T) * (size_t)B.nnz, s) == cudaSuccess
                                            ? CSRK_OK : CSRK_ERR_CUDA) : CSRK_OK;
        if (B.nnz / 32 + B.nrows >= (int64_t)UINT32_MAX) return CSRK_ERR_INDEX_OVERFLOW;
        CSRK_CUDA(cudaMemsetAsync(lng.ctr, 0, sizeof(unsigned long long), s));
        const int64_t warps = cdiv(B.nrows, 32);
        const int64_t cap = (int64_t)kNumSMs * 8 * (kDbTPB / 32);
        const int64_t grid = cdiv(warps < cap ? warps : cap, kDbTPB / 32);
        if (B.nrows > 0)
            CSRK_LAUNCH(k_gemm_bwd_rows<T>, (unsigned)grid, kDbTPB, 0, s, B.nrows, B.indptr, B.indices, Bv, AT->indptr,
                        AT->indices, perm, Av, C.indptr, C.indices, dC, dA, dB, lng);
        CSRK_LAUNCH(k_gemm_dB_long<T>, (unsigned)(kNumSMs * 8), kDbTPB, 0, s, B.indptr, B.indices, AT->indptr,
                    AT->indices, perm, Av, C.indptr, C.indices, dC, dB, lng);
        CSRK_LAUNCH(k_gemm_dA_long<T>, (unsigned)(kNumSMs * 4), kDbTPB, 0, s, B.indptr, B.indices, Bv, AT->indptr,
                    AT->indices, perm, C.indptr, C.indices, dC, dA, lng);
        return CSRK_OK;
    }
    // dA by the row traversal (no dB), then the dB gather; they run in order on one stream and
    // share the scratch
    Bump w2 = ws;
    if (dA || ws.sizing()) CSRK_TRY(spgemm_values_t<T>(PH_BWD, A, Av, B, Bv, C, nullptr, dC, dA, nullptr, w2, s));
    if (ws.sizing()) {
        CSRK_TRY(launch_dB_gather<T>(B, *AT, perm, Av, C, dC, dB, ws, s));
        ws.used = w2.used > ws.used ? w2.used : ws.used;
        ws.used = fused_used > ws.used ? fused_used : ws.used;
        return CSRK_OK;
    }
    if (!dB) return CSRK_OK;
    return launch_dB_gather<T>(B, *AT, perm, Av, C, dC, dB, ws, s);
}

int spgemm_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
               const csrk_pattern &B, const void *B_val, const csrk_pattern &C, const void *dC, void *dA, void *dB,
               Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return spgemm_bwd_t<double>(A, (const double *)A_val, AT, perm, B, (const double *)B_val, C,
                                    (const double *)dC, (double *)dA, (double *)dB, ws, s);
    return spgemm_bwd_t<float>(A, (const float *)A_val, AT, perm, B, (const float *)B_val, C, (const float *)dC,
                               (float *)dA, (float *)dB, ws, s);
}

}  // namespace csrk
