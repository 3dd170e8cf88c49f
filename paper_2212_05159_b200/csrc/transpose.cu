// transpose.cu -- CSR transpose with position map ("take the sparse transpose of A";
// S:53-61).  A counting sort by column:
//   1. column histogram (int64 atomics into AT_indptr[1..n])
//   2. int64 prefix scan -> AT_indptr
//   3. row-tile scatter (tile.cuh, MODE_TRANSPOSE): every nonzero claims a slot of its column
//      with an atomic cursor and stores ONE packed key  (p << 31) | row  (p = its position in
//      A).  Within a column rows are distinct and p grows with the row, so ordering keys
//      orders rows.
//   4. per-column sort of the keys (register network for <= 16, warp / CTA bitonic in shared
//      memory, merge sort through a workspace buffer beyond 8192), then unpack into
//      AT_indices (row) and AT_perm (p) -- canonical CSR, bit-identical to the stable
//      counting sort of the oracle regardless of the atomic order.
//   5. AT_val[q] = A_val[perm[q]] (optional)
// Matrices with scattered columns use the stable radix sort of radix.cu instead (use_radix).
// Packing needs nnz < 2^33 (checked).
//
// Structurally symmetric patterns (every stored (i, j) has a stored (j, i): Poisson stencils, the
// paper's PDE operators, undirected graphs) are tried first (k_tr_sym): then A^T has A's pattern,
// row j of A^T lists the same columns as row j of A, and the A^T slot of A's entry p = (i, j) is
// the position q of i inside row j -- one binary search per entry, no counting, no sort:
// AT_indptr = A_indptr, AT_indices = A_indices, AT_perm[q] = p.  A failed search marks the
// pattern unsymmetric (device flag), and the general kernels above, which are launched behind it
// and read the flag, then run; on success they return at once.  Exact either way.

#include "condgraph.cuh"
#include "ops.cuh"
#include "rows.cuh"
#include "tile.cuh"

namespace csrk {

constexpr int kRegMax = 16;
constexpr int kWarpMax = 1024;
constexpr int kBlockMax = 8192;
constexpr int kSortTPB = 256;
constexpr uint64_t kKeyPad = ~0ull;

__device__ __forceinline__ int32_t key_row(uint64_t k) { return (int32_t)(k & 0x7fffffffull); }
__device__ __forceinline__ int64_t key_pos(uint64_t k) { return (int64_t)(k >> 31); }

// Column histogram (plain atomics: warp aggregation with __match_any_sync measured 2x slower).
__global__ void k_col_count(int64_t nnz, const int32_t *__restrict__ indices, unsigned long long *__restrict__ cnt,
                            const int *run_if)
{
    pdl_wait();
    if (run_if && *(volatile const int *)run_if == 0) return;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[indices[p]], 1ULL);
}

struct SortLists {
    int32_t *mid, *big, *huge;
    int *count;  // [3]
};

template <int N>
__device__ __forceinline__ void reg_sort(uint64_t (&k)[N])
{
#pragma unroll
    for (int size = 2; size <= N; size <<= 1)
#pragma unroll
        for (int stride = size / 2; stride > 0; stride >>= 1)
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool asc = (i & size) == 0;
                    const uint64_t a = k[i], b = k[j];
                    if ((a > b) == asc) { k[i] = b; k[j] = a; }
                }
            }
}

template <int N>
__device__ __forceinline__ void sort_unpack_regs(const uint64_t *__restrict__ keys, int64_t s, int len,
                                                 int32_t *__restrict__ ATi, int64_t *__restrict__ perm)
{
    uint64_t k[N];
#pragma unroll
    for (int i = 0; i < N; ++i) k[i] = i < len ? keys[s + i] : kKeyPad;
    reg_sort<N>(k);
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (i < len) {
            ATi[s + i] = key_row(k[i]);
            perm[s + i] = key_pos(k[i]);
        }
}

// Sort one short column held in shared memory (keys s[0..len)) in registers, in place.
template <int N>
__device__ __forceinline__ void sort_smem_regs(uint64_t *s, int len)
{
    uint64_t k[N];
#pragma unroll
    for (int i = 0; i < N; ++i) k[i] = i < len ? s[i] : kKeyPad;
    reg_sort<N>(k);
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (i < len) s[i] = k[i];
}

constexpr int kShortWarps = 8;
constexpr int kShortBuf = 512;   // keys staged per warp

// A warp owns 32 consecutive columns.  When they are all short (<= 16) and their keys fit the
// warp's buffer, the keys are loaded coalesced into shared memory, each lane sorts its column
// there with a register network, and the unpacked rows / positions are stored coalesced.
// Otherwise each lane sorts its short column straight from global memory; longer columns are
// queued for the warp / CTA / merge-sort kernels.
__global__ __launch_bounds__(32 * kShortWarps) void k_sort_short(int64_t n, const int64_t *__restrict__ ATp,
                                                                 const uint64_t *__restrict__ keys,
                                                                 int32_t *__restrict__ ATi,
                                                                 int64_t *__restrict__ perm, SortLists L,
                                                                 const int *run_if)
{
    pdl_wait();
    if (run_if && *(volatile const int *)run_if == 0) return;
    __shared__ uint64_t s_key[kShortWarps][kShortBuf];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t j0 = ((int64_t)blockIdx.x * kShortWarps + w) * 32; j0 < n;
         j0 += (int64_t)gridDim.x * kShortWarps * 32) {
        const int64_t j = j0 + lane;
        const bool valid = j < n;
        const int64_t s = valid ? ATp[j] : 0, e = valid ? ATp[j + 1] : 0;
        const int len = (int)(e - s);
        const int64_t lastj = (n - j0 < 32 ? n - j0 : 32) - 1;
        const int64_t R0 = __shfl_sync(0xffffffffu, s, 0), R1 = __shfl_sync(0xffffffffu, e, (int)lastj);
        const bool fast = __all_sync(0xffffffffu, len <= kRegMax) && R1 - R0 <= kShortBuf;
        if (fast) {
            const int span = (int)(R1 - R0);
            for (int i = lane; i < span; i += 32) s_key[w][i] = keys[R0 + i];
            __syncwarp();
            if (len > 1) {
                if (len <= 8) sort_smem_regs<8>(&s_key[w][s - R0], len);
                else sort_smem_regs<16>(&s_key[w][s - R0], len);
            }
            __syncwarp();
            for (int i = lane; i < span; i += 32) {
                const uint64_t k = s_key[w][i];
                ATi[R0 + i] = key_row(k);
                perm[R0 + i] = key_pos(k);
            }
            __syncwarp();
            continue;
        }
        if (len == 0) continue;
        if (len <= 8) {
            sort_unpack_regs<8>(keys, s, len, ATi, perm);
        } else if (len <= kRegMax) {
            sort_unpack_regs<16>(keys, s, len, ATi, perm);
        } else if (len <= kWarpMax) {
            L.mid[atomicAdd(&L.count[0], 1)] = (int32_t)j;
        } else if (len <= kBlockMax) {
            L.big[atomicAdd(&L.count[1], 1)] = (int32_t)j;
        } else {
            L.huge[atomicAdd(&L.count[2], 1)] = (int32_t)j;
        }
    }
}

// Bitonic sort of u64 keys in shared memory; `nt` threads cooperate.
template <bool WARP>
__device__ __forceinline__ void smem_bitonic(uint64_t *key, int P, int t, int nt)
{
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = t; i < P; i += nt) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool asc = (i & k) == 0;
                    const uint64_t a = key[i], b = key[ixj];
                    if ((a > b) == asc) { key[i] = b; key[ixj] = a; }
                }
            }
            if (WARP) __syncwarp(); else __syncthreads();
        }
}

__device__ __forceinline__ int pow2ceil(int x)
{
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

constexpr int kWarpsPerSortCTA = 4;

__global__ __launch_bounds__(32 * kWarpsPerSortCTA) void k_sort_warp(const int64_t *__restrict__ ATp,
                                                                     const uint64_t *__restrict__ keys,
                                                                     int32_t *__restrict__ ATi,
                                                                     int64_t *__restrict__ perm, SortLists L)
{
    pdl_wait();
    __shared__ uint64_t s_key[kWarpsPerSortCTA][kWarpMax];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cnt = *(volatile int *)&L.count[0];
    for (int it = blockIdx.x * kWarpsPerSortCTA + w; it < cnt; it += gridDim.x * kWarpsPerSortCTA) {
        const int64_t j = L.mid[it];
        const int64_t s = ATp[j];
        const int len = (int)(ATp[j + 1] - s);
        const int P = pow2ceil(len);
        for (int i = lane; i < P; i += 32) s_key[w][i] = i < len ? keys[s + i] : kKeyPad;
        __syncwarp();
        smem_bitonic<true>(s_key[w], P, lane, 32);
        for (int i = lane; i < len; i += 32) {
            ATi[s + i] = key_row(s_key[w][i]);
            perm[s + i] = key_pos(s_key[w][i]);
        }
        __syncwarp();
    }
}

__global__ __launch_bounds__(kSortTPB) void k_sort_block(const int64_t *__restrict__ ATp,
                                                         const uint64_t *__restrict__ keys, int32_t *__restrict__ ATi,
                                                         int64_t *__restrict__ perm, SortLists L)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *s_key = reinterpret_cast<uint64_t *>(smem);
    const int cnt = *(volatile int *)&L.count[1];
    for (int it = blockIdx.x; it < cnt; it += gridDim.x) {
        const int64_t j = L.big[it];
        const int64_t s = ATp[j];
        const int len = (int)(ATp[j + 1] - s);
        const int P = pow2ceil(len);
        for (int i = threadIdx.x; i < P; i += kSortTPB) s_key[i] = i < len ? keys[s + i] : kKeyPad;
        __syncthreads();
        smem_bitonic<false>(s_key, P, threadIdx.x, kSortTPB);
        for (int i = threadIdx.x; i < len; i += kSortTPB) {
            ATi[s + i] = key_row(s_key[i]);
            perm[s + i] = key_pos(s_key[i]);
        }
        __syncthreads();
    }
}

// Huge columns: runs of kBlockMax sorted in shared memory, then pairwise merge passes
// (merge-path split across the CTA) ping-ponging between `keys` and `buf`.
__global__ __launch_bounds__(kSortTPB) void k_sort_huge(const int64_t *__restrict__ ATp, uint64_t *__restrict__ keys,
                                                        uint64_t *__restrict__ buf, int32_t *__restrict__ ATi,
                                                        int64_t *__restrict__ perm, SortLists L)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *s_key = reinterpret_cast<uint64_t *>(smem);
    const int cnt = *(volatile int *)&L.count[2];
    for (int it = blockIdx.x; it < cnt; it += gridDim.x) {
        const int64_t j = L.huge[it];
        const int64_t s = ATp[j];
        const int64_t len = ATp[j + 1] - s;
        for (int64_t r = 0; r < len; r += kBlockMax) {
            const int rl = (int)(len - r < kBlockMax ? len - r : kBlockMax);
            const int P = pow2ceil(rl);
            for (int i = threadIdx.x; i < P; i += kSortTPB) s_key[i] = i < rl ? keys[s + r + i] : kKeyPad;
            __syncthreads();
            smem_bitonic<false>(s_key, P, threadIdx.x, kSortTPB);
            for (int i = threadIdx.x; i < rl; i += kSortTPB) keys[s + r + i] = s_key[i];
            __syncthreads();
        }
        uint64_t *src = keys + s, *dst = buf + s;
        for (int64_t width = kBlockMax; width < len; width <<= 1) {
            for (int64_t lo = 0; lo < len; lo += 2 * width) {
                const int64_t mid = lo + width < len ? lo + width : len;
                const int64_t hi = lo + 2 * width < len ? lo + 2 * width : len;
                const int64_t na = mid - lo, nb = hi - mid, tot = na + nb;
                const int64_t per = cdiv(tot, kSortTPB);
                const int64_t d0 = (int64_t)threadIdx.x * per < tot ? (int64_t)threadIdx.x * per : tot;
                const int64_t d1 = d0 + per < tot ? d0 + per : tot;
                int64_t a_lo = d0 - nb > 0 ? d0 - nb : 0, a_hi = d0 < na ? d0 : na;
                while (a_lo < a_hi) {
                    const int64_t piv = (a_lo + a_hi) >> 1;
                    if (src[lo + piv] < src[mid + d0 - piv - 1]) a_lo = piv + 1;
                    else a_hi = piv;
                }
                int64_t ia = a_lo, ib = d0 - a_lo;
                for (int64_t d = d0; d < d1; ++d) {
                    if (ib >= nb || (ia < na && src[lo + ia] < src[mid + ib])) dst[lo + d] = src[lo + ia++];
                    else dst[lo + d] = src[mid + ib++];
                }
            }
            __syncthreads();
            uint64_t *t = src; src = dst; dst = t;
        }
        for (int64_t i = threadIdx.x; i < len; i += kSortTPB) {
            const uint64_t k = src[i];
            ATi[s + i] = key_row(k);
            perm[s + i] = key_pos(k);
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void k_gather_vals(int64_t nnz, const int64_t *__restrict__ perm, const T *__restrict__ A_val,
                              T *__restrict__ AT_val)
{
    pdl_wait();
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
        AT_val[q] = A_val[perm[q]];
}

// ---------------------------------------------------------------- structurally symmetric patterns
constexpr int kSymTPB = 256;
constexpr int kSymShort = 32;
#ifndef CSRK_SYM_U
#define CSRK_SYM_U 4
#endif
constexpr int kSymU = CSRK_SYM_U;   // k_tr_sym: entries searched in lock step (A/B via CSRK_NVCC_EXTRA)

// position of v in the sorted c[lo, hi), or -1
__device__ __forceinline__ int64_t sym_find(const int32_t *__restrict__ c, int64_t lo, int64_t hi, int32_t v)
{
    int64_t l = lo, h = hi;
    while (l < h) {
        const int64_t mid = (l + h) >> 1;
        if (__ldg(c + mid) < v) l = mid + 1; else h = mid;
    }
    return (l < hi && __ldg(c + l) == v) ? l : -1;
}

// One thread per row of A (rows longer than kSymShort: the warp, lanes over the entries).  For
// every entry p = (i, j): q = position of i in row j (binary search; kSymU entries of a row at a
// time, their searches in flight together); AT_perm[q] = p, AT_indices[p] = j.  `bad` is set
// when some (j, i) is missing; warps stop early once it is.
__global__ __launch_bounds__(kSymTPB) void k_tr_sym(int64_t m, const int64_t *__restrict__ Ap,
                                                    const int32_t *__restrict__ Ai, int64_t *__restrict__ ATp,
                                                    int32_t *__restrict__ ATi, int64_t *__restrict__ perm, int *bad)
{
    pdl_wait();
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * kSymTPB + threadIdx.x;
    if (__any_sync(FULL, *(volatile int *)bad != 0)) return;
    const bool valid = i < m;
    int64_t s = 0, e = 0;
    if (valid) {
        s = Ap[i];
        e = Ap[i + 1];
        ATp[i] = s;
        if (i == m - 1) ATp[m] = e;
    }
    bool miss = false;
    const bool lng = e - s > kSymShort;
    if (!lng)
        for (int64_t p0 = s; p0 < e; p0 += kSymU) {
            int64_t lo[kSymU], end[kSymU];
            int32_t len[kSymU];
#pragma unroll
            for (int u = 0; u < kSymU; ++u) {
                lo[u] = end[u] = 0;
                len[u] = 0;
                if (p0 + u < e) {
                    const int32_t j = Ai[p0 + u];
                    ATi[p0 + u] = j;
                    lo[u] = __ldg(Ap + j);
                    end[u] = __ldg(Ap + j + 1);
                    len[u] = (int32_t)(end[u] - lo[u]);
                }
            }
            bool any = true;
            while (any) {   // lower bound of i in row j: len = entries left to the right of lo
                any = false;
#pragma unroll
                for (int u = 0; u < kSymU; ++u) {
                    if (len[u] > 0) {
                        const int32_t half = len[u] >> 1;
                        if (__ldg(Ai + lo[u] + half) < (int32_t)i) {
                            lo[u] += half + 1;
                            len[u] -= half + 1;
                        } else {
                            len[u] = half;
                        }
                        any = true;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kSymU; ++u) {
                if (p0 + u >= e) continue;
                const bool hit = lo[u] < end[u] && __ldg(Ai + lo[u]) == (int32_t)i;
                if (!hit) miss = true; else perm[lo[u]] = p0 + u;
            }
        }
    unsigned lm = __ballot_sync(FULL, lng);
    while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const int64_t rs = __shfl_sync(FULL, s, src), re = __shfl_sync(FULL, e, src);
        const int32_t r = (int32_t)(i - lane + src);
        for (int64_t p = rs + lane; p < re; p += 32) {
            const int32_t j = Ai[p];
            ATi[p] = j;
            const int64_t q = sym_find(Ai, Ap[j], Ap[j + 1], r);
            if (q < 0) miss = true; else perm[q] = p;
        }
    }
    if (__any_sync(FULL, miss) && lane == 0) atomicExch(bad, 1);
}

// x[0..n) = 0 / dst[0..n) = src[0..n), unless *run_if == 0
__global__ void k_zero_i64_if(int64_t *__restrict__ x, int64_t n, const int *run_if)
{
    pdl_wait();
    if (*(volatile const int *)run_if == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = 0;
}
__global__ void k_copy_i64_if(int64_t *__restrict__ dst, const int64_t *__restrict__ src, int64_t n, const int *run_if)
{
    pdl_wait();
    if (*(volatile const int *)run_if == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

static unsigned grid_for(int64_t work, int tpb)
{
    int64_t g = cdiv(work, tpb);
    const int64_t cap = (int64_t)kNumSMs * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

int transpose_radix(const csrk_pattern &A, int64_t *ATp, int32_t *ATi, int64_t *perm, Bump &ws, cudaStream_t s);

// Scattered columns (many columns, many entries each: config 4) take the radix sort of radix.cu;
// banded / stencil matrices keep the atomic-cursor scatter + per-column sort (measured faster
// there).  CSRK_TRANSPOSE_RADIX=0/1 forces either.
static bool use_radix(const csrk_pattern &A)
{
    static int k = knob("TRANSPOSE_RADIX", -1);
    if (k >= 0) return k != 0;
    return A.ncols >= (int64_t(1) << 22) && A.nnz >= 8 * A.ncols;
}

int transpose_impl(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t *ATp, int32_t *ATi,
                   void *AT_val, int64_t *perm, Bump &ws, cudaStream_t s)
{
    const int64_t n = A.ncols, nnz = A.nnz;
    if (nnz >= (int64_t(1) << 33)) return CSRK_ERR_INDEX_OVERFLOW;
    if (use_radix(A)) {
        int64_t *pm = perm ? perm : ws.take<int64_t>(nnz > 0 ? nnz : 1);
        CSRK_TRY(transpose_radix(A, ATp, ATi, pm, ws, s));
        if (ws.sizing() || !AT_val || nnz == 0) return CSRK_OK;
        if (dt == CSRK_F64)
            CSRK_LAUNCH(k_gather_vals<double>, grid_for(nnz, 256), 256, 0, s, nnz, (const int64_t *)pm,
                        (const double *)A_val, (double *)AT_val);
        else
            CSRK_LAUNCH(k_gather_vals<float>, grid_for(nnz, 256), 256, 0, s, nnz, (const int64_t *)pm,
                        (const float *)A_val, (float *)AT_val);
        return CSRK_OK;
    }
    int64_t *cursor = ws.take<int64_t>(n > 0 ? n : 1);
    uint64_t *keys = ws.take<uint64_t>(nnz > 0 ? nnz : 1);
    int64_t *pm = perm ? perm : ws.take<int64_t>(nnz > 0 ? nnz : 1);
    SortLists L{};
    L.mid = ws.take<int32_t>(nnz / (kRegMax + 1) + 1);
    L.big = ws.take<int32_t>(nnz / (kWarpMax + 1) + 1);
    L.huge = ws.take<int32_t>(nnz / (kBlockMax + 1) + 1);
    L.count = ws.take<int>(4);
    uint64_t *buf = ws.take<uint64_t>(nnz > kBlockMax ? nnz : 1);
    RowList RL{};
    carve_rowlist(A.nrows, RL, ws);
    int *sym_bad = ws.take<int>(1);
    if (ws.sizing()) return scan_counts_i64(nullptr, n, ws, s);  // carve the scan scratch

    const size_t big_smem = sizeof(uint64_t) * kBlockMax;
    static DevOnce attr;
    if (attr.need()) {
        CSRK_CUDA(cudaFuncSetAttribute(k_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
        CSRK_CUDA(cudaFuncSetAttribute(k_sort_huge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
        attr.done();
    }
    // The general counting-sort path on stream st.  gate (device flag, nullable): every kernel
    // returns at once unless *gate != 0 -- how it runs behind the symmetric attempt on a plain stream.
    auto general = [&](cudaStream_t st, const int *gate, Bump &w) -> int {
        if (gate) CSRK_LAUNCH(k_zero_i64_if, grid_for(n + 1, 256), 256, 0, st, ATp, n + 1, gate);
        else CSRK_CUDA(cudaMemsetAsync(ATp, 0, sizeof(int64_t) * (size_t)(n + 1), st));
        if (nnz > 0)
            CSRK_LAUNCH(k_col_count, grid_for(nnz, 256), 256, 0, st, nnz, A.indices,
                        reinterpret_cast<unsigned long long *>(ATp + 1), gate);
        CSRK_TRY(scan_counts_i64(ATp, n, w, st, gate));
        if (nnz == 0) return CSRK_OK;
        if (gate) CSRK_LAUNCH(k_copy_i64_if, grid_for(n, 256), 256, 0, st, cursor, (const int64_t *)ATp, n, gate);
        else CSRK_CUDA(cudaMemcpyAsync(cursor, ATp, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToDevice, st));
        CSRK_CUDA(cudaMemsetAsync(L.count, 0, sizeof(int) * 4, st));
        {
            TileArgs<double> a{};
            a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
            a.cursor = cursor; a.out_keys = keys;
            a.R = tile_rows(A.nrows, nnz);
            a.run_if = gate;
            if (knob("SPMV_TILE", 0)) CSRK_TRY((launch_tile<double, MODE_TRANSPOSE, false, false>(a, st)));
            else CSRK_TRY((launch_rows<double, MODE_TRANSPOSE, false, false>(a, RL, st)));
        }
        CSRK_LAUNCH(k_sort_short, grid_for(cdiv(n, 32) * 32, 32 * kShortWarps), 32 * kShortWarps, 0, st, n,
                    (const int64_t *)ATp, (const uint64_t *)keys, ATi, pm, L, gate);
        if (nnz > kRegMax)
            CSRK_LAUNCH(k_sort_warp, (unsigned)(kNumSMs * 4), 32 * kWarpsPerSortCTA, 0, st, (const int64_t *)ATp,
                        (const uint64_t *)keys, ATi, pm, L);
        if (nnz > kWarpMax)
            CSRK_LAUNCH(k_sort_block, (unsigned)kNumSMs, kSortTPB, big_smem, st, (const int64_t *)ATp,
                        (const uint64_t *)keys, ATi, pm, L);
        if (nnz > kBlockMax)
            CSRK_LAUNCH(k_sort_huge, (unsigned)kNumSMs, kSortTPB, big_smem, st, (const int64_t *)ATp, keys, buf, ATi,
                        pm, L);
        return CSRK_OK;
    };
    auto sym = [&](cudaStream_t st) -> int {
        CSRK_CUDA(cudaMemsetAsync(sym_bad, 0, sizeof(int), st));
        CSRK_LAUNCH(k_tr_sym, (unsigned)cdiv(A.nrows, kSymTPB), kSymTPB, 0, st, A.nrows, A.indptr, A.indices, ATp,
                    ATi, pm, sym_bad);
        return CSRK_OK;
    };
    // Symmetric pattern first (square, not the SPMV_TILE A/B path).  Default: one CUDA graph whose
    // conditional node runs the general path only if k_tr_sym found a missing mirror (no launches
    // at all otherwise); fallback / CSRK_TRANSPOSE_GRAPH=0: the general kernels gated on the flag.
    const bool try_sym = A.nrows == A.ncols && nnz > 0 && knob("TRANSPOSE_SYM", 1) && !knob("SPMV_TILE", 0);
    bool done = false;
    // not while the caller's stream is being captured (e.g. inside the PCG step's graph): a graph
    // cannot be captured and launched inside another capture -- the flag-gated kernels are captured
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(s, &cap_st) != cudaSuccess || cap_st != cudaStreamCaptureStatusNone;
    if (try_sym && knob("TRANSPOSE_GRAPH", 1) && !capturing) {
        int dev = 0;
        cudaGetDevice(&dev);
        const CondKey key = cond_key({(uint64_t)A.indptr, (uint64_t)A.indices, (uint64_t)A.nrows, (uint64_t)nnz,
                                      (uint64_t)ATp, (uint64_t)ATi, (uint64_t)pm, (uint64_t)ws.base, (uint64_t)ws.cap,
                                      (uint64_t)dev});
        Bump wb = ws;
        done = cond_graph_run(1, key, s, sym_bad, sym, [&](cudaStream_t cs) { return general(cs, nullptr, wb); }) ==
               CSRK_OK;
    }
    if (!done) {
        if (try_sym) CSRK_TRY(sym(s));
        CSRK_TRY(general(s, try_sym ? sym_bad : nullptr, ws));
    }
    if (nnz == 0) return CSRK_OK;
    if (AT_val) {
        if (dt == CSRK_F64)
            CSRK_LAUNCH(k_gather_vals<double>, grid_for(nnz, 256), 256, 0, s, nnz, (const int64_t *)pm,
                        (const double *)A_val, (double *)AT_val);
        else
            CSRK_LAUNCH(k_gather_vals<float>, grid_for(nnz, 256), 256, 0, s, nnz, (const int64_t *)pm,
                        (const float *)A_val, (float *)AT_val);
    }
    return CSRK_OK;
}

int csr_transpose(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t *AT_indptr, int32_t *AT_indices,
                  void *AT_val, int64_t *perm, Bump &ws, cudaStream_t s)
{
    return transpose_impl(dt, A, A_val, AT_indptr, AT_indices, AT_val, perm, ws, s);
}

}  // namespace csrk
