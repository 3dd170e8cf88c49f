// rows.cuh -- thread-per-row CSR traversal with a warp-per-row pass for long rows.
//
// k_rows: one thread per row.  Rows of at most kShortRow nonzeros are processed by their
// thread; the thread's index/value loads are contiguous, and across a warp the L1 serves the
// neighbouring rows' lines, so short-row matrices (stencils) stream at near copy bandwidth
// without staging or block synchronisation.  Rows of kShortRow < l <= kHugeRow are then taken
// by the whole warp one at a time (coalesced over the row); longer rows by the whole CTA once
// its block is done (no second kernel launch).  Per-element
// modes (scatter, transpose) stream the warp's element range instead, unless it holds a
// huge row.
// Modes (same semantics as tile.cuh):
//   REDUCE    y[row] = sum_p val(pv) v[idx p]  (in p order -- the oracle's order -- for short
//             rows; lane-strided + fixed shuffle tree for long rows; both deterministic)
//             SIDE: D[pv] = v[idx p] * u[row]
//   SCATTER   w = u[row]; SIDE: D[p] = w v[idx p]; y64 (nullable): y64[idx p] += val[p] w (fp64 atomic)
//   TRANSPOSE slot = cursor[idx p]++ (atomic); keys[slot] = (p << 31) | row
#pragma once

#include "csrk_internal.cuh"
#include "tile.cuh"

namespace csrk {

#ifndef CSRK_STREAM_UNROLL
#define CSRK_STREAM_UNROLL 4
#endif
constexpr int kStreamUnroll = CSRK_STREAM_UNROLL;  // A/B via CSRK_NVCC_EXTRA
constexpr int kShortRow = 32;
constexpr int kHugeRow = 4096;
constexpr int kRowsTPB = 256;

struct RowList {
    int32_t *rows;
    int *count;
};

// D += product, the product rounded first (no contraction): the same bits as forming the product
// into a scratch array and adding it afterwards
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// REDUCE output: y[row] = acc, or y[row] += acc (accY, internal: the PCG's adjoint accumulation)
// dotw (internal): dp += y_row * dotw[row] for the thread that stores the row (fused dot product)
template <typename T>
__device__ __forceinline__ void store_y(const TileArgs<T> &a, int64_t row, double acc, double &dp)
{
    const T y = a.accY ? add_rn(a.y[row], (T)acc) : (T)acc;
    a.y[row] = y;
    if (a.dotw) dp = fma((double)y, (double)a.dotw[row], dp);
}

template <typename T, int MODE, bool PERM, bool SIDE>
__device__ __forceinline__ void row_elem(const TileArgs<T> &a, int64_t row, int64_t p, double &acc)
{
    const int32_t c = a.indices[p];
    if (MODE == MODE_REDUCE) {
        const int64_t pv = PERM ? a.perm[p] : p;
        const T vc = a.v[c];
        acc = fma((double)a.vals[pv], (double)vc, acc);
        if (SIDE) a.D[pv] = a.accD ? add_rn(a.D[pv], mul_rn(vc, a.u[row])) : (T)(vc * a.u[row]);
    } else if (MODE == MODE_SCATTER) {
        const T w = a.u[row];
        if (SIDE) a.D[p] = a.accD ? add_rn(a.D[p], mul_rn(w, a.v[c])) : (T)(w * a.v[c]);
        if (a.y64) atomicAdd(&a.y64[c], (double)a.vals[p] * (double)w);
    } else {
        const int64_t slot = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(&a.cursor[c]), 1ULL);
        a.out_keys[slot] = ((uint64_t)p << 31) | (uint64_t)row;
    }
}

template <typename T, int MODE, bool PERM, bool SIDE>
__device__ __forceinline__ void rows_block(const TileArgs<T> &a, int64_t vb, int *s_nh, int32_t *s_h, double &dp)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t row = vb * kRowsTPB + threadIdx.x;
    const bool valid = row < a.nrows;
    int64_t s = 0, e = 0;
    if (valid) {
        s = a.indptr[row];
        e = a.indptr[row + 1];
    }
    const bool huge = valid && e - s > kHugeRow;
    const unsigned hm = __ballot_sync(FULL, huge);
    if (hm) {  // rows longer than kHugeRow: taken by the whole CTA afterwards (rows_huge)
        int base = 0;
        if (lane == 0) base = atomicAdd(s_nh, __popc(hm));
        base = __shfl_sync(FULL, base, 0);
        if (huge) s_h[base + __popc(hm & ((1u << lane) - 1))] = (int32_t)row;
    }
    const bool lng = valid && e - s > kShortRow && !huge;
    if (MODE != MODE_REDUCE && !hm) {
        // per-element outputs (scatter / transpose): stream the warp's contiguous element range
        // coalesced; element -> row by a shuffle binary search over the 32 row starts
        const int64_t s_eff = valid ? s : INT64_MAX;
        const int64_t e0 = __shfl_sync(FULL, s, 0);
        int64_t e1 = valid ? e : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t y = __shfl_xor_sync(FULL, e1, o);
            e1 = y > e1 ? y : e1;
        }
        const int64_t r0 = row - lane;
        double dummy = 0.0;
        if (!__any_sync(FULL, lng)) {
            // all rows short: element -> lane map in shared memory (<= 32 x kShortRow elements)
            __shared__ uint8_t s_rw[kRowsTPB / 32][32 * kShortRow];
            const int w = threadIdx.x >> 5;
            for (int64_t p = s; p < e; ++p) s_rw[w][p - e0] = (uint8_t)lane;
            __syncwarp();
#pragma unroll kStreamUnroll
            for (int64_t p = e0 + lane; p < e1; p += 32) row_elem<T, MODE, PERM, SIDE>(a, r0 + s_rw[w][p - e0], p, dummy);
            return;
        }
        for (int64_t pb = e0; pb < e1; pb += 32) {
            const int64_t p = pb + lane;
            int lo = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const int64_t sc = __shfl_sync(FULL, s_eff, lo + st);
                if (sc <= p) lo += st;
            }
            if (p < e1) row_elem<T, MODE, PERM, SIDE>(a, r0 + lo, p, dummy);
        }
        return;
    }
    bool done = false;
    if (MODE == MODE_REDUCE && !hm) {
        // long average rows (power-law bodies, config 4: 8..32 entries): a 4-lane group per row so
        // the index / value loads of a warp instruction cover 8 rows instead of 32 (the per-thread
        // walk is bound by L1 wavefronts there); lane-strided sums + a fixed 2-step shuffle tree
        const int len = valid && !lng ? (int)(e - s) : 0;
        const int tot = (int)__reduce_add_sync(FULL, (unsigned)len);
        if (tot > 32 * 8) {
            const int g = lane >> 2, sub = lane & 3;
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
                const int src = 4 * g + k;
                const int64_t rs = __shfl_sync(FULL, s, src), re = __shfl_sync(FULL, e, src);
                const bool own = __shfl_sync(FULL, (int)(valid && !lng), src) != 0;
                double acc = 0.0;
                if (own)
#pragma unroll 2
                    for (int64_t p = rs + sub; p < re; p += 4) row_elem<T, MODE, PERM, SIDE>(a, row - lane + src, p, acc);
                acc += __shfl_xor_sync(FULL, acc, 1);
                acc += __shfl_xor_sync(FULL, acc, 2);
                if (own && sub == 0) store_y(a, row - lane + src, acc, dp);
            }
            done = true;
        }
    }
    if (valid && !lng && !huge && !done) {
        double acc = 0.0;
#pragma unroll 4
        for (int64_t p = s; p < e; ++p) row_elem<T, MODE, PERM, SIDE>(a, row, p, acc);
        if (MODE == MODE_REDUCE) store_y(a, row, acc, dp);
    }
    // rows of kShortRow < l <= kHugeRow: the warp takes them one by one (coalesced over the row,
    // fixed shuffle tree -- deterministic)
    unsigned lm = __ballot_sync(FULL, lng);
    while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const int64_t rs = __shfl_sync(FULL, s, src), re = __shfl_sync(FULL, e, src);
        const int64_t r = row - lane + src;
        double acc = 0.0;
#pragma unroll 4
        for (int64_t p = rs + lane; p < re; p += 32) row_elem<T, MODE, PERM, SIDE>(a, r, p, acc);
        if (MODE == MODE_REDUCE) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
            if (lane == 0) store_y(a, r, acc, dp);
        }
    }
}

// One row longer than kHugeRow, by the whole CTA (lane-strided; REDUCE: fixed warp and block
// trees -- deterministic)
template <typename T, int MODE, bool PERM, bool SIDE>
__device__ __forceinline__ void rows_huge(const TileArgs<T> &a, int64_t row, double *s_red, double &dp)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t s = a.indptr[row], e = a.indptr[row + 1];
    double acc = 0.0;
#pragma unroll 4
    for (int64_t p = s + threadIdx.x; p < e; p += kRowsTPB) row_elem<T, MODE, PERM, SIDE>(a, row, p, acc);
    if (MODE == MODE_REDUCE) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) s_red[w] = acc;
        __syncthreads();
        if (w == 0) {
            acc = lane < kRowsTPB / 32 ? s_red[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) store_y(a, row, acc, dp);
        }
        __syncthreads();
    }
}

// One CTA per block of kRowsTPB rows, which then takes the block's rows longer than kHugeRow
// together (no second kernel); the transpose scatter (MODE_TRANSPOSE, which runs gated behind the
// symmetric-pattern transpose) grid-strides over the blocks with a resident-sized grid instead,
// so that skipping it costs a few CTAs, not one per 256 rows.
template <int MODE> constexpr bool rows_persistent() { return MODE == MODE_TRANSPOSE; }

template <typename T, int MODE, bool PERM, bool SIDE>
__global__ __launch_bounds__(kRowsTPB, 8) void k_rows(TileArgs<T> a)
{
    pdl_wait();
    if (a.run_if && *(volatile const int *)a.run_if == 0) return;
    __shared__ int s_nh;
    __shared__ int32_t s_h[kRowsTPB];
    __shared__ double s_red[kRowsTPB / 32];
    double dp = 0.0;   // fused dot product (dotw): this thread's rows
    auto block = [&](int64_t vb) {
        if (threadIdx.x == 0) s_nh = 0;
        __syncthreads();
        rows_block<T, MODE, PERM, SIDE>(a, vb, &s_nh, s_h, dp);
        __syncthreads();
        const int nh = s_nh;
        for (int h = 0; h < nh; ++h) rows_huge<T, MODE, PERM, SIDE>(a, s_h[h], s_red, dp);
    };
    if constexpr (rows_persistent<MODE>()) {
        const int64_t nvb = cdiv(a.nrows, kRowsTPB);
        for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
            block(vb);
            __syncthreads();   // s_nh, s_h and the warps' s_rw maps are reused by the next block
        }
    } else {
        block(blockIdx.x);
    }
    if (MODE == MODE_REDUCE && a.dotw) {   // the CTA's partial, fixed shuffle + warp-order tree
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
        __syncthreads();
        if (lane == 0) s_red[w] = dp;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < kRowsTPB / 32; ++q) t += s_red[q];
            a.dotpart[blockIdx.x] = t;
        }
    }
}

// *out = sum of the nb CTA partials of a fused dot product, in a fixed order
static __global__ __launch_bounds__(256) void k_dot_finish(const double *__restrict__ part, int64_t nb, double *out)
{
    pdl_wait();
    __shared__ double s[8];
    double acc = 0.0;
    for (int64_t q = threadIdx.x; q < nb; q += 256) acc += part[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += s[q];
        *out = t;
    }
}

// Workspace: the long-row list (int32 per row + a counter).
inline void carve_rowlist(int64_t nrows, RowList &L, Bump &ws)
{
    L.rows = ws.take<int32_t>(nrows > 0 ? nrows : 1);
    L.count = ws.take<int>(1);
}

template <typename T, int MODE, bool PERM, bool SIDE>
int launch_rows(const TileArgs<T> &a, const RowList &, cudaStream_t s)
{
    if (a.nrows <= 0) return CSRK_OK;
    const int64_t nvb = cdiv(a.nrows, kRowsTPB);
    const int64_t cap = rows_persistent<MODE>() ? (int64_t)kNumSMs * 8 : nvb;
    const int64_t grid = nvb < cap ? nvb : cap;
    CSRK_LAUNCH((k_rows<T, MODE, PERM, SIDE>), (unsigned)grid, kRowsTPB, 0, s, a);
    if (MODE == MODE_REDUCE && a.dotw) CSRK_LAUNCH(k_dot_finish, 1, 256, 0, s, (const double *)a.dotpart, grid, a.dotout);
    return CSRK_OK;
}

}  // namespace csrk
