// radix.cu -- CSR transpose as a stable LSD radix sort of the nonzeros by column ("take the
// sparse transpose of A"), for matrices whose columns are scattered (config
// 4: uniform random columns, where claiming slots with atomic cursors and sorting every column
// afterwards costs ~15 ms).
//
// The nonzeros arrive sorted by row; a STABLE sort by column therefore leaves every column's
// rows ascending -- exactly the oracle's counting sort.  Keys are the column indices, values
// the packed (p << 31) | row (p = position in A).  8-bit digits, ceil(log2 ncols / 8) passes;
// each pass is
//   k_rs_up    per-tile digit histogram (4096 items per tile), stored digit-major;
//   scan       exclusive int64 scan of the 256 x ntiles counts (utils.cu);
//   k_rs_down  the tile again: per-warp ranking with __match_any_sync in item order, per-digit
//              warp prefixes in shared memory, scatter to offset + rank (stable).
// The last pass unpacks into AT_indices / AT_perm; AT_indptr is read off the sorted keys.
#include "ops.cuh"

namespace csrk {

constexpr int kRsTPB = 256;
constexpr int kRsWarps = kRsTPB / 32;
constexpr int kRsItems = 8;                     // per lane
constexpr int kRsTile = kRsTPB * kRsItems;      // 2048 items
constexpr int kRsBins = 256;

// row id of every nonzero (a thread per row; rows longer than 32 by the whole warp)
__global__ __launch_bounds__(256) void k_rs_rows(int64_t m, const int64_t *__restrict__ indptr,
                                                 int32_t *__restrict__ rows)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t s = 0, e = 0;
    if (i < m) {
        s = indptr[i];
        e = indptr[i + 1];
    }
    const bool lng = e - s > 32;
    if (!lng)
        for (int64_t p = s; p < e; ++p) rows[p] = (int32_t)i;
    unsigned lm = __ballot_sync(0xffffffffu, lng);
    while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const int64_t rs = __shfl_sync(0xffffffffu, s, src), re = __shfl_sync(0xffffffffu, e, src);
        const int32_t r = (int32_t)__shfl_sync(0xffffffffu, i, src);
        for (int64_t p = rs + lane; p < re; p += 32) rows[p] = r;
    }
}

__device__ __forceinline__ int64_t rs_item(int64_t tile, int warp, int r, int lane)
{
    return tile * kRsTile + (int64_t)warp * (32 * kRsItems) + r * 32 + lane;
}

// per-tile digit counts -> cnt[1 + d * ntiles + tile]
__global__ __launch_bounds__(kRsTPB) void k_rs_up(int64_t nnz, int64_t ntiles, int shift,
                                                  const int32_t *__restrict__ keys, int64_t *__restrict__ cnt)
{
    pdl_wait();
    __shared__ int s_h[kRsBins];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    s_h[tid] = 0;
    __syncthreads();
    int32_t k[kRsItems];
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int64_t p = rs_item(tile, warp, r, lane);
        k[r] = p < nnz ? keys[p] : -1;
    }
#pragma unroll
    for (int r = 0; r < kRsItems; ++r)
        if (k[r] >= 0) atomicAdd(&s_h[(k[r] >> shift) & 0xff], 1);
    __syncthreads();
    cnt[1 + (int64_t)tid * ntiles + tile] = s_h[tid];
}

#ifndef CSRK_RS_MINB
#define CSRK_RS_MINB 1
#endif
template <bool FIRST, bool LAST>
__global__ __launch_bounds__(kRsTPB, CSRK_RS_MINB) void k_rs_down(int64_t nnz, int64_t ntiles, int shift,
                                                    const int32_t *__restrict__ kin, const uint64_t *__restrict__ vin,
                                                    const int32_t *__restrict__ rows, const int64_t *__restrict__ cnt,
                                                    int32_t *__restrict__ kout, uint64_t *__restrict__ vout,
                                                    int32_t *__restrict__ ATi, int64_t *__restrict__ perm)
{
    pdl_wait();
    __shared__ int s_w[kRsWarps][kRsBins];  // per-warp digit counts, then per-warp prefixes
    __shared__ int64_t s_base[kRsBins];
    __shared__ int s_tot[kRsBins], s_start[kRsBins];
    __shared__ int32_t s_key[kRsTile];
    __shared__ uint64_t s_val[kRsTile];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    for (int q = tid; q < kRsWarps * kRsBins; q += kRsTPB) (&s_w[0][0])[q] = 0;
    s_base[tid] = cnt[(int64_t)tid * ntiles + tile];
    int32_t key[kRsItems];
    uint64_t val[kRsItems];
    int rank[kRsItems];
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int64_t p = rs_item(tile, warp, r, lane);
        key[r] = -1;
        val[r] = 0;
        if (p < nnz) {
            key[r] = kin[p];
            val[r] = FIRST ? (((uint64_t)p << 31) | (uint64_t)rows[p]) : vin[p];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int d = key[r] < 0 ? kRsBins : (key[r] >> shift) & 0xff;
        const unsigned peers = __match_any_sync(FULL, d);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader && d < kRsBins) {
            base = s_w[warp][d];
            s_w[warp][d] = base + __popc(peers);
        }
        base = __shfl_sync(FULL, base, leader);
        rank[r] = base + __popc(peers & ((1u << lane) - 1u));
        __syncwarp();
    }
    __syncthreads();
    {   // exclusive prefix over the warps (item order) for digit tid, and the digit's tile offset
        int run = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) {
            const int t = s_w[w][tid];
            s_w[w][tid] = run;
            run += t;
        }
        s_tot[tid] = run;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the digit totals: tile-local start of every digit
        int v[kRsBins / 32], acc = 0;
#pragma unroll
        for (int q = 0; q < kRsBins / 32; ++q) {
            v[q] = s_tot[tid * (kRsBins / 32) + q];
            acc += v[q];
        }
        int x = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, x, o);
            if (tid >= o) x += y;
        }
        int st = x - acc;
#pragma unroll
        for (int q = 0; q < kRsBins / 32; ++q) {
            s_start[tid * (kRsBins / 32) + q] = st;
            st += v[q];
        }
    }
    __syncthreads();
    // tile-local sorted order in shared memory, then coalesced runs to the global positions
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        if (key[r] < 0) continue;
        const int d = (key[r] >> shift) & 0xff;
        const int L = s_start[d] + s_w[warp][d] + rank[r];
        s_key[L] = key[r];
        s_val[L] = val[r];
    }
    __syncthreads();
    const int64_t tb = tile * kRsTile;
    const int nt = (int)(nnz - tb < kRsTile ? nnz - tb : kRsTile);
    for (int L = tid; L < nt; L += kRsTPB) {
        const int32_t kk = s_key[L];
        const int d = (kk >> shift) & 0xff;
        const int64_t pos = s_base[d] + (L - s_start[d]);
        const uint64_t vv = s_val[L];
        if (LAST) {
            ATi[pos] = (int32_t)(vv & 0x7fffffffull);
            perm[pos] = (int64_t)(vv >> 31);
        } else {
            vout[pos] = vv;
        }
        kout[pos] = kk;
    }
}

// AT_indptr from the sorted columns: ATp[c] = first position with column >= c
__global__ void k_rs_indptr(int64_t nnz, int64_t n, const int32_t *__restrict__ keys, int64_t *__restrict__ ATp)
{
    pdl_wait();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q > nnz) return;
    const int64_t c = q < nnz ? keys[q] : n;
    const int64_t cp = q > 0 ? keys[q - 1] : -1;
    for (int64_t cc = cp + 1; cc <= c; ++cc) ATp[cc] = q;
}

int transpose_radix(const csrk_pattern &A, int64_t *ATp, int32_t *ATi, int64_t *perm, Bump &ws, cudaStream_t s)
{
    const int64_t nnz = A.nnz, n = A.ncols;
    const int64_t ntiles = cdiv(nnz > 0 ? nnz : 1, kRsTile);
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < n) ++bits;
    const int passes = (bits + 7) / 8;
    int32_t *rows = ws.take<int32_t>(nnz > 0 ? nnz : 1);
    int32_t *k0 = ws.take<int32_t>(nnz > 0 ? nnz : 1);
    int32_t *k1 = ws.take<int32_t>(nnz > 0 ? nnz : 1);
    uint64_t *v0 = ws.take<uint64_t>(nnz > 0 ? nnz : 1);
    uint64_t *v1 = ws.take<uint64_t>(nnz > 0 ? nnz : 1);
    int64_t *cnt = ws.take<int64_t>(kRsBins * ntiles + 1);
    if (ws.sizing()) return scan_counts_i64(nullptr, kRsBins * ntiles, ws, s);
    if (nnz == 0) {
        CSRK_CUDA(cudaMemsetAsync(ATp, 0, sizeof(int64_t) * (size_t)(n + 1), s));
        return CSRK_OK;
    }
    CSRK_LAUNCH(k_rs_rows, (unsigned)cdiv(A.nrows, 256), 256, 0, s, A.nrows, A.indptr, rows);
    const int32_t *kin = A.indices;
    const uint64_t *vin = nullptr;
    for (int ps = 0; ps < passes; ++ps) {
        const int shift = 8 * ps;
        const bool first = ps == 0, last = ps == passes - 1;
        int32_t *kout = (ps & 1) ? k1 : k0;
        uint64_t *vout = (ps & 1) ? v1 : v0;
        CSRK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t), s));
        CSRK_LAUNCH(k_rs_up, (unsigned)ntiles, kRsTPB, 0, s, nnz, ntiles, shift, kin, cnt);
        const size_t mark = ws.used;  // every pass reuses the same scan scratch
        CSRK_TRY(scan_counts_i64(cnt, kRsBins * ntiles, ws, s));
        ws.used = mark;
        if (first && last)
            CSRK_LAUNCH((k_rs_down<true, true>), (unsigned)ntiles, kRsTPB, 0, s, nnz, ntiles, shift, kin, vin, rows,
                        cnt, kout, vout, ATi, perm);
        else if (first)
            CSRK_LAUNCH((k_rs_down<true, false>), (unsigned)ntiles, kRsTPB, 0, s, nnz, ntiles, shift, kin, vin, rows,
                        cnt, kout, vout, ATi, perm);
        else if (last)
            CSRK_LAUNCH((k_rs_down<false, true>), (unsigned)ntiles, kRsTPB, 0, s, nnz, ntiles, shift, kin, vin, rows,
                        cnt, kout, vout, ATi, perm);
        else
            CSRK_LAUNCH((k_rs_down<false, false>), (unsigned)ntiles, kRsTPB, 0, s, nnz, ntiles, shift, kin, vin, rows,
                        cnt, kout, vout, ATi, perm);
        kin = kout;
        vin = vout;
    }
    CSRK_LAUNCH(k_rs_indptr, (unsigned)cdiv(nnz + 1, 256), 256, 0, s, nnz, n, kin, ATp);
    return CSRK_OK;
}

}  // namespace csrk
