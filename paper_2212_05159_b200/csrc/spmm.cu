// spmm.cu -- SpDMM forward and backward (PAPER 3.1.3; Table 1).
//
// A CTA owns a tile of RT consecutive rows (of A, or of A^T for the transposed backward).
// For each of the tile's nonzeros the byte offset of the dense row it gathers and its value
// (for the transposed traversal: A[perm q], and perm q) are staged in shared memory with
// coalesced loads.  A group of G = 8 lanes then walks one row at a time and accumulates the
// k-wide dense rows in 32-column passes.  Lane map (vector path): in each pass lane l owns the
// 16-byte chunks l and l + 8 of the 256-byte (fp64) pass, i.e. columns {2l, 2l+1, 16+2l, 17+2l},
// or chunk l (fp32, 128-byte pass) -- so every load / store instruction of a group covers 128
// contiguous bytes and each 32-byte sector crosses L1 once.  Accumulation is fp64.
//
//   FWD      Y[i,:]  = sum_p A[p] X[idx p,:]
//   FWD_PERM same over the cached transpose, values A[perm q]      (dX = A^T dY)
//   SDDMM    dA[p]   = <dY[i,:], X[idx p,:]>                        ((dY X^T)(.)mask(A))
//   FUSED_T  row j of A^T: dX[j,:] = sum_q A[perm q] dY[i_q,:] and, from the same dY row,
//            dA[perm q] = <dY[i_q,:], X[j,:]>  -- both gradients in one pass.
// Rows that are not 16-byte aligned / k not a multiple of 4 use the scalar map (G = 32 lanes x
// 1 column).  An experimental TMA bulk-gather forward (cp.async.bulk into shared memory) is
// kept behind CSRK_SPMM_BULK=1; it measured slower.
#include "async.cuh"
#include "ops.cuh"
#include "vec.cuh"

namespace csrk {

enum { SP_FWD = 0, SP_FWD_PERM = 1, SP_SDDMM = 2, SP_FUSED_T = 3 };

template <typename T>
struct SpmmArgs {
    int64_t nrows;
    const int64_t *indptr;
    const int32_t *indices;
    const T *vals;
    const int64_t *perm;
    int64_t k;
    const T *X;  int64_t ldx;   // gathered operand (FWD: X, FUSED_T/FWD_PERM: dY, SDDMM: X)
    const T *W;  int64_t ldw;   // row operand (SDDMM: dY[i,:], FUSED_T: X[j,:])
    T *Y;        int64_t ldy;   // dense output (FWD: Y, FUSED_T / FWD_PERM: dX)
    T *D;                       // dA (SDDMM, FUSED_T)
    int64_t xrows;              // rows of the gathered operand (= ncols of the traversed matrix)
};

constexpr int kSpmmTPB = 256;
constexpr int kSpmmRPG = 4;        // rows per group per tile
constexpr int kSpmmCAP = 1536;     // staged nonzeros per tile
constexpr int kPass = 32;          // columns per pass (both maps)
constexpr int kFusedMaxPasses = 2;

// ---------------------------------------------------------------- lane maps
// Vector map (G = 8, W = 4 elements per lane per pass) or scalar map (G = 32, W = 1).
template <typename T, int G, int W>
struct LaneMap {
    static constexpr int E = W == 1 ? 1 : 16 / (int)sizeof(T);   // elements per chunk
    static constexpr int NCH = W / E;                             // chunks per lane
    // column (within a pass) of chunk ch of lane l
    __device__ static int col(int l, int ch) { return (l + ch * G) * E; }
};

// Load lane l's W elements of a pass starting at p (kleft = columns left in the row).
// GLOBAL: read-only global path (__ldg); otherwise a generic load (shared-memory staging).
template <typename T, int G, int W, bool GLOBAL = true>
__device__ __forceinline__ void ldl(const T *p, int l, int64_t kleft, double (&r)[W])
{
    using M = LaneMap<T, G, W>;
#pragma unroll
    for (int ch = 0; ch < M::NCH; ++ch) {
        const int c = M::col(l, ch);
        if constexpr (M::E == 1) {
            r[ch] = c < kleft ? (double)(GLOBAL ? __ldg(p + c) : p[c]) : 0.0;
        } else if constexpr (sizeof(T) == 8) {
            double2 v = make_double2(0.0, 0.0);
            if (c < kleft) {
                const double2 *q = reinterpret_cast<const double2 *>(p + c);
                v = GLOBAL ? __ldg(q) : *q;
            }
            r[ch * 2] = v.x;
            r[ch * 2 + 1] = v.y;
        } else {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < kleft) {
                const float4 *q = reinterpret_cast<const float4 *>(p + c);
                v = GLOBAL ? __ldg(q) : *q;
            }
            r[ch * 4] = v.x; r[ch * 4 + 1] = v.y; r[ch * 4 + 2] = v.z; r[ch * 4 + 3] = v.w;
        }
    }
}

template <typename T, int G, int W>
__device__ __forceinline__ void stl(T *p, int l, int64_t kleft, const double (&r)[W])
{
    using M = LaneMap<T, G, W>;
#pragma unroll
    for (int ch = 0; ch < M::NCH; ++ch) {
        const int c = M::col(l, ch);
        if (c >= kleft) continue;
        if constexpr (M::E == 1) {
            p[c] = (T)r[ch];
        } else if constexpr (sizeof(T) == 8) {
            *reinterpret_cast<double2 *>(p + c) = make_double2(r[ch * 2], r[ch * 2 + 1]);
        } else {
            *reinterpret_cast<float4 *>(p + c) =
                make_float4((float)r[ch * 4], (float)r[ch * 4 + 1], (float)r[ch * 4 + 2], (float)r[ch * 4 + 3]);
        }
    }
}

template <int G>
__device__ __forceinline__ double group_sum(double v)
{
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

// ---------------------------------------------------------------- tile kernel
// Rows [r0, r0 + nr) of a tile.  STAGED: the tile's nonzeros are in shared memory as
// (byte offset of the gathered row, value[, perm]); otherwise they are read from global.
template <typename T, int G, int W, int MODE, bool STAGED>
__device__ __forceinline__ void spmm_rows(const SpmmArgs<T> &a, const int64_t *s_ptr, const int64_t *s_off,
                                          const double *s_val, const int64_t *s_perm, int64_t r0, int nr,
                                          int64_t base)
{
    constexpr int NG = kSpmmTPB / G;
    constexpr bool PERM = MODE == SP_FWD_PERM || MODE == SP_FUSED_T;
    const int tid = threadIdx.x, g = tid / G, lane = tid % G;
    const int64_t rowbytes = a.ldx * (int64_t)sizeof(T);
    auto off_of = [&](int64_t e) -> int64_t {
        if constexpr (STAGED) return s_off[e];
        else return (int64_t)(uint32_t)a.indices[base + e] * rowbytes;
    };
    auto val_of = [&](int64_t e) -> double {
        if constexpr (STAGED) return s_val[e];
        else return (double)a.vals[PERM ? a.perm[base + e] : base + e];
    };
    auto perm_of = [&](int64_t e) -> int64_t {
        if constexpr (STAGED) return s_perm[e];
        else return a.perm[base + e];
    };
    const int npass = (int)((a.k + kPass - 1) / kPass);
    const char *Xb = reinterpret_cast<const char *>(a.X);

    for (int j = 0; j < kSpmmRPG; ++j) {
        const int rl = g + j * NG;   // adjacent groups take adjacent rows
        const bool valid = rl < nr;
        const int64_t row = r0 + rl;
        const int s = valid ? (int)(s_ptr[rl] - base) : 0, e = valid ? (int)(s_ptr[rl + 1] - base) : 0;
        if (MODE == SP_SDDMM || MODE == SP_FUSED_T) {
            // warp-uniform trip count: the group reductions below shuffle across the warp
            const int len = e - s;
            const int maxlen = (int)__reduce_max_sync(0xffffffffu, (unsigned)len);
            if (!__any_sync(0xffffffffu, valid)) break;
            if (MODE == SP_SDDMM) {
                for (int t = 0; t < maxlen; ++t) {
                    const bool on = t < len;
                    const int64_t off = on ? off_of(s + t) : 0;
                    double dot = 0.0;
                    for (int ps = 0; ps < npass; ++ps) {
                        const int64_t pc = (int64_t)ps * kPass;
                        if (on) {
                            double xv[W], wv[W];
                            ldl<T, G, W>(reinterpret_cast<const T *>(Xb + off) + pc, lane, a.k - pc, xv);
                            ldl<T, G, W>(a.W + row * a.ldw + pc, lane, a.k - pc, wv);
#pragma unroll
                            for (int i = 0; i < W; ++i) dot = fma(wv[i], xv[i], dot);
                        }
                    }
                    dot = group_sum<G>(dot);
                    if (on && lane == 0) a.D[base + s + t] = (T)dot;
                }
            } else {
                double xj[kFusedMaxPasses][W], acc[kFusedMaxPasses][W];
#pragma unroll
                for (int ps = 0; ps < kFusedMaxPasses; ++ps) {
#pragma unroll
                    for (int i = 0; i < W; ++i) { xj[ps][i] = 0.0; acc[ps][i] = 0.0; }
                    if (valid && ps < npass)
                        ldl<T, G, W>(a.W + row * a.ldw + (int64_t)ps * kPass, lane, a.k - (int64_t)ps * kPass, xj[ps]);
                }
#pragma unroll 4
                for (int t = 0; t < maxlen; ++t) {
                    const bool on = t < len;
                    const int64_t off = on ? off_of(s + t) : 0;
                    const double av = on ? val_of(s + t) : 0.0;
                    double dot = 0.0;
#pragma unroll
                    for (int ps = 0; ps < kFusedMaxPasses; ++ps) {
                        if (on && ps < npass) {
                            const int64_t pc = (int64_t)ps * kPass;
                            double gv[W];
                            ldl<T, G, W>(reinterpret_cast<const T *>(Xb + off) + pc, lane, a.k - pc, gv);
#pragma unroll
                            for (int i = 0; i < W; ++i) {
                                acc[ps][i] = fma(av, gv[i], acc[ps][i]);
                                dot = fma(gv[i], xj[ps][i], dot);
                            }
                        }
                    }
                    dot = group_sum<G>(dot);
                    if (on && a.D && lane == 0) a.D[perm_of(s + t)] = (T)dot;
                }
#pragma unroll
                for (int ps = 0; ps < kFusedMaxPasses; ++ps)
                    if (valid && ps < npass)
                        stl<T, G, W>(a.Y + row * a.ldy + (int64_t)ps * kPass, lane, a.k - (int64_t)ps * kPass, acc[ps]);
            }
            continue;
        }
        if (!valid) break;
        // FWD / FWD_PERM
        for (int ps = 0; ps < npass; ++ps) {
            const int64_t pc = (int64_t)ps * kPass;
            double acc[W];
#pragma unroll
            for (int i = 0; i < W; ++i) acc[i] = 0.0;
            const char *Xc = reinterpret_cast<const char *>(a.X + pc);
#pragma unroll 4
            for (int q = s; q < e; ++q) {
                const double av = val_of(q);
                double xv[W];
                ldl<T, G, W>(reinterpret_cast<const T *>(Xc + off_of(q)), lane, a.k - pc, xv);
#pragma unroll
                for (int i = 0; i < W; ++i) acc[i] = fma(av, xv[i], acc[i]);
            }
            stl<T, G, W>(a.Y + row * a.ldy + pc, lane, a.k - pc, acc);
        }
    }
}

template <typename T, int G, int W, int MODE>
__global__ __launch_bounds__(kSpmmTPB, MODE == SP_FUSED_T ? 4 : 5) void k_spmm(SpmmArgs<T> a)
{
    pdl_wait();
    constexpr int NG = kSpmmTPB / G;           // groups per CTA
    constexpr int RT = NG * kSpmmRPG;          // rows per tile
    constexpr bool PERM = MODE == SP_FWD_PERM || MODE == SP_FUSED_T;
    __shared__ int64_t s_ptr[RT + 1];
    __shared__ int64_t s_off[kSpmmCAP];
    __shared__ double s_val[MODE == SP_SDDMM ? 1 : kSpmmCAP];
    __shared__ int64_t s_perm[MODE == SP_FUSED_T ? kSpmmCAP : 1];

    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * RT;
    const int nr = (int)(a.nrows - r0 < RT ? a.nrows - r0 : RT);
    for (int i = tid; i <= nr; i += kSpmmTPB) s_ptr[i] = a.indptr[r0 + i];
    __syncthreads();
    const int64_t base = s_ptr[0];
    const int64_t tnz = s_ptr[nr] - base;
    if (tnz > kSpmmCAP) {   // tile-uniform: nonzeros read from global memory
        spmm_rows<T, G, W, MODE, false>(a, s_ptr, s_off, s_val, s_perm, r0, nr, base);
        return;
    }
    const int64_t rowbytes = a.ldx * (int64_t)sizeof(T);
    for (int e = tid; e < (int)tnz; e += kSpmmTPB) {
        const int64_t p = base + e;
        s_off[e] = (int64_t)(uint32_t)a.indices[p] * rowbytes;
        if (MODE != SP_SDDMM) {
            const int64_t pv = PERM ? a.perm[p] : p;
            s_val[e] = (double)a.vals[pv];
            if (MODE == SP_FUSED_T) s_perm[e] = pv;
        }
    }
    __syncthreads();
    spmm_rows<T, G, W, MODE, true>(a, s_ptr, s_off, s_val, s_perm, r0, nr, base);
}

template <typename T, int G, int W, int MODE>
static int launch_spmm(const SpmmArgs<T> &a, cudaStream_t s)
{
    if (a.nrows <= 0) return CSRK_OK;
    constexpr int RT = (kSpmmTPB / G) * kSpmmRPG;
    CSRK_LAUNCH((k_spmm<T, G, W, MODE>), (unsigned)cdiv(a.nrows, RT), kSpmmTPB, 0, s, a);
    return CSRK_OK;
}

// ---------------------------------------------------------------- lean row kernel (no staging)
// One G-lane group per row, RPW rows per group strided by the grid; index and value read with
// group-broadcast loads (one L1 request per group), no shared memory, no block barrier.
template <typename T, int G, int W, bool PERM>
__global__ __launch_bounds__(256) void k_spmm_lean(SpmmArgs<T> a)
{
    pdl_wait();
    const int lane = threadIdx.x % G;
    const int64_t ngroups = (int64_t)gridDim.x * (256 / G);
    const int npass = (int)((a.k + kPass - 1) / kPass);
    for (int64_t row = (int64_t)blockIdx.x * (256 / G) + threadIdx.x / G; row < a.nrows; row += ngroups) {
        const int64_t s = a.indptr[row], e = a.indptr[row + 1];
        for (int ps = 0; ps < npass; ++ps) {
            const int64_t pc = (int64_t)ps * kPass;
            double acc[W];
#pragma unroll
            for (int i = 0; i < W; ++i) acc[i] = 0.0;
            const T *Xc = a.X + pc;
#pragma unroll 4
            for (int64_t q = s; q < e; ++q) {
                const double av = (double)a.vals[PERM ? a.perm[q] : q];
                double xv[W];
                ldl<T, G, W>(Xc + (int64_t)(uint32_t)a.indices[q] * a.ldx, lane, a.k - pc, xv);
#pragma unroll
                for (int i = 0; i < W; ++i) acc[i] = fma(av, xv[i], acc[i]);
            }
            stl<T, G, W>(a.Y + row * a.ldy + pc, lane, a.k - pc, acc);
        }
    }
}

// ---------------------------------------------------------------- experimental TMA bulk gather
// One CTA = 32 rows.  Every nonzero's gathered dense row (k*sizeof(T) bytes, a multiple of 16)
// is fetched into shared memory by a 1D bulk copy (cp.async.bulk) completing on one mbarrier;
// the 8-lane groups then accumulate from shared memory.  Off by default (slower).
constexpr int kBulkTPB = 256;
constexpr int kBulkG = 8;
constexpr int kBulkRT = kBulkTPB / kBulkG;
constexpr int kBulkBytes = 40 * 1024;

// Persistent CTAs, two buffers: the bulk copies of tile t+grid are issued before tile t is
// computed from shared memory, so the TMA gathers of one tile overlap the math of the other.
template <typename T>
__global__ __launch_bounds__(kBulkTPB) void k_spmm_bulk(SpmmArgs<T> a, int cap, int64_t ntiles)
{
    pdl_wait();
    constexpr int W = 4;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int64_t s_ptr[2][kBulkRT + 1];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int s_fits[2];
    const int rb = (int)(a.k * (int64_t)sizeof(T));
    const size_t bufb = (size_t)cap * rb + (size_t)cap * sizeof(double);
    const int tid = threadIdx.x, g = tid / kBulkG, lane = tid % kBulkG;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const char *Xb = reinterpret_cast<const char *>(a.X);
    const int64_t ldb = a.ldx * (int64_t)sizeof(T);
    auto issue = [&](int64_t t, int b) {
        const int64_t r0 = t * kBulkRT;
        const int nr = (int)(a.nrows - r0 < kBulkRT ? a.nrows - r0 : kBulkRT);
        for (int i = tid; i <= nr; i += kBulkTPB) s_ptr[b][i] = a.indptr[r0 + i];
        __syncthreads();
        const int64_t base = s_ptr[b][0];
        const int64_t tnz = s_ptr[b][nr] - base;
        const bool fits = tnz <= cap;
        if (tid == 0) s_fits[b] = fits;
        if (!fits) return;
        if (tid == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(tnz * rb));
        __syncthreads();
        unsigned char *s_g = smem + b * bufb;
        double *s_val = reinterpret_cast<double *>(s_g + (size_t)cap * rb);
        for (int e = tid; e < (int)tnz; e += kBulkTPB) {
            const int64_t p = base + e;
            bulk_g2s(s_g + (size_t)e * rb, Xb + (int64_t)(uint32_t)a.indices[p] * ldb, (uint32_t)rb, &bar[b]);
            s_val[e] = (double)a.vals[p];
        }
    };
    uint32_t phase[2] = {0u, 0u};
    int64_t t = blockIdx.x;
    if (t < ntiles) issue(t, 0);
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        if (t + gridDim.x < ntiles) issue(t + gridDim.x, b ^ 1);
        __syncthreads();                        // s_val / s_fits of buffer b visible
        const bool fits = s_fits[b];
        if (fits) {
            mbar_wait(&bar[b], phase[b]);
            phase[b] ^= 1u;
        }
        const unsigned char *s_g = smem + b * bufb;
        const double *s_val = reinterpret_cast<const double *>(s_g + (size_t)cap * rb);
        const int64_t r0 = t * kBulkRT;
        const int nr = (int)(a.nrows - r0 < kBulkRT ? a.nrows - r0 : kBulkRT);
        if (g < nr) {
            const int64_t base = s_ptr[b][0];
            const int64_t row = r0 + g;
            const int64_t s = s_ptr[b][g] - base, e = s_ptr[b][g + 1] - base;
            for (int64_t pc = 0; pc < a.k; pc += kPass) {
                double acc[W] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
                for (int64_t q = s; q < e; ++q) {
                    double xv[W];
                    double av;
                    if (fits) {
                        ldl<T, kBulkG, W, false>(reinterpret_cast<const T *>(s_g + (size_t)q * rb) + pc, lane,
                                                 a.k - pc, xv);
                        av = s_val[q];
                    } else {
                        ldl<T, kBulkG, W>(a.X + (int64_t)a.indices[base + q] * a.ldx + pc, lane, a.k - pc, xv);
                        av = (double)a.vals[base + q];
                    }
#pragma unroll
                    for (int i = 0; i < W; ++i) acc[i] = fma(av, xv[i], acc[i]);
                }
                stl<T, kBulkG, W>(a.Y + row * a.ldy + pc, lane, a.k - pc, acc);
            }
        }
        __syncthreads();                        // buffer b free for tile t + 2 grid
    }
}

template <typename T>
static int launch_spmm_bulk(const SpmmArgs<T> &a, cudaStream_t s)
{
    if (a.nrows <= 0) return CSRK_OK;
    const int rb = (int)(a.k * (int64_t)sizeof(T));
    const int cap = kBulkBytes / rb;
    const size_t smem = 2 * ((size_t)cap * rb + (size_t)cap * sizeof(double));
    static DevOnce attr;
    if (attr.need()) {
        CSRK_CUDA(cudaFuncSetAttribute(k_spmm_bulk<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr.done();
    }
    const int64_t ntiles = cdiv(a.nrows, kBulkRT);
    const int64_t grid = ntiles < (int64_t)kNumSMs * 2 ? ntiles : (int64_t)kNumSMs * 2;
    CSRK_LAUNCH(k_spmm_bulk<T>, (unsigned)grid, kBulkTPB, smem, s, a, cap, ntiles);
    return CSRK_OK;
}

// ---------------------------------------------------------------- wide path (256-bit vectors)
// For dense rows of exactly 128 or 256 bytes (fp64 k = 16 / 32, fp32 k = 32): a group of 4
// lanes owns a row, each lane holding NV 32-byte vectors, so one load / store instruction of a
// group covers a whole 128-byte line.  A group walks the CONTIGUOUS nonzero stream of its
// kWRPG consecutive rows in batches of 4: the 4 gathers of a batch are issued before any is
// consumed (memory-level parallelism), row transitions flush the accumulator, and the 4 dot
// products of a batch (SDDMM / fused backward) are finished by one transpose-reduction, after
// which lane l stores dA of the batch's l-th nonzero.
constexpr int kWG = 4;
constexpr int kWRPG = 4;
constexpr int kWCAP = 1536;
// CTA size per mode (measured, config 2): 256 threads with the band for the forward modes,
// 128 threads (more, smaller CTAs per SM) for the dot-product modes.
template <int MODE> constexpr int wide_tpb() { return MODE == SP_FWD || MODE == SP_FWD_PERM ? 256 : 128; }
#ifndef CSRK_WIDE_MINB_FWD
#define CSRK_WIDE_MINB_FWD 2
#endif
#ifndef CSRK_WIDE_MINB_DOT
#define CSRK_WIDE_MINB_DOT 4
#endif
// occupancy hint (CTAs per SM) per mode; A/B via CSRK_NVCC_EXTRA
template <int MODE> constexpr int wide_minb()
{
    return MODE == SP_FWD || MODE == SP_FWD_PERM ? CSRK_WIDE_MINB_FWD : CSRK_WIDE_MINB_DOT;
}

struct __align__(16) WideNz {
    double val;
    int64_t off;   // element offset of the gathered dense row
};

// Near-diagonal band (BAND): the gathered operand's rows [b0, b1) around the tile's own row
// range (scaled to the column space, +-kBandH) are brought into shared memory by ONE TMA bulk
// copy per tile; gathers inside the band read shared memory.  On a stencil 3 of 5 gathers per
// row fall in the band, so the L2 traffic of the gathers drops from 5 to ~3 dense rows per row.
constexpr int kBandH = 8;
template <int MODE> constexpr int band_cap() { return wide_tpb<MODE>() / kWG * kWRPG + 2 * kBandH + 1; }

template <typename T, int NV, int MODE, bool BAND>
__global__ __launch_bounds__(wide_tpb<MODE>(), wide_minb<MODE>()) void k_spmm_wide(SpmmArgs<T> a)
{
    pdl_wait();
    constexpr int kWTPB = wide_tpb<MODE>();
    constexpr int kWRT = kWTPB / kWG * kWRPG;
    constexpr int kBandCap = band_cap<MODE>();
    constexpr int E = V32<T>::E;
    constexpr int NE = NV * E;
    constexpr bool PERM = MODE == SP_FWD_PERM || MODE == SP_FUSED_T;
    constexpr bool ACC = MODE != SP_SDDMM;
    constexpr bool DOT = MODE == SP_SDDMM || MODE == SP_FUSED_T;
    __shared__ int64_t s_ptr[kWRT + 1];
    __shared__ WideNz s_nz[kWCAP];
    __shared__ int64_t s_perm[MODE == SP_FUSED_T ? kWCAP : 1];

    constexpr int RB = NV * 128;   // bytes per dense row
    extern __shared__ __align__(128) unsigned char s_band[];
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kWRT;
    const int nr = (int)(a.nrows - r0 < kWRT ? a.nrows - r0 : kWRT);
    int64_t b0 = 0, b1 = 0;
    if (BAND) {
        const double sc = (double)a.xrows / (double)a.nrows;
        b0 = (int64_t)((double)r0 * sc) - kBandH;
        b0 = b0 < 0 ? 0 : b0;
        b1 = (int64_t)((double)(r0 + nr) * sc) + kBandH + 1;
        b1 = b1 > a.xrows ? a.xrows : b1;
        b1 = b1 > b0 + kBandCap ? b0 + kBandCap : b1;
        b1 = b1 < b0 ? b0 : b1;
        if (tid == 0) {
            mbar_init(&s_bar, 1);
            mbar_fence_init();
        }
    }
    for (int i = tid; i <= nr; i += kWTPB) s_ptr[i] = a.indptr[r0 + i];
    __syncthreads();
    if (BAND && tid == 0 && b1 > b0) {
        const uint32_t bytes = (uint32_t)((b1 - b0) * RB);
        mbar_arrive_expect_tx(&s_bar, bytes);
        bulk_g2s(s_band, a.X + b0 * a.ldx, bytes, &s_bar);
    }
    // element offset of a gathered row in global memory, or (band) -1 - its shared byte offset
    auto where = [&](int64_t c) -> int64_t {
        if (BAND && c >= b0 && c < b1) return -1 - (c - b0) * RB;
        return c * a.ldx;
    };
    const int64_t base = s_ptr[0];
    const bool staged = s_ptr[nr] - base <= kWCAP;   // tile-uniform
    if (staged) {
        const int tnz = (int)(s_ptr[nr] - base);
        for (int e = tid; e < tnz; e += kWTPB) {
            const int64_t p = base + e;
            const int64_t pv = PERM ? a.perm[p] : p;
            WideNz z;
            z.off = where((int64_t)(uint32_t)a.indices[p]);
            z.val = ACC ? (double)a.vals[pv] : 0.0;
            s_nz[e] = z;
            if (MODE == SP_FUSED_T) s_perm[e] = pv;
        }
        __syncthreads();
    }
    auto meta = [&](int64_t e) -> WideNz {
        if (staged) return s_nz[e];
        WideNz z;
        z.off = where((int64_t)(uint32_t)a.indices[base + e]);
        z.val = ACC ? (double)a.vals[PERM ? a.perm[base + e] : base + e] : 0.0;
        return z;
    };

    const int g = tid / kWG, l = tid % kWG;
    const int rb = g * kWRPG < nr ? g * kWRPG : nr;
    const int re = rb + kWRPG < nr ? rb + kWRPG : nr;
    const int64_t sb = s_ptr[rb] - base, se = s_ptr[re] - base;   // the group's nonzero stream
    const int nbw = (int)__reduce_max_sync(0xffffffffu, (unsigned)((se - sb + 3) >> 2));
    const int lo = l * E;   // this lane's first element; vector v at lo + v * kWG * E

    double acc[NE], xr[NE];
    int cur = rb;
    int64_t cend = rb < re ? s_ptr[rb + 1] - base : 0;
    auto begin = [&]() {
        if (ACC) {
#pragma unroll
            for (int i = 0; i < NE; ++i) acc[i] = 0.0;
        }
        if (DOT) {
            const T *w = a.W + (r0 + cur) * a.ldw + lo;
#pragma unroll
            for (int v = 0; v < NV; ++v) ldv32(w + v * kWG * E, xr + v * E);
        }
    };
    auto finish = [&]() {
        if (ACC) {
            T *y = a.Y + (r0 + cur) * a.ldy + lo;
#pragma unroll
            for (int v = 0; v < NV; ++v) stv32(y + v * kWG * E, acc + v * E);
        }
    };
    if (BAND && b1 > b0) mbar_wait(&s_bar, 0);
    const int h = g & 1;   // shared-memory half order (bank spread between the 2 groups of a phase)
    if (rb < re) begin();
    for (int t = 0; t < nbw; ++t) {
        const int64_t e0 = sb + 4 * t;
        WideNz z[4];
        double gv[4][NE];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (e0 + b < se) {
                z[b] = meta(e0 + b);
                if (!BAND || z[b].off >= 0) {
                    const T *xp = a.X + z[b].off + lo;
#pragma unroll
                    for (int v = 0; v < NV; ++v) ldv32(xp + v * kWG * E, gv[b] + v * E);
                } else {
                    const T *xp = reinterpret_cast<const T *>(s_band + (-1 - z[b].off)) + lo;
#pragma unroll
                    for (int v = 0; v < NV; ++v) lds32(xp + v * kWG * E, gv[b] + v * E, h);
                }
            } else {
                z[b].val = 0.0;
#pragma unroll
                for (int i = 0; i < NE; ++i) gv[b][i] = 0.0;
            }
        }
        double d[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (e0 + b < se) {
                while (e0 + b >= cend) {   // row transition (skips empty rows)
                    finish();
                    ++cur;
                    cend = s_ptr[cur + 1] - base;
                    begin();
                }
            }
            if (ACC) {
#pragma unroll
                for (int i = 0; i < NE; ++i) acc[i] = fma(z[b].val, gv[b][i], acc[i]);
            }
            if (DOT) {
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < NE; ++i) s = fma(gv[b][i], xr[i], s);
                d[b] = s;
            }
        }
        if (DOT) {
            const double dd = transpose_reduce4(d, l);
            const int64_t e = e0 + l;
            if (e < se) a.D[MODE == SP_FUSED_T ? (staged ? s_perm[e] : a.perm[base + e]) : base + e] = (T)dd;
        }
    }
    if (rb < re) {   // the current row and any trailing empty rows
        finish();
        while (++cur < re) {
            if (ACC) {
#pragma unroll
                for (int i = 0; i < NE; ++i) acc[i] = 0.0;
            }
            finish();
        }
    }
}

// ---------------------------------------------------------------- persistent pipelined wide path
// k_spmm_wide stages each tile's metadata (indptr slice, then indices / values / perm slices)
// with dependent loads at the start of the CTA: ncu attributed ~25 % of the backward's stall
// samples to that chain.  Here persistent CTAs walk tiles t = blockIdx.x + k gridDim.x and the
// metadata arrives by TMA bulk copies issued AHEAD: the indptr slice two tiles ahead, the
// index / perm / value slices and the near-diagonal band one tile ahead (their range comes from
// the indptr slice), each completing on an mbarrier.  Slices are copied as the 16-byte-aligned
// superset of their range; a tile whose superset would run past the end of an array or that
// holds more than kPCAP nonzeros reads its metadata from global memory instead ("direct").
// Values of the transposed traversal are gathered through perm in the compute batch (with the
// dense-row gathers), not in the staging chain.  The compute is k_spmm_wide's.
constexpr int kPTPB = 128;
constexpr int kPRPG = 4;
constexpr int kPRT = kPTPB / kWG * kPRPG;   // 128 rows per tile
constexpr int kPCAP = 1024;                 // staged nonzeros per tile

template <typename T, int NV, int MODE, bool BAND>
struct PipeLayout {
    static constexpr bool PERM = MODE == SP_FWD_PERM || MODE == SP_FUSED_T;
    static constexpr bool VAL = MODE == SP_FWD;      // contiguous values staged
    static constexpr int RB = NV * 128;
    static constexpr int kBand = kPRT + 2 * kBandH + 1;
    static constexpr size_t ptr = 0;                                            // int64 [3][kPRT + 4]
    static constexpr size_t idx = ptr + 3 * (kPRT + 4) * 8;                     // int32 [2][kPCAP + 8]
    static constexpr size_t perm = idx + 2 * (kPCAP + 8) * 4;                   // int64 [2][kPCAP + 4]
    static constexpr size_t val = perm + (PERM ? 2 * (kPCAP + 4) * 8 : 0);      // T [2][kPCAP + 32/sizeof T]
    static constexpr size_t band = (val + (VAL ? 2 * (kPCAP + 32 / sizeof(T)) * sizeof(T) : 0) + 127) & ~size_t(127);
    static constexpr size_t wrow = band + (BAND ? 2 * (size_t)kBand * RB : 0);   // staged W rows [2][kPRT]
    static constexpr size_t total_nw = wrow;
    static constexpr size_t total_w = wrow + 2 * (size_t)kPRT * RB;
};

#ifndef CSRK_PIPE_MINB_FWD
#define CSRK_PIPE_MINB_FWD 4   // measured: config-2 forward 473 -> 445 us (5: spills)
#endif
#ifndef CSRK_PIPE_MINB_G8
#define CSRK_PIPE_MINB_G8 5
#endif
#ifndef CSRK_PIPE_MINB_DOT
#define CSRK_PIPE_MINB_DOT 3   // measured 3 / 4 / 5: 805 / 817 / 1460 us (4: small spills, 5: heavy)
#endif
template <int MODE, int G> constexpr int pipe_minb()
{
    return G == 8 ? CSRK_PIPE_MINB_G8 : (MODE == SP_FWD || MODE == SP_FWD_PERM ? CSRK_PIPE_MINB_FWD : CSRK_PIPE_MINB_DOT);
}

template <typename T, int NV, int MODE, bool BAND, int G, bool WST, bool L1G = false>
__global__ __launch_bounds__(kPTPB, pipe_minb<MODE, G>()) void k_spmm_pipe(SpmmArgs<T> a, int64_t ntiles)
{
    pdl_wait();
    using PL = PipeLayout<T, NV, MODE, BAND>;
    constexpr bool PERM = PL::PERM;
    constexpr bool ACC = MODE != SP_SDDMM;
    constexpr bool DOT = MODE == SP_SDDMM || MODE == SP_FUSED_T;
    constexpr int E = V32<T>::E;
    constexpr int NVL = NV * kWG / G;   // 32-byte vectors per lane (a row is NV * 4 vectors)
    constexpr int NE = NVL * E;
    constexpr int RPG = kPRT * G / kPTPB;   // rows per group per tile
    constexpr int RB = PL::RB;
    constexpr int kBand = PL::kBand;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bp[3], bm[2];
    __shared__ int s_off_ptr[3], s_off_idx[2], s_off_perm[2], s_off_val[2], s_direct[2];
    __shared__ int64_t s_b0[2], s_b1[2];
    int64_t *ptr_buf = reinterpret_cast<int64_t *>(smem + PL::ptr);
    int32_t *idx_buf = reinterpret_cast<int32_t *>(smem + PL::idx);
    int64_t *perm_buf = reinterpret_cast<int64_t *>(smem + PL::perm);
    T *val_buf = reinterpret_cast<T *>(smem + PL::val);
    unsigned char *band_buf = smem + PL::band;
    unsigned char *w_buf = smem + PL::wrow;     // WST: the tile's W rows (dot modes), by TMA

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(&bp[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&bm[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t nptr = a.nrows + 1;
    const int64_t nnz_all = a.indptr[a.nrows] - a.indptr[0];   // indptr[0] = 0 (canonical)
    auto tile_of = [&](int64_t k) { return (int64_t)blockIdx.x + k * (int64_t)gridDim.x; };
    auto rows_of = [&](int64_t t, int64_t &r0, int &nr) {
        r0 = t * kPRT;
        nr = (int)(a.nrows - r0 < kPRT ? a.nrows - r0 : kPRT);
    };
    // thread 0: indptr slice of tile t into ptr stage ps (aligned superset, or a plain copy)
    auto issue_ptr = [&](int64_t t, int ps) {
        int64_t r0;
        int nr;
        rows_of(t, r0, nr);
        const int64_t lo = r0 & ~int64_t(1), hi = (r0 + nr + 1 + 1) & ~int64_t(1);
        int64_t *dst = ptr_buf + ps * (kPRT + 4);
        s_off_ptr[ps] = (int)(r0 - lo);
        if (hi <= nptr) {
            mbar_arrive_expect_tx(&bp[ps], (uint32_t)((hi - lo) * 8));
            bulk_g2s(dst, a.indptr + lo, (uint32_t)((hi - lo) * 8), &bp[ps]);
        } else {   // the array's last entries: plain loads (this thread), then arrive
            for (int64_t i = lo; i < r0 + nr + 1; ++i) dst[i - lo] = a.indptr[i];
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bp[ps])) : "memory");
        }
    };
    // thread 0: index / perm / value slices and the band of tile t (its ptr stage ps ready) into
    // metadata stage ms
    auto issue_meta = [&](int64_t t, int ps, int ms) {
        int64_t r0;
        int nr;
        rows_of(t, r0, nr);
        const int64_t *P = ptr_buf + ps * (kPRT + 4) + s_off_ptr[ps];
        const int64_t e0 = P[0], e1 = P[nr];
        const int64_t ilo = e0 & ~int64_t(3), ihi = (e1 + 3) & ~int64_t(3);
        const int64_t plo = e0 & ~int64_t(1), phi = (e1 + 1) & ~int64_t(1);
        constexpr int VE = 16 / (int)sizeof(T);
        const int64_t vlo = e0 & ~int64_t(VE - 1), vhi = (e1 + VE - 1) & ~int64_t(VE - 1);
        bool direct = e1 - e0 > kPCAP || ihi > nnz_all || (PERM && phi > nnz_all) || (PL::VAL && vhi > nnz_all);
        uint32_t bytes = 0;
        int64_t b0 = 0, b1 = 0;
        if (BAND) {
            const double sc = (double)a.xrows / (double)a.nrows;
            b0 = (int64_t)((double)r0 * sc) - kBandH;
            b0 = b0 < 0 ? 0 : b0;
            b1 = (int64_t)((double)(r0 + nr) * sc) + kBandH + 1;
            b1 = b1 > a.xrows ? a.xrows : b1;
            b1 = b1 > b0 + kBand ? b0 + kBand : b1;
            b1 = b1 < b0 ? b0 : b1;
            bytes += (uint32_t)((b1 - b0) * RB);
        }
        s_b0[ms] = b0;
        s_b1[ms] = b1;
        if (WST) bytes += (uint32_t)(nr * RB);
        if (!direct && e1 > e0) {
            bytes += (uint32_t)((ihi - ilo) * 4);
            if (PERM) bytes += (uint32_t)((phi - plo) * 8);
            if (PL::VAL) bytes += (uint32_t)((vhi - vlo) * sizeof(T));
        }
        s_direct[ms] = direct;
        s_off_idx[ms] = (int)(e0 - ilo);
        s_off_perm[ms] = (int)(e0 - plo);
        s_off_val[ms] = (int)(e0 - vlo);
        if (bytes == 0) {
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bm[ms])) : "memory");
            return;
        }
        mbar_arrive_expect_tx(&bm[ms], bytes);
        if (BAND && b1 > b0) bulk_g2s(band_buf + (size_t)ms * kBand * RB, a.X + b0 * a.ldx, (uint32_t)((b1 - b0) * RB), &bm[ms]);
        if (WST && nr > 0) bulk_g2s(w_buf + (size_t)ms * kPRT * RB, a.W + r0 * a.ldw, (uint32_t)(nr * RB), &bm[ms]);
        if (!direct && e1 > e0) {
            bulk_g2s(idx_buf + ms * (kPCAP + 8), a.indices + ilo, (uint32_t)((ihi - ilo) * 4), &bm[ms]);
            if (PERM) bulk_g2s(perm_buf + ms * (kPCAP + 4), a.perm + plo, (uint32_t)((phi - plo) * 8), &bm[ms]);
            if (PL::VAL)
                bulk_g2s(val_buf + ms * (kPCAP + 32 / sizeof(T)), a.vals + vlo, (uint32_t)((vhi - vlo) * sizeof(T)),
                         &bm[ms]);
        }
    };
    // prologue: indptr of the first two tiles, then the metadata of the first
    if (tid == 0) {
        if (tile_of(0) < ntiles) issue_ptr(tile_of(0), 0);
        if (tile_of(1) < ntiles) issue_ptr(tile_of(1), 1);
        if (tile_of(0) < ntiles) {
            mbar_wait(&bp[0], 0);
            issue_meta(tile_of(0), 0, 0);
        }
    }
    const int g = tid / G, l = tid % G;
    const int lo_e = l * E;
    const int h = g & 1;
    for (int64_t k = 0; tile_of(k) < ntiles; ++k) {
        const int ps = (int)(k % 3), ms = (int)(k & 1);
        if (tid == 0) {
            if (tile_of(k + 2) < ntiles) issue_ptr(tile_of(k + 2), (int)((k + 2) % 3));
            if (tile_of(k + 1) < ntiles) {
                mbar_wait(&bp[(k + 1) % 3], (uint32_t)(((k + 1) / 3) & 1));
                issue_meta(tile_of(k + 1), (int)((k + 1) % 3), (int)((k + 1) & 1));
            }
        }
        mbar_wait(&bp[ps], (uint32_t)((k / 3) & 1));
        mbar_wait(&bm[ms], (uint32_t)((k >> 1) & 1));
        const int64_t t = tile_of(k);
        int64_t r0;
        int nr;
        rows_of(t, r0, nr);
        const int64_t *s_ptr = ptr_buf + ps * (kPRT + 4) + s_off_ptr[ps];
        const int32_t *s_idx = idx_buf + ms * (kPCAP + 8) + s_off_idx[ms];
        const int64_t *s_perm = perm_buf + ms * (kPCAP + 4) + s_off_perm[ms];
        const T *s_val = val_buf + ms * (kPCAP + 32 / sizeof(T)) + s_off_val[ms];
        const unsigned char *s_band = band_buf + (size_t)ms * kBand * RB;
        const bool staged = !s_direct[ms];
        const int64_t b0 = s_b0[ms], b1 = s_b1[ms];
        const int64_t base = s_ptr[0];
        auto where = [&](int64_t c) -> int64_t {
            if (BAND && c >= b0 && c < b1) return -1 - (c - b0) * RB;
            return c * a.ldx;
        };
        auto meta = [&](int64_t e) -> WideNz {
            WideNz z;
            const int64_t c = staged ? (int64_t)(uint32_t)s_idx[e] : (int64_t)(uint32_t)a.indices[base + e];
            z.off = where(c);
            if (!ACC) z.val = 0.0;
            else if (PERM) z.val = (double)a.vals[staged ? s_perm[e] : a.perm[base + e]];
            else z.val = (double)(staged ? s_val[e] : a.vals[base + e]);
            return z;
        };
        const int rb = g * RPG < nr ? g * RPG : nr;
        const int re = rb + RPG < nr ? rb + RPG : nr;
        const int64_t sb = s_ptr[rb] - base, se = s_ptr[re] - base;
        const int nbw = (int)__reduce_max_sync(0xffffffffu, (unsigned)((se - sb + G - 1) / G));
        double acc[NE], xr[NE];
        int cur = rb;
        int64_t cend = rb < re ? s_ptr[rb + 1] - base : 0;
        auto begin = [&]() {
            if (ACC) {
#pragma unroll
                for (int i = 0; i < NE; ++i) acc[i] = 0.0;
            }
            if (DOT) {
                if (WST) {
                    const T *w = reinterpret_cast<const T *>(w_buf + ((size_t)ms * kPRT + cur) * RB) + lo_e;
#pragma unroll
                    for (int v = 0; v < NVL; ++v) lds32(w + v * G * E, xr + v * E, h);
                } else {
                    const T *w = a.W + (r0 + cur) * a.ldw + lo_e;
#pragma unroll
                    for (int v = 0; v < NVL; ++v) ldv32(w + v * G * E, xr + v * E);
                }
            }
        };
        auto finish = [&]() {
            if (ACC) {
                T *y = a.Y + (r0 + cur) * a.ldy + lo_e;
#pragma unroll
                for (int v = 0; v < NVL; ++v) stv32(y + v * G * E, acc + v * E);
            }
        };
        if (rb < re) begin();
        for (int tb = 0; tb < nbw; ++tb) {
            const int64_t e0 = sb + (int64_t)G * tb;
            WideNz z[G];
            double gv[G][NE];
#pragma unroll
            for (int b = 0; b < G; ++b) {
                if (e0 + b < se) {
                    z[b] = meta(e0 + b);
                    if (!BAND || z[b].off >= 0) {
                        const T *xp = a.X + z[b].off + lo_e;
#pragma unroll
                        for (int v = 0; v < NVL; ++v) {
                            if (L1G) ldv32_l1(xp + v * G * E, gv[b] + v * E);
                            else ldv32(xp + v * G * E, gv[b] + v * E);
                        }
                    } else {
                        const T *xp = reinterpret_cast<const T *>(s_band + (-1 - z[b].off)) + lo_e;
#pragma unroll
                        for (int v = 0; v < NVL; ++v) lds32(xp + v * G * E, gv[b] + v * E, h);
                    }
                } else {
                    z[b].val = 0.0;
#pragma unroll
                    for (int i = 0; i < NE; ++i) gv[b][i] = 0.0;
                }
            }
            double d[G];
#pragma unroll
            for (int b = 0; b < G; ++b) {
                if (e0 + b < se) {
                    while (e0 + b >= cend) {
                        finish();
                        ++cur;
                        cend = s_ptr[cur + 1] - base;
                        begin();
                    }
                }
                if (ACC) {
#pragma unroll
                    for (int i = 0; i < NE; ++i) acc[i] = fma(z[b].val, gv[b][i], acc[i]);
                }
                if (DOT) {
                    double sdot = 0.0;
#pragma unroll
                    for (int i = 0; i < NE; ++i) sdot = fma(gv[b][i], xr[i], sdot);
                    d[b] = sdot;
                }
            }
            if (DOT) {
                const double dd = transpose_reduce<G>(d, l);
                const int64_t e = e0 + l;
                if (e < se)
                    a.D[MODE == SP_FUSED_T ? (staged ? s_perm[e] : a.perm[base + e]) : base + e] = (T)dd;
            }
        }
        if (rb < re) {
            finish();
            while (++cur < re) {
                if (ACC) {
#pragma unroll
                    for (int i = 0; i < NE; ++i) acc[i] = 0.0;
                }
                finish();
            }
        }
        __syncthreads();   // the stages of tile k are free for tiles k + 2 (metadata) / k + 3 (indptr)
    }
}

template <typename T, int NV, int MODE>
static int launch_pipe(const SpmmArgs<T> &a, bool band, cudaStream_t s)
{
    const int64_t ntiles = cdiv(a.nrows, kPRT);
    auto go = [&](auto kern, size_t smem) -> int {
        int per = 0;
        CSRK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CSRK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kPTPB, smem));
        per = per < 1 ? 1 : per;
        const int64_t grid = ntiles < (int64_t)kNumSMs * per ? ntiles : (int64_t)kNumSMs * per;
        CSRK_LAUNCH(kern, (unsigned)grid, kPTPB, smem, s, a, ntiles);
        return CSRK_OK;
    };
    // lanes per row: 8 (one 32-byte vector each, batches of 8 gathers) for 256-byte rows when asked;
    // WST: the W rows of a dot mode by TMA with the tile's metadata (needs contiguous W rows)
    const int g8 = NV == 2 ? knob(MODE == SP_FUSED_T || MODE == SP_SDDMM ? "SPMM_G8_DOT" : "SPMM_G8_FWD", 0) : 0;
    const bool wst = (MODE == SP_FUSED_T || MODE == SP_SDDMM) && knob("SPMM_PIPE_W", 0) && a.ldw == a.k &&
                     !(reinterpret_cast<uintptr_t>(a.W) & 15);
    using PLn = PipeLayout<T, NV, MODE, false>;
    using PLb = PipeLayout<T, NV, MODE, true>;
    if constexpr (NV == 2) {
        if (g8) {
            if (band) return go(k_spmm_pipe<T, NV, MODE, true, 8, false>, PLb::total_nw);
            return go(k_spmm_pipe<T, NV, MODE, false, 8, false>, PLn::total_nw);
        }
    }
    if (wst) {
        if (band) return go(k_spmm_pipe<T, NV, MODE, true, 4, true>, PLb::total_w);
        return go(k_spmm_pipe<T, NV, MODE, false, 4, true>, PLn::total_w);
    }
    if (band) return go(k_spmm_pipe<T, NV, MODE, true, 4, false>, PLb::total_nw);
    if (knob(MODE == SP_FUSED_T || MODE == SP_SDDMM ? "SPMM_L1_DOT" : "SPMM_L1_FWD", 0))
        return go(k_spmm_pipe<T, NV, MODE, false, 4, false, true>, PLn::total_nw);
    return go(k_spmm_pipe<T, NV, MODE, false, 4, false>, PLn::total_nw);
}

template <typename T, int MODE>
static bool launch_wide(const SpmmArgs<T> &a, cudaStream_t s, int &st)
{
    if (!knob("SPMM_WIDE", 1)) return false;
    const int64_t rb = a.k * (int64_t)sizeof(T);
    const int nv = rb == 128 ? 1 : rb == 256 && sizeof(T) == 8 ? 2 : 0;
    if (!nv) return false;
    auto al = [](const void *p, int64_t ld) {
        return !p || (!(reinterpret_cast<uintptr_t>(p) & 31) && !((ld * (int64_t)sizeof(T)) & 31));
    };
    if (!al(a.X, a.ldx) || !al(a.W, a.ldw) || !al(a.Y, a.ldy)) return false;
    st = CSRK_OK;
    if (a.nrows <= 0) return true;
    constexpr int kWTPB = wide_tpb<MODE>();
    const unsigned grid = (unsigned)cdiv(a.nrows, kWTPB / kWG * kWRPG);
    // band staging needs contiguous dense rows (one bulk copy)
    const bool band = knob("SPMM_BAND", 1) && (MODE == SP_FWD || MODE == SP_FWD_PERM) && a.ldx == a.k && a.xrows > 0;
    // persistent pipelined path (bulk copies of 16-byte aligned slices: every operand 16-byte
    // aligned, indptr / indices / perm / values as allocated by the caller)
    if (knob("SPMM_PIPE", 1) && a.nrows >= (int64_t)kNumSMs * kPRT) {
        // (the band costs the pipelined kernel occupancy: fwd 1.16 vs 0.47 ms, bwd 2.08 vs 0.84 ms on config 2)
        const int pband = knob("SPMM_PIPE_BAND", 0) && a.ldx == a.k && a.xrows > 0;
        const bool al16 = !(reinterpret_cast<uintptr_t>(a.indptr) & 15) && !(reinterpret_cast<uintptr_t>(a.indices) & 15) &&
                          (!a.perm || !(reinterpret_cast<uintptr_t>(a.perm) & 15)) &&
                          (!a.vals || !(reinterpret_cast<uintptr_t>(a.vals) & 15));
        if (al16) {
            if (nv == 1) st = launch_pipe<T, 1, MODE>(a, pband, s);
            else st = launch_pipe<T, sizeof(T) == 8 ? 2 : 1, MODE>(a, pband, s);
            return true;
        }
    }
    auto go = [&](auto kern, bool bnd) -> int {
        const size_t smem = bnd ? (size_t)band_cap<MODE>() * rb : 0;
        if (bnd) CSRK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CSRK_LAUNCH(kern, grid, kWTPB, smem, s, a);
        return CSRK_OK;
    };
    constexpr int NV2 = sizeof(T) == 8 ? 2 : 1;
    if (nv == 1) st = band ? go(k_spmm_wide<T, 1, MODE, true>, true) : go(k_spmm_wide<T, 1, MODE, false>, false);
    else st = band ? go(k_spmm_wide<T, NV2, MODE, true>, true) : go(k_spmm_wide<T, NV2, MODE, false>, false);
    return true;
}

// ---------------------------------------------------------------- dispatch
// Vector map: 16-byte aligned row starts and k a multiple of 4.  Otherwise the scalar map.
template <typename T>
static bool vec_ok(int64_t k, std::initializer_list<std::pair<const void *, int64_t>> ops)
{
    if (k % 4) return false;
    for (auto &o : ops)
        if (o.first && ((reinterpret_cast<uintptr_t>(o.first) & 15) || ((o.second * (int64_t)sizeof(T)) % 16)))
            return false;
    return true;
}

template <typename T, int MODE>
static int dispatch(bool vec, const SpmmArgs<T> &a, cudaStream_t s)
{
    int st = CSRK_OK;
    if (vec && launch_wide<T, MODE>(a, s, st)) return st;
    const int lean = knob("SPMM_LEAN", 0);
    if (vec && lean && (MODE == SP_FWD || MODE == SP_FWD_PERM) && a.nrows > 0) {
        const int64_t groups = 256 / 8;
        int64_t grid = cdiv(a.nrows, groups * lean);
        CSRK_LAUNCH((k_spmm_lean<T, 8, 4, MODE == SP_FWD_PERM>), (unsigned)grid, 256, 0, s, a);
        return CSRK_OK;
    }
    if (vec) return launch_spmm<T, 8, 4, MODE>(a, s);
    return launch_spmm<T, 32, 1, MODE>(a, s);
}

template <typename T>
static int spmm_fwd_t(const csrk_pattern &A, const T *A_val, int64_t k, const T *X, int64_t ldx, T *Y,
                      int64_t ldy, Bump &ws, cudaStream_t s)
{
    if (ws.sizing() || A.nrows == 0 || k == 0) return CSRK_OK;
    SpmmArgs<T> a{};
    a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices; a.vals = A_val;
    a.k = k; a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.xrows = A.ncols;
    const bool vec = vec_ok<T>(k, {{X, ldx}, {Y, ldy}});
    if (vec && knob("SPMM_BULK", 0) && (k * (int64_t)sizeof(T)) % 16 == 0 && k * (int64_t)sizeof(T) <= 1024)
        return launch_spmm_bulk<T>(a, s);
    return dispatch<T, SP_FWD>(vec, a, s);
}

template <typename T>
static int spmm_bwd_t(const csrk_pattern &A, const T *A_val, const csrk_pattern *AT, const int64_t *perm,
                      int64_t k, const T *X, int64_t ldx, const T *dY, int64_t lddy, T *dA, T *dX, int64_t lddx,
                      Bump &ws, cudaStream_t s)
{
    const bool vec = vec_ok<T>(k, {{X, ldx}, {dY, lddy}, {dX, lddx}});
    const int64_t np = cdiv(k, kPass);
    // Transpose plan: the caller's, or built in the workspace.
    csrk_pattern ATl{};
    const int64_t *permu = perm;
    if (dX && !AT) {
        int64_t *ATp = ws.take<int64_t>(A.ncols + 1);
        int32_t *ATi = ws.take<int32_t>(A.nnz > 0 ? A.nnz : 1);
        int64_t *pm = ws.take<int64_t>(A.nnz > 0 ? A.nnz : 1);
        CSRK_TRY(transpose_impl(CSRK_F64, A, nullptr, ATp, ATi, nullptr, pm, ws, s));
        ATl = csrk_pattern{A.ncols, A.nrows, A.nnz, ATp, ATi};
        AT = &ATl;
        permu = pm;
    }
    if (ws.sizing() || k == 0) return CSRK_OK;
    SpmmArgs<T> a{};
    a.k = k; a.vals = A_val;
    if (dX && dA && np <= kFusedMaxPasses) {
        // fused transposed traversal: dX and dA in one pass
        a.nrows = AT->nrows; a.indptr = AT->indptr; a.indices = AT->indices; a.perm = permu;
        a.xrows = AT->ncols;
        a.X = dY; a.ldx = lddy; a.W = X; a.ldw = ldx; a.Y = dX; a.ldy = lddx; a.D = dA;
        return dispatch<T, SP_FUSED_T>(vec, a, s);
    }
    if (dX) {
        SpmmArgs<T> b = a;
        b.nrows = AT->nrows; b.indptr = AT->indptr; b.indices = AT->indices; b.perm = permu;
        b.xrows = AT->ncols;
        b.X = dY; b.ldx = lddy; b.Y = dX; b.ldy = lddx;
        CSRK_TRY((dispatch<T, SP_FWD_PERM>(vec, b, s)));
    }
    if (dA && A.nrows > 0) {
        a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices; a.xrows = A.ncols;
        a.X = X; a.ldx = ldx; a.W = dY; a.ldw = lddy; a.D = dA;
        CSRK_TRY((dispatch<T, SP_SDDMM>(vec, a, s)));
    }
    return CSRK_OK;
}

int spmm_fwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t k, const void *X, int64_t ldx,
             void *Y, int64_t ldy, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return spmm_fwd_t<double>(A, (const double *)A_val, k, (const double *)X, ldx, (double *)Y, ldy, ws, s);
    return spmm_fwd_t<float>(A, (const float *)A_val, k, (const float *)X, ldx, (float *)Y, ldy, ws, s);
}

int spmm_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
             int64_t k, const void *X, int64_t ldx, const void *dY, int64_t lddy, void *dA, void *dX, int64_t lddx,
             Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return spmm_bwd_t<double>(A, (const double *)A_val, AT, perm, k, (const double *)X, ldx, (const double *)dY,
                                  lddy, (double *)dA, (double *)dX, lddx, ws, s);
    return spmm_bwd_t<float>(A, (const float *)A_val, AT, perm, k, (const float *)X, ldx, (const float *)dY, lddy,
                             (float *)dA, (float *)dX, lddx, ws, s);
}

}  // namespace csrk
