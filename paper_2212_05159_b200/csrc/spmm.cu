// spmm.cu -- SpDMM forward and backward (PAPER 3.1.3; Table 1).
//
// A CTA owns a tile of RT consecutive rows (of A, or of A^T for the transposed backward).
// The tile's row pointers, column indices and values (for the transposed traversal: the
// values gathered through perm, A[perm q], and perm itself) are staged in shared memory
// with coalesced loads.  A group of G lanes then walks one row at a time; each lane owns W
// consecutive columns of the k-wide dense rows (two 16-byte vectors when the rows are
// aligned), so every gathered X / dY row is one coalesced G*W*sizeof(T)-byte transaction,
// and the loop over a row's nonzeros is unrolled so its gathers are in flight together.
// Accumulation is fp64 for both dtypes.
//
//   FWD      Y[i,:]  = sum_p A[p] X[idx p,:]
//   FWD_PERM same over the cached transpose, values A[perm q]      (dX = A^T dY)
//   SDDMM    dA[p]   = <dY[i,:], X[idx p,:]>                        ((dY X^T)(.)mask(A))
//   FUSED_T  row j of A^T: dX[j,:] = sum_q A[perm q] dY[i_q,:] and, from the same dY row,
//            dA[perm q] = <dY[i_q,:], X[j,:]>  -- both gradients in one pass.
#include "ops.cuh"

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
};

constexpr int kSpmmTPB = 256;
constexpr int kSpmmRPG = 4;        // rows per group per tile
constexpr int kSpmmCAP = 1536;     // staged nonzeros per tile
constexpr int kFusedMaxPasses = 2;

// W consecutive elements of T, as fp64.
template <typename T, int W>
__device__ __forceinline__ void ldw(const T *p, double (&r)[W])
{
    if constexpr (W * sizeof(T) == 32) {
        using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        constexpr int E = 16 / sizeof(T);
        V a = __ldg(reinterpret_cast<const V *>(p));
        V b = __ldg(reinterpret_cast<const V *>(p) + 1);
        const T *ea = reinterpret_cast<const T *>(&a), *eb = reinterpret_cast<const T *>(&b);
#pragma unroll
        for (int i = 0; i < E; ++i) { r[i] = (double)ea[i]; r[E + i] = (double)eb[i]; }
    } else if constexpr (W * sizeof(T) == 16) {
        using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        V a = __ldg(reinterpret_cast<const V *>(p));
        const T *ea = reinterpret_cast<const T *>(&a);
#pragma unroll
        for (int i = 0; i < W; ++i) r[i] = (double)ea[i];
    } else {
#pragma unroll
        for (int i = 0; i < W; ++i) r[i] = (double)__ldg(p + i);
    }
}

template <typename T, int W>
__device__ __forceinline__ void stw(T *p, const double (&r)[W])
{
    if constexpr (W * sizeof(T) == 32) {
        using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        constexpr int E = 16 / sizeof(T);
        V a, b;
        T *ea = reinterpret_cast<T *>(&a), *eb = reinterpret_cast<T *>(&b);
#pragma unroll
        for (int i = 0; i < E; ++i) { ea[i] = (T)r[i]; eb[i] = (T)r[E + i]; }
        reinterpret_cast<V *>(p)[0] = a;
        reinterpret_cast<V *>(p)[1] = b;
    } else if constexpr (W * sizeof(T) == 16) {
        using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
        V a;
        T *ea = reinterpret_cast<T *>(&a);
#pragma unroll
        for (int i = 0; i < W; ++i) ea[i] = (T)r[i];
        *reinterpret_cast<V *>(p) = a;
    } else {
#pragma unroll
        for (int i = 0; i < W; ++i) p[i] = (T)r[i];
    }
}

template <int G>
__device__ __forceinline__ double group_sum(double v)
{
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

// Reduce four per-lane values d[0..3] across a group of G (>= 4) lanes at once ("transpose
// reduce"): the first two butterfly steps exchange halves of the vector, the rest reduce one
// value.  Lane l ends with the group sum of d[v], v = l / (G/4).  8 shuffles for G = 8
// instead of 4 x 6 for four separate reductions.
template <int G>
__device__ __forceinline__ double group_sum4(const double (&d)[4], int lane)
{
    constexpr int o1 = G >> 1, o2 = G >> 2;
    const bool lo1 = (lane & o1) == 0;
    const double s0 = lo1 ? d[2] : d[0], s1 = lo1 ? d[3] : d[1];
    const double k0 = (lo1 ? d[0] : d[2]) + __shfl_xor_sync(0xffffffffu, s0, o1, G);
    const double k1 = (lo1 ? d[1] : d[3]) + __shfl_xor_sync(0xffffffffu, s1, o1, G);
    const bool lo2 = (lane & o2) == 0;
    double v = (lo2 ? k0 : k1) + __shfl_xor_sync(0xffffffffu, lo2 ? k1 : k0, o2, G);
#pragma unroll
    for (int o = o2 >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

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
    const int64_t stride = (int64_t)G * W;
    const int npass = (int)((a.k + stride - 1) / stride);

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
                        const int64_t col = ps * stride + (int64_t)lane * W;
                        if (on && col < a.k) {
                            double xv[W], wv[W];
                            ldw<T, W>(reinterpret_cast<const T *>(reinterpret_cast<const char *>(a.X + col) + off), xv);
                            ldw<T, W>(a.W + row * a.ldw + col, wv);
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
                    const int64_t col = ps * stride + (int64_t)lane * W;
#pragma unroll
                    for (int i = 0; i < W; ++i) { xj[ps][i] = 0.0; acc[ps][i] = 0.0; }
                    if (valid && ps < npass && col < a.k) ldw<T, W>(a.W + row * a.ldw + col, xj[ps]);
                }
                const char *Xl = reinterpret_cast<const char *>(a.X + (int64_t)lane * W);
#pragma unroll 2
                for (int t = 0; t < maxlen; ++t) {
                    const bool on = t < len;
                    const int64_t off = on ? off_of(s + t) : 0;
                    const double av = on ? val_of(s + t) : 0.0;
                    double dot = 0.0;
#pragma unroll
                    for (int ps = 0; ps < kFusedMaxPasses; ++ps) {
                        const int64_t col = ps * stride + (int64_t)lane * W;
                        if (on && ps < npass && col < a.k) {
                            double gv[W];
                            ldw<T, W>(reinterpret_cast<const T *>(Xl + off) + ps * stride, gv);
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
                for (int ps = 0; ps < kFusedMaxPasses; ++ps) {
                    const int64_t col = ps * stride + (int64_t)lane * W;
                    if (valid && ps < npass && col < a.k) stw<T, W>(a.Y + row * a.ldy + col, acc[ps]);
                }
            }
            continue;
        }
        if (!valid) break;
        // FWD / FWD_PERM
        for (int ps = 0; ps < npass; ++ps) {
            const int64_t col = ps * stride + (int64_t)lane * W;
            if (col >= a.k) break;
            double acc[W];
#pragma unroll
            for (int i = 0; i < W; ++i) acc[i] = 0.0;
            const char *Xc = reinterpret_cast<const char *>(a.X + col);
#pragma unroll 4
            for (int q = s; q < e; ++q) {
                const double av = val_of(q);
                double xv[W];
                ldw<T, W>(reinterpret_cast<const T *>(Xc + off_of(q)), xv);
#pragma unroll
                for (int i = 0; i < W; ++i) acc[i] = fma(av, xv[i], acc[i]);
            }
            stw<T, W>(a.Y + row * a.ldy + col, acc);
        }
    }
}

template <typename T, int G, int W, int MODE>
__global__ __launch_bounds__(kSpmmTPB, MODE == SP_FUSED_T ? 4 : 5) void k_spmm(SpmmArgs<T> a)
{
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

// Vector path: each lane owns 4 consecutive columns (16 or 32 bytes; 8 lanes cover 32 columns);
// needs 16-byte aligned row starts and k a multiple of 4.  Otherwise the scalar path (32 x 1).
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
    a.k = k; a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy;
    return dispatch<T, SP_FWD>(vec_ok<T>(k, {{X, ldx}, {Y, ldy}}), a, s);
}

template <typename T>
static int spmm_bwd_t(const csrk_pattern &A, const T *A_val, const csrk_pattern *AT, const int64_t *perm,
                      int64_t k, const T *X, int64_t ldx, const T *dY, int64_t lddy, T *dA, T *dX, int64_t lddx,
                      Bump &ws, cudaStream_t s)
{
    const bool vec = vec_ok<T>(k, {{X, ldx}, {dY, lddy}, {dX, lddx}});
    const int64_t stride = 32;  // columns per pass: 8 lanes x 4 (vector) or 32 lanes x 1
    const int64_t np = cdiv(k, stride);
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
    if (dX && np <= kFusedMaxPasses) {
        // fused transposed traversal: dX and (optionally) dA in one pass
        a.nrows = AT->nrows; a.indptr = AT->indptr; a.indices = AT->indices; a.perm = permu;
        a.X = dY; a.ldx = lddy; a.W = X; a.ldw = ldx; a.Y = dX; a.ldy = lddx; a.D = dA;
        return dispatch<T, SP_FUSED_T>(vec, a, s);
    }
    if (dX) {
        SpmmArgs<T> b = a;
        b.nrows = AT->nrows; b.indptr = AT->indptr; b.indices = AT->indices; b.perm = permu;
        b.X = dY; b.ldx = lddy; b.Y = dX; b.ldy = lddx;
        CSRK_TRY((dispatch<T, SP_FWD_PERM>(vec, b, s)));
    }
    if (dA && A.nrows > 0) {
        a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
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
