// spmm.cu -- SpDMM forward and backward (PAPER 3.1.3; Table 1).
//
// A group of G lanes owns one row (of A, or of A^T for the backward); each lane owns V
// consecutive columns of the k-wide dense rows (16-byte vectors when aligned), so every
// gathered X/dY row is one coalesced G*V*sizeof(T)-byte transaction.  Row nonzeros are
// fetched G at a time (coalesced) and broadcast with shuffles.  Accumulation is fp64.
//
//   FWD      Y[i,:]  = sum_p A[p] X[idx p,:]
//   FWD_PERM same over the cached transpose with values A[perm q]  (dX = A^T dY)
//   SDDMM    dA[p]   = <dY[i,:], X[idx p,:]>                        ((dY X^T)(.)mask(A))
//   FUSED_T  over row j of A^T: dX[j,:] = sum_q A[perm q] dY[i_q,:] and, from the same
//            dY row, dA[perm q] = <dY[i_q,:], X[j,:]>  -- one pass for both gradients.
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
    T *Y;        int64_t ldy;   // dense output (FWD: Y, FUSED_T: dX)
    T *D;                       // dA (SDDMM, FUSED_T)
    int G;                      // lanes per row (power of two, <= 32)
};

template <typename T, int V> struct VecT;
template <> struct VecT<double, 1> { using type = double; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<float, 4> { using type = float4; };

template <typename T, int V>
__device__ __forceinline__ void vload(const T *p, double (&r)[V])
{
    using VT = typename VecT<T, V>::type;
    VT v = __ldg(reinterpret_cast<const VT *>(p));
    const T *e = reinterpret_cast<const T *>(&v);
#pragma unroll
    for (int i = 0; i < V; ++i) r[i] = (double)e[i];
}

template <typename T, int V>
__device__ __forceinline__ void vstore(T *p, const double (&r)[V])
{
    using VT = typename VecT<T, V>::type;
    VT v;
    T *e = reinterpret_cast<T *>(&v);
#pragma unroll
    for (int i = 0; i < V; ++i) e[i] = (T)r[i];
    *reinterpret_cast<VT *>(p) = v;
}

constexpr int kSpmmTPB = 256;

template <typename T, int V, int MODE, int NP>
__global__ __launch_bounds__(kSpmmTPB) void k_spmm(SpmmArgs<T> a)
{
    const int G = a.G;
    const int lane = threadIdx.x & (G - 1);
    const int64_t row = ((int64_t)blockIdx.x * kSpmmTPB + threadIdx.x) / G;
    if (row >= a.nrows) return;  // whole group leaves together
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const int64_t s = a.indptr[row], e = a.indptr[row + 1];
    const int64_t stride = (int64_t)G * V;

    if (MODE == SP_FWD || MODE == SP_FWD_PERM) {
        for (int64_t col0 = 0; col0 < a.k; col0 += stride) {
            const int64_t col = col0 + (int64_t)lane * V;
            const bool act = col < a.k;
            double acc[V];
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] = 0.0;
            for (int64_t p0 = s; p0 < e; p0 += G) {
                const int nb = (int)(e - p0 < G ? e - p0 : G);
                int c_l = 0;
                double a_l = 0.0;
                if (lane < nb) {
                    c_l = a.indices[p0 + lane];
                    a_l = (double)a.vals[MODE == SP_FWD_PERM ? a.perm[p0 + lane] : p0 + lane];
                }
#pragma unroll 4
                for (int b = 0; b < nb; ++b) {
                    const int cb = __shfl_sync(gmask, c_l, b, G);
                    const double ab = __shfl_sync(gmask, a_l, b, G);
                    if (act) {
                        double xv[V];
                        vload<T, V>(a.X + (int64_t)cb * a.ldx + col, xv);
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[i] = fma(ab, xv[i], acc[i]);
                    }
                }
            }
            if (act) vstore<T, V>(a.Y + row * a.ldy + col, acc);
        }
    } else if (MODE == SP_SDDMM) {
        for (int64_t p0 = s; p0 < e; p0 += G) {
            const int nb = (int)(e - p0 < G ? e - p0 : G);
            const int c_l = lane < nb ? a.indices[p0 + lane] : 0;
            double mine = 0.0;
            for (int b = 0; b < nb; ++b) {
                const int cb = __shfl_sync(gmask, c_l, b, G);
                double dot = 0.0;
                for (int64_t col0 = 0; col0 < a.k; col0 += stride) {
                    const int64_t col = col0 + (int64_t)lane * V;
                    if (col < a.k) {
                        double xv[V], wv[V];
                        vload<T, V>(a.X + (int64_t)cb * a.ldx + col, xv);
                        vload<T, V>(a.W + row * a.ldw + col, wv);
#pragma unroll
                        for (int i = 0; i < V; ++i) dot = fma(wv[i], xv[i], dot);
                    }
                }
                for (int o = G >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(gmask, dot, o, G);
                if (lane == b) mine = dot;
            }
            if (lane < nb) a.D[p0 + lane] = (T)mine;
        }
    } else {  // SP_FUSED_T: row `row` of A^T (= column j of A)
        double xj[NP][V], acc[NP][V];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int64_t col = q * stride + (int64_t)lane * V;
#pragma unroll
            for (int i = 0; i < V; ++i) { xj[q][i] = 0.0; acc[q][i] = 0.0; }
            if (col < a.k) vload<T, V>(a.W + row * a.ldw + col, xj[q]);
        }
        for (int64_t p0 = s; p0 < e; p0 += G) {
            const int nb = (int)(e - p0 < G ? e - p0 : G);
            int i_l = 0;
            int64_t pv_l = 0;
            double a_l = 0.0;
            if (lane < nb) {
                i_l = a.indices[p0 + lane];
                pv_l = a.perm[p0 + lane];
                a_l = (double)a.vals[pv_l];
            }
            double mine = 0.0;
#pragma unroll 2
            for (int b = 0; b < nb; ++b) {
                const int ib = __shfl_sync(gmask, i_l, b, G);
                const double ab = __shfl_sync(gmask, a_l, b, G);
                double dot = 0.0;
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const int64_t col = q * stride + (int64_t)lane * V;
                    if (col < a.k) {
                        double g[V];
                        vload<T, V>(a.X + (int64_t)ib * a.ldx + col, g);
#pragma unroll
                        for (int i = 0; i < V; ++i) {
                            acc[q][i] = fma(ab, g[i], acc[q][i]);
                            dot = fma(g[i], xj[q][i], dot);
                        }
                    }
                }
                for (int o = G >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(gmask, dot, o, G);
                if (lane == b) mine = dot;
            }
            if (a.D && lane < nb) a.D[pv_l] = (T)mine;
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int64_t col = q * stride + (int64_t)lane * V;
            if (col < a.k) vstore<T, V>(a.Y + row * a.ldy + col, acc[q]);
        }
    }
}

template <typename T, int V, int MODE, int NP>
static int launch_spmm(const SpmmArgs<T> &a, cudaStream_t s)
{
    if (a.nrows <= 0) return CSRK_OK;
    const int64_t per_cta = kSpmmTPB / a.G;
    CSRK_LAUNCH((k_spmm<T, V, MODE, NP>), (unsigned)cdiv(a.nrows, per_cta), kSpmmTPB, 0, s, a);
    return CSRK_OK;
}

// Vector width: 16-byte lanes when every dense row start is 16-byte aligned.
template <typename T>
static int pick_v(int64_t k, std::initializer_list<std::pair<const void *, int64_t>> ops)
{
    const int vmax = 16 / (int)sizeof(T);
    if (k % vmax) return 1;
    for (auto &o : ops) {
        if (o.first && ((reinterpret_cast<uintptr_t>(o.first) & 15) || (o.second % vmax))) return 1;
    }
    return vmax;
}

static int pick_g(int64_t k, int V)
{
    int64_t need = cdiv(k, V);
    int G = 4;
    while (G < 32 && G < need) G <<= 1;
    return G;
}

template <typename T, int MODE, int NP>
static int dispatch_v(int V, const SpmmArgs<T> &a, cudaStream_t s)
{
    if (V == 1) return launch_spmm<T, 1, MODE, NP>(a, s);
    return launch_spmm<T, 16 / sizeof(T), MODE, NP>(a, s);
}

template <typename T>
static int spmm_fwd_t(const csrk_pattern &A, const T *A_val, int64_t k, const T *X, int64_t ldx, T *Y,
                      int64_t ldy, Bump &ws, cudaStream_t s)
{
    if (ws.sizing() || A.nrows == 0 || k == 0) return CSRK_OK;
    SpmmArgs<T> a{};
    a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices; a.vals = A_val;
    a.k = k; a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy;
    const int V = pick_v<T>(k, {{X, ldx}, {Y, ldy}});
    a.G = pick_g(k, V);
    return dispatch_v<T, SP_FWD, 1>(V, a, s);
}

template <typename T>
static int spmm_bwd_t(const csrk_pattern &A, const T *A_val, const csrk_pattern *AT, const int64_t *perm,
                      int64_t k, const T *X, int64_t ldx, const T *dY, int64_t lddy, T *dA, T *dX, int64_t lddx,
                      Bump &ws, cudaStream_t s)
{
    const int V = pick_v<T>(k, {{X, ldx}, {dY, lddy}, {dX, lddx}});
    const int G = pick_g(k, V);
    const int64_t np = cdiv(k, (int64_t)G * V);
    // Transpose plan: the caller's, or built in the workspace.
    csrk_pattern ATl{};
    const int64_t *permu = perm;
    if (dX && !AT) {
        int64_t *ATp = ws.take<int64_t>(A.ncols + 1);
        int32_t *ATi = ws.take<int32_t>(A.nnz);
        int64_t *pm = ws.take<int64_t>(A.nnz);
        CSRK_TRY(transpose_impl(CSRK_F64, A, nullptr, ATp, ATi, nullptr, pm, ws, s));
        ATl = csrk_pattern{A.ncols, A.nrows, A.nnz, ATp, ATi};
        AT = &ATl;
        permu = pm;
    }
    if (ws.overflow) return CSRK_ERR_WORKSPACE;
    if (ws.sizing() || k == 0) return CSRK_OK;
    SpmmArgs<T> a{};
    a.k = k; a.G = G; a.vals = A_val;
    if (dX && np <= 4) {
        // fused transposed traversal: dX and (optionally) dA in one pass
        a.nrows = AT->nrows; a.indptr = AT->indptr; a.indices = AT->indices; a.perm = permu;
        a.X = dY; a.ldx = lddy; a.W = X; a.ldw = ldx; a.Y = dX; a.ldy = lddx; a.D = dA;
        if (np == 1) return dispatch_v<T, SP_FUSED_T, 1>(V, a, s);
        if (np == 2) return dispatch_v<T, SP_FUSED_T, 2>(V, a, s);
        return dispatch_v<T, SP_FUSED_T, 4>(V, a, s);
    }
    if (dX) {
        SpmmArgs<T> b = a;
        b.nrows = AT->nrows; b.indptr = AT->indptr; b.indices = AT->indices; b.perm = permu;
        b.X = dY; b.ldx = lddy; b.Y = dX; b.ldy = lddx;
        CSRK_TRY((dispatch_v<T, SP_FWD_PERM, 1>(V, b, s)));
    }
    if (dA && A.nrows > 0) {
        a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
        a.X = X; a.ldx = ldx; a.W = dY; a.ldw = lddy; a.D = dA;
        CSRK_TRY((dispatch_v<T, SP_SDDMM, 1>(V, a, s)));
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
