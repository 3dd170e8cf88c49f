// gcn.cu -- the GCN layer of PAPER 4.4, Eq. gcn_update
// evaluated right to left as the paper's listing does (Fig. 12):
//
//   D       = (graph.row_sum() + 1.) ** -0.5             k_gcn_deg
//   XTheta  = X @ weights                                k_rowgemm        (csrk_dense_gemm_nn)
//   C       = D[:, None] * (graph @ (D Z) + D Z) + bias  k_gcn_prop       (csrk_gcn_fwd)
//
// The propagation is one SpMM with the D scalings fused into its gather (a_p D_j per neighbour)
// and epilogue (D_i, the identity term D_i Z_i of A~ = A + I, the bias): Z is read once per
// stored entry and Y written once.  Backward (csrk_gcn_bwd): dZ = D (A^T (D dY) + D dY) -- the
// same kernel over the rows of A^T (cached plan, or a transpose built in the workspace; values
// gathered through perm) -- and dbias = column sums of dY.  dTheta = X^T dZ (k_gemm_tn) and
// dX = dZ Theta^T (k_rowgemm) close the layer.  Rows of width F are handled by G = F / V lanes
// (V = 4 values per lane), 32 / G rows per warp; rows with more than kGcnLong
// neighbours (power-law hubs) are queued for a CTA each.  All reductions in fp64.
#include "ops.cuh"
#include "rows.cuh"

namespace csrk {

constexpr int kGcnTPB = 256;
constexpr int kGcnLong = 64;
constexpr int kV = 4;

// D_i = (row sum + 1)^-1/2: a thread per row of <= 32 entries, the warp together for longer
// rows (power-law hubs), fixed shuffle tree
__global__ __launch_bounds__(256) void k_gcn_deg(int64_t n, const int64_t *__restrict__ indptr,
                                                 const float *__restrict__ vf, const double *__restrict__ vd,
                                                 double *__restrict__ D)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    int64_t s = 0, e = 0;
    if (valid) {
        s = indptr[i];
        e = indptr[i + 1];
    }
    const bool lng = valid && e - s > 32;
    if (valid && !lng) {
        double sum = 1.0;  // the + 1 of A~ = A + I
        for (int64_t p = s; p < e; ++p) sum += vd ? vd[p] : (double)vf[p];
        D[i] = 1.0 / sqrt(sum);
    }
    unsigned lm = __ballot_sync(0xffffffffu, lng);
    while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const int64_t rs = __shfl_sync(0xffffffffu, s, src), re = __shfl_sync(0xffffffffu, e, src);
        double sum = 0.0;
        for (int64_t p = rs + lane; p < re; p += 32) sum += vd ? vd[p] : (double)vf[p];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == src) D[i] = 1.0 / sqrt(1.0 + sum);
    }
}

template <typename T>
struct GcnArgs {
    int64_t n, F;
    const int64_t *indptr;
    const int32_t *indices;
    const T *vals;
    const int64_t *perm;  // nullable: value of entry p is vals[perm[p]]
    const double *D;
    const T *Z;           // gathered operand (Z fwd, dY bwd)
    int64_t ldz;
    const T *bias;        // nullable
    T *Y;
    int64_t ldy;
    RowList L;
};

template <typename T>
__device__ __forceinline__ void gcn_load(const T *p, int64_t c, int64_t F, double (&v)[kV])
{
#pragma unroll
    for (int q = 0; q < kV; ++q) v[q] = c + q < F ? (double)p[c + q] : 0.0;
}

// the lane's kV values of a row as one 16-byte (fp32) / two 16-byte (fp64) loads: F % 4 == 0 and
// 16-byte aligned rows (checked on the host)
__device__ __forceinline__ void gcn_load_vec(const float *p, int64_t c, double (&v)[kV])
{
    const float4 f = __ldg(reinterpret_cast<const float4 *>(p + c));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}
__device__ __forceinline__ void gcn_load_vec(const double *p, int64_t c, double (&v)[kV])
{
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p + c));
    const double2 b = __ldg(reinterpret_cast<const double2 *>(p + c) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// out row i = D_i (sum_p a_p D_j Z_j + D_i Z_i) + bias, lanes [g*G, g*G + G) of a warp own row i
template <typename T>
__device__ __forceinline__ void gcn_finish(const GcnArgs<T> &a, int64_t i, int64_t c, double (&acc)[kV])
{
    const double di = a.D[i];
    double z[kV];
    gcn_load(a.Z + i * a.ldz, c, a.F, z);
#pragma unroll
    for (int q = 0; q < kV; ++q) {
        if (c + q < a.F) {
            double y = di * fma(di, z[q], acc[q]);
            if (a.bias) y += (double)a.bias[c + q];
            a.Y[i * a.ldy + c + q] = (T)y;
        }
    }
}

#ifndef CSRK_GCN_MINB
#define CSRK_GCN_MINB 4   // measured (1 / 4 / 6 / 8): fwd 356 / 324 / 344 / 445 us on the f4 workload
#endif
template <typename T, int G, bool VEC>
__global__ __launch_bounds__(kGcnTPB, CSRK_GCN_MINB) void k_gcn_prop(GcnArgs<T> a)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int sub = lane % G;            // lane within the row group
    const int64_t c = (int64_t)sub * kV; // first column of this lane
    const int64_t gid = ((int64_t)blockIdx.x * kGcnTPB + threadIdx.x) / G;
    const int64_t ngroups = (int64_t)gridDim.x * kGcnTPB / G;
    for (int64_t i = gid; i < a.n; i += ngroups) {
        const int64_t s = a.indptr[i], e = a.indptr[i + 1];
        if (e - s > kGcnLong) {
            if (sub == 0) a.L.rows[atomicAdd(a.L.count, 1)] = (int32_t)i;
            continue;
        }
        double acc[kV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int64_t p = s; p < e; ++p) {
            const int32_t j = a.indices[p];
            const double w = (double)a.vals[a.perm ? a.perm[p] : p] * a.D[j];
            double z[kV];
            if (VEC) gcn_load_vec(a.Z + (int64_t)j * a.ldz, c, z);
            else gcn_load(a.Z + (int64_t)j * a.ldz, c, a.F, z);
#pragma unroll
            for (int q = 0; q < kV; ++q) acc[q] = fma(w, z[q], acc[q]);
        }
        gcn_finish(a, i, c, acc);
    }
}

// hubs: one CTA per row; the kGcnTPB / G groups split the neighbours (unrolled gathers), then a
// shuffle tree inside each warp and a fixed-order sum over the warps
template <typename T, int G>
__global__ __launch_bounds__(kGcnTPB) void k_gcn_prop_long(GcnArgs<T> a)
{
    pdl_wait();
    __shared__ double s_part[kGcnTPB / 32][32 * kV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane % G;
    const int grp = threadIdx.x / G;
    constexpr int NG = kGcnTPB / G;
    const int64_t c = (int64_t)sub * kV;
    const int n = *(volatile int *)a.L.count;
    for (int it = blockIdx.x; it < n; it += gridDim.x) {
        const int64_t i = a.L.rows[it];
        double acc[kV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int64_t p = a.indptr[i] + grp; p < a.indptr[i + 1]; p += NG) {
            const int32_t j = a.indices[p];
            const double w = (double)a.vals[a.perm ? a.perm[p] : p] * a.D[j];
            double z[kV];
            gcn_load(a.Z + (int64_t)j * a.ldz, c, a.F, z);
#pragma unroll
            for (int q = 0; q < kV; ++q) acc[q] = fma(w, z[q], acc[q]);
        }
#pragma unroll
        for (int o = G; o < 32; o <<= 1)
#pragma unroll
            for (int q = 0; q < kV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (lane < G)
#pragma unroll
            for (int q = 0; q < kV; ++q) s_part[warp][lane * kV + q] = acc[q];
        __syncthreads();
        if (warp == 0) {
            if (lane < G) {
#pragma unroll
                for (int q = 0; q < kV; ++q) {
                    double t = 0.0;
                    for (int w = 0; w < kGcnTPB / 32; ++w) t += s_part[w][lane * kV + q];
                    acc[q] = t;
                }
                gcn_finish(a, i, c, acc);
            }
        }
        __syncthreads();
    }
}

// column sums of dY (n x F) into acc[F] (fp64 atomics; one partial per CTA and column)
template <typename T>
__global__ __launch_bounds__(kGcnTPB) void k_colsum(int64_t n, int64_t F, const T *__restrict__ Y, int64_t ld,
                                                    double *__restrict__ acc)
{
    pdl_wait();
    const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = r0 + rows_per < n ? r0 + rows_per : n;
    const int64_t lanes = kGcnTPB - kGcnTPB % F;  // threads (row slot, column)
    if (threadIdx.x >= lanes) return;
    const int64_t f = threadIdx.x % F, rs = threadIdx.x / F, rstep = lanes / F;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t r = r0 + rs;
    for (; r + 3 * rstep < r1; r += 4 * rstep) {
        s0 += (double)Y[r * ld + f];
        s1 += (double)Y[(r + rstep) * ld + f];
        s2 += (double)Y[(r + 2 * rstep) * ld + f];
        s3 += (double)Y[(r + 3 * rstep) * ld + f];
    }
    for (; r < r1; r += rstep) s0 += (double)Y[r * ld + f];
    atomicAdd(&acc[f], (s0 + s1) + (s2 + s3));
}

template <typename T>
__global__ void k_to_dtype(int64_t m, const double *__restrict__ a, T *__restrict__ out)
{
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = (T)a[i];
}

// ---------------------------------------------------------------- small dense GEMMs
// Z[n x F] = X[n x C] W (W: C x F row-major) or X W^T (W: F x C), W staged in shared memory;
// one thread per (row, 16-column chunk), fp64 accumulation.
constexpr int kGemmChunk = 16;

template <typename T>
__global__ __launch_bounds__(kGcnTPB) void k_rowgemm(int64_t n, int64_t C, int64_t F, const T *__restrict__ X,
                                                     int64_t ldx, const T *__restrict__ W, int transW,
                                                     T *__restrict__ Z, int64_t ldz, int vec)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char s_raw[];
    double *sW = reinterpret_cast<double *>(s_raw);  // C x F, [c * F + f]
    for (int64_t q = threadIdx.x; q < C * F; q += kGcnTPB) {
        const int64_t cc = q / F, f = q % F;
        sW[q] = (double)(transW ? W[f * C + cc] : W[cc * F + f]);
    }
    __syncthreads();
    const int64_t nch = (F + kGemmChunk - 1) / kGemmChunk;
    const int64_t t = (int64_t)blockIdx.x * kGcnTPB + threadIdx.x;
    const int64_t r = t / nch, ch = t % nch;
    if (r >= n) return;
    const int64_t f0 = ch * kGemmChunk;
    double acc[kGemmChunk];
#pragma unroll
    for (int q = 0; q < kGemmChunk; ++q) acc[q] = 0.0;
    if (vec) {  // fp32, C % 4 == 0, F % 16 == 0, 16-byte aligned rows: float4 loads and stores
        const float4 *xr = reinterpret_cast<const float4 *>(X + r * ldx);
        for (int64_t c4 = 0; c4 < C / 4; ++c4) {
            const float4 xv = xr[c4];
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const double *w = sW + (c4 * 4 + h) * F + f0;
#pragma unroll
                for (int q = 0; q < kGemmChunk; ++q) acc[q] = fma((double)xs[h], w[q], acc[q]);
            }
        }
        float4 *zr = reinterpret_cast<float4 *>(Z + r * ldz + f0);
#pragma unroll
        for (int q = 0; q < kGemmChunk / 4; ++q)
            zr[q] = make_float4((float)acc[4 * q], (float)acc[4 * q + 1], (float)acc[4 * q + 2], (float)acc[4 * q + 3]);
        return;
    }
    for (int64_t cc = 0; cc < C; ++cc) {
        const double x = (double)X[r * ldx + cc];
        const double *w = sW + cc * F + f0;
#pragma unroll
        for (int q = 0; q < kGemmChunk; ++q)
            if (f0 + q < F) acc[q] = fma(x, w[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < kGemmChunk; ++q)
        if (f0 + q < F) Z[r * ldz + f0 + q] = (T)acc[q];
}

// dW[C x F] += X^T dZ: a thread owns (c, 16-column chunk of F) for one row slot; the CTA's row
// slots stride its slice of rows; partials reduced in shared memory, then one fp64 atomic per
// output and CTA.  X[r, c] and dZ[r, chunk] are shared by the threads of a row (broadcast).
// dW = X^T dZ (C x F) for tall X (n x C), dZ (n x F): each CTA sums a contiguous block of rows;
// its 256 threads are `slots` row slots x (C x ceil(F/16)) column blocks, each thread owning 16
// fp64 accumulators.  The slots' partials are added in slot order in shared memory and the
// CTA's C x F partial is written to part[blockIdx]; k_tn_sum adds the CTAs' partials in block
// order.  No atomics: the result is the same bits on every run.
template <typename T>
__global__ __launch_bounds__(kGcnTPB) void k_gemm_tn(int64_t n, int64_t C, int64_t F, const T *__restrict__ X,
                                                     int64_t ldx, const T *__restrict__ dZ, int64_t lddz,
                                                     double *__restrict__ part)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char s_raw[];
    double *s_part = reinterpret_cast<double *>(s_raw);  // [slots][C x F]
    const int64_t nch = (F + kGemmChunk - 1) / kGemmChunk;
    const int64_t per_row = C * nch;                        // threads per row slot (<= kGcnTPB)
    const int64_t slots = kGcnTPB / per_row;
    const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = r0 + rows_per < n ? r0 + rows_per : n;
    const int64_t slot = threadIdx.x / per_row, w = threadIdx.x % per_row;
    const int64_t cc = w / nch, f0 = (w % nch) * kGemmChunk;
    const int64_t CF = C * F;
    if (slot < slots) {
        double a[kGemmChunk];
#pragma unroll
        for (int q = 0; q < kGemmChunk; ++q) a[q] = 0.0;
#pragma unroll 2
        for (int64_t r = r0 + slot; r < r1; r += slots) {
            const double x = (double)X[r * ldx + cc];
            const T *z = dZ + r * lddz + f0;
#pragma unroll
            for (int q = 0; q < kGemmChunk; ++q)
                if (f0 + q < F) a[q] = fma(x, (double)z[q], a[q]);
        }
#pragma unroll
        for (int q = 0; q < kGemmChunk; ++q)
            if (f0 + q < F) s_part[slot * CF + cc * F + f0 + q] = a[q];
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < CF; q += kGcnTPB) {
        double t = 0.0;
        for (int64_t sl = 0; sl < slots; ++sl) t += s_part[sl * CF + q];
        part[(int64_t)blockIdx.x * CF + q] = t;
    }
}

// dW[q] = sum_b part[b][q] in a fixed order: a warp per output, lane-strided partial sums then a
// fixed shuffle tree (a single thread's chain over all CTAs' partials would be ~600 dependent loads)
template <typename T>
__global__ __launch_bounds__(kGcnTPB) void k_tn_sum(int64_t CF, int nb, const double *__restrict__ part,
                                                    T *__restrict__ dW)
{
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (kGcnTPB / 32);
    for (int64_t q = (int64_t)blockIdx.x * (kGcnTPB / 32) + (threadIdx.x >> 5); q < CF; q += warps) {
        double t = 0.0;
        for (int b = lane; b < nb; b += 32) t += part[(int64_t)b * CF + q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) dW[q] = (T)t;
    }
}

// ---------------------------------------------------------------- host side
template <typename T, int G>
static int launch_prop(GcnArgs<T> &a, cudaStream_t s)
{
    CSRK_CUDA(cudaMemsetAsync(a.L.count, 0, sizeof(int), s));
    const int64_t groups = cdiv(a.n, 1);
    int64_t grid = cdiv(groups * G, kGcnTPB);
    if (grid > kNumSMs * 16) grid = kNumSMs * 16;
    const bool vec = a.F % kV == 0 && (a.ldz * (int64_t)sizeof(T)) % 16 == 0 &&
                     !(reinterpret_cast<uintptr_t>(a.Z) & 15) && knob("GCN_VEC", 1);
    if (vec) CSRK_LAUNCH((k_gcn_prop<T, G, true>), (unsigned)grid, kGcnTPB, 0, s, a);
    else CSRK_LAUNCH((k_gcn_prop<T, G, false>), (unsigned)grid, kGcnTPB, 0, s, a);
    CSRK_LAUNCH((k_gcn_prop_long<T, G>), (unsigned)(kNumSMs * 4), kGcnTPB, 0, s, a);
    return CSRK_OK;
}

template <typename T>
static int run_prop(GcnArgs<T> &a, cudaStream_t s)
{
    if (a.n == 0) return CSRK_OK;
    const int64_t lanes = cdiv(a.F, kV);
    if (lanes <= 1) return launch_prop<T, 1>(a, s);
    if (lanes <= 2) return launch_prop<T, 2>(a, s);
    if (lanes <= 4) return launch_prop<T, 4>(a, s);
    if (lanes <= 8) return launch_prop<T, 8>(a, s);
    if (lanes <= 16) return launch_prop<T, 16>(a, s);
    return launch_prop<T, 32>(a, s);  // F <= 128 (checked at the ABI)
}

template <typename T>
static int gcn_fwd_t(const csrk_pattern &A, const T *Av, int64_t F, const T *Z, int64_t ldz, const T *bias, T *Y,
                     int64_t ldy, double *D, Bump &ws, cudaStream_t s)
{
    GcnArgs<T> a{};
    carve_rowlist(A.nrows, a.L, ws);
    if (ws.sizing()) return CSRK_OK;
    if (A.nrows == 0) return CSRK_OK;
    const bool f64 = sizeof(T) == 8;
    CSRK_LAUNCH(k_gcn_deg, (unsigned)cdiv(A.nrows, 256), 256, 0, s, A.nrows, A.indptr,
                f64 ? nullptr : (const float *)Av, f64 ? (const double *)Av : nullptr, D);
    a.n = A.nrows; a.F = F; a.indptr = A.indptr; a.indices = A.indices; a.vals = Av; a.D = D;
    a.Z = Z; a.ldz = ldz; a.bias = bias; a.Y = Y; a.ldy = ldy;
    return run_prop(a, s);
}

template <typename T>
static int gcn_bwd_t(const csrk_pattern &A, const T *Av, const csrk_pattern *AT, const int64_t *perm, int64_t F,
                     const double *D, const T *dY, int64_t lddy, T *dZ, int64_t lddz, T *dbias, Bump &ws,
                     cudaStream_t s)
{
    const int64_t n = A.nrows;
    csrk_pattern Tt{};
    int64_t *tp = nullptr;
    if (AT) {
        Tt = *AT;
    } else {
        int64_t *ATp = ws.take<int64_t>(n + 1);
        int32_t *ATi = ws.take<int32_t>(A.nnz > 0 ? A.nnz : 1);
        tp = ws.take<int64_t>(A.nnz > 0 ? A.nnz : 1);
        Tt = csrk_pattern{n, n, A.nnz, ATp, ATi};
    }
    double *bacc = ws.take<double>(F > 0 ? F : 1);
    GcnArgs<T> a{};
    carve_rowlist(n, a.L, ws);
    if (!AT && dZ) CSRK_TRY(transpose_impl(sizeof(T) == 8 ? CSRK_F64 : CSRK_F32, A, nullptr,
                                           const_cast<int64_t *>(Tt.indptr), const_cast<int32_t *>(Tt.indices),
                                           nullptr, tp, ws, s));
    if (ws.sizing()) return CSRK_OK;
    if (dbias) {
        CSRK_CUDA(cudaMemsetAsync(bacc, 0, sizeof(double) * (size_t)F, s));
        if (n > 0) CSRK_LAUNCH(k_colsum<T>, (unsigned)(kNumSMs * 4), kGcnTPB, 0, s, n, F, dY, lddy, bacc);
        CSRK_LAUNCH(k_to_dtype<T>, (unsigned)cdiv(F, 256), 256, 0, s, F, bacc, dbias);
    }
    if (!dZ || n == 0) return CSRK_OK;
    a.n = n; a.F = F; a.indptr = Tt.indptr; a.indices = Tt.indices; a.vals = Av; a.perm = AT ? perm : tp;
    a.D = D; a.Z = dY; a.ldz = lddy; a.bias = nullptr; a.Y = dZ; a.ldy = lddz;
    return run_prop(a, s);
}

int gcn_fwd(csrk_dtype dt, const csrk_pattern &A, const void *Av, int64_t F, const void *Z, int64_t ldz,
            const void *bias, void *Y, int64_t ldy, double *D, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return gcn_fwd_t<double>(A, (const double *)Av, F, (const double *)Z, ldz, (const double *)bias, (double *)Y,
                                 ldy, D, ws, s);
    return gcn_fwd_t<float>(A, (const float *)Av, F, (const float *)Z, ldz, (const float *)bias, (float *)Y, ldy, D,
                            ws, s);
}

int gcn_bwd(csrk_dtype dt, const csrk_pattern &A, const void *Av, const csrk_pattern *AT, const int64_t *perm,
            int64_t F, const double *D, const void *dY, int64_t lddy, void *dZ, int64_t lddz, void *dbias, Bump &ws,
            cudaStream_t s)
{
    if (dt == CSRK_F64)
        return gcn_bwd_t<double>(A, (const double *)Av, AT, perm, F, D, (const double *)dY, lddy, (double *)dZ, lddz,
                                 (double *)dbias, ws, s);
    return gcn_bwd_t<float>(A, (const float *)Av, AT, perm, F, D, (const float *)dY, lddy, (float *)dZ, lddz,
                            (float *)dbias, ws, s);
}

template <typename T>
static int gemm_nn_t(int64_t n, int64_t C, int64_t F, const T *X, int64_t ldx, const T *W, int transW, T *Z,
                     int64_t ldz, cudaStream_t s)
{
    if (n == 0 || F == 0) return CSRK_OK;
    const size_t smem = sizeof(double) * (size_t)(C * F);
    if (smem > 48 * 1024) CSRK_CUDA(cudaFuncSetAttribute(k_rowgemm<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)smem));
    const int64_t threads = n * cdiv(F, kGemmChunk);
    const bool al = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Z)) & 15) == 0;
    const int vec = sizeof(T) == 4 && al && C % 4 == 0 && ldx % 4 == 0 && F % kGemmChunk == 0 && ldz % 4 == 0;
    CSRK_LAUNCH(k_rowgemm<T>, (unsigned)cdiv(threads, kGcnTPB), kGcnTPB, smem, s, n, C, F, X, ldx, W, transW, Z, ldz,
                vec);
    return CSRK_OK;
}

int dense_gemm_nn(csrk_dtype dt, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *W,
                  int transW, void *Z, int64_t ldz, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return gemm_nn_t<double>(n, C, F, (const double *)X, ldx, (const double *)W, transW, (double *)Z, ldz, s);
    return gemm_nn_t<float>(n, C, F, (const float *)X, ldx, (const float *)W, transW, (float *)Z, ldz, s);
}

template <typename T>
static int gemm_tn_t(int64_t n, int64_t C, int64_t F, const T *X, int64_t ldx, const T *dZ, int64_t lddz, T *dW,
                     Bump &ws, cudaStream_t s)
{
    constexpr int nb = kNumSMs * 4;
    double *part = ws.take<double>((size_t)nb * (C * F > 0 ? C * F : 1));
    if (ws.sizing()) return CSRK_OK;
    if (C * F == 0) return CSRK_OK;
    if (n == 0) return cudaMemsetAsync(dW, 0, sizeof(T) * (size_t)(C * F), s) == cudaSuccess ? CSRK_OK : CSRK_ERR_CUDA;
    const int64_t per_row = C * ((F + kGemmChunk - 1) / kGemmChunk);
    const size_t smem = sizeof(double) * (size_t)(kGcnTPB / per_row) * (size_t)(C * F);
    if (smem > 48 * 1024) CSRK_CUDA(cudaFuncSetAttribute(k_gemm_tn<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)smem));
    CSRK_LAUNCH(k_gemm_tn<T>, (unsigned)nb, kGcnTPB, smem, s, n, C, F, X, ldx, dZ, lddz, part);
    CSRK_LAUNCH(k_tn_sum<T>, (unsigned)cdiv(C * F, kGcnTPB / 32), kGcnTPB, 0, s, C * F, nb, (const double *)part,
                dW);
    return CSRK_OK;
}

int dense_gemm_tn(csrk_dtype dt, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *dZ,
                  int64_t lddz, void *dW, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return gemm_tn_t<double>(n, C, F, (const double *)X, ldx, (const double *)dZ, lddz, (double *)dW, ws, s);
    return gemm_tn_t<float>(n, C, F, (const float *)X, ldx, (const float *)dZ, lddz, (float *)dW, ws, s);
}

}  // namespace csrk
