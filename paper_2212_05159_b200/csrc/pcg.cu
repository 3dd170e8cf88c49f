// pcg.cu -- config-5 composition: training step of the learned PCG
// preconditioner M = L L^T (PAPER 4.3).
//
// Forward (x0 = 0, so x never influences the loss and is not formed):
//   r0 = b, u0 = L^T r0, z0 = L u0, p0 = z0, rho0 = r0.z0
//   for i = 1..N:  q_i = A p_{i-1};  s_i = p_{i-1}.q_i;  alpha_i = rho_{i-1}/s_i
//                  r_i = r_{i-1} - alpha_i q_i   (and ||r_i||^2 in the same pass)
//                  u_i = L^T r_i;  z_i = L u_i;  rho_i = r_i.z_i
//                  p_i = z_i + (rho_i/rho_{i-1}) p_{i-1}      (skipped for i = N: unused)
//   loss = sum_i w_i ||r_i|| / ||b||,  w_i = gamma^(N-i) / sum_j gamma^(N-j)
// Reverse: the adjoint of each step above, in reverse order (see pcg_loss_grad below); L's
// gradient comes from the SpMV VJPs of z = L u (op N) and u = L^T r (op T), A's products use
// A^T = the op-T SpMV.  Vectors saved: p_{i-1}, q_i, r_i; u_i, z_i are recomputed.
// precond = 1: M = (L L^T)^{-1} applied exactly, u = L^{-1} r, z = L^{-T} u, by
// the SpTRSV kernels; their VJPs (a solve, a transposed solve and two masked outer products)
// replace the SpMV VJPs.
// All reductions are fixed-grid, fixed-order (deterministic).
#include <cmath>
#include <vector>

#include "ops.cuh"

namespace csrk {

constexpr int kVecTPB = 256;
constexpr int kVecGrid = kNumSMs * 4;

// coefficient = c * (num ? *num : 1) / (den ? *den : 1), read on the device
struct Cf {
    double c;
    const double *num;
    const double *den;
};
__device__ __forceinline__ double cfv(const Cf &a)
{
    double v = a.c;
    if (a.num) v *= *a.num;
    if (a.den) v /= *a.den;
    return v;
}

__device__ __forceinline__ double block_sum(double v)
{
    __shared__ double s[kVecTPB / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kVecTPB / 32; ++i) t += s[i];
    return t;
}

// out = a x + b y + c z  (null vectors skipped); part[blk] = sum out * w (w null: out * out)
__global__ __launch_bounds__(kVecTPB) void k_lin3(int64_t n, double *out, Cf a, const double *x, Cf b,
                                                  const double *y, Cf c, const double *z, const double *w,
                                                  double *part)
{
    pdl_wait();
    const double ca = cfv(a), cb = cfv(b), cc = cfv(c);
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kVecTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kVecTPB) {
        double v = 0.0;
        if (x) v = ca * x[i];
        if (y) v = fma(cb, y[i], v);
        if (z) v = fma(cc, z[i], v);
        out[i] = v;
        if (part) acc = fma(v, w ? w[i] : v, acc);
    }
    if (part) {
        const double t = block_sum(acc);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

__global__ __launch_bounds__(kVecTPB) void k_dot(int64_t n, const double *x, const double *y, double *part)
{
    pdl_wait();
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kVecTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kVecTPB)
        acc = fma(x[i], y[i], acc);
    const double t = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// dst = sign * sum part[0..nb)  (fixed order)
__global__ __launch_bounds__(kVecTPB) void k_finish(const double *part, int nb, double *dst, double sign)
{
    pdl_wait();
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += kVecTPB) acc += part[i];
    const double t = block_sum(acc);
    if (threadIdx.x == 0) *dst = sign * t;
}

struct Scal {         // device scalar layout
    double *rho;      // [N+1]
    double *s;        // [N+1] (index i)
    double *nr2;      // [N+1]
    double *cn;       // [N+1] loss-adjoint coefficients w_i / (||b|| ||r_i||)
    double *rhobar;   // [N+1]
    double *bb;       // b.b
    double *loss;
    double *betabar, *alphabar, *sbar;
};

__global__ void k_loss(Scal S, int N, double gamma)
{
    pdl_wait();
    double wsum = 0.0;
    for (int j = 1; j <= N; ++j) wsum += pow(gamma, (double)(N - j));
    const double nb = sqrt(*S.bb);
    double loss = 0.0;
    for (int i = 1; i <= N; ++i) {
        const double w = pow(gamma, (double)(N - i)) / wsum;
        const double nr = sqrt(S.nr2[i]);
        loss += w * nr / nb;
        S.cn[i] = nr > 0.0 ? w / (nb * nr) : 0.0;
        S.rhobar[i] = 0.0;
    }
    S.rhobar[0] = 0.0;
    *S.loss = loss;
}

// beta_i = rho_i / rho_{i-1}:  rhobar_i += betabar / rho_{i-1};  rhobar_{i-1} -= betabar rho_i / rho_{i-1}^2
__global__ void k_bwd_beta(Scal S, int i)
{
    pdl_wait();
    const double bb = *S.betabar, rm = S.rho[i - 1];
    S.rhobar[i] += bb / rm;
    S.rhobar[i - 1] -= bb * S.rho[i] / (rm * rm);
}

// alpha_i = rho_{i-1} / s_i:  rhobar_{i-1} += alphabar / s_i;  sbar = -alphabar rho_{i-1} / s_i^2
__global__ void k_bwd_alpha(Scal S, int i)
{
    pdl_wait();
    const double ab = *S.alphabar, si = S.s[i];
    S.rhobar[i - 1] += ab / si;
    *S.sbar = -ab * S.rho[i - 1] / (si * si);
}

struct PcgWs {
    double *pb, *rb, *qb;                                   // saved p_{0..N-1}, r_{0..N}, q_{1..N}
    double *u, *z, *rbar, *pbar, *zbar, *ubar, *qbar, *tmp; // n each
    double *dAt;                                            // nnz(L)
    double *part;
    csrk_pattern LT;                                        // precond = solve: L^T pattern + perm
    int64_t *LTperm;
    Scal S;
    void *sub;
    size_t sub_bytes;
};

static size_t spmv_ws_bytes(const csrk_pattern &M)
{
    Bump b(nullptr, 0);
    spmv_fwd(CSRK_F64, CSRK_OP_N, M, nullptr, nullptr, nullptr, nullptr, nullptr, b, 0);
    return b.used + 256;
}

static size_t solve_ws_bytes(const csrk_pattern &L)
{
    size_t m = 0;
    {
        Bump b(nullptr, 0);
        sptrsv_fwd(CSRK_F64, L, nullptr, 0, 0, nullptr, nullptr, b, 0);
        m = b.used > m ? b.used : m;
    }
    {
        Bump b(nullptr, 0);
        csrk_pattern T{L.ncols, L.nrows, L.nnz, L.indptr, L.indices};
        sptrsv_bwd(CSRK_F64, L, nullptr, &T, L.indptr, 0, 0, nullptr, nullptr, nullptr, nullptr, b, 0);
        m = b.used > m ? b.used : m;
    }
    {
        Bump b(nullptr, 0);
        transpose_impl(CSRK_F64, L, nullptr, nullptr, nullptr, nullptr, nullptr, b, 0);
        m = b.used > m ? b.used : m;
    }
    return m + 256;
}

static void carve_pcg(const csrk_pattern &A, const csrk_pattern &L, int N, int precond, PcgWs &w, Bump &ws)
{
    const int64_t n = A.nrows;
    w.pb = ws.take<double>((size_t)N * n);
    w.rb = ws.take<double>((size_t)(N + 1) * n);
    w.qb = ws.take<double>((size_t)N * n);
    double **tv[] = {&w.u, &w.z, &w.rbar, &w.pbar, &w.zbar, &w.ubar, &w.qbar, &w.tmp};
    for (auto p : tv) *p = ws.take<double>(n);
    w.dAt = ws.take<double>(L.nnz > 0 ? L.nnz : 1);
    w.part = ws.take<double>(kVecGrid);
    double *sc = ws.take<double>(5 * (size_t)(N + 1) + 8);
    w.S.rho = sc;
    w.S.s = sc + (N + 1);
    w.S.nr2 = sc + 2 * (N + 1);
    w.S.cn = sc + 3 * (N + 1);
    w.S.rhobar = sc + 4 * (N + 1);
    w.S.bb = sc + 5 * (N + 1);
    w.S.loss = w.S.bb + 1;
    w.S.betabar = w.S.bb + 2;
    w.S.alphabar = w.S.bb + 3;
    w.S.sbar = w.S.bb + 4;
    w.sub_bytes = spmv_ws_bytes(A) > spmv_ws_bytes(L) ? spmv_ws_bytes(A) : spmv_ws_bytes(L);
    w.LTperm = nullptr;
    w.LT = csrk_pattern{L.ncols, L.nrows, L.nnz, nullptr, nullptr};
    if (precond) {
        w.LT.indptr = ws.take<int64_t>(L.ncols + 1);
        w.LT.indices = ws.take<int32_t>(L.nnz > 0 ? L.nnz : 1);
        w.LTperm = ws.take<int64_t>(L.nnz > 0 ? L.nnz : 1);
        const size_t sb = solve_ws_bytes(L);
        w.sub_bytes = sb > w.sub_bytes ? sb : w.sub_bytes;
    }
    w.sub = ws.take<char>(w.sub_bytes);
}

static const Cf ONE{1.0, nullptr, nullptr};

// helpers ------------------------------------------------------------------------------------
#define LIN3(n_, out, a, x, b, y, c, z, wv, part)                                                   \
    CSRK_LAUNCH(k_lin3, (unsigned)kVecGrid, kVecTPB, 0, s, (int64_t)(n_), out, a, x, b, y, c, z, wv, part)

static int dot_to(int64_t n, const double *x, const double *y, double *dst, double sign, double *part,
                  cudaStream_t s)
{
    CSRK_LAUNCH(k_dot, (unsigned)kVecGrid, kVecTPB, 0, s, n, x, y, part);
    CSRK_LAUNCH(k_finish, 1, kVecTPB, 0, s, (const double *)part, kVecGrid, dst, sign);
    return CSRK_OK;
}

int pcg_loss_grad(const csrk_pattern &A, const double *Av, const csrk_pattern &L, const double *Lv, const double *b,
                  int N, double gamma, int precond, double *loss_host, double *resid_host, double *dL, Bump &ws,
                  cudaStream_t s)
{
    PcgWs w{};
    carve_pcg(A, L, N, precond, w, ws);
    if (ws.sizing()) return CSRK_OK;
    const int64_t n = A.nrows;
    auto sub = [&]() { return Bump(w.sub, w.sub_bytes); };
    auto Lt = [&](const double *in, double *out) {   // out = L^T in
        Bump bw = sub();
        return spmv_fwd(CSRK_F64, CSRK_OP_T, L, Lv, nullptr, nullptr, in, out, bw, s);
    };
    auto Ln = [&](const double *in, double *out) {   // out = L in
        Bump bw = sub();
        return spmv_fwd(CSRK_F64, CSRK_OP_N, L, Lv, nullptr, nullptr, in, out, bw, s);
    };
    if (precond) {  // L^T (pattern + perm) once per call, for the transposed solves
        Bump bw = sub();
        CSRK_TRY(transpose_impl(CSRK_F64, L, nullptr, const_cast<int64_t *>(w.LT.indptr),
                                const_cast<int32_t *>(w.LT.indices), nullptr, w.LTperm, bw, s));
    }
    // z = M r with the intermediate in w.u:  M = L L^T: u = L^T r, z = L u;
    // precond = solve: M = (L L^T)^{-1}: u = L^{-1} r, z = L^{-T} u
    auto applyM = [&](const double *r, double *z) -> int {
        if (!precond) {
            CSRK_TRY(Lt(r, w.u));
            return Ln(w.u, z);
        }
        {
            Bump bw = sub();
            CSRK_TRY(sptrsv_fwd(CSRK_F64, L, Lv, 0, 0, r, w.u, bw, s));
        }
        Bump bw = sub();
        return sptrsv_bwd(CSRK_F64, L, Lv, &w.LT, w.LTperm, 0, 0, w.u, w.u, nullptr, z, bw, s);
    };
    // adjoint of z = M r given w.zbar (w.u, z of the same r): dL += ..., rbar += M^T zbar (if asked)
    auto adjM = [&](const double *r, const double *z, bool want_rbar) -> int {
        if (!precond) {
            // z = L u:  Lbar += zbar u^T (.) mask(L);  ubar = L^T zbar
            {
                Bump bw = sub();
                CSRK_TRY(spmv_bwd(CSRK_F64, CSRK_OP_N, L, Lv, nullptr, nullptr, w.u, w.zbar, w.dAt, w.ubar, bw, s));
            }
            LIN3(L.nnz, dL, ONE, dL, ONE, w.dAt, ONE, nullptr, nullptr, nullptr);
            // u = L^T r:  Lbar += r ubar^T (.) mask(L);  rbar += L ubar
            {
                Bump bw = sub();
                CSRK_TRY(spmv_bwd(CSRK_F64, CSRK_OP_T, L, Lv, nullptr, nullptr, r, w.ubar, w.dAt,
                                  want_rbar ? w.tmp : nullptr, bw, s));
            }
            LIN3(L.nnz, dL, ONE, dL, ONE, w.dAt, ONE, nullptr, nullptr, nullptr);
        } else {
            // z = L^{-T} u:  ubar = L^{-1} zbar;  Lbar += -z ubar^T (.) mask(L)
            {
                Bump bw = sub();
                CSRK_TRY(sptrsv_fwd(CSRK_F64, L, Lv, 0, 0, w.zbar, w.ubar, bw, s));
            }
            CSRK_TRY(trsv_outer(L, z, w.ubar, w.dAt, s));
            LIN3(L.nnz, dL, ONE, dL, ONE, w.dAt, ONE, nullptr, nullptr, nullptr);
            // u = L^{-1} r:  rbar += L^{-T} ubar;  Lbar += -(L^{-T} ubar) u^T (.) mask(L)
            {
                Bump bw = sub();
                CSRK_TRY(sptrsv_bwd(CSRK_F64, L, Lv, &w.LT, w.LTperm, 0, 0, w.u, w.ubar, w.dAt, w.tmp, bw, s));
            }
            LIN3(L.nnz, dL, ONE, dL, ONE, w.dAt, ONE, nullptr, nullptr, nullptr);
        }
        if (want_rbar) LIN3(n, w.rbar, ONE, w.rbar, ONE, w.tmp, ONE, nullptr, nullptr, nullptr);
        return CSRK_OK;
    };
    const Scal &S = w.S;
    double *part = w.part;
    auto P = [&](int i) { return w.pb + (size_t)i * n; };       // p_i, i = 0..N-1
    auto R = [&](int i) { return w.rb + (size_t)i * n; };       // r_i, i = 0..N
    auto Q = [&](int i) { return w.qb + (size_t)(i - 1) * n; }; // q_i, i = 1..N

    // ---------------- forward
    CSRK_TRY(dot_to(n, b, b, S.bb, 1.0, part, s));
    LIN3(n, R(0), ONE, b, ONE, nullptr, ONE, nullptr, nullptr, nullptr);
    CSRK_TRY(applyM(b, P(0)));                                 // p0 = z0
    CSRK_TRY(dot_to(n, b, P(0), &S.rho[0], 1.0, part, s));
    for (int i = 1; i <= N; ++i) {
        {
            Bump bw = sub();
            CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_N, A, Av, nullptr, nullptr, P(i - 1), Q(i), bw, s));
        }
        CSRK_TRY(dot_to(n, P(i - 1), Q(i), &S.s[i], 1.0, part, s));
        // r_i = r_{i-1} - (rho_{i-1}/s_i) q_i ; nr2_i = r_i.r_i
        LIN3(n, R(i), ONE, R(i - 1), (Cf{-1.0, &S.rho[i - 1], &S.s[i]}), Q(i), ONE, nullptr, nullptr, part);
        CSRK_LAUNCH(k_finish, 1, kVecTPB, 0, s, (const double *)part, kVecGrid, &S.nr2[i], 1.0);
        if (i == N) break;                                     // rho_N, p_N do not reach the loss
        CSRK_TRY(applyM(R(i), w.z));
        CSRK_TRY(dot_to(n, R(i), w.z, &S.rho[i], 1.0, part, s));
        // p_i = z_i + (rho_i / rho_{i-1}) p_{i-1}
        LIN3(n, P(i), ONE, w.z, (Cf{1.0, &S.rho[i], &S.rho[i - 1]}), P(i - 1), ONE, nullptr, nullptr, nullptr);
    }
    CSRK_LAUNCH(k_loss, 1, 1, 0, s, S, N, gamma);

    // ---------------- reverse
    CSRK_CUDA(cudaMemsetAsync(dL, 0, sizeof(double) * (size_t)L.nnz, s));
    CSRK_CUDA(cudaMemsetAsync(w.rbar, 0, sizeof(double) * (size_t)n, s));
    CSRK_CUDA(cudaMemsetAsync(w.pbar, 0, sizeof(double) * (size_t)n, s));
    for (int i = N; i >= 1; --i) {
        if (i < N) {
            // p_i = z_i + beta_i p_{i-1}:  betabar = pbar . p_{i-1}
            CSRK_TRY(dot_to(n, w.pbar, P(i - 1), S.betabar, 1.0, part, s));
            CSRK_LAUNCH(k_bwd_beta, 1, 1, 0, s, S, i);
            CSRK_TRY(applyM(R(i), w.z));                       // recompute u_i, z_i
            // zbar = pbar + rhobar_i r_i ;  rbar += cn_i r_i + rhobar_i z_i
            LIN3(n, w.zbar, ONE, w.pbar, (Cf{1.0, &S.rhobar[i], nullptr}), R(i), ONE, nullptr, nullptr, nullptr);
            LIN3(n, w.rbar, ONE, w.rbar, (Cf{1.0, &S.cn[i], nullptr}), R(i), (Cf{1.0, &S.rhobar[i], nullptr}), w.z,
                 nullptr, nullptr);
            CSRK_TRY(adjM(R(i), w.z, true));
        } else {
            LIN3(n, w.rbar, ONE, w.rbar, (Cf{1.0, &S.cn[i], nullptr}), R(i), ONE, nullptr, nullptr, nullptr);
        }
        // r_i = r_{i-1} - alpha_i q_i:  alphabar = -rbar . q_i ;  qbar = -alpha_i rbar + sbar p_{i-1}
        CSRK_TRY(dot_to(n, w.rbar, Q(i), S.alphabar, -1.0, part, s));
        CSRK_LAUNCH(k_bwd_alpha, 1, 1, 0, s, S, i);
        LIN3(n, w.qbar, (Cf{-1.0, &S.rho[i - 1], &S.s[i]}), w.rbar, (Cf{1.0, S.sbar, nullptr}), P(i - 1), ONE,
             nullptr, nullptr, nullptr);
        // pbar_{i-1} = beta_i pbar_i + sbar q_i + A^T qbar
        {
            Bump bw = sub();
            CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_T, A, Av, nullptr, nullptr, w.qbar, w.tmp, bw, s));
        }
        const Cf beta = i < N ? Cf{1.0, &S.rho[i], &S.rho[i - 1]} : Cf{0.0, nullptr, nullptr};
        LIN3(n, w.pbar, beta, w.pbar, (Cf{1.0, S.sbar, nullptr}), Q(i), ONE, w.tmp, nullptr, nullptr);
    }
    // p0 = z0, rho0 = r0.z0 (r0 = b):  zbar = pbar + rhobar_0 b
    LIN3(n, w.zbar, ONE, w.pbar, (Cf{1.0, &S.rhobar[0], nullptr}), b, ONE, nullptr, nullptr, nullptr);
    CSRK_TRY(applyM(b, w.z));                                  // recompute u_0, z_0
    CSRK_TRY(adjM(b, w.z, false));

    CSRK_CUDA(cudaMemcpyAsync(loss_host, S.loss, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (resid_host) {
        std::vector<double> nr2(N + 1);
        CSRK_CUDA(cudaMemcpyAsync(nr2.data(), S.nr2, sizeof(double) * (N + 1), cudaMemcpyDeviceToHost, s));
        CSRK_CUDA(cudaStreamSynchronize(s));
        for (int i = 1; i <= N; ++i) resid_host[i - 1] = std::sqrt(nr2[i]);
    }
    CSRK_CUDA(cudaStreamSynchronize(s));
    return CSRK_OK;
}

}  // namespace csrk
