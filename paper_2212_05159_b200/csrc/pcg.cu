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
#include <mutex>
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
    double *dpart;                                          // fused-dot CTA partials (cdiv(m, 256))
    csrk_pattern LT;                                        // precond = solve: L^T pattern + perm
    int64_t *LTperm;
    Scal S;
    void *sub;
    size_t sub_bytes;
};

static size_t spmv_ws_bytes(const csrk_pattern &M)
{
    size_t m = 0;
    const void *d = M.indptr;
    for (int op = 0; op < 2; ++op) {
        Bump f(nullptr, 0), g(nullptr, 0);
        spmv_fwd(CSRK_F64, (csrk_op)op, M, d, nullptr, nullptr, d, (void *)d, f, 0);
        spmv_bwd(CSRK_F64, (csrk_op)op, M, d, nullptr, nullptr, d, d, (void *)d, (void *)d, g, 0);
        m = f.used > m ? f.used : m;
        m = g.used > m ? g.used : m;
    }
    return m + 256;
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

// Vectors of length n_ext (extended layout of a row-sharded rank; n_ext = n on one GPU): the
// owned part is [off, off + m).  Saved per iteration: p_{i-1} (extended: the halo-gathered input of
// A p), r_i and q_i (owned).
static void carve_pcg(const csrk_pattern &A, const csrk_pattern &L, int N, int precond, PcgWs &w, Bump &ws)
{
    const int64_t m = A.nrows, ne = A.ncols > m ? A.ncols : m;
    w.pb = ws.take<double>((size_t)N * ne);
    w.rb = ws.take<double>((size_t)(N + 1) * m);
    w.qb = ws.take<double>((size_t)N * m);
    double **tv[] = {&w.u, &w.z, &w.rbar, &w.pbar, &w.zbar, &w.ubar, &w.qbar, &w.tmp};
    for (auto p : tv) *p = ws.take<double>(ne);
    w.dAt = ws.take<double>(L.nnz > 0 ? L.nnz : 1);
    w.part = ws.take<double>(kVecGrid);
    w.dpart = ws.take<double>((size_t)cdiv(m > 0 ? m : 1, 256));
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

// The whole step enqueued on `s` (no synchronisation; capturable when the comm is).
static int pcg_enqueue(const csrk_comm *comm, int64_t off, const csrk_pattern &A, const double *Av,
                       const csrk_pattern &L, const double *Lv, const double *b, int N, double gamma, int precond,
                       double *dL, PcgWs &w, cudaStream_t s)
{
    const int64_t m = A.nrows;                 // owned rows
    auto own = [&](double *v) { return v + off; };
    auto sub = [&]() { return Bump(w.sub, w.sub_bytes); };
    // exchanges (no-ops on one GPU)
    auto gather = [&](double *v) -> int { return comm ? comm->halo(comm->ctx, v, 0, (csrk_stream_t)s) : CSRK_OK; };
    auto reduce = [&](double *v) -> int { return comm ? comm->halo(comm->ctx, v, 1, (csrk_stream_t)s) : CSRK_OK; };
    auto allred = [&](double *v, int64_t c) -> int {
        return comm ? comm->allreduce_sum(comm->ctx, v, c, (csrk_stream_t)s) : CSRK_OK;
    };
    if (precond) {  // L^T (pattern + perm) once per call, for the transposed solves (one GPU only)
        Bump bw = sub();
        CSRK_TRY(transpose_impl(CSRK_F64, L, nullptr, const_cast<int64_t *>(w.LT.indptr),
                                const_cast<int32_t *>(w.LT.indices), nullptr, w.LTperm, bw, s));
    }
    // z = M r (owned r, owned z) with the intermediate u (extended) in w.u:
    //   M = L L^T: u = L^T r (op T: an extended partial, halo-reduced, then halo-gathered
    //   for the op-N product), z = L u;   precond = solve: u = L^{-1} r, z = L^{-T} u
    // rz (nullable): also *rz = r.z over the owned rows, fused into the last product (M = L L^T)
    auto applyM = [&](const double *r, double *z, double *rz = nullptr) -> int {
        if (!precond) {
            {
                Bump bw = sub();
                CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_T, L, Lv, nullptr, nullptr, r, w.u, bw, s));
            }
            CSRK_TRY(reduce(w.u));
            CSRK_TRY(gather(w.u));
            Bump bw = sub();
            const FusedDot fd{r, w.dpart, rz};
            return spmv_fwd(CSRK_F64, CSRK_OP_N, L, Lv, nullptr, nullptr, w.u, z, bw, s, 0, rz ? &fd : nullptr);
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
        double *rb_add = own(w.tmp);           // owned-length contribution to rbar
        if (!precond) {
            // z = L gather(u):  Lbar += zbar u^T (.) mask(L);  ubar = reduce(L^T zbar)
            // (the masked gradients are added into dL by the SpMV VJP kernels themselves)
            {
                Bump bw = sub();
                CSRK_TRY(spmv_bwd(CSRK_F64, CSRK_OP_N, L, Lv, nullptr, nullptr, w.u, w.zbar, dL, w.ubar, bw, s, 1));
            }
            CSRK_TRY(reduce(w.ubar));
            CSRK_TRY(gather(w.ubar));
            // u = reduce(L^T r):  Lbar += r ubar^T (.) mask(L);  rbar += L gather(ubar)
            {   // (rbar += L gather(ubar) straight into rbar: accumulate mode)
                Bump bw = sub();
                CSRK_TRY(spmv_bwd(CSRK_F64, CSRK_OP_T, L, Lv, nullptr, nullptr, r, w.ubar, dL,
                                  want_rbar ? w.rbar : nullptr, bw, s, 1, 1));
            }
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
                CSRK_TRY(sptrsv_bwd(CSRK_F64, L, Lv, &w.LT, w.LTperm, 0, 0, w.u, w.ubar, w.dAt, rb_add, bw, s));
            }
            LIN3(L.nnz, dL, ONE, dL, ONE, w.dAt, ONE, nullptr, nullptr, nullptr);
        }
        if (want_rbar && precond) LIN3(m, w.rbar, ONE, w.rbar, ONE, rb_add, ONE, nullptr, nullptr, nullptr);
        return CSRK_OK;
    };
    const Scal &S = w.S;
    double *part = w.part;
    const int64_t ne = A.ncols > m ? A.ncols : m;
    auto Pe = [&](int i) { return w.pb + (size_t)i * ne; };     // p_i extended, i = 0..N-1
    auto P = [&](int i) { return Pe(i) + off; };                // its owned part
    auto R = [&](int i) { return w.rb + (size_t)i * m; };       // r_i, i = 0..N (owned)
    auto Q = [&](int i) { return w.qb + (size_t)(i - 1) * m; }; // q_i, i = 1..N (owned)
    // dot over the owned rows, then summed over ranks
    auto gdot = [&](const double *x, const double *y, double *dst, double sign) -> int {
        CSRK_TRY(dot_to(m, x, y, dst, sign, part, s));
        return allred(dst, 1);
    };

    // ---------------- forward
    CSRK_TRY(gdot(b, b, S.bb, 1.0));
    LIN3(m, R(0), ONE, b, ONE, nullptr, ONE, nullptr, nullptr, nullptr);
    CSRK_TRY(applyM(b, P(0)));                                 // p0 = z0
    CSRK_TRY(gdot(b, P(0), &S.rho[0], 1.0));
    for (int i = 1; i <= N; ++i) {
        CSRK_TRY(gather(Pe(i - 1)));
        {   // q_i = A p_{i-1} with s_i = p_{i-1}.q_i fused into the product
            Bump bw = sub();
            const FusedDot fd{P(i - 1), w.dpart, &S.s[i]};
            CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_N, A, Av, nullptr, nullptr, Pe(i - 1), Q(i), bw, s, 0, &fd));
        }
        CSRK_TRY(allred(&S.s[i], 1));
        // r_i = r_{i-1} - (rho_{i-1}/s_i) q_i ; nr2_i = r_i.r_i (summed over ranks once, at the end)
        LIN3(m, R(i), ONE, R(i - 1), (Cf{-1.0, &S.rho[i - 1], &S.s[i]}), Q(i), ONE, nullptr, nullptr, part);
        CSRK_LAUNCH(k_finish, 1, kVecTPB, 0, s, (const double *)part, kVecGrid, &S.nr2[i], 1.0);
        if (i == N) break;                                     // rho_N, p_N do not reach the loss
        if (!precond) {
            CSRK_TRY(applyM(R(i), own(w.z), &S.rho[i]));        // rho_i = r_i.z_i fused into z = L u
            CSRK_TRY(allred(&S.rho[i], 1));
        } else {
            CSRK_TRY(applyM(R(i), own(w.z)));
            CSRK_TRY(gdot(R(i), own(w.z), &S.rho[i], 1.0));
        }
        // p_i = z_i + (rho_i / rho_{i-1}) p_{i-1}
        LIN3(m, P(i), ONE, own(w.z), (Cf{1.0, &S.rho[i], &S.rho[i - 1]}), P(i - 1), ONE, nullptr, nullptr, nullptr);
    }
    CSRK_TRY(allred(S.nr2 + 1, N));
    CSRK_LAUNCH(k_loss, 1, 1, 0, s, S, N, gamma);

    // ---------------- reverse
    CSRK_CUDA(cudaMemsetAsync(dL, 0, sizeof(double) * (size_t)L.nnz, s));
    CSRK_CUDA(cudaMemsetAsync(w.rbar, 0, sizeof(double) * (size_t)m, s));
    CSRK_CUDA(cudaMemsetAsync(w.pbar, 0, sizeof(double) * (size_t)m, s));
    for (int i = N; i >= 1; --i) {
        if (i < N) {
            // p_i = z_i + beta_i p_{i-1}:  betabar = pbar . p_{i-1}
            CSRK_TRY(gdot(w.pbar, P(i - 1), S.betabar, 1.0));
            CSRK_LAUNCH(k_bwd_beta, 1, 1, 0, s, S, i);
            CSRK_TRY(applyM(R(i), own(w.z)));                  // recompute u_i, z_i
            // zbar = pbar + rhobar_i r_i ;  rbar += cn_i r_i + rhobar_i z_i
            LIN3(m, w.zbar, ONE, w.pbar, (Cf{1.0, &S.rhobar[i], nullptr}), R(i), ONE, nullptr, nullptr, nullptr);
            LIN3(m, w.rbar, ONE, w.rbar, (Cf{1.0, &S.cn[i], nullptr}), R(i), (Cf{1.0, &S.rhobar[i], nullptr}),
                 own(w.z), nullptr, nullptr);
            CSRK_TRY(adjM(R(i), own(w.z), true));
        } else {
            LIN3(m, w.rbar, ONE, w.rbar, (Cf{1.0, &S.cn[i], nullptr}), R(i), ONE, nullptr, nullptr, nullptr);
        }
        // r_i = r_{i-1} - alpha_i q_i:  alphabar = -rbar . q_i ;  qbar = -alpha_i rbar + sbar p_{i-1}
        CSRK_TRY(gdot(w.rbar, Q(i), S.alphabar, -1.0));
        CSRK_LAUNCH(k_bwd_alpha, 1, 1, 0, s, S, i);
        LIN3(m, w.qbar, (Cf{-1.0, &S.rho[i - 1], &S.s[i]}), w.rbar, (Cf{1.0, S.sbar, nullptr}), P(i - 1), ONE,
             nullptr, nullptr, nullptr);
        // q_i = A gather(p_{i-1}):  pbar_{i-1} = beta_i pbar_i + sbar q_i + reduce(A^T qbar)
        const Cf beta = i < N ? Cf{1.0, &S.rho[i], &S.rho[i - 1]} : Cf{0.0, nullptr, nullptr};
        if (!comm) {
            // one GPU: pbar = beta pbar + sbar q first, then A^T qbar scattered straight into it
            // (no zeroed scratch, no third pass)
            LIN3(m, w.pbar, beta, w.pbar, (Cf{1.0, S.sbar, nullptr}), Q(i), ONE, nullptr, nullptr, nullptr);
            Bump bw = sub();
            CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_T, A, Av, nullptr, nullptr, w.qbar, w.pbar, bw, s, 1));
        } else {
            {
                Bump bw = sub();
                CSRK_TRY(spmv_fwd(CSRK_F64, CSRK_OP_T, A, Av, nullptr, nullptr, w.qbar, w.tmp, bw, s));
            }
            CSRK_TRY(reduce(w.tmp));
            LIN3(m, w.pbar, beta, w.pbar, (Cf{1.0, S.sbar, nullptr}), Q(i), ONE, own(w.tmp), nullptr, nullptr);
        }
    }
    // p0 = z0, rho0 = r0.z0 (r0 = b):  zbar = pbar + rhobar_0 b
    LIN3(m, w.zbar, ONE, w.pbar, (Cf{1.0, &S.rhobar[0], nullptr}), b, ONE, nullptr, nullptr, nullptr);
    CSRK_TRY(applyM(b, own(w.z)));                             // recompute u_0, z_0
    CSRK_TRY(adjM(b, own(w.z), false));
    return CSRK_OK;
}

// One CUDA graph per argument set (stream capture of pcg_enqueue), replayed on later calls.
struct PcgGraphKey {
    const void *ptr[10];
    int64_t sz[6];
    int N;
    double gamma;
    bool operator==(const PcgGraphKey &o) const
    {
        for (int i = 0; i < 10; ++i)
            if (ptr[i] != o.ptr[i]) return false;
        for (int i = 0; i < 6; ++i)
            if (sz[i] != o.sz[i]) return false;
        return N == o.N && gamma == o.gamma;
    }
};
struct PcgGraph {
    PcgGraphKey key;
    int dev;
    cudaGraphExec_t exec;
    uint64_t kernels;   // csrk kernels captured (counted once per replay by csrk_launch_count)
};
static std::mutex g_graph_mu;
static std::vector<PcgGraph> g_graphs;

static cudaStream_t capture_stream(int dev)
{
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    std::lock_guard<std::mutex> g(mu);
    if (!streams[dev & 63] && cudaStreamCreateWithFlags(&streams[dev & 63], cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    return streams[dev & 63];
}

int pcg_loss_grad(const csrk_comm *comm, int64_t off, const csrk_pattern &A, const double *Av, const csrk_pattern &L,
                  const double *Lv, const double *b, int N, double gamma, int precond, double *loss_host,
                  double *resid_host, double *dL, Bump &ws, cudaStream_t s)
{
    PcgWs w{};
    carve_pcg(A, L, N, precond, w, ws);
    if (ws.sizing()) return CSRK_OK;
    const bool graph = knob("PCG_GRAPH", 1) && (!comm || comm->capturable);
    if (!graph) {
        CSRK_TRY(pcg_enqueue(comm, off, A, Av, L, Lv, b, N, gamma, precond, dL, w, s));
    } else {
        PcgGraphKey key{{A.indptr, A.indices, Av, L.indptr, L.indices, Lv, b, dL, ws.base, comm ? comm->ctx : nullptr},
                        {A.nrows, A.ncols, A.nnz, L.nnz, off, (int64_t)ws.cap + precond},
                        N, gamma};
        const int dev = DevOnce::dev();
        cudaGraphExec_t exec = nullptr;
        {
            std::lock_guard<std::mutex> g(g_graph_mu);
            for (auto &e : g_graphs)
                if (e.dev == dev && e.key == key) exec = e.exec;
        }
        uint64_t nk = 0;
        {
            std::lock_guard<std::mutex> g(g_graph_mu);
            for (auto &e : g_graphs)
                if (e.dev == dev && e.key == key) nk = e.kernels;
        }
        if (exec) {
            g_launches.fetch_add(nk, std::memory_order_relaxed);   // the graph's kernels run again
        } else {
            // capture on a private non-blocking stream (the caller's may be the legacy default
            // stream, which cannot be captured); the graph is then launched on the caller's stream
            cudaStream_t cs = capture_stream(dev);
            if (!cs) return CSRK_ERR_CUDA;
            cudaGraph_t gr = nullptr;
            const uint64_t before = g_launches.load(std::memory_order_relaxed);
            CSRK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            const int st = pcg_enqueue(comm, off, A, Av, L, Lv, b, N, gamma, precond, dL, w, cs);
            const cudaError_t ce = cudaStreamEndCapture(cs, &gr);
            if (st != CSRK_OK || ce != cudaSuccess) {
                if (gr) cudaGraphDestroy(gr);
                (void)cudaGetLastError();
                return st != CSRK_OK ? st : CSRK_ERR_CUDA;
            }
            const cudaError_t ie = cudaGraphInstantiate(&exec, gr, 0);
            cudaGraphDestroy(gr);
            if (ie != cudaSuccess) return CSRK_ERR_CUDA;
            std::lock_guard<std::mutex> g(g_graph_mu);
            if (g_graphs.size() >= 8) {     // a handful of argument sets in flight: drop the oldest
                cudaGraphExecDestroy(g_graphs.front().exec);
                g_graphs.erase(g_graphs.begin());
            }
            g_graphs.push_back(PcgGraph{key, dev, exec, g_launches.load(std::memory_order_relaxed) - before});
        }
        CSRK_CUDA(cudaGraphLaunch(exec, s));
    }
    const Scal &S = w.S;
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
