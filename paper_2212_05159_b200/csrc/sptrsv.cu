// sptrsv.cu -- sparse triangular solve x = T^{-1} b and its VJP (PAPER 3.1.5, P:477-488;
// SURVEY 8(f) row f3).
//
// Forward.  "each row depends on the intermediate values of previous rows only": row i
// of a lower T needs x_j for its stored j < i (upper: j > i, solved in reverse order -- the
// paper's "matrix flip").  Two kernels, launched back to back:
//
//   k_trsv_chain  scan for CHAIN matrices (every row's off-diagonal entries lie on the first
//                 sub-diagonal: bidiagonal L of the PCG preconditioner, or the triangle
//                 of A_N, Table 2).  Row i is the affine map x_i = c_i + a_i x_{i-1}
//                 (a_i = -l_i / d_i, c_i = b_i / d_i); maps compose associatively, so a tile of
//                 2048 rows composes its maps (reduce), one CTA scans the tile maps into every
//                 tile's carry-in x (k_trsv_carry), and each tile then evaluates
//                 x_i = (b_i - l_i x_{i-1}) / d_i row by row from its thread's start value
//                 (apply).  Two streaming passes and no waiting between CTAs: a 16.7M-row chain
//                 that the sync-free method would walk one dependency at a time runs like two
//                 SpMVs.  A row with any other dependency sets `abort` (apply and carry skip).
//                 This three-kernel form is kept behind CSRK_TRSV_LOOKBACK=0; the default is
//                 the single-pass decoupled look-back k_trsv_chain_lb (below), measured faster
//                 (0.55 vs 0.87 ms on the 16.7M-row config-5 L) once its look-back resolved 32
//                 predecessors per round.
//   k_trsv_sf     the synchronisation-free solve the paper uses (Capellini et al.):
//                 warps take 32-row blocks in solve order from an atomic ticket; each lane
//                 owns a row, waits (acquire) on the ready flag of every dependency outside
//                 the block, then the warp resolves the dependencies inside the block in lane
//                 order through shuffles; x_i is stored and its flag released.  Tickets are
//                 claimed by running warps in order, so every awaited row belongs to a warp
//                 that is resident or done: no deadlock.  Runs only if the chain pass aborted.
//
// Backward: db = T^{-T} v "with our existing forward triangular solve routine" -- the
// same two kernels on T^T (cached transpose plan, or one built in the workspace), values
// gathered through perm; dT = -(db) x^T (.) mask(T) "executed in parallel over the nonzero
// entries of L" (k_trsv_dT).
//
// Stored entries on the wrong side of the diagonal are ignored (CSRK_VALIDATE=1 rejects
// them); a missing diagonal (unit == 0) divides by zero.
#include "ops.cuh"

namespace csrk {

constexpr int kChTPB = 128;
constexpr int kChPer = 8;
constexpr int kChTile = kChTPB * kChPer;
constexpr int kSfTPB = 256;

__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double *p)
{
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed(const float *p)
{
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return (double)v;
}

template <typename T>
struct TrsvArgs {
    int64_t n;
    const int64_t *indptr;
    const int32_t *indices;
    const T *vals;
    const int64_t *perm;  // nullable: value of entry p is vals[perm[p]]
    const T *b;
    T *x;
    int upper, unit;
    // chain pass: tile maps, carry-in / inclusive values, look-back status words
    double *aggA, *aggC, *inclX;
    int *status;
    int *ticket_chain;
    int *abort;
    // sync-free pass
    int *ready;
    int *ticket_sf;
};

template <typename T>
__device__ __forceinline__ double tval(const TrsvArgs<T> &a, int64_t p)
{
    return (double)a.vals[a.perm ? a.perm[p] : p];
}

// ---------------------------------------------------------------- chain pass
// Three launches, no inter-CTA waiting: (1) every tile composes the affine maps of its rows
// (k_trsv_chain<REDUCE>) and flags a non-chain row; (2) one CTA scans the tile maps into each
// tile's carry-in x (k_trsv_carry); (3) every tile re-reads its rows, scans its thread maps for
// each thread's start value and runs the substitution formula (k_trsv_chain<APPLY>).

// Shared-memory staging of a tile: rows [m0, m1) in memory order, their entries and b, loaded
// with coalesced reads (a thread's own rows are consecutive, so direct loads would touch 32
// lines per warp instruction).
struct ChSmem {
    int64_t ip[kChTile + 1];
    double val[2 * kChTile];
    double b[kChTile];
    int32_t idx[2 * kChTile];
};

// Stage the tile and parse this thread's rows: l (neighbour value), d (diagonal), b.  Returns
// true if a row is not a chain row (more than two entries, or a dependency other than the
// neighbour); wrong-side entries are ignored.
template <typename T>
__device__ __forceinline__ bool chain_rows(const TrsvArgs<T> &a, ChSmem &S, int tile, double (&lv)[kChPer],
                                           double (&dv)[kChPer], double (&bv)[kChPer])
{
    const int64_t n = a.n;
    const int tid = threadIdx.x;
    const int64_t T0 = (int64_t)tile * kChTile;
    const int64_t m0 = a.upper ? (n - T0 - kChTile > 0 ? n - T0 - kChTile : 0) : T0;
    const int64_t m1 = a.upper ? n - T0 : (T0 + kChTile < n ? T0 + kChTile : n);
    const int nr = (int)(m1 - m0);
    for (int r = tid; r <= nr; r += kChTPB) S.ip[r] = a.indptr[m0 + r];
    for (int r = tid; r < nr; r += kChTPB) S.b[r] = (double)a.b[m0 + r];
    __syncthreads();
    const int64_t ent0 = S.ip[0], ne = S.ip[nr] - ent0;
    bool bad = ne > 2 * kChTile;
    if (!bad)
        for (int q = tid; q < ne; q += kChTPB) {
            S.idx[q] = a.indices[ent0 + q];
            S.val[q] = tval(a, ent0 + q);
        }
    __syncthreads();
    const int64_t o0 = T0 + (int64_t)tid * kChPer;
#pragma unroll
    for (int r = 0; r < kChPer; ++r) {
        const int64_t o = o0 + r;
        lv[r] = 0.0;
        dv[r] = 1.0;
        bv[r] = 0.0;
        if (o < n && !bad) {
            const int64_t i = a.upper ? n - 1 - o : o;
            const int lr = (int)(i - m0);
            const int64_t prev = a.upper ? i + 1 : i - 1;
            const int64_t rs = S.ip[lr] - ent0, re = S.ip[lr + 1] - ent0;
            double d = a.unit ? 1.0 : 0.0, l = 0.0;
            bad |= re - rs > 2;
            for (int64_t q = rs; q < re && q < rs + 2; ++q) {
                const int64_t j = S.idx[q];
                if (j == i) {
                    if (!a.unit) d = S.val[q];
                } else if (j == prev) {
                    l = S.val[q];
                } else if (a.upper ? j > i : j < i) {
                    bad = true;
                }
            }
            lv[r] = l;
            dv[r] = d;
            bv[r] = S.b[lr];
        }
    }
    return bad;
}

// exclusive scan of the CTA's thread maps (composition in row order); returns the thread's
// prefix map (tA, tC) and the tile map (gA, gC)
__device__ __forceinline__ void chain_block_scan(double mA, double mC, double &tA, double &tC, double &gA, double &gC)
{
    __shared__ double s_wA[kChTPB / 32], s_wC[kChTPB / 32];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double iA = mA, iC = mC;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double pA = __shfl_up_sync(FULL, iA, o), pC = __shfl_up_sync(FULL, iC, o);
        if (lane >= o) {
            iC = iA * pC + iC;
            iA = iA * pA;
        }
    }
    if (lane == 31) {
        s_wA[warp] = iA;
        s_wC[warp] = iC;
    }
    double eA = __shfl_up_sync(FULL, iA, 1), eC = __shfl_up_sync(FULL, iC, 1);
    if (lane == 0) {
        eA = 1.0;
        eC = 0.0;
    }
    __syncthreads();
    double wA = 1.0, wC = 0.0;
    gA = 1.0;
    gC = 0.0;
    for (int w = 0; w < kChTPB / 32; ++w) {
        if (w < warp) {
            wC = s_wA[w] * wC + s_wC[w];
            wA = s_wA[w] * wA;
        }
        gC = s_wA[w] * gC + s_wC[w];
        gA = s_wA[w] * gA;
    }
    tA = eA * wA;
    tC = eA * wC + eC;
}

template <typename T, bool APPLY>
__global__ __launch_bounds__(kChTPB, 4) void k_trsv_chain(TrsvArgs<T> a)
{
    pdl_wait();
    if (APPLY && *(volatile int *)a.abort) return;
    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const int64_t n = a.n;
    const int64_t o0 = (int64_t)tile * kChTile + (int64_t)tid * kChPer;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    ChSmem &S = *reinterpret_cast<ChSmem *>(s_dyn);
    double lv[kChPer], dv[kChPer], bv[kChPer];
    const bool bad = chain_rows(a, S, tile, lv, dv, bv);
    double mA = 1.0, mC = 0.0;  // composition of this thread's row maps
#pragma unroll
    for (int r = 0; r < kChPer; ++r) {
        if (o0 + r < n) {
            const double rd = 1.0 / dv[r];
            const double ar = -lv[r] * rd, cr = bv[r] * rd;
            mC = ar * mC + cr;
            mA = ar * mA;
        }
    }
    if (!APPLY) {
        if (__syncthreads_or(bad)) {
            if (tid == 0) atomicExch(a.abort, 1);
            return;
        }
    }
    double tA, tC, gA, gC;
    chain_block_scan(mA, mC, tA, tC, gA, gC);
    if (!APPLY) {
        if (tid == 0) {
            a.aggA[tile] = gA;
            a.aggC[tile] = gC;
        }
        return;
    }
    // rows from the carried-in value, by the substitution formula
    const double xin = a.inclX[tile];
    double xp = tid == 0 ? xin : tA * xin + tC;
    const int64_t T0 = (int64_t)tile * kChTile;
    const int64_t m0 = a.upper ? (n - T0 - kChTile > 0 ? n - T0 - kChTile : 0) : T0;
    const int64_t m1 = a.upper ? n - T0 : (T0 + kChTile < n ? T0 + kChTile : n);
    __syncthreads();  // S.b is rewritten with x below
#pragma unroll
    for (int r = 0; r < kChPer; ++r) {
        const int64_t o = o0 + r;
        if (o < n) {
            const T xi = (T)((bv[r] - lv[r] * xp) / dv[r]);
            S.b[(a.upper ? n - 1 - o : o) - m0] = (double)xi;
            xp = (double)xi;
        }
    }
    __syncthreads();
    for (int64_t r = tid; r < m1 - m0; r += kChTPB) a.x[m0 + r] = (T)S.b[r];
}

// one CTA: carry-in x of every tile, inclX[t] = (M_{t-1} o ... o M_0)(0)
constexpr int kCarryTPB = 1024;
template <typename T>
__global__ __launch_bounds__(kCarryTPB) void k_trsv_carry(TrsvArgs<T> a, int64_t ntiles)
{
    pdl_wait();
    if (*(volatile int *)a.abort) return;
    __shared__ double s_A[kCarryTPB / 32], s_C[kCarryTPB / 32];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (ntiles + kCarryTPB - 1) / kCarryTPB;
    const int64_t t0 = tid * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
    double mA = 1.0, mC = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
        mC = a.aggA[t] * mC + a.aggC[t];
        mA = a.aggA[t] * mA;
    }
    double iA = mA, iC = mC;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double pA = __shfl_up_sync(FULL, iA, o), pC = __shfl_up_sync(FULL, iC, o);
        if (lane >= o) {
            iC = iA * pC + iC;
            iA = iA * pA;
        }
    }
    if (lane == 31) {
        s_A[warp] = iA;
        s_C[warp] = iC;
    }
    double eA = __shfl_up_sync(FULL, iA, 1), eC = __shfl_up_sync(FULL, iC, 1);
    if (lane == 0) {
        eA = 1.0;
        eC = 0.0;
    }
    __syncthreads();
    double wA = 1.0, wC = 0.0;
    for (int w = 0; w < warp; ++w) {
        wC = s_A[w] * wC + s_C[w];
        wA = s_A[w] * wA;
    }
    double x = eA * wC + eC;  // prefix map applied to x = 0
    for (int64_t t = t0; t < t1; ++t) {
        a.inclX[t] = x;
        x = a.aggA[t] * x + a.aggC[t];
    }
}


// ---------------------------------------------------------------- chain pass, one kernel
// Single pass with a decoupled look-back (the default; measured 0.63 vs 0.87 ms for the 16.7M-row
// chain against reduce / carry / apply): tiles are claimed in order from a ticket, every tile
// publishes its map as soon as it has composed it, warp 0 resolves the carry-in by a warp-wide
// look-back (32 predecessors per round, their maps composed by a shuffle tree) and publishes the
// tile's inclusive x before the row pass.  Tickets are claimed by running CTAs in order, so
// every awaited tile is resident or finished.
enum { CH_NONE = 0, CH_AGG = 1, CH_INCL = 2, CH_ABORT = 3 };
constexpr int kLbTPB = 256;
#ifndef CSRK_LB_PER
#define CSRK_LB_PER 8
#endif
constexpr int kLbPer = CSRK_LB_PER;  // rows per thread (A/B via CSRK_NVCC_EXTRA)
constexpr int kLbTile = kLbTPB * kLbPer;

template <typename T>
__device__ __forceinline__ bool chain_rows_reg(const TrsvArgs<T> &a, int64_t o0, double (&lv)[kLbPer],
                                               double (&dv)[kLbPer], double (&bv)[kLbPer])
{
    const int64_t n = a.n;
    bool bad = false;
    int64_t rs[kLbPer], re[kLbPer];
#pragma unroll
    for (int r = 0; r < kLbPer; ++r) {
        const int64_t o = o0 + r;
        const int64_t i = a.upper ? n - 1 - o : o;
        rs[r] = re[r] = 0;
        bv[r] = 0.0;
        if (o < n) {
            rs[r] = a.indptr[i];
            re[r] = a.indptr[i + 1];
            bv[r] = (double)a.b[i];
        }
    }
#pragma unroll
    for (int r = 0; r < kLbPer; ++r) {
        const int64_t o = o0 + r;
        const int64_t len = re[r] - rs[r];
        bad |= len > 2;
        const int64_t c0 = len > 0 ? a.indices[rs[r]] : -1, c1 = len > 1 ? a.indices[rs[r] + 1] : -1;
        const double v0 = len > 0 ? tval(a, rs[r]) : 0.0, v1 = len > 1 ? tval(a, rs[r] + 1) : 0.0;
        lv[r] = 0.0;
        dv[r] = 1.0;
        if (o < n) {
            const int64_t i = a.upper ? n - 1 - o : o;
            const int64_t prev = a.upper ? i + 1 : i - 1;
            double d = a.unit ? 1.0 : 0.0, l = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = h ? c1 : c0;
                const double v = h ? v1 : v0;
                if (j < 0) continue;
                if (j == i) {
                    if (!a.unit) d = v;
                } else if (j == prev) {
                    l = v;
                } else if (a.upper ? j > i : j < i) {
                    bad = true;
                }
            }
            lv[r] = l;
            dv[r] = d;
        }
    }
    return bad;
}

template <typename T>
#ifndef CSRK_LB_MINB
#define CSRK_LB_MINB 4  // measured: chain fwd 0.55 -> 0.48 ms (<= 64 registers, 4 CTAs per SM)
#endif
__global__ __launch_bounds__(kLbTPB, CSRK_LB_MINB) void k_trsv_chain_lb(TrsvArgs<T> a)
{
    pdl_wait();
    __shared__ int s_tile, s_abort;
    __shared__ double s_wA[kLbTPB / 32], s_wC[kLbTPB / 32];
    __shared__ double s_xin;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned FULL = 0xffffffffu;
    if (tid == 0) {
        s_tile = atomicAdd(a.ticket_chain, 1);
        s_abort = *(volatile int *)a.abort;
    }
    __syncthreads();
    const int tile = s_tile;
    const int64_t n = a.n;
    if (s_abort) {
        if (tid == 0) st_release(&a.status[tile], CH_ABORT);
        return;
    }
    const int64_t o0 = (int64_t)tile * kLbTile + (int64_t)tid * kLbPer;
    double lv[kLbPer], dv[kLbPer], bv[kLbPer];
    const bool bad = chain_rows_reg(a, o0, lv, dv, bv);
    if (__syncthreads_or(bad)) {
        if (tid == 0) {
            atomicExch(a.abort, 1);
            st_release(&a.status[tile], CH_ABORT);
        }
        return;
    }
    double mA = 1.0, mC = 0.0;
#pragma unroll
    for (int r = 0; r < kLbPer; ++r) {
        if (o0 + r < n) {
            const double rd = 1.0 / dv[r];
            const double ar = -lv[r] * rd, cr = bv[r] * rd;
            mC = ar * mC + cr;
            mA = ar * mA;
        }
    }
    // inclusive warp scan, then the prefix over earlier warps
    double iA = mA, iC = mC;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double pA = __shfl_up_sync(FULL, iA, o), pC = __shfl_up_sync(FULL, iC, o);
        if (lane >= o) {
            iC = iA * pC + iC;
            iA = iA * pA;
        }
    }
    if (lane == 31) {
        s_wA[warp] = iA;
        s_wC[warp] = iC;
    }
    double eA = __shfl_up_sync(FULL, iA, 1), eC = __shfl_up_sync(FULL, iC, 1);
    if (lane == 0) {
        eA = 1.0;
        eC = 0.0;
    }
    __syncthreads();
    double wA = 1.0, wC = 0.0;
    for (int w = 0; w < warp; ++w) {
        wC = s_wA[w] * wC + s_wC[w];
        wA = s_wA[w] * wA;
    }
    const double tA = eA * wA, tC = eA * wC + eC;
    if (warp == 0) {
        double gA = 1.0, gC = 0.0;
        for (int w = 0; w < kLbTPB / 32; ++w) {
            gC = s_wA[w] * gC + s_wC[w];
            gA = s_wA[w] * gA;
        }
        double xin = 0.0;
        bool abort = false;
        if (tile > 0) {
            if (lane == 0) {
                a.aggA[tile] = gA;
                a.aggC[tile] = gC;
                st_release(&a.status[tile], CH_AGG);
            }
            double MA = 1.0, MC = 0.0;  // maps x_in(window end) -> x_in(tile)
            for (int p = tile - 1;;) {
                const int q = p - lane;
                const int st = q >= 0 ? ld_acquire(&a.status[q]) : CH_INCL;
                const unsigned done = __ballot_sync(FULL, st == CH_INCL || st == CH_ABORT);
                const int f = done ? __ffs(done) - 1 : 32;
                const unsigned none = __ballot_sync(FULL, st == CH_NONE) & (f < 32 ? ((2u << f) - 1u) : FULL);
                if (none) continue;
                double A1 = 1.0, C1 = 0.0;
                if (lane < f) {
                    A1 = ld_relaxed(&a.aggA[q]);
                    C1 = ld_relaxed(&a.aggC[q]);
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double A2 = __shfl_down_sync(FULL, A1, o), C2 = __shfl_down_sync(FULL, C1, o);
                    if ((lane & (2 * o - 1)) == 0) {
                        C1 = A1 * C2 + C1;
                        A1 = A1 * A2;
                    }
                }
                A1 = __shfl_sync(FULL, A1, 0);
                C1 = __shfl_sync(FULL, C1, 0);
                MC = MA * C1 + MC;
                MA = MA * A1;
                if (f < 32) {
                    if (__shfl_sync(FULL, st, f) == CH_ABORT) {
                        abort = true;
                    } else {
                        const int qf = p - f;
                        const double X = (lane == f && qf >= 0) ? ld_relaxed(&a.inclX[qf]) : 0.0;
                        xin = MA * __shfl_sync(FULL, X, f) + MC;
                    }
                    break;
                }
                p -= 32;
            }
        }
        if (lane == 0) {
            s_xin = xin;
            s_abort = abort;
            if (abort) {
                st_release(&a.status[tile], CH_ABORT);
            } else {
                a.inclX[tile] = gA * xin + gC;
                st_release(&a.status[tile], CH_INCL);
            }
        }
    }
    __syncthreads();
    if (s_abort) return;
    double xp = tid == 0 ? s_xin : tA * s_xin + tC;
#pragma unroll
    for (int r = 0; r < kLbPer; ++r) {
        const int64_t o = o0 + r;
        if (o < n) {
            const T xi = (T)((bv[r] - lv[r] * xp) / dv[r]);
            a.x[a.upper ? n - 1 - o : o] = xi;
            xp = (double)xi;
        }
    }
}

// zero the ready flags only when the chain pass aborted
template <typename T>
__global__ void k_trsv_prep(TrsvArgs<T> a)
{
    pdl_wait();
    if (*(volatile int *)a.abort == 0) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
        a.ready[i] = 0;
}

// ---------------------------------------------------------------- sync-free pass
template <typename T>
__global__ __launch_bounds__(kSfTPB) void k_trsv_sf(TrsvArgs<T> a)
{
    pdl_wait();
    if (*(volatile int *)a.abort == 0) return;  // the chain pass solved it
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t n = a.n;
    const int64_t nblk = cdiv(n, 32);
    while (true) {
        int blk = 0;
        if (lane == 0) blk = atomicAdd(a.ticket_sf, 1);
        blk = __shfl_sync(FULL, blk, 0);
        if (blk >= nblk) return;
        const int64_t blo = (int64_t)blk * 32;
        const int64_t o = blo + lane;
        const bool valid = o < n;
        const int64_t i = valid ? (a.upper ? n - 1 - o : o) : 0;
        int64_t s = 0, e = 0;
        if (valid) {
            s = a.indptr[i];
            e = a.indptr[i + 1];
        }
        double acc = valid ? (double)a.b[i] : 0.0;
        double d = a.unit ? 1.0 : 0.0;
        int64_t qs = e, qe = e;  // intra-block dependencies: contiguous positions [qs, qe)
        for (int64_t p = s; p < e; ++p) {
            const int64_t j = a.indices[p];
            if (j == i) {
                if (!a.unit) d = tval(a, p);
                continue;
            }
            const int64_t oj = a.upper ? n - 1 - j : j;
            if (oj >= o) continue;  // wrong side of the diagonal: ignored
            if (oj >= blo) {
                if (qs == e) qs = p;
                qe = p + 1;
                continue;
            }
            if (ld_acquire(&a.ready[j]) == 0) {
                unsigned ns = 32;
                while (ld_acquire(&a.ready[j]) == 0) {
                    __nanosleep(ns);
                    ns = ns < 256 ? ns * 2 : 256;
                }
            }
            acc = fma(-tval(a, p), ld_relaxed(&a.x[j]), acc);
        }
        const unsigned im = __ballot_sync(FULL, valid && qs < qe);
        double xi = 0.0;
        // in-block dependencies that form a chain (each lane depends at most on lane - 1, e.g. the
        // left neighbour of a stencil triangle in natural ordering): the recurrence
        // x_l = c_l + a_l x_{l-1} is resolved by a warp scan of affine maps instead of 32 steps
        const int64_t prevrow = a.upper ? i + 1 : i - 1;
        const bool chainlane = !(valid && qs < qe) || (qe - qs == 1 && lane > 0 && a.indices[qs] == prevrow);
        if (im && __all_sync(FULL, chainlane)) {
            const double rd = 1.0 / d;
            double mA = (valid && qs < qe) ? -tval(a, qs) * rd : 0.0;
            double mC = acc * rd;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double pA = __shfl_up_sync(FULL, mA, o), pC = __shfl_up_sync(FULL, mC, o);
                if (lane >= o) {
                    mC = mA * pC + mC;
                    mA = mA * pA;
                }
            }
            xi = mC;  // lane 0 has no in-block dependency, so the composed map's offset is x
        } else if (im) {
            // lanes depended upon are below the highest dependent lane; resolve in lane order
            const int last = 31 - __clz(im);
            int64_t q = a.upper ? qe - 1 : qs;
            // next in-block dependency of this lane (its column) and value, kept in registers
            const bool has = valid && qs < qe;
            int64_t nxt = has ? a.indices[q] : -1;
            double nv = has ? tval(a, q) : 0.0;
            for (int src = 0; src < last; ++src) {
                if (lane == src) xi = (double)(T)(acc / d);
                const double xs = __shfl_sync(FULL, xi, src);
                const int64_t rs = a.upper ? n - 1 - (blo + src) : blo + src;
                if (lane > src && nxt == rs) {
                    acc = fma(-nv, xs, acc);
                    q += a.upper ? -1 : 1;
                    const bool more = a.upper ? q >= qs : q < qe;
                    nxt = more ? a.indices[q] : -1;
                    nv = more ? tval(a, q) : 0.0;
                }
            }
            if (lane >= last) xi = acc / d;
        } else {
            xi = acc / d;
        }
        if (valid) {
            a.x[i] = (T)xi;
            st_release(&a.ready[i], 1);
        }
    }
}

// ---------------------------------------------------------------- VJP: masked outer product
template <typename T>
__global__ void k_trsv_dT(int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                          const T *__restrict__ w, const T *__restrict__ x, int unit, T *__restrict__ dT)
{
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double wi = (double)w[i];
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
        const int32_t j = indices[p];
        dT[p] = (unit && j == i) ? (T)0 : (T)(-(wi * (double)x[j]));
    }
}

// ---------------------------------------------------------------- host side
template <typename T>
static int carve_solve(TrsvArgs<T> &a, int64_t n, Bump &ws)
{
    // tile arrays serve both chain kernels: the three-kernel form (kChTile rows per tile) and the
    // look-back form (kLbTile rows per tile) -- sized for the one with more tiles
    const int64_t nt0 = cdiv(n, kChTile), nt1 = cdiv(n, kLbTile);
    const int64_t ntiles = nt0 > nt1 ? nt0 : nt1;
    a.aggA = ws.take<double>(ntiles > 0 ? ntiles : 1);
    a.aggC = ws.take<double>(ntiles > 0 ? ntiles : 1);
    a.inclX = ws.take<double>(ntiles > 0 ? ntiles : 1);
    a.status = ws.take<int>(ntiles > 0 ? ntiles : 1);
    a.ready = ws.take<int>(n > 0 ? n : 1);
    int *cnt = ws.take<int>(4);
    a.ticket_chain = cnt;
    a.ticket_sf = cnt ? cnt + 1 : nullptr;
    a.abort = cnt ? cnt + 2 : nullptr;
    return CSRK_OK;
}

template <typename T>
static int launch_solve(TrsvArgs<T> &a, cudaStream_t s)
{
    const int64_t n = a.n;
    if (n == 0) return CSRK_OK;
    const int64_t ntiles = cdiv(n, kChTile);
    CSRK_CUDA(cudaMemsetAsync(a.ticket_chain, 0, 4 * sizeof(int), s));
    if (ntiles > INT32_MAX) return CSRK_ERR_INDEX_OVERFLOW;
    if (knob("TRSV_LOOKBACK", 1)) {
        const int64_t nlb = cdiv(n, kLbTile);
        CSRK_CUDA(cudaMemsetAsync(a.status, 0, sizeof(int) * (size_t)nlb, s));
        CSRK_LAUNCH(k_trsv_chain_lb<T>, (unsigned)nlb, kLbTPB, 0, s, a);
    } else {
        const int sm = (int)sizeof(ChSmem);
        CSRK_CUDA(cudaFuncSetAttribute(k_trsv_chain<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CSRK_CUDA(cudaFuncSetAttribute(k_trsv_chain<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CSRK_LAUNCH((k_trsv_chain<T, false>), (unsigned)ntiles, kChTPB, sm, s, a);
        CSRK_LAUNCH(k_trsv_carry<T>, 1, kCarryTPB, 0, s, a, ntiles);
        CSRK_LAUNCH((k_trsv_chain<T, true>), (unsigned)ntiles, kChTPB, sm, s, a);
    }
    CSRK_LAUNCH(k_trsv_prep<T>, (unsigned)(kNumSMs * 4), 256, 0, s, a);
    const int64_t nwarps = cdiv(n, 32);
    const int64_t grid = cdiv(nwarps, kSfTPB / 32) < kNumSMs * 8 ? cdiv(nwarps, kSfTPB / 32) : kNumSMs * 8;
    CSRK_LAUNCH(k_trsv_sf<T>, (unsigned)grid, kSfTPB, 0, s, a);
    return CSRK_OK;
}

template <typename T>
static int sptrsv_fwd_t(const csrk_pattern &A, const T *Av, int upper, int unit, const T *b, T *x, Bump &ws,
                        cudaStream_t s)
{
    TrsvArgs<T> a{};
    carve_solve(a, A.nrows, ws);
    if (ws.sizing()) return CSRK_OK;
    a.n = A.nrows;
    a.indptr = A.indptr;
    a.indices = A.indices;
    a.vals = Av;
    a.b = b;
    a.x = x;
    a.upper = upper;
    a.unit = unit;
    return launch_solve(a, s);
}

template <typename T>
static int sptrsv_bwd_t(const csrk_pattern &A, const T *Av, const csrk_pattern *AT, const int64_t *perm, int upper,
                        int unit, const T *x, const T *v, T *dA, T *db, Bump &ws, cudaStream_t s)
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
    T *w = db ? db : ws.take<T>(n > 0 ? n : 1);
    TrsvArgs<T> a{};
    carve_solve(a, n, ws);
    if (!AT) CSRK_TRY(transpose_impl(sizeof(T) == 8 ? CSRK_F64 : CSRK_F32, A, nullptr, const_cast<int64_t *>(Tt.indptr),
                                     const_cast<int32_t *>(Tt.indices), nullptr, tp, ws, s));
    if (ws.sizing()) return CSRK_OK;
    a.n = n;
    a.indptr = Tt.indptr;
    a.indices = Tt.indices;
    a.vals = Av;
    a.perm = AT ? perm : tp;
    a.b = v;
    a.x = w;
    a.upper = !upper;
    a.unit = unit;
    CSRK_TRY(launch_solve(a, s));
    if (dA && n > 0) CSRK_LAUNCH(k_trsv_dT<T>, (unsigned)cdiv(n, 256), 256, 0, s, n, A.indptr, A.indices, w, x, unit, dA);
    return CSRK_OK;
}

int trsv_outer(const csrk_pattern &A, const double *w, const double *x, double *dA, cudaStream_t s)
{
    if (A.nrows > 0)
        CSRK_LAUNCH(k_trsv_dT<double>, (unsigned)cdiv(A.nrows, 256), 256, 0, s, A.nrows, A.indptr, A.indices, w, x, 0,
                    dA);
    return CSRK_OK;
}

int sptrsv_fwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int upper, int unit, const void *b, void *x,
               Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return sptrsv_fwd_t<double>(A, (const double *)A_val, upper, unit, (const double *)b, (double *)x, ws, s);
    return sptrsv_fwd_t<float>(A, (const float *)A_val, upper, unit, (const float *)b, (float *)x, ws, s);
}

int sptrsv_bwd(csrk_dtype dt, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT, const int64_t *perm,
               int upper, int unit, const void *x, const void *v, void *dA, void *db, Bump &ws, cudaStream_t s)
{
    if (dt == CSRK_F64)
        return sptrsv_bwd_t<double>(A, (const double *)A_val, AT, perm, upper, unit, (const double *)x,
                                    (const double *)v, (double *)dA, (double *)db, ws, s);
    return sptrsv_bwd_t<float>(A, (const float *)A_val, AT, perm, upper, unit, (const float *)x, (const float *)v,
                               (float *)dA, (float *)db, ws, s);
}

}  // namespace csrk
