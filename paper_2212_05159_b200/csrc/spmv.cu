// spmv.cu -- SpMV forward and backward (PAPER 3.1.1; Table 1).
//
// Traversal: rows.cuh (thread per row, warp per long row) by default; the row-tile /
// merge-path kernel of tile.cuh is kept behind CSRK_SPMV_TILE=1 (measured 135 vs 70 us for
// the config-2 forward).
#include "ops.cuh"
#include "rows.cuh"
#include "tile.cuh"

namespace csrk {

template <typename T, int MODE, bool PERM, bool SIDE>
static int run(TileArgs<T> a, const RowList &L, cudaStream_t s)
{
    if (knob("SPMV_TILE", 0) && !a.accD && !a.accY && !a.dotw) return launch_tile<T, MODE, PERM, SIDE>(a, s);
    return launch_rows<T, MODE, PERM, SIDE>(a, L, s);
}

// fp64 target of an atomic A^T scatter into y[n]: y itself for fp64 data, workspace scratch for
// fp32 data (rounded once by round_scatter; reading A5)
template <typename T>
static double *scatter_target(T *y, int64_t n, Bump &ws)
{
    if constexpr (sizeof(T) == sizeof(double)) return reinterpret_cast<double *>(y);
    else return ws.take<double>(n > 0 ? n : 1);
}
template <typename T>
static int round_scatter(const double *acc, T *y, int64_t n, cudaStream_t s)
{
    if constexpr (sizeof(T) == sizeof(double)) return CSRK_OK;
    else return f64_to_f32(acc, y, n, s);
}

// Plan-path SpMV backward with dA split off into the row traversal: for matrices with scattered
// columns (the radix-transpose regime, config 4), where writing dA through perm is random.
// CSRK_SPMV_PLAN_SPLIT=0/1 forces either.
static bool split_plan(const csrk_pattern &A)
{
    static int k = knob("SPMV_PLAN_SPLIT", -1);
    if (k >= 0) return k != 0;
    return A.ncols >= (int64_t(1) << 22) && A.nnz >= 8 * A.ncols;
}

template <typename T>
static int spmv_fwd_t(csrk_op op, const csrk_pattern &A, const T *A_val, const csrk_pattern *AT,
                      const int64_t *perm, const T *x, T *y, Bump &ws, cudaStream_t s, int accY, const FusedDot *fd)
{
    if (accY && sizeof(T) != sizeof(double)) return CSRK_ERR_INVALID_ARG;   // internal, fp64 only
    RowList L{};
    carve_rowlist(A.nrows > A.ncols ? A.nrows : A.ncols, L, ws);
    double *acc = (op == CSRK_OP_T && !AT) ? scatter_target(y, A.ncols, ws) : nullptr;
    if (ws.sizing()) return CSRK_OK;
    TileArgs<T> a{};
    a.accY = accY;
    if (op == CSRK_OP_N) {
        // y_i = sum_{p in row i} A[p] x[idx p]
        a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
        a.vals = A_val; a.v = x; a.y = y;
        if (fd) {
            a.dotw = static_cast<const T *>(fd->w);
            a.dotpart = fd->part;
            a.dotout = fd->out;
        }
        a.R = tile_rows(A.nrows, A.nnz);
        return run<T, MODE_REDUCE, false, false>(a, L, s);
    }
    if (AT) {
        // y = A^T x as row inner products of the cached transpose, values gathered via perm
        a.nrows = AT->nrows; a.indptr = AT->indptr; a.indices = AT->indices;
        a.vals = A_val; a.perm = perm; a.v = x; a.y = y;
        a.R = tile_rows(AT->nrows, AT->nnz);
        return run<T, MODE_REDUCE, true, false>(a, L, s);
    }
    // y = A^T x by atomic scatter of A_ij x_i into y_j (fp64 target, reading A5); accY: into y as is
    if (!accY) CSRK_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * (size_t)A.ncols, s));
    a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
    a.vals = A_val; a.u = x; a.y64 = acc;
    a.R = tile_rows(A.nrows, A.nnz);
    CSRK_TRY((run<T, MODE_SCATTER, false, false>(a, L, s)));
    return round_scatter(acc, y, A.ncols, s);
}

template <typename T>
static int spmv_bwd_t(csrk_op op, const csrk_pattern &A, const T *A_val, const csrk_pattern *AT,
                      const int64_t *perm, const T *x, const T *dy, T *dA, T *dx, Bump &ws, cudaStream_t s,
                      int accD, int accY)
{
    if (accY && sizeof(T) != sizeof(double)) return CSRK_ERR_INVALID_ARG;   // internal, fp64 only
    RowList L{};
    carve_rowlist(A.nrows > A.ncols ? A.nrows : A.ncols, L, ws);
    // atomic dx (op N without a plan): fp64 target (sized whenever the call could need it)
    double *acc = (op == CSRK_OP_N && !(AT && dx) && (dx || ws.sizing())) ? scatter_target(dx, A.ncols, ws) : nullptr;
    if (ws.sizing()) return CSRK_OK;
    TileArgs<T> a{};
    a.accD = accD;
    a.accY = accY;
    if (op == CSRK_OP_T) {
        // y = A^T x:  dx = A dy (row inner products),  dA[p] = x_i dy_{idx p}
        a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
        a.vals = A_val; a.v = dy; a.u = x;
        a.R = tile_rows(A.nrows, A.nnz);
        if (dx) {
            a.y = dx;
            if (dA) {
                a.D = dA;
                return run<T, MODE_REDUCE, false, true>(a, L, s);
            }
            return run<T, MODE_REDUCE, false, false>(a, L, s);
        }
        a.D = dA;  // dA only: scatter mode without the atomic output
        return run<T, MODE_SCATTER, false, true>(a, L, s);
    }
    // op N (y = A x)
    if (AT && dx) {
        // transposed traversal: dx_j = sum_q A[perm q] dy[AT idx q];  dA[perm q] = dy[AT idx q] x_j.
        // Scattered patterns (use_split_plan): dA through perm would be one random sector write per
        // entry, so dA takes the coalesced row traversal instead and the transposed pass only
        // gathers dx (config 4: 10.2 -> ~2 ms).
        if (dA && split_plan(A)) {
            TileArgs<T> r = a;
            r.nrows = A.nrows; r.indptr = A.indptr; r.indices = A.indices;
            r.vals = A_val; r.u = dy; r.v = x; r.D = dA;
            r.R = tile_rows(A.nrows, A.nnz);
            CSRK_TRY((run<T, MODE_SCATTER, false, true>(r, L, s)));
            dA = nullptr;
        }
        a.nrows = AT->nrows; a.indptr = AT->indptr; a.indices = AT->indices;
        a.vals = A_val; a.perm = perm; a.v = dy; a.u = x; a.y = dx;
        a.R = tile_rows(AT->nrows, AT->nnz);
        if (dA) {
            a.D = dA;
            return run<T, MODE_REDUCE, true, true>(a, L, s);
        }
        return run<T, MODE_REDUCE, true, false>(a, L, s);
    }
    // row traversal: dA[p] = dy_i x[idx p] (coalesced), dx[idx p] += A[p] dy_i (fp64 atomic)
    if (dx && !accY) CSRK_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * (size_t)A.ncols, s));
    a.nrows = A.nrows; a.indptr = A.indptr; a.indices = A.indices;
    a.vals = A_val; a.u = dy; a.v = x; a.y64 = dx ? acc : nullptr; a.D = dA;
    a.R = tile_rows(A.nrows, A.nnz);
    if (dA) CSRK_TRY((run<T, MODE_SCATTER, false, true>(a, L, s)));
    else CSRK_TRY((run<T, MODE_SCATTER, false, false>(a, L, s)));
    return dx ? round_scatter(acc, dx, A.ncols, s) : CSRK_OK;
}

int spmv_fwd(csrk_dtype dt, csrk_op op, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT,
             const int64_t *perm, const void *x, void *y, Bump &ws, cudaStream_t s, int accumulate_y,
             const FusedDot *dot)
{
    if (dot && (op != CSRK_OP_N || dt != CSRK_F64)) return CSRK_ERR_INVALID_ARG;   // internal, fp64 op N
    if (dt == CSRK_F64)
        return spmv_fwd_t<double>(op, A, (const double *)A_val, AT, perm, (const double *)x, (double *)y, ws, s,
                                  accumulate_y, dot);
    return spmv_fwd_t<float>(op, A, (const float *)A_val, AT, perm, (const float *)x, (float *)y, ws, s,
                             accumulate_y, nullptr);
}

int spmv_bwd(csrk_dtype dt, csrk_op op, const csrk_pattern &A, const void *A_val, const csrk_pattern *AT,
             const int64_t *perm, const void *x, const void *dy, void *dA, void *dx, Bump &ws, cudaStream_t s,
             int accumulate_dA, int accumulate_dx)
{
    if (dt == CSRK_F64)
        return spmv_bwd_t<double>(op, A, (const double *)A_val, AT, perm, (const double *)x, (const double *)dy,
                                  (double *)dA, (double *)dx, ws, s, accumulate_dA, accumulate_dx);
    return spmv_bwd_t<float>(op, A, (const float *)A_val, AT, perm, (const float *)x, (const float *)dy,
                             (float *)dA, (float *)dx, ws, s, accumulate_dA, accumulate_dx);
}

}  // namespace csrk
