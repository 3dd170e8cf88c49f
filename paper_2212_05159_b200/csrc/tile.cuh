// tile.cuh -- the row-tile / merge-path CSR traversal shared by SpMV (fwd, bwd), the
// atomic A^T scatter and the transpose scatter.
//
// A CTA owns R consecutive rows (R chosen from the mean row length so a tile is about one
// chunk of CAP = TPB*IPT merge items).  The tile's merge path over (row ends, nonzeros)
// is cut into chunks of CAP items; every thread takes IPT consecutive items, so rows of
// any length are spread evenly over the CTA (power-law rows, empty rows).  Index and
// value loads are coalesced over the chunk; the x gather is the only irregular read.
//
// MODE_REDUCE  : y[row] = sum_p val(p) * v[idx p]      (SpMV; the A^T-plan
//                traversal of the backward pass).  Deterministic: partial sums of
//                rows spanning several threads/chunks are combined in thread order.
//                SIDE adds D[pv] = v[idx p] * u[row]    (the masked outer product).
// MODE_SCATTER : w = u[row]; SIDE: D[p] = w * v[idx p]; y64 (nullable): y64[idx p] += val[p]*w
//                (atomic A^T v, "atomically reduced into correct entries").
// MODE_TRANSPOSE: slot = cursor[idx p]++; ATi[slot] = row; perm[slot] = p  (counting-sort
//                scatter of csr_transpose; order inside a column fixed by a later sort).
#pragma once

#include "csrk_internal.cuh"

namespace csrk {

enum { MODE_REDUCE = 0, MODE_SCATTER = 1, MODE_TRANSPOSE = 2 };

constexpr int kTileTPB = 256;
constexpr int kTileIPT = 6;
constexpr int kTileCAP = kTileTPB * kTileIPT;
constexpr int kTileShortRow = 256;   // fast path: all rows of the tile at most this long
constexpr int kTileMaxRPT = 4;        // rows per thread in the fast path (R <= 1024)

template <typename T>
struct TileArgs {
    int64_t nrows;
    const int64_t *indptr;
    const int32_t *indices;
    const T *vals;          // REDUCE/SCATTER values (indexed by pv / p)
    const int64_t *perm;    // REDUCE with PERM: value position = perm[p]
    const T *v;             // column-gathered vector
    T *y;                   // REDUCE: y[row]
    double *y64;            // SCATTER: y64[col] += val * w, fp64 atomics (nullable); fp32 data
                            // accumulates here too and is rounded once afterwards (reading A5)
    const T *u;             // row vector (SIDE / SCATTER)
    T *D;                   // SIDE output aligned with the values
    int64_t *cursor;        // TRANSPOSE
    uint64_t *out_keys;     // TRANSPOSE: packed (p << 31) | row per claimed slot
    int R;                  // rows per tile
    const int *run_if;      // non-null: k_rows does nothing unless *run_if != 0
    int accD;               // k_rows SIDE: D += instead of D = (internal: the PCG's dL accumulation)
    int accY;               // k_rows REDUCE y += / SCATTER into y as is (internal: PCG adjoint sums)
    const T *dotw;          // k_rows REDUCE (internal): also *dotout = sum_row y_row dotw_row
    double *dotpart;        //   per-CTA partials, cdiv(nrows, 256) of them
    double *dotout;
};

// Dynamic shared-memory layout (bytes offsets), identical on host and device.
struct TileSmem {
    size_t ptr, y, u, prod, row, crow, cval, total;
};

template <typename T>
__host__ __device__ inline TileSmem tile_smem(int R, int mode, bool side)
{
    TileSmem L;
    size_t o = 0;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    L.ptr = o;  o = al(o + sizeof(int64_t) * (R + 1));
    L.y = o;    if (mode == MODE_REDUCE) o = al(o + sizeof(double) * R);
    L.u = o;    if (side || mode == MODE_SCATTER) o = al(o + sizeof(T) * R);
    L.prod = o; if (mode == MODE_REDUCE) o = al(o + sizeof(double) * kTileCAP);
    L.row = o;  if (side || mode != MODE_REDUCE) o = al(o + sizeof(int) * kTileCAP);
    L.crow = o; if (mode == MODE_REDUCE) o = al(o + sizeof(int) * kTileTPB);
    L.cval = o; if (mode == MODE_REDUCE) o = al(o + sizeof(double) * kTileTPB);
    L.total = o;
    return L;
}

__device__ __forceinline__ int64_t tile_merge_rows(int64_t d, int64_t nr, int64_t Z, const int64_t *s_ptr, int64_t base)
{
    int64_t lo = d - Z > 0 ? d - Z : 0;
    int64_t hi = d < nr ? d : nr;
    while (lo < hi) {
        int64_t piv = (lo + hi) >> 1;
        if (s_ptr[piv + 1] - base <= d - piv - 1) lo = piv + 1;
        else hi = piv;
    }
    return lo;
}

template <typename T, int MODE, bool PERM, bool SIDE>
__global__ __launch_bounds__(kTileTPB) void k_csr_tile(TileArgs<T> a)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool NEED_ROW = SIDE || MODE != MODE_REDUCE;
    constexpr bool NEED_U = SIDE || MODE == MODE_SCATTER;
    const int R = a.R;
    const TileSmem L = tile_smem<T>(R, MODE, SIDE);
    int64_t *s_ptr = reinterpret_cast<int64_t *>(smem + L.ptr);
    double *s_y = reinterpret_cast<double *>(smem + L.y);
    T *s_u = reinterpret_cast<T *>(smem + L.u);
    double *s_prod = reinterpret_cast<double *>(smem + L.prod);
    int *s_row = reinterpret_cast<int *>(smem + L.row);
    int *s_crow = reinterpret_cast<int *>(smem + L.crow);
    double *s_cval = reinterpret_cast<double *>(smem + L.cval);
    __shared__ int64_t s_chunk[2];
    __shared__ int s_cc_row;
    __shared__ double s_cc_val;

    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int64_t nr = a.nrows - r0 < R ? a.nrows - r0 : R;
    for (int i = tid; i <= nr; i += kTileTPB) s_ptr[i] = a.indptr[r0 + i];
    if (NEED_U)
        for (int i = tid; i < nr; i += kTileTPB) s_u[i] = a.u[r0 + i];
    __syncthreads();
    const int64_t nzb = s_ptr[0];
    const int64_t Z = s_ptr[nr] - nzb;
    const int64_t total = nr + Z;
    int cc_row = -1;
    double cc_val = 0.0;

    // ---- fast path: every row of the tile is short -> a thread owns its rows (tid + i*TPB)
    bool mine_short = true;
    for (int i = tid; i < nr; i += kTileTPB) mine_short &= (s_ptr[i + 1] - s_ptr[i]) <= kTileShortRow;
    if (__syncthreads_and(mine_short)) {
        double acc[kTileMaxRPT];
#pragma unroll
        for (int j = 0; j < kTileMaxRPT; ++j) acc[j] = 0.0;
        for (int64_t c0 = 0; c0 < Z; c0 += kTileCAP) {
            const int64_t c1 = c0 + kTileCAP < Z ? c0 + kTileCAP : Z;
            if (MODE == MODE_REDUCE) {
#pragma unroll 2
                for (int64_t e = c0 + tid; e < c1; e += kTileTPB) {
                    const int64_t p = nzb + e;
                    const int64_t pv = PERM ? a.perm[p] : p;
                    s_prod[e - c0] = (double)a.vals[pv] * (double)a.v[a.indices[p]];
                }
            }
            if (NEED_ROW) {
#pragma unroll
                for (int j = 0; j < kTileMaxRPT; ++j) {
                    const int r = tid + j * kTileTPB;
                    if (r < nr) {
                        const int64_t s = s_ptr[r] - nzb, e = s_ptr[r + 1] - nzb;
                        for (int64_t q = (s > c0 ? s : c0); q < (e < c1 ? e : c1); ++q) s_row[q - c0] = r;
                    }
                }
            }
            __syncthreads();
            if (MODE == MODE_REDUCE) {
#pragma unroll
                for (int j = 0; j < kTileMaxRPT; ++j) {
                    const int r = tid + j * kTileTPB;
                    if (r < nr) {
                        const int64_t s = s_ptr[r] - nzb, e = s_ptr[r + 1] - nzb;
                        double t = acc[j];
                        for (int64_t q = (s > c0 ? s : c0); q < (e < c1 ? e : c1); ++q) t += s_prod[q - c0];
                        acc[j] = t;
                    }
                }
            }
            if (NEED_ROW) {
#pragma unroll 4
                for (int64_t e = c0 + tid; e < c1; e += kTileTPB) {
                    const int64_t p = nzb + e;
                    const int r = s_row[e - c0];
                    const int32_t c = a.indices[p];
                    if (MODE == MODE_SCATTER) {
                        const T w = s_u[r];
                        if (SIDE) a.D[p] = w * a.v[c];
                        if (a.y64) atomicAdd(&a.y64[c], (double)a.vals[p] * (double)w);
                    } else if (MODE == MODE_REDUCE) {
                        const int64_t pv = PERM ? a.perm[p] : p;
                        a.D[pv] = a.v[c] * s_u[r];
                    } else {
                        const int64_t slot =
                            (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(&a.cursor[c]), 1ULL);
                        a.out_keys[slot] = ((uint64_t)p << 31) | (uint64_t)(r0 + r);
                    }
                }
            }
            __syncthreads();
        }
        if (MODE == MODE_REDUCE) {
#pragma unroll
            for (int j = 0; j < kTileMaxRPT; ++j) {
                const int r = tid + j * kTileTPB;
                if (r < nr) a.y[r0 + r] = (T)acc[j];
            }
        }
        return;
    }

    for (int64_t D0 = 0; D0 < total; D0 += kTileCAP) {
        const int64_t D1 = D0 + kTileCAP < total ? D0 + kTileCAP : total;
        int64_t d = D0 + (int64_t)tid * kTileIPT;
        if (d > D1) d = D1;
        int64_t row = tile_merge_rows(d, nr, Z, s_ptr, nzb);
        int64_t nz = d - row;
        if (tid == 0) {
            s_chunk[0] = nz;
            s_chunk[1] = D1 - tile_merge_rows(D1, nr, Z, s_ptr, nzb);
        }
        __syncthreads();
        const int64_t nzA = s_chunk[0], nzB = s_chunk[1];

        if (MODE == MODE_REDUCE) {
            for (int64_t e = nzA + tid; e < nzB; e += kTileTPB) {
                const int64_t p = nzb + e;
                const int64_t pv = PERM ? a.perm[p] : p;
                s_prod[e - nzA] = (double)a.vals[pv] * (double)a.v[a.indices[p]];
            }
            __syncthreads();
        }

        // ---- consume this thread's merge items
        const int64_t first_row = row;
        bool first_done = false;
        double first_val = 0.0, acc = 0.0;
        const int nitems = (int)((d + kTileIPT < D1 ? d + kTileIPT : D1) - d);
        int64_t rend = row < nr ? s_ptr[row + 1] - nzb : INT64_MAX;
        for (int it = 0; it < nitems; ++it) {
            if (nz < rend) {
                if (MODE == MODE_REDUCE) acc += s_prod[nz - nzA];
                if (NEED_ROW) s_row[nz - nzA] = (int)row;
                ++nz;
            } else {
                if (MODE == MODE_REDUCE) {
                    if (row == first_row) {
                        first_done = true;
                        first_val = acc;
                    } else {
                        s_y[row] = acc;
                    }
                    acc = 0.0;
                }
                ++row;
                rend = row < nr ? s_ptr[row + 1] - nzb : INT64_MAX;
            }
        }
        if (MODE == MODE_REDUCE) {
            s_crow[tid] = (int)row;
            s_cval[tid] = acc;
        }
        __syncthreads();

        if (MODE == MODE_REDUCE) {
            if (first_done) {  // combine the partial sums of first_row in thread order
                int t0 = tid;
                while (t0 > 0 && s_crow[t0 - 1] == (int)first_row) --t0;
                double s = (t0 == 0 && cc_row == (int)first_row) ? cc_val : 0.0;
                for (int t = t0; t < tid; ++t) s += s_cval[t];
                s_y[first_row] = s + first_val;
            }
            if (tid == 0) {  // carry of the row still open at the end of the chunk
                const int rl = s_crow[kTileTPB - 1];
                int t0 = kTileTPB - 1;
                while (t0 > 0 && s_crow[t0 - 1] == rl) --t0;
                double s = (t0 == 0 && cc_row == rl) ? cc_val : 0.0;
                for (int t = t0; t < kTileTPB; ++t) s += s_cval[t];
                s_cc_row = rl;
                s_cc_val = s;
            }
        }

        if (NEED_ROW) {
            for (int64_t e = nzA + tid; e < nzB; e += kTileTPB) {
                const int64_t p = nzb + e;
                const int r = s_row[e - nzA];
                const int32_t c = a.indices[p];
                if (MODE == MODE_SCATTER) {
                    const T w = s_u[r];
                    if (SIDE) a.D[p] = w * a.v[c];
                    if (a.y64) atomicAdd(&a.y64[c], (double)a.vals[p] * (double)w);
                } else if (MODE == MODE_REDUCE) {  // SIDE
                    const int64_t pv = PERM ? a.perm[p] : p;
                    a.D[pv] = a.v[c] * s_u[r];
                } else {  // TRANSPOSE
                    const int64_t slot = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(&a.cursor[c]), 1ULL);
                    a.out_keys[slot] = ((uint64_t)p << 31) | (uint64_t)(r0 + r);
                }
            }
        }
        __syncthreads();
        if (MODE == MODE_REDUCE) {
            cc_row = s_cc_row;
            cc_val = s_cc_val;
        }
    }
    if (MODE == MODE_REDUCE) {
        __syncthreads();
        for (int i = tid; i < nr; i += kTileTPB) a.y[r0 + i] = (T)s_y[i];
    }
}

// Rows per tile from the mean row length: about one chunk of merge items per tile.
inline int tile_rows(int64_t nrows, int64_t nnz)
{
    double avg = nrows > 0 ? (double)nnz / (double)nrows : 0.0;
    int R = 1024;
    while (R > 32 && (double)R * (1.0 + avg) > 1.5 * kTileCAP) R >>= 1;
    return R;
}

template <typename T, int MODE, bool PERM, bool SIDE>
int launch_tile(const TileArgs<T> &a, cudaStream_t s)
{
    if (a.nrows <= 0) return CSRK_OK;
    const size_t smem = tile_smem<T>(a.R, MODE, SIDE).total;
    static DevOnce attr;
    if (attr.need()) {
        if (cudaFuncSetAttribute(k_csr_tile<T, MODE, PERM, SIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 64 * 1024) != cudaSuccess)
            return CSRK_ERR_CUDA;
        attr.done();
    }
    const int64_t grid = cdiv(a.nrows, a.R);
    CSRK_LAUNCH((k_csr_tile<T, MODE, PERM, SIDE>), (unsigned)grid, kTileTPB, smem, s, a);
    return CSRK_OK;
}

}  // namespace csrk
