// utils.cu -- int64 prefix scan, optional pattern validation, launch counter.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "condgraph.cuh"
#include "csrk_internal.cuh"

namespace csrk {

std::atomic<uint64_t> g_launches{0};

bool pdl_enabled()
{
    static const bool on = knob("PDL", 1) != 0;
    return on;
}

int knob(const char *name, int def)
{
    char key[96];
    snprintf(key, sizeof(key), "CSRK_%s", name);
    const char *v = getenv(key);
    return v ? atoi(v) : def;
}

// ---------------------------------------------------------------- inclusive int64 scan
// Three phases (tile sums, recursive scan of the sums, tile scan + offset).  A tile is
// 256 threads x 16 items; loads/stores are coalesced through shared memory.
constexpr int kScanTPB = 256;
constexpr int kScanIPT = 16;
constexpr int kScanTile = kScanTPB * kScanIPT;

__device__ __forceinline__ int scan_pad(int i) { return i + (i >> 4); }

__device__ __forceinline__ int64_t block_incl_scan(int64_t v, int64_t *s_warp, int64_t &total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < kScanTPB / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < kScanTPB / 32) s_warp[lane] = w;
    }
    __syncthreads();
    if (warp > 0) v += s_warp[warp - 1];
    total = s_warp[kScanTPB / 32 - 1];
    return v;
}

__global__ __launch_bounds__(kScanTPB) void k_scan_tile_sums(const int64_t *__restrict__ x, int64_t n,
                                                             int64_t *__restrict__ sums, const int *run_if)
{
    pdl_wait();
    if (run_if && *(volatile const int *)run_if == 0) return;
    __shared__ int64_t s_warp[kScanTPB / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    int64_t v = 0;
#pragma unroll 4
    for (int i = 0; i < kScanIPT; ++i) {
        int64_t g = base + i * kScanTPB + threadIdx.x;
        if (g < n) v += x[g];
    }
    int64_t total;
    block_incl_scan(v, s_warp, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ __launch_bounds__(kScanTPB) void k_scan_tiles(int64_t *__restrict__ x, int64_t n,
                                                         const int64_t *__restrict__ offsets, const int *run_if)
{
    pdl_wait();
    if (run_if && *(volatile const int *)run_if == 0) return;
    __shared__ int64_t s[kScanTile + kScanTile / 16];
    __shared__ int64_t s_warp[kScanTPB / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    for (int i = 0; i < kScanIPT; ++i) {
        int li = i * kScanTPB + threadIdx.x;
        int64_t g = base + li;
        s[scan_pad(li)] = g < n ? x[g] : 0;
    }
    __syncthreads();
    int64_t loc[kScanIPT];
    int64_t run = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        run += s[scan_pad(threadIdx.x * kScanIPT + i)];
        loc[i] = run;
    }
    int64_t total;
    int64_t incl = block_incl_scan(run, s_warp, total);
    int64_t excl = incl - run + (offsets && blockIdx.x > 0 ? offsets[blockIdx.x - 1] : 0);
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) s[scan_pad(threadIdx.x * kScanIPT + i)] = loc[i] + excl;
    __syncthreads();
    for (int i = 0; i < kScanIPT; ++i) {
        int li = i * kScanTPB + threadIdx.x;
        int64_t g = base + li;
        if (g < n) x[g] = s[scan_pad(li)];
    }
}

static int incl_scan_i64(int64_t *x, int64_t n, Bump &ws, cudaStream_t s, const int *run_if)
{
    if (n <= 0) return CSRK_OK;
    int64_t nb = cdiv(n, kScanTile);
    if (nb == 1) {
        if (ws.sizing()) return CSRK_OK;
        CSRK_LAUNCH(k_scan_tiles, 1, kScanTPB, 0, s, x, n, (const int64_t *)nullptr, run_if);
        return CSRK_OK;
    }
    int64_t *sums = ws.take<int64_t>(nb);
    if (!ws.sizing()) CSRK_LAUNCH(k_scan_tile_sums, (unsigned)nb, kScanTPB, 0, s, x, n, sums, run_if);
    CSRK_TRY(incl_scan_i64(sums, nb, ws, s, run_if));
    if (!ws.sizing()) CSRK_LAUNCH(k_scan_tiles, (unsigned)nb, kScanTPB, 0, s, x, n, (const int64_t *)sums, run_if);
    return CSRK_OK;
}

int scan_counts_i64(int64_t *indptr, int64_t n, Bump &ws, cudaStream_t s, const int *run_if)
{
    if (ws.overflow) return CSRK_ERR_WORKSPACE;
    return incl_scan_i64(indptr ? indptr + 1 : nullptr, n, ws, s, run_if);
}

size_t scan_ws_bytes(int64_t n)
{
    Bump b(nullptr, 0);
    scan_counts_i64(nullptr, n, b, 0);
    return b.used;
}

// ---------------------------------------------------------------- fp64 accumulation -> fp32
__global__ __launch_bounds__(256) void k_f64_to_f32(const double *__restrict__ src, float *__restrict__ dst, int64_t n)
{
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
        dst[i] = (float)src[i];
}

int f64_to_f32(const double *src, float *dst, int64_t n, cudaStream_t s)
{
    if (n <= 0) return CSRK_OK;
    const int64_t g = cdiv(n, 256);
    CSRK_LAUNCH(k_f64_to_f32, (unsigned)(g < kNumSMs * 8 ? g : kNumSMs * 8), 256, 0, s, src, dst, n);
    return CSRK_OK;
}

// ---------------------------------------------------------------- validation (CSRK_VALIDATE=1)
__device__ int g_bad_pattern;

__global__ void k_validate(int64_t m, int64_t n, int64_t nnz, const int64_t *__restrict__ indptr,
                           const int32_t *__restrict__ indices)
{
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = indptr[i], e = indptr[i + 1];
        bool bad = (i == 0 && s != 0) || (i == m - 1 && e != nnz) || e < s;
        for (int64_t p = s; !bad && p < e; ++p) {
            int32_t c = indices[p];
            if (c < 0 || c >= n || (p > s && indices[p - 1] >= c)) bad = true;
        }
        if (bad) g_bad_pattern = 1;
    }
}

static bool validate_on()
{
    static int mode = -1;
    if (mode < 0) {
        const char *e = getenv("CSRK_VALIDATE");
        mode = (e && strcmp(e, "1") == 0) ? 1 : 0;
    }
    return mode == 1;
}

// triangular structure (PAPER 3.1.5 P:482 "L_ij != 0 if i >= j"): no entry on the
// wrong side of the diagonal, and a stored diagonal in every row unless unit
__global__ void k_validate_tri(int64_t m, const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                               int upper, int unit)
{
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        bool diag = false, bad = false;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            const int64_t c = indices[p];
            diag |= c == i;
            bad |= upper ? c < i : c > i;
        }
        if (bad || (!unit && !diag)) g_bad_pattern = 1;
    }
}

int validate_triangular(const csrk_pattern &A, int upper, int unit, cudaStream_t s)
{
    if (!validate_on() || A.nrows == 0) return CSRK_OK;
    int zero = 0, bad = 0;
    CSRK_CUDA(cudaMemcpyToSymbolAsync(g_bad_pattern, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CSRK_LAUNCH(k_validate_tri, 1024, 256, 0, s, A.nrows, A.indptr, A.indices, upper, unit);
    CSRK_CUDA(cudaMemcpyFromSymbolAsync(&bad, g_bad_pattern, sizeof(int), 0, cudaMemcpyDeviceToHost, s));
    CSRK_CUDA(cudaStreamSynchronize(s));
    return bad ? CSRK_ERR_PATTERN : CSRK_OK;
}

int validate_pattern(const csrk_pattern &A, cudaStream_t s)
{
    if (!validate_on() || A.nrows == 0) return CSRK_OK;
    int zero = 0, bad = 0;
    CSRK_CUDA(cudaMemcpyToSymbolAsync(g_bad_pattern, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CSRK_LAUNCH(k_validate, 1024, 256, 0, s, A.nrows, A.ncols, A.nnz, A.indptr, A.indices);
    CSRK_CUDA(cudaMemcpyFromSymbolAsync(&bad, g_bad_pattern, sizeof(int), 0, cudaMemcpyDeviceToHost, s));
    CSRK_CUDA(cudaStreamSynchronize(s));
    return bad ? CSRK_ERR_PATTERN : CSRK_OK;
}

// ---------------------------------------------------------------- conditional graphs (condgraph.cuh)
__global__ void k_set_cond(cudaGraphConditionalHandle h, const int *flag)
{
    cudaGraphSetConditional(h, *(volatile const int *)flag != 0 ? 1u : 0u);
}

cudaStream_t cond_capture_stream(int which)
{
    static std::mutex mu;
    static cudaStream_t streams[64][2] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    cudaStream_t &st = streams[dev & 63][which & 1];
    if (!st && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    return st;
}

}  // namespace csrk
