// csrk_internal.cuh -- shared device/host utilities of the sm_100a CSR kernel library.
// Nothing here is visible through the C-ABI (include/csrk.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <atomic>

#include "csrk.h"

namespace csrk {

// ---------------------------------------------------------------- launches / status
extern std::atomic<uint64_t> g_launches;

#define CSRK_TRY(expr)                          \
    do {                                        \
        int _st = (expr);                       \
        if (_st != CSRK_OK) return _st;         \
    } while (0)

#define CSRK_CUDA(expr)                                         \
    do {                                                        \
        if ((expr) != cudaSuccess) return CSRK_ERR_CUDA;        \
    } while (0)

// Programmatic dependent launch (PDL): every kernel is launched with programmatic stream
// serialization, so its CTAs may be scheduled while the previous kernel on the stream drains,
// and every kernel begins with pdl_wait() (griddepcontrol.wait), which blocks until that
// previous grid has completed and its writes are visible.  The launch latency of kernel N+1
// overlaps the tail of kernel N; the data dependence is unchanged.  CSRK_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();

// Launch a kernel, count it, and surface launch-configuration errors.
#define CSRK_LAUNCH(kernel, grid_, block_, smem_, stream_, ...)                    \
    do {                                                                         \
        cudaLaunchConfig_t _cfg = {};                                            \
        _cfg.gridDim = dim3(grid_);                                               \
        _cfg.blockDim = dim3(block_);                                            \
        _cfg.dynamicSmemBytes = (size_t)(smem_);                                \
        _cfg.stream = (stream_);                                                  \
        cudaLaunchAttribute _attr[1];                                            \
        _attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;        \
        _attr[0].val.programmaticStreamSerializationAllowed = 1;                 \
        _cfg.attrs = _attr;                                                      \
        _cfg.numAttrs = ::csrk::pdl_enabled() ? 1 : 0;                           \
        const cudaError_t _e = cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__);   \
        ::csrk::g_launches.fetch_add(1, std::memory_order_relaxed);              \
        if (_e != cudaSuccess) {                                                 \
            (void)cudaGetLastError();                                            \
            return CSRK_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)

constexpr int kNumSMs = 148;

// One-time setup per CUDA device (kernel attributes such as the dynamic shared-memory limit are
// per device): need() stays true on the current device until done() is called there.  Setting an
// attribute twice is harmless, so callers racing on a first call may both set it.
struct DevOnce {
    std::atomic<uint64_t> bits{0};
    static int dev()
    {
        int d = 0;
        cudaGetDevice(&d);
        return d & 63;
    }
    bool need() const { return !(bits.load(std::memory_order_acquire) & (1ull << dev())); }
    void done() { bits.fetch_or(1ull << dev(), std::memory_order_acq_rel); }
};

// ---------------------------------------------------------------- workspace carving
// One planning routine per op carves its scratch from `ws` through a Bump.  In size
// mode (base == nullptr) it only counts, so csrk_workspace_size and the op agree.
struct Bump {
    char *base;
    size_t cap;
    size_t used = 0;
    bool overflow = false;
    Bump(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
    template <typename U>
    U *take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        size_t bytes = count * sizeof(U);
        used = off + bytes;
        if (base && used > cap) overflow = true;
        return base ? reinterpret_cast<U *>(base + off) : nullptr;
    }
    bool sizing() const { return base == nullptr; }
};

// ---------------------------------------------------------------- dtype helpers
template <typename T> struct Acc { using type = double; };   // fp32 and fp64 data accumulate in fp64

// Atomic scatters (A^T v without a plan, SpGEMM dB, big-row SpGEMM dA) always add fp64 terms into
// an fp64 target: for fp32 data that target is workspace scratch, rounded once to fp32 at the end
// (f64_to_f32 / the ops' epilogues) -- reading A5: fp32 and fp64 data both accumulate in fp64.

// ---------------------------------------------------------------- merge-path search
// Merge of (row-end offsets a[0..nr), nnz indices 0..Z-1): at state (i, j) the next item
// is the end of row i if a[i] <= j, else nnz j.  Returns i (rows consumed) for diagonal d.
__device__ __forceinline__ int merge_path_rows(int d, int nr, int Z, const int64_t *s_ptr, int64_t base)
{
    int lo = d - Z > 0 ? d - Z : 0;
    int hi = d < nr ? d : nr;
    while (lo < hi) {
        int piv = (lo + hi) >> 1;
        if (s_ptr[piv + 1] - base <= (int64_t)(d - piv - 1)) lo = piv + 1;
        else hi = piv;
    }
    return lo;
}

// ---------------------------------------------------------------- host utilities (utils.cu)
// In-place int64 prefix sum: data[0] := 0 is NOT written; data[1..n] := inclusive scan of
// data[1..n].  Used to turn counts stored at indptr[1..] into a CSR indptr.
// run_if (nullable, device): the kernels do nothing unless *run_if != 0.
int scan_counts_i64(int64_t *indptr, int64_t n, Bump &ws, cudaStream_t s, const int *run_if = nullptr);
// dst[i] = (float)src[i], i < n (the single rounding of an fp64 accumulation of fp32 data)
int f64_to_f32(const double *src, float *dst, int64_t n, cudaStream_t s);
size_t scan_ws_bytes(int64_t n);

// Row-length classification etc.
int validate_pattern(const csrk_pattern &A, cudaStream_t s);  // honours CSRK_VALIDATE
int validate_triangular(const csrk_pattern &A, int upper, int unit, cudaStream_t s);  // honours CSRK_VALIDATE

// Internal transpose (pattern + perm, optional values) used by ops that need A^T when
// the caller passes no plan.  ws sized by transpose_ws(A).
int transpose_impl(csrk_dtype dt, const csrk_pattern &A, const void *A_val, int64_t *AT_indptr,
                   int32_t *AT_indices, void *AT_val, int64_t *perm, Bump &ws, cudaStream_t s);

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Tuning knob read once from the environment (CSRK_<name>), default `def`.  Used to A/B
// kernel variants on the GPU box; the defaults are the measured-best choices.
int knob(const char *name, int def);

}  // namespace csrk
