/* abi_demo.c -- a plain C consumer of the C-ABI (include/csrk.h), no Python, no torch.
 *
 * Builds the 1D Poisson matrix A_N = tridiag(-1, 2, -1) (PAPER Eq. mat_1d_fd) for N = 1000 on
 * the device, runs
 *   csrk_spmv_fwd:  y = A 1, whose closed form is e_0 + e_{N-1} (interior rows sum to 0), and
 *   csrk_spgemm_symbolic (two-call protocol) + csrk_spgemm_numeric: C = A A, the pentadiagonal
 *     matrix with rows (1, -4, 6, -4, 1) inside and nnz(C) = 5N - 6,
 * and checks both exactly (integer-valued fp64).  Prints "abi_demo OK" on success.
 * Compiled by tests/test_abi_cpu.py (gcc, C99) and run on the GPU by tests/test_gpu_validate.py.
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "csrk.h"

#define CK(x)                                                                        \
    do {                                                                             \
        int st_ = (x);                                                               \
        if (st_ != 0) {                                                              \
            fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, st_,    \
                    csrk_status_string(st_));                                        \
            return 1;                                                                \
        }                                                                            \
    } while (0)
#define CU(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x,              \
                    cudaGetErrorString(e_));                                         \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void)
{
    const int64_t n = 1000, nnz = 3 * n - 2;
    int64_t *hp = malloc(sizeof(int64_t) * (n + 1));
    int32_t *hi = malloc(sizeof(int32_t) * nnz);
    double *hv = malloc(sizeof(double) * nnz), *hx = malloc(sizeof(double) * n), *hy = malloc(sizeof(double) * n);
    int64_t q = 0;
    for (int64_t i = 0; i < n; ++i) {
        hp[i] = q;
        for (int64_t j = i - 1; j <= i + 1; ++j)
            if (j >= 0 && j < n) {
                hi[q] = (int32_t)j;
                hv[q++] = j == i ? 2.0 : -1.0;
            }
        hx[i] = 1.0;
    }
    hp[n] = q;

    int64_t *dp;
    int32_t *di;
    double *dv, *dx, *dy;
    CU(cudaMalloc((void **)&dp, sizeof(int64_t) * (n + 1)));
    CU(cudaMalloc((void **)&di, sizeof(int32_t) * nnz));
    CU(cudaMalloc((void **)&dv, sizeof(double) * nnz));
    CU(cudaMalloc((void **)&dx, sizeof(double) * n));
    CU(cudaMalloc((void **)&dy, sizeof(double) * n));
    CU(cudaMemcpy(dp, hp, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(di, hi, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dv, hv, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dx, hx, sizeof(double) * n, cudaMemcpyHostToDevice));
    csrk_pattern A = {n, n, nnz, dp, di};

    /* y = A 1 */
    size_t wsb = 0;
    CK(csrk_workspace_size(CSRK_WS_SPMV_FWD, CSRK_F64, &A, NULL, 0, 0, &wsb));
    void *ws = NULL;
    if (wsb) CU(cudaMalloc(&ws, wsb));
    CK(csrk_spmv_fwd(CSRK_F64, CSRK_OP_N, A, dv, NULL, NULL, dx, dy, ws, wsb, NULL));
    CU(cudaMemcpy(hy, dy, sizeof(double) * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
        const double want = (i == 0 || i == n - 1) ? 1.0 : 0.0;
        if (hy[i] != want) {
            fprintf(stderr, "spmv: y[%ld] = %g, want %g\n", (long)i, hy[i], want);
            return 1;
        }
    }
    if (ws) CU(cudaFree(ws));

    /* C = A A: count (host sync, nnz), allocate, fill, numeric */
    int64_t *cp;
    CU(cudaMalloc((void **)&cp, sizeof(int64_t) * (n + 1)));
    CK(csrk_workspace_size(CSRK_WS_SPGEMM_SYMBOLIC, CSRK_F64, &A, &A, 0, 0, &wsb));
    CU(cudaMalloc(&ws, wsb));
    int64_t nnzc = -1;
    CK(csrk_spgemm_symbolic(A, A, cp, NULL, &nnzc, ws, wsb, NULL));
    if (nnzc != 5 * n - 6) {
        fprintf(stderr, "spgemm: nnz(C) = %ld, want %ld\n", (long)nnzc, (long)(5 * n - 6));
        return 1;
    }
    int32_t *ci;
    double *cv;
    CU(cudaMalloc((void **)&ci, sizeof(int32_t) * nnzc));
    CU(cudaMalloc((void **)&cv, sizeof(double) * nnzc));
    CK(csrk_spgemm_symbolic(A, A, cp, ci, NULL, ws, wsb, NULL));
    CU(cudaFree(ws));
    csrk_pattern C = {n, n, nnzc, cp, ci};
    CK(csrk_workspace_size(CSRK_WS_SPGEMM_NUMERIC, CSRK_F64, &A, &A, 0, 0, &wsb));
    ws = NULL;
    if (wsb) CU(cudaMalloc(&ws, wsb));
    CK(csrk_spgemm_numeric(CSRK_F64, A, dv, A, dv, C, cv, ws, wsb, NULL));
    CU(cudaDeviceSynchronize());
    int64_t *hcp = malloc(sizeof(int64_t) * (n + 1));
    int32_t *hci = malloc(sizeof(int32_t) * nnzc);
    double *hcv = malloc(sizeof(double) * nnzc);
    CU(cudaMemcpy(hcp, cp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(hci, ci, sizeof(int32_t) * nnzc, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(hcv, cv, sizeof(double) * nnzc, cudaMemcpyDeviceToHost));
    const double stencil[5] = {1.0, -4.0, 6.0, -4.0, 1.0};
    for (int64_t i = 2; i < n - 2; ++i) {   /* interior rows: columns i-2..i+2 */
        if (hcp[i + 1] - hcp[i] != 5) {
            fprintf(stderr, "spgemm: row %ld has %ld entries\n", (long)i, (long)(hcp[i + 1] - hcp[i]));
            return 1;
        }
        for (int t = 0; t < 5; ++t)
            if (hci[hcp[i] + t] != i - 2 + t || hcv[hcp[i] + t] != stencil[t]) {
                fprintf(stderr, "spgemm: C[%ld, %d] = %g\n", (long)i, hci[hcp[i] + t], hcv[hcp[i] + t]);
                return 1;
            }
    }
    printf("abi_demo OK (%s)\n", csrk_version());
    return 0;
}
