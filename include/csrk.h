/*
 * csrk.h -- C-ABI of the B200 (sm_100a) CSR kernel library for the hot path of
 * Nytko et al., "Optimized Sparse Matrix Operations for Reverse Mode Automatic
 * Differentiation" (arXiv 2212.05159).  "P:n" = PAPER.md line n (with section /
 * table), "S:n" = SPEC.md line n.
 *
 * CONVENTIONS (apply to every entry point)
 *   Memory     Every array argument is a DEVICE pointer on the current CUDA device,
 *              owned by the caller.  The library never allocates device memory;
 *              scratch is the caller's `ws` (size from csrk_workspace_size()).
 *              The only host pointer is csrk_spgemm_symbolic's `nnzC_host`.
 *   Streams    Every call enqueues on `stream` (0 = legacy default) and returns
 *              without synchronising, except csrk_spgemm_symbolic's count phase.
 *   Outputs    Overwritten (beta = 0); gradients are NOT accumulated into
 *              (reading A16).  A NULL optional output skips its work
 *              (mirrors requires_grad = False).
 *   CSR        indptr int64[nrows+1], indices int32[nnz]; canonical: indptr[0] = 0,
 *              nondecreasing, indptr[nrows] = nnz, indices strictly increasing
 *              within a row and in [0, ncols).  Stored zeros are structural
 *              entries (reading A1).  Canonical form is the caller's contract; it
 *              is checked (CSRK_ERR_PATTERN) only when env CSRK_VALIDATE=1.
 *   Values     dtype CSRK_F32 or CSRK_F64; values and dense operands share dtype.
 *              Reductions accumulate in fp64 for both dtypes (reading A5/A18): register /
 *              shared-memory sums are fp64, and atomic scatters (A^T v without a plan,
 *              SpGEMM dB, multi-window big-row SpGEMM dA) add fp64 terms into an fp64
 *              target -- for fp32 data a workspace scratch rounded once to fp32 at the end.
 *   Dense      row-major, leading dimension ld >= k (elements).
 *   Transpose  Ops that need A^T accept an optional cached transpose plan
 *              (AT = pattern of A^T, AT_perm[q] = position in A of A^T's q-th
 *              entry), as produced by csrk_csr_transpose.  With a plan, A^T work is
 *              a deterministic gather ("take the sparse transpose of A and re-execute
 *              the forward routine"); without one it is an atomic scatter
 *              ("atomically reduced into correct entries"; reading A7/A8).
 *   Errors     Every call returns a csrk_status (0 = OK, negative = error) and
 *              launches nothing on error.  Asynchronous device faults surface at the
 *              caller's next synchronisation.
 *   Threads    Stateless and reentrant; safe on concurrent streams.
 */
#ifndef CSRK_H
#define CSRK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *csrk_stream_t; /* == cudaStream_t */

typedef enum {
    CSRK_OK = 0,
    CSRK_ERR_INVALID_ARG = -1,   /* NULL where required, negative size, unknown dtype/op */
    CSRK_ERR_DIM_MISMATCH = -2,  /* e.g. A.ncols != B.nrows ("dimension mismatch") */
    CSRK_ERR_PATTERN = -3,       /* non-canonical CSR, or patterns that do not match (CSRK_VALIDATE=1) */
    CSRK_ERR_WORKSPACE = -4,     /* ws_bytes smaller than csrk_workspace_size() */
    CSRK_ERR_INDEX_OVERFLOW = -5,/* a size exceeds the index types (ncols > INT32_MAX, ...) */
    CSRK_ERR_CUDA = -6           /* a CUDA launch or runtime call failed */
} csrk_status;

typedef enum { CSRK_F32 = 0, CSRK_F64 = 1 } csrk_dtype;
typedef enum { CSRK_OP_N = 0, CSRK_OP_T = 1 } csrk_op;

/* Pattern (structure) of an nrows x ncols CSR matrix; indptr/indices are device pointers. */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;
    const int64_t *indptr;
    const int32_t *indices;
} csrk_pattern;

/* Operation ids for csrk_workspace_size. */
typedef enum {
    CSRK_WS_SPMV_FWD = 0,
    CSRK_WS_SPMV_BWD = 1,
    CSRK_WS_SPMM_FWD = 2,
    CSRK_WS_SPMM_BWD = 3,
    CSRK_WS_CSR_TRANSPOSE = 4,
    CSRK_WS_SPGEMM_SYMBOLIC = 5,
    CSRK_WS_SPGEMM_NUMERIC = 6,
    CSRK_WS_SPGEMM_BWD = 7,
    CSRK_WS_PCG = 8,         /* B = L, k = n_it, have_plan = precond */
    CSRK_WS_SPADD_SYMBOLIC = 9,/* numeric / bwd need no workspace */
    CSRK_WS_SPAI = 10,       /* A = C = pattern(M A), B = R = pattern(I) U C, k = n */
    CSRK_WS_SPTRSV_FWD = 11, /* A = T */
    CSRK_WS_SPTRSV_BWD = 12, /* A = T; have_plan = 1 if T^T (pattern + perm) is passed */
    CSRK_WS_GCN_FWD = 13,    /* A = graph, k = F */
    CSRK_WS_GCN_BWD = 14,    /* A = graph, k = F, have_plan */
    CSRK_WS_DENSE_GEMM_TN = 15,/* A->nrows = n, A->ncols = C, k = F (only the sizes are read) */
    CSRK_WS_PCG_DIST = 16    /* A, B = L: the rank's m x n_ext blocks, k = n_it */
} csrk_ws_op;

/*
 * SpMV forward (PAPER 3.1.1; Table 1).
 *   op = N:  y[m] = A x,    y_i = sum_{p in row i} A[p] x[idx p]   ("inner products of each
 *            row of A and x ... executed in parallel")
 *   op = T:  y[n] = A^T x,  y_j = sum_{(i,j) in A} A_ij x_i
 * A_val[nnz]; x[n] (op N) or x[m] (op T); y overwritten.  AT/AT_perm: optional plan,
 * used only for op T (both NULL or both set).
 */
int csrk_spmv_fwd(csrk_dtype dtype, csrk_op op, csrk_pattern A, const void *A_val,
                  const csrk_pattern *AT, const int64_t *AT_perm,
                  const void *x, void *y, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpMV backward = VJP of y = op(A) x (Table 1).
 *   op = N:  dA[p] = dy_i x_{idx p}  at stored p ONLY ("masked to a sparse matrix, only
 *            requiring computation of nonzero entries of A") -- one multiply,
 *            bit-exact;  dx[n] = A^T dy.
 *   op = T:  dA[p] = x_i dy_{idx p};  dx[m] = A dy.
 * dA_val (nullable) is aligned with A's indices; dx (nullable).  x, dy as in forward.
 * AT/AT_perm optional (op N only): deterministic transposed traversal computing dx and
 * dA together; without a plan dx uses atomic adds.
 */
int csrk_spmv_bwd(csrk_dtype dtype, csrk_op op, csrk_pattern A, const void *A_val,
                  const csrk_pattern *AT, const int64_t *AT_perm,
                  const void *x, const void *dy, void *dA_val, void *dx,
                  void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpMM (SpDMM) forward (PAPER 3.1.3; Table 1; reading A10/A21).
 *   Y[m x k] = A X,  X[n x k] row-major with leading dimension ldx >= k, Y with ldy >= k.
 */
int csrk_spmm_fwd(csrk_dtype dtype, csrk_pattern A, const void *A_val, int64_t k,
                  const void *X, int64_t ldx, void *Y, int64_t ldy,
                  void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpMM backward = VJP of Y = A X (Table 1).
 *   dA[p]   = sum_c dY[i,c] X[idx p, c]     ((dY X^T) (.) mask(A), an SDDMM)
 *   dX[n x k] = A^T dY                      ("take the sparse transpose of A and re-execute
 *                                             the forward routine")
 * dA_val, dX nullable.  AT/AT_perm: optional plan.  With a plan, one fused transposed
 * traversal produces dA and dX; without one, dA is a row traversal and dX builds the
 * transpose in `ws` first (workspace size accounts for it).
 */
int csrk_spmm_bwd(csrk_dtype dtype, csrk_pattern A, const void *A_val,
                  const csrk_pattern *AT, const int64_t *AT_perm, int64_t k,
                  const void *X, int64_t ldx, const void *dY, int64_t lddy,
                  void *dA_val, void *dX, int64_t lddx,
                  void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * CSR transpose.  Writes A^T (n x m) in canonical CSR:
 *   AT_indptr[n+1], AT_indices[nnz] (rows of A, ascending within each A^T row),
 *   AT_perm[nnz] (nullable): position in A of A^T's q-th entry,
 *   AT_val[nnz]  (nullable; A_val may then be NULL): A_val[AT_perm[q]].
 * Pattern outputs are bit-exact against the stable counting sort of the oracle.
 */
int csrk_csr_transpose(csrk_dtype dtype, csrk_pattern A, const void *A_val,
                       int64_t *AT_indptr, int32_t *AT_indices, void *AT_val, int64_t *AT_perm,
                       void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpGEMM symbolic phase (PAPER 3.1.2):
 *   pattern(C) = {(i,j) : exists k, (i,k) in A and (k,j) in B}, STRUCTURAL (values never
 *   consulted; entries that would cancel are kept -- reading A2), columns ascending.
 * Two calls with the same arguments:
 *   (1) C_indices == NULL: writes C_indptr[m+1] (int64, reading A4), synchronises `stream`,
 *       and stores nnz(C) in *nnzC_host (host pointer, required).
 *   (2) C_indices != NULL (caller allocated nnz(C) int32): fills the sorted indices
 *       (C_indptr must hold the result of call 1).  Does not synchronise.
 * A is m x n, B is n x p.
 * Call (1) also leaves the columns of every short row in `ws`; call (2) copies them instead of
 * merging again when it is the first fill after the latest count with the same A, B and `ws`
 * (tracked on the host).  Any other csrk call given a workspace overlapping that `ws` in between
 * invalidates the copy (call (2) then merges again).  Writes to `ws` by anything other than
 * csrk between the calls, or changes to A's / B's patterns, are outside the contract (call (2)
 * needs the patterns of call (1) anyway); CSRK_GEMM_FILL_CACHE=0 disables the copy.
 */
int csrk_spgemm_symbolic(csrk_pattern A, csrk_pattern B, int64_t *C_indptr, int32_t *C_indices,
                         int64_t *nnzC_host, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpGEMM numeric phase: C_ij = sum_k A_ik B_kj over the symbolic pattern C
 * (C.indptr / C.indices from csrk_spgemm_symbolic).  C_val[nnz(C)] overwritten.
 */
int csrk_spgemm_numeric(csrk_dtype dtype, csrk_pattern A, const void *A_val,
                        csrk_pattern B, const void *B_val, csrk_pattern C, void *C_val,
                        void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpGEMM backward = VJP of C = A B (Table 1; Fig. 3):
 *   dA_ik = sum_{j in row k of B} dC_ij B_kj        ((dC B^T) (.) mask(A))
 *   dB_kj = sum_{i : (i,k) in A}   A_ik dC_ij        ((A^T dC) (.) mask(B))
 * dC_val[nnz(C)] aligned with C's pattern (reading A15); dA_val[nnz(A)], dB_val[nnz(B)]
 * nullable.  When B aliases A the caller sums dA + dB (reading A13).
 */
int csrk_spgemm_bwd(csrk_dtype dtype, csrk_pattern A, const void *A_val,
                    csrk_pattern B, const void *B_val, csrk_pattern C, const void *dC_val,
                    void *dA_val, void *dB_val, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * csrk_spgemm_bwd with A's transpose plan (AT pattern + AT_perm from csrk_csr_transpose; both
 * NULL = csrk_spgemm_bwd).  With a plan, dB is computed as the paper's "modified version of the
 * SpGEMM algorithm that operates on columns of A": each stored (k, j) of B gathers
 * sum_{i in row k of A^T} A_ik dC_ij in ascending i (fp64, rounded once) -- no atomics, so dB is
 * bit-identical from run to run (reading A7/A9).  C must be the structural product pattern of
 * csrk_spgemm_symbolic(A, B) (entries of C_i missing for some j of B_k count as dC_ij = 0).
 * dA as in csrk_spgemm_bwd.  Workspace: CSRK_WS_SPGEMM_BWD with have_plan = 1 (no dB scratch).
 */
int csrk_spgemm_bwd_plan(csrk_dtype dtype, csrk_pattern A, const void *A_val,
                         const csrk_pattern *AT, const int64_t *AT_perm,
                         csrk_pattern B, const void *B_val, csrk_pattern C, const void *dC_val,
                         void *dA_val, void *dB_val, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Sp + Sp symbolic phase (PAPER 3.1.4):
 *   pattern(C) = pattern(A) U pattern(B) ("mask(C) = mask(A) U mask(B) ... a union over the
 *   rows"), columns ascending, structural (an entry whose values would sum to 0 is
 *   kept).  A and B are m x n.  Same two-call protocol as csrk_spgemm_symbolic:
 *   (1) C_indices == NULL: writes C_indptr[m+1], synchronises `stream`, stores nnz(C) in
 *       *nnzC_host;  (2) C_indices != NULL: fills the sorted indices (no synchronisation).
 */
int csrk_spadd_symbolic(csrk_pattern A, csrk_pattern B, int64_t *C_indptr, int32_t *C_indices,
                        int64_t *nnzC_host, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Sp + Sp numeric phase:  C_ij = alpha A_ij + beta B_ij on C's pattern (absent
 * entries count as 0), formed in fp64 and rounded once to dtype.  C MUST be the pattern
 * returned by csrk_spadd_symbolic for (A, B) (CSRK_ERR_PATTERN if nnz(C) < nnz(A) or nnz(B));
 * C_val[nnz(C)] overwritten.
 */
int csrk_spadd_numeric(csrk_dtype dtype, double alpha, csrk_pattern A, const void *A_val, double beta,
                       csrk_pattern B, const void *B_val, csrk_pattern C, void *C_val,
                       void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Sp + Sp backward = VJP of C = alpha A + beta B (Table 1):
 *   dA = alpha dC (.) mask(A),  dB = beta dC (.) mask(B)
 * ("the row-wise reduction from V to the sparsity mask of A or B"): each stored entry of A (B)
 * takes dC at the same (i, j) times alpha (beta) -- one fp64 multiply, rounded once (bit-exact
 * against the oracle).  dC_val aligned with C = csrk_spadd_symbolic(A, B); dA_val[nnz(A)],
 * dB_val[nnz(B)] nullable.
 */
int csrk_spadd_bwd(csrk_dtype dtype, double alpha, csrk_pattern A, double beta, csrk_pattern B,
                   csrk_pattern C, const void *dC_val, void *dA_val, void *dB_val,
                   void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SPAI loss and gradient -- the SURVEY 8(f) row-f2 workload (PAPER 4.6):
 *     loss = || I - M A ||_F^2   (Eq. spai_loss),
 *     dM_val[nnz(M)] = d loss / d M.values on M's fixed pattern.
 * Composed from this library's kernels (C = M A by csrk_spgemm_numeric, R = I - C by
 * csrk_spadd_numeric, loss = sum R^2 and dR = 2R, dC by csrk_spadd_bwd, dM by the left VJP of
 * csrk_spgemm_bwd); deterministic.  fp64.  A, M: n x n.  Cached patterns, built once by the
 * caller: C = csrk_spgemm_symbolic(M, A); I = the n x n identity pattern (indptr[i] = i,
 * indices[i] = i); R = csrk_spadd_symbolic(I, C).  loss_host: host pointer (required); the
 * call synchronises `stream` once at the end.
 * Workspace: csrk_workspace_size(CSRK_WS_SPAI, CSRK_F64, &C, &R, n, 0, &bytes).
 */
int csrk_spai_loss_grad(csrk_pattern A, const double *A_val, csrk_pattern M, const double *M_val,
                        csrk_pattern C, csrk_pattern R, csrk_pattern I, double *loss_host, double *dM_val,
                        void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Sparse triangular solve (PAPER 3.1.5):  x = T^{-1} b.
 *   upper = 0: T lower triangular ("L_ij != 0 if i >= j"); forward substitution
 *              x_i = (b_i - sum_{j<i} T_ij x_j) / T_ii ("each row depends on the intermediate
 *              values of previous rows only").
 *   upper = 1: T upper triangular, solved in reverse row order (the "matrix flip" of P:482).
 *   unit_diag: the diagonal is taken as 1 (a stored diagonal entry is then unused).
 * T is n x n, canonical CSR; b[n], x[n] (overwritten; must not alias b).  Method: a one-pass
 * decoupled look-back scan when every row depends only on its neighbour (bidiagonal chains),
 * otherwise the synchronisation-free solve of P:487 (see sptrsv.cu).  Stored entries on the
 * wrong side of the diagonal are ignored, a missing / zero diagonal (unit_diag = 0) divides
 * by zero; with CSRK_VALIDATE=1 both are rejected (CSRK_ERR_PATTERN).
 * Workspace: csrk_workspace_size(CSRK_WS_SPTRSV_FWD, dtype, &T, NULL, 0, 0, &bytes).
 */
int csrk_sptrsv_fwd(csrk_dtype dtype, csrk_pattern T, const void *T_val, int upper, int unit_diag, const void *b,
                    void *x, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * SpTRSV backward = VJP of x = T^{-1} b (Table 1 SpSolve row P:290-293):
 *   db = T^{-T} v                 ("we first find L^{-T} v with our existing forward triangular
 *                                   solve routine": the same solve on T^T, triangular on the
 *                                   other side)
 *   dT = -(db) x^T (.) mask(T)    (dT[p] = -(db_i x_j) at stored (i, j); "the masked
 *                                   outer-product can be executed in parallel over the nonzero
 *                                   entries"); with unit_diag a stored diagonal gets 0.
 * x = the forward solution (saved operand), v = dL/dx.  dT_val[nnz] and db[n] nullable (both
 * NULL: no-op); db must not alias v.  TT / TT_perm: optional cached transpose plan of T from
 * csrk_csr_transpose (both NULL: T^T is built in the workspace).
 * Workspace: csrk_workspace_size(CSRK_WS_SPTRSV_BWD, dtype, &T, NULL, 0, have_plan, &bytes).
 */
int csrk_sptrsv_bwd(csrk_dtype dtype, csrk_pattern T, const void *T_val, const csrk_pattern *TT,
                    const int64_t *TT_perm, int upper, int unit_diag, const void *x, const void *v, void *dT_val,
                    void *db, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * GCN propagation -- the sparse part of the GCN layer (PAPER 4.4, Eq. gcn_update),
 * evaluated as the paper's listing (Fig. 12) from XTheta on:
 *     D_i = (sum of the stored values of row i + 1)^(-1/2)   ("D = (graph.row_sum() + 1.) ** -0.5")
 *     Y   = D (A (D Z) + D Z) + bias                          ("C = D[:, None] * (graph @ DXTheta
 *                                                              + DXTheta)", "return C + bias")
 * A: n x n graph (values = edge weights; the + I of A~ = A + I is implicit, never stored).
 * Z = X Theta and Y: n x F row-major (ld >= F), 1 <= F <= 128; bias[F] nullable; D[n] (fp64,
 * required) receives D for the backward.  One fused SpMM (the scalings in its gather and
 * epilogue).  Y must not alias Z.  Workspace: CSRK_WS_GCN_FWD (k = F).
 */
int csrk_gcn_fwd(csrk_dtype dtype, csrk_pattern A, const void *A_val, int64_t F, const void *Z, int64_t ldz,
                 const void *bias, void *Y, int64_t ldy, double *D, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * GCN propagation backward (VJP of csrk_gcn_fwd with the graph constant, as in the paper's
 * training where only Theta and bias are parameters):
 *     dZ    = D (A^T (D dY) + D dY)     (the transposed propagation; "a matrix transpose is
 *                                         needed to compute the VJP in the backward pass")
 *     dbias = sum_i dY_i                (column sums, fp64)
 * D from csrk_gcn_fwd.  dZ, dbias nullable (both NULL: no-op).  AT / AT_perm: optional cached
 * transpose plan of A (else built in the workspace).  Workspace: CSRK_WS_GCN_BWD.
 */
int csrk_gcn_bwd(csrk_dtype dtype, csrk_pattern A, const void *A_val, const csrk_pattern *AT, const int64_t *AT_perm,
                 int64_t F, const double *D, const void *dY, int64_t lddy, void *dZ, int64_t lddz, void *dbias,
                 void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Small dense products of the GCN layer (Fig. 12 "XTheta = X @ self.weights" and its VJP):
 *   csrk_dense_gemm_nn:  Z[n x F] = X[n x C] W        (transW = 0, W: C x F row-major)
 *                        Z[n x F] = X[n x C] W^T      (transW = 1, W: F x C row-major; dX = dZ Theta^T)
 *                        W is staged in shared memory (C F <= 25600); no workspace.
 *   csrk_dense_gemm_tn:  dW[C x F] = X^T dZ           (dTheta; fp64 accumulation in a fixed order --
 *                        per-CTA partials summed in block order, no atomics, so the same bits on
 *                        every run; workspace CSRK_WS_DENSE_GEMM_TN; C * ceil(F / 16) <= 256).
 * Row-major, ld >= the row width.  Memory-bound tall-skinny products (C, F ~ 16): one pass over
 * the n rows, no tensor cores.
 */
int csrk_dense_gemm_nn(csrk_dtype dtype, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *W,
                       int transW, void *Z, int64_t ldz, csrk_stream_t stream);
int csrk_dense_gemm_tn(csrk_dtype dtype, int64_t n, int64_t C, int64_t F, const void *X, int64_t ldx, const void *dZ,
                       int64_t lddz, void *dW, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Learned-preconditioner PCG training step -- the config-5 composition of SURVEY 8(a) row a14
 * (PAPER 4.3).  Runs n_it iterations of preconditioned CG on A x = b with x0 = 0 and
 * M = L L^T (L lower triangular, e.g. the lower-bidiagonal L of P:857), records the
 * residuals r^(1..n_it), evaluates the weighted loss
 *     loss = sum_i w_i ||r^(i)||_2 / ||b||_2,   w_i = gamma^(n_it - i) / sum_j gamma^(n_it - j),
 * and back-propagates to dL_val[nnz(L)] = d loss / d L.values (on L's pattern).
 * The reverse pass is the adjoint of every CG step (SpMV VJPs for L, L^T and A; dot / axpy
 * adjoints), run with the same kernels as the forward.  fp64 only.  All vectors are device
 * arrays of length n = A.nrows; loss_host (required) and resid_host (nullable, n_it entries,
 * ||r^(i)||) are host pointers: the call synchronises `stream` once at the end.
 * precond = 0: M = L L^T as in the paper (two SpMVs per application).  precond = 1 (SURVEY 8(f)
 * row f3): M = (L L^T)^{-1} applied exactly by two triangular solves, u = L^{-1} r, z = L^{-T} u
 * (csrk_sptrsv_*; L must be lower triangular with its diagonal, CSRK_VALIDATE=1 checks), the
 * reverse pass through the SpTRSV VJPs.
 * Workspace: csrk_workspace_size(CSRK_WS_PCG, CSRK_F64, &A, &L, n_it, precond, &bytes) -- the
 * saved p, q, r vectors of every iteration, (3 n_it + 12) n doubles (+ L^T for precond = 1).
 */
int csrk_pcg_loss_grad(csrk_pattern A, const double *A_val, csrk_pattern L, const double *L_val,
                       const double *b, int n_it, double gamma, int precond, double *loss_host, double *resid_host,
                       double *dL_val, void *ws, size_t ws_bytes, csrk_stream_t stream);

/*
 * Row-sharded multi-GPU execution (north_star "rows of A are partitioned across the
 * GPUs ... partial gradients combined by NCCL").  One process per GPU.  A rank owns m consecutive
 * rows; its vectors are EXTENDED: n_ext entries holding the owned rows at [own_off, own_off + m)
 * and ghost copies of the neighbours' entries its rows reference around them.  Local matrices
 * are the rank's rows with columns in extended coordinates (m x n_ext).
 *
 * csrk_comm: the three exchanges a sharded step needs, stream-ordered on `stream`:
 *   allreduce_sum(ctx, buf, count, stream)  in-place sum over ranks of `count` doubles (device)
 *   halo(ctx, vec, mode, stream)            on an extended vector: mode 0 = GATHER (every ghost
 *                                           entry receives its owner's value), mode 1 = REDUCE
 *                                           (every ghost entry is added into its owner's entry;
 *                                           ghosts are then undefined)
 *   capturable                              nonzero if both may be captured in a CUDA graph
 * csrk_comm_nccl_create builds one over NCCL (libnccl.so.2, loaded at run time) from a halo
 * description; any other implementation (e.g. a host-staged one for tests) may fill the struct.
 */
typedef struct {
    void *ctx;
    int (*allreduce_sum)(void *ctx, double *buf, int64_t count, csrk_stream_t stream);
    int (*halo)(void *ctx, double *vec, int mode, csrk_stream_t stream);
    int capturable;
} csrk_comm;

/* Halo description of one rank (host arrays of npeers entries, extended coordinates): peer q
 * holds my owned entries [own_off[q], +own_len[q]) as its ghosts, and my ghost entries
 * [ghost_off[q], +ghost_len[q]) are owned by peer q.  Ranges are in matching order on both sides
 * (my own range for q is, element for element, q's ghost range for me). */
typedef struct {
    int npeers;
    const int *peer;
    const int64_t *own_off, *own_len;
    const int64_t *ghost_off, *ghost_len;
} csrk_halo;

/* NCCL unique id (128 bytes) for csrk_comm_nccl_create; call on one rank and broadcast it. */
int csrk_comm_nccl_unique_id(void *id128);
/* Collective over the `world` ranks: creates the NCCL communicator and a csrk_comm whose halo
 * follows `halo` (copied).  Allocates its own device scratch (the max received ghost total) --
 * the only csrk object that owns device memory; csrk_comm_nccl_destroy frees it. */
int csrk_comm_nccl_create(const void *id128, int rank, int world, const csrk_halo *halo, csrk_comm *out);
int csrk_comm_nccl_destroy(csrk_comm *comm);

/*
 * Config-5 training step, row-sharded (the multi-GPU form of csrk_pcg_loss_grad, M = L L^T):
 * A and L are this rank's m rows (m x n_ext, columns in extended coordinates), b its owned m
 * entries, dL_val[nnz(L)] the gradient on its rows.  Every SpMV with A or L reads a halo-gathered
 * extended input (op N) or produces an extended partial that is halo-reduced (op T); the dot
 * products are local sums followed by comm->allreduce_sum (p.q and r.z per iteration and their
 * adjoints; the ||r^(i)||^2 once at the end).  loss_host / resid_host are the global values on
 * every rank.  comm == NULL (with n_ext == m, own_off == 0) is the single-GPU call.  precond must
 * be 0.  If comm is NULL or capturable, the whole forward + reverse pass is captured once in a
 * CUDA graph (per argument set) and replayed (CSRK_PCG_GRAPH=0 disables).
 * Workspace: csrk_workspace_size(CSRK_WS_PCG_DIST, CSRK_F64, &A, &L, n_it, 0, &bytes) with
 * A.ncols = L.ncols = n_ext.
 */
int csrk_pcg_loss_grad_dist(const csrk_comm *comm, int64_t own_off, csrk_pattern A, const double *A_val,
                            csrk_pattern L, const double *L_val, const double *b, int n_it, double gamma,
                            double *loss_host, double *resid_host, double *dL_val, void *ws, size_t ws_bytes,
                            csrk_stream_t stream);

/*
 * Scratch bytes needed by operation `op` for operands A (and B for SpGEMM, or the
 * output pattern C for numeric/bwd passed as B), width k (SpMM) and dtype.
 * have_plan = 1 if a transpose plan will be passed.  Writes *bytes; host-only, no launch.
 */
int csrk_workspace_size(csrk_ws_op op, csrk_dtype dtype, const csrk_pattern *A,
                        const csrk_pattern *B, int64_t k, int have_plan, size_t *bytes);

/* Static text for a status code. */
const char *csrk_status_string(int status);

/* Number of kernels this library has launched in this process (all devices). */
uint64_t csrk_launch_count(void);

/* Library version, e.g. "csrk 0.1 sm_100a". */
const char *csrk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CSRK_H */
