/*
 * oracle/csr_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the hot path of
 * Nytko et al., "Optimized Sparse Matrix Operations for Reverse Mode Automatic
 * Differentiation" (arXiv 2212.05159).  Citations "P:n" are lines of the paper
 * text, "S:n" lines of SPEC.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares NO code with the CUDA path
 * (paper_2212_05159_b200/csrc/) and includes none of its headers.
 *
 * Conventions:
 *   - CSR: indptr int64[nrows+1], indices int32[nnz], canonical (A3, A4).
 *   - Values arrive as double.  fp32 data is widened exactly by the caller and the
 *     result rounded once to float by the caller (oracle/__init__.py).
 *   - Every reduction accumulates in long double (x87 80-bit) and rounds once
 *     (SURVEY 8(c) c.2).  Alongside each reduced output e the oracle returns
 *     S_e = sum |term| for the S-scaled tolerance rule (reading A6).
 *   - Single products (spmv dA) are one IEEE double multiply -- no accumulator,
 *     so they are bit-comparable (reading A18).
 *   - Patterns are structural: stored zeros are kept, cancellation is kept
 *     (readings A1, A2).
 *   - Outputs are overwritten, never accumulated into (reading A16).
 *
 * Parallelism: single-threaded unless orc_set_threads(t>1); then row loops whose
 * outputs are disjoint use OpenMP.  Scatter loops (A^T products) stay serial.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double acc_t;

static int g_threads = 1;

void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int orc_get_threads(void) { return g_threads; }
int orc_sizeof_long_double_mantissa(void) { return __LDBL_MANT_DIG__; }

/* ------------------------------------------------------------------------ */
/* SpMV  (PAPER 3.1.1; Table 1)                          */
/* ------------------------------------------------------------------------ */

/* op = 0: y = A x,  y_i = sum_{p in row i} A[p] x[idx p]
 * op = 1: y = A^T x, y_j = sum_{(i,j) in A} A_ij x_i            (the Table 1 P:273 product)
 * S (nullable) receives sum |A[p] x[.]| per output. */
void orc_spmv(int op, int64_t m, int64_t n, const int64_t *indptr, const int32_t *indices,
              const double *val, const double *x, double *y, double *S)
{
    if (op == 0) {
        #pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads) if (g_threads > 1)
        for (int64_t i = 0; i < m; ++i) {
            acc_t s = 0, a = 0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                acc_t t = (acc_t)val[p] * (acc_t)x[indices[p]];
                s += t;
                a += fabsl(t);
            }
            y[i] = (double)s;
            if (S) S[i] = (double)a;
        }
    } else {
        acc_t *s = (acc_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(acc_t));
        acc_t *a = (acc_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(acc_t));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                acc_t t = (acc_t)val[p] * (acc_t)x[i];
                s[indices[p]] += t;
                a[indices[p]] += fabsl(t);
            }
        for (int64_t j = 0; j < n; ++j) {
            y[j] = (double)s[j];
            if (S) S[j] = (double)a[j];
        }
        free(s);
        free(a);
    }
}

/* VJP of SpMV (Table 1).
 * op = 0 (y = A x, dy in R^m, x in R^n):
 *     dA[p] = dy_i * x_{idx p}   at stored p only ("masked to a sparse matrix, only
 *                                 requiring computation of nonzero entries of A")
 *     dx    = A^T dy             ("atomically reduced into correct entries", P:448 -- reading A8)
 * op = 1 (y = A^T x, x in R^m, dy in R^n):
 *     dA[p] = x_i * dy_{idx p},   dx = A dy.
 * dA, dx nullable (skip).  S_dx nullable. */
void orc_spmv_bwd(int op, int64_t m, int64_t n, const int64_t *indptr, const int32_t *indices,
                  const double *val, const double *x, const double *dy,
                  double *dA, double *dx, double *S_dx)
{
    if (dA) {
        #pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads) if (g_threads > 1)
        for (int64_t i = 0; i < m; ++i)
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
                dA[p] = (op == 0) ? dy[i] * x[indices[p]] : x[i] * dy[indices[p]];
    }
    if (dx) {
        /* op 0: dx = A^T dy (scatter);  op 1: dx = A dy (row inner products) */
        orc_spmv(op == 0 ? 1 : 0, m, n, indptr, indices, val, dy, dx, S_dx);
    }
}

/* ------------------------------------------------------------------------ */
/* SpDMM (PAPER 3.1.3; Table 1)                          */
/* Dense operands are row-major with leading dimension ld >= k (reading A10). */
/* ------------------------------------------------------------------------ */

/* Y[i,c] = sum_{p in row i} A[p] X[idx p, c] */
void orc_spmm(int64_t m, int64_t n, int64_t k, const int64_t *indptr, const int32_t *indices,
              const double *val, const double *X, int64_t ldx, double *Y, int64_t ldy, double *S)
{
    (void)n;
    #pragma omp parallel for schedule(dynamic, 256) num_threads(g_threads) if (g_threads > 1)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t c = 0; c < k; ++c) {
            acc_t s = 0, a = 0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                acc_t t = (acc_t)val[p] * (acc_t)X[(int64_t)indices[p] * ldx + c];
                s += t;
                a += fabsl(t);
            }
            Y[i * ldy + c] = (double)s;
            if (S) S[i * k + c] = (double)a;
        }
}

/* VJP of SpDMM (Table 1):
 *   dA[p]   = sum_c dY[i,c] X[idx p, c]        = ((dY X^T) (.) mask(A))_{i, idx p}, c ascending
 *   dX[j,c] = sum_{(i,j) in A} A_ij dY[i,c]    = (A^T dY)_{j,c}
 * dA / dX nullable; S_dA [nnz], S_dX [n*k] nullable. */
void orc_spmm_bwd(int64_t m, int64_t n, int64_t k, const int64_t *indptr, const int32_t *indices,
                  const double *val, const double *X, int64_t ldx, const double *dY, int64_t lddy,
                  double *dA, double *S_dA, double *dX, int64_t lddx, double *S_dX)
{
    if (dA) {
        #pragma omp parallel for schedule(dynamic, 256) num_threads(g_threads) if (g_threads > 1)
        for (int64_t i = 0; i < m; ++i)
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                acc_t s = 0, a = 0;
                for (int64_t c = 0; c < k; ++c) {
                    acc_t t = (acc_t)dY[i * lddy + c] * (acc_t)X[(int64_t)indices[p] * ldx + c];
                    s += t;
                    a += fabsl(t);
                }
                dA[p] = (double)s;
                if (S_dA) S_dA[p] = (double)a;
            }
    }
    if (dX) {
        size_t cnt = (size_t)(n * k > 0 ? n * k : 1);
        acc_t *s = (acc_t *)calloc(cnt, sizeof(acc_t));
        acc_t *a = (acc_t *)calloc(cnt, sizeof(acc_t));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                int64_t j = indices[p];
                for (int64_t c = 0; c < k; ++c) {
                    acc_t t = (acc_t)val[p] * (acc_t)dY[i * lddy + c];
                    s[j * k + c] += t;
                    a[j * k + c] += fabsl(t);
                }
            }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t c = 0; c < k; ++c) {
                dX[j * lddx + c] = (double)s[j * k + c];
                if (S_dX) S_dX[j * k + c] = (double)a[j * k + c];
            }
        free(s);
        free(a);
    }
}

/* ------------------------------------------------------------------------ */
/* Sparse transpose ("take the sparse transpose of A")         */
/* ------------------------------------------------------------------------ */

/* Counting sort of the entries by column, stable in row order, so each row of
 * A^T lists its columns (= rows of A) ascending.  perm[q] = position in A of the
 * q-th entry of A^T.  AT_val, perm nullable. */
void orc_csr_transpose(int64_t m, int64_t n, const int64_t *indptr, const int32_t *indices,
                       const double *val, int64_t *AT_indptr, int32_t *AT_indices,
                       double *AT_val, int64_t *perm)
{
    int64_t nnz = indptr[m];
    memset(AT_indptr, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t p = 0; p < nnz; ++p) AT_indptr[indices[p] + 1] += 1;      /* column counts */
    for (int64_t j = 0; j < n; ++j) AT_indptr[j + 1] += AT_indptr[j];       /* prefix sum */
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) next[j] = AT_indptr[j];
    for (int64_t i = 0; i < m; ++i)                                          /* rows ascending => stable */
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            int64_t q = next[indices[p]]++;
            AT_indices[q] = (int32_t)i;
            if (AT_val) AT_val[q] = val[p];
            if (perm) perm[q] = p;
        }
    free(next);
}

/* ------------------------------------------------------------------------ */
/* SpGEMM  C = A B  (PAPER 3.1.2; Table 1)               */
/* ------------------------------------------------------------------------ */

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Symbolic phase.  pattern(C) = {(i,j) : exists k, (i,k) in A and (k,j) in B} --
 * structural: values are never consulted (reading A1/A2).
 * Per row i, mark the columns of every row k of B for k in row i of A (a marker
 * over the p columns of B), then emit the marked columns ascending.
 * C_indices == NULL: fills C_indptr and returns nnz(C).
 * C_indices != NULL: also fills the sorted column indices.  Returns nnz(C). */
int64_t orc_spgemm_symbolic(int64_t m, int64_t n, int64_t p,
                            const int64_t *A_indptr, const int32_t *A_indices,
                            const int64_t *B_indptr, const int32_t *B_indices,
                            int64_t *C_indptr, int32_t *C_indices)
{
    (void)n;
    int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p > 0 ? p : 1));
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p > 0 ? p : 1));
    for (int64_t j = 0; j < p; ++j) mark[j] = -1;
    C_indptr[0] = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t cnt = 0;
        for (int64_t a = A_indptr[i]; a < A_indptr[i + 1]; ++a) {
            int64_t kk = A_indices[a];
            for (int64_t b = B_indptr[kk]; b < B_indptr[kk + 1]; ++b) {
                int32_t j = B_indices[b];
                if (mark[j] != i) {
                    mark[j] = i;
                    row[cnt++] = j;
                }
            }
        }
        if (C_indices) {
            qsort(row, (size_t)cnt, sizeof(int32_t), cmp_i32);
            memcpy(C_indices + C_indptr[i], row, sizeof(int32_t) * (size_t)cnt);
        }
        C_indptr[i + 1] = C_indptr[i] + cnt;
    }
    free(mark);
    free(row);
    return C_indptr[m];
}

/* Numeric phase: C_ij = sum_{k ascending in row i of A} A_ik B_kj over the
 * symbolic pattern.  Dense long-double accumulator per row.  S nullable.
 * Returns 0, or -1 if a product falls outside C's pattern. */
int orc_spgemm_numeric(int64_t m, int64_t n, int64_t p,
                       const int64_t *A_indptr, const int32_t *A_indices, const double *A_val,
                       const int64_t *B_indptr, const int32_t *B_indices, const double *B_val,
                       const int64_t *C_indptr, const int32_t *C_indices, double *C_val, double *S)
{
    (void)n;
    int bad = 0;
    #pragma omp parallel num_threads(g_threads) if (g_threads > 1)
    {
        acc_t *s = (acc_t *)calloc((size_t)(p > 0 ? p : 1), sizeof(acc_t));
        acc_t *a = (acc_t *)calloc((size_t)(p > 0 ? p : 1), sizeof(acc_t));
        unsigned char *in = (unsigned char *)calloc((size_t)(p > 0 ? p : 1), 1);
        #pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t c = C_indptr[i]; c < C_indptr[i + 1]; ++c) in[C_indices[c]] = 1;
            for (int64_t e = A_indptr[i]; e < A_indptr[i + 1]; ++e) {
                int64_t kk = A_indices[e];
                for (int64_t b = B_indptr[kk]; b < B_indptr[kk + 1]; ++b) {
                    int32_t j = B_indices[b];
                    acc_t t = (acc_t)A_val[e] * (acc_t)B_val[b];
                    if (!in[j]) bad = 1;
                    s[j] += t;
                    a[j] += fabsl(t);
                }
            }
            for (int64_t c = C_indptr[i]; c < C_indptr[i + 1]; ++c) {
                int32_t j = C_indices[c];
                C_val[c] = (double)s[j];
                if (S) S[c] = (double)a[j];
                s[j] = 0;
                a[j] = 0;
                in[j] = 0;
            }
        }
        free(s);
        free(a);
        free(in);
    }
    return bad ? -1 : 0;
}

/* VJP of SpGEMM (Table 1; Fig. 3), V = dC on pattern(C):
 *   dA_ik = sum_{j in row k of B} V_ij B_kj         = ((V B^T) (.) mask(A))_ik
 *   dB_kj = sum_{i : (i,k) in A}  A_ik V_ij         = ((A^T V) (.) mask(B))_kj
 * V_ij is looked up at (i,j) in C's pattern (always present: row k of B is a
 * subset of row i of C).  dA, dB, S_dA, S_dB nullable.  Returns 0, or -1 if some
 * (i,j) is missing from C's pattern. */
int orc_spgemm_bwd(int64_t m, int64_t n, int64_t p,
                   const int64_t *A_indptr, const int32_t *A_indices, const double *A_val,
                   const int64_t *B_indptr, const int32_t *B_indices, const double *B_val,
                   const int64_t *C_indptr, const int32_t *C_indices, const double *dC,
                   double *dA, double *S_dA, double *dB, double *S_dB)
{
    (void)n;
    int bad = 0;
    int64_t nnzB = B_indptr[n];
    double *Vrow = (double *)calloc((size_t)(p > 0 ? p : 1), sizeof(double));
    unsigned char *in = (unsigned char *)calloc((size_t)(p > 0 ? p : 1), 1);
    acc_t *sB = NULL, *aB = NULL;
    if (dB) {
        sB = (acc_t *)calloc((size_t)(nnzB > 0 ? nnzB : 1), sizeof(acc_t));
        aB = (acc_t *)calloc((size_t)(nnzB > 0 ? nnzB : 1), sizeof(acc_t));
    }
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t c = C_indptr[i]; c < C_indptr[i + 1]; ++c) {
            Vrow[C_indices[c]] = dC[c];
            in[C_indices[c]] = 1;
        }
        for (int64_t e = A_indptr[i]; e < A_indptr[i + 1]; ++e) {
            int64_t kk = A_indices[e];
            acc_t s = 0, a = 0;
            for (int64_t b = B_indptr[kk]; b < B_indptr[kk + 1]; ++b) {
                int32_t j = B_indices[b];
                if (!in[j]) bad = 1;
                acc_t t = (acc_t)Vrow[j] * (acc_t)B_val[b];
                s += t;
                a += fabsl(t);
                if (dB) {
                    acc_t u = (acc_t)A_val[e] * (acc_t)Vrow[j];
                    sB[b] += u;
                    aB[b] += fabsl(u);
                }
            }
            if (dA) {
                dA[e] = (double)s;
                if (S_dA) S_dA[e] = (double)a;
            }
        }
        for (int64_t c = C_indptr[i]; c < C_indptr[i + 1]; ++c) {
            Vrow[C_indices[c]] = 0;
            in[C_indices[c]] = 0;
        }
    }
    if (dB) {
        for (int64_t b = 0; b < nnzB; ++b) {
            dB[b] = (double)sB[b];
            if (S_dB) S_dB[b] = (double)aB[b];
        }
        free(sB);
        free(aB);
    }
    free(Vrow);
    free(in);
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Sp + Sp  C = alpha A + beta B  (PAPER 3.1.4; Table 1) */
/* ------------------------------------------------------------------------ */

/* Symbolic: mask(C) = mask(A) U mask(B) ("the computation of C is viewed as a union over
 * the rows of A and B").  Per row, the sorted union of the two column lists
 * (structural: a sum that is 0 keeps its entry).  C_indices == NULL: counts only.
 * Returns nnz(C). */
int64_t orc_spadd_symbolic(int64_t m, const int64_t *A_indptr, const int32_t *A_indices,
                           const int64_t *B_indptr, const int32_t *B_indices,
                           int64_t *C_indptr, int32_t *C_indices)
{
    C_indptr[0] = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t a = A_indptr[i], ae = A_indptr[i + 1], b = B_indptr[i], be = B_indptr[i + 1];
        int64_t c = C_indptr[i];
        while (a < ae || b < be) {
            int32_t j;
            if (b >= be || (a < ae && A_indices[a] < B_indices[b])) j = A_indices[a++];
            else if (a >= ae || B_indices[b] < A_indices[a]) j = B_indices[b++];
            else { j = A_indices[a]; ++a; ++b; }
            if (C_indices) C_indices[c] = j;
            ++c;
        }
        C_indptr[i + 1] = c;
    }
    return C_indptr[m];
}

/* value of row i of M at column j, or 0 with *found = 0 (linear scan: plain and slow) */
static double orc_row_value(const int64_t *Mp, const int32_t *Mi, const double *Mv, int64_t i, int32_t j,
                            int64_t *pos)
{
    for (int64_t q = Mp[i]; q < Mp[i + 1]; ++q)
        if (Mi[q] == j) { *pos = q; return Mv ? Mv[q] : 0.0; }
    *pos = -1;
    return 0.0;
}

/* Numeric: C_ij = alpha A_ij + beta B_ij over C's pattern (absent entries are 0).  The two
 * products and their sum are formed in long double and rounded once; S = |alpha A_ij| +
 * |beta B_ij|.  Returns -1 if an entry of A or B is missing from C's pattern. */
int orc_spadd_numeric(int64_t m, double alpha, double beta,
                      const int64_t *A_indptr, const int32_t *A_indices, const double *A_val,
                      const int64_t *B_indptr, const int32_t *B_indices, const double *B_val,
                      const int64_t *C_indptr, const int32_t *C_indices, double *C_val, double *S)
{
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t c = C_indptr[i]; c < C_indptr[i + 1]; ++c) {
            int64_t pa, pb;
            const double a = orc_row_value(A_indptr, A_indices, A_val, i, C_indices[c], &pa);
            const double b = orc_row_value(B_indptr, B_indices, B_val, i, C_indices[c], &pb);
            const acc_t ta = (acc_t)alpha * (acc_t)a, tb = (acc_t)beta * (acc_t)b;
            C_val[c] = (double)(ta + tb);
            if (S) S[c] = (double)(fabsl(ta) + fabsl(tb));
        }
        /* every stored entry of A and B must appear in C */
        for (int64_t q = A_indptr[i]; q < A_indptr[i + 1]; ++q) {
            int64_t pc;
            orc_row_value(C_indptr, C_indices, NULL, i, A_indices[q], &pc);
            if (pc < 0) return -1;
        }
        for (int64_t q = B_indptr[i]; q < B_indptr[i + 1]; ++q) {
            int64_t pc;
            orc_row_value(C_indptr, C_indices, NULL, i, B_indices[q], &pc);
            if (pc < 0) return -1;
        }
    }
    return 0;
}

/* VJP (Table 1): dA = alpha V (.) mask(A), dB = beta V (.) mask(B) --
 * "the row-wise reduction from V to the sparsity mask of A or B": each stored entry picks
 * V at the same (i,j) (one IEEE double multiply, no accumulation).  dA / dB nullable.
 * Returns -1 if V's pattern (= C's) misses an entry of A or B. */
int orc_spadd_bwd(int64_t m, double alpha, double beta,
                  const int64_t *A_indptr, const int32_t *A_indices,
                  const int64_t *B_indptr, const int32_t *B_indices,
                  const int64_t *C_indptr, const int32_t *C_indices, const double *dC,
                  double *dA, double *dB)
{
    for (int64_t i = 0; i < m; ++i) {
        if (dA)
            for (int64_t q = A_indptr[i]; q < A_indptr[i + 1]; ++q) {
                int64_t pc;
                orc_row_value(C_indptr, C_indices, NULL, i, A_indices[q], &pc);
                if (pc < 0) return -1;
                dA[q] = alpha * dC[pc];
            }
        if (dB)
            for (int64_t q = B_indptr[i]; q < B_indptr[i + 1]; ++q) {
                int64_t pc;
                orc_row_value(C_indptr, C_indices, NULL, i, B_indices[q], &pc);
                if (pc < 0) return -1;
                dB[q] = beta * dC[pc];
            }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* SpTRSV  x = T^{-1} b, T triangular  (PAPER 3.1.5; Table 2) */
/* ------------------------------------------------------------------------ */

/* Forward: "each row depends on the intermediate values of previous rows only".
 *   lower (upper == 0): for i = 0, 1, ..., n-1   x_i = (b_i - sum_{p in row i, j < i} T[p] x_j) / d_i
 *   upper (upper == 1): for i = n-1, ..., 0      x_i = (b_i - sum_{p in row i, j > i} T[p] x_j) / d_i
 *     (P:482 converts U x = b by "matrix flip operations" into a lower system; the flip
 *      reverses the row and column order, i.e. this backward substitution -- SPEC S:202)
 *   d_i = the stored diagonal T_ii, or 1 when unit != 0 (a stored diagonal is then unused).
 * The numerator is accumulated in long double (p ascending) and divided there; x_i is rounded
 * once to double.  S (nullable) receives the componentwise forward-error magnitude
 *   S = M(T)^{-1} (|T| |x|),   M(T) = comparison matrix (|d_i| on the diagonal, -|T_ij| off it),
 * the textbook bound |x - x_computed| <= gamma * M(T)^{-1}|T||x| for substitution (reading
 * R-TRSV in DESIGN.md).  Returns 0, -2 if an entry lies on the wrong side of the diagonal
 * ("L_ij != 0 if i >= j"; SPEC S:203 shape error), -3 if a diagonal is missing and
 * unit == 0 (singular).  A zero stored diagonal divides by zero (IEEE). */
int orc_sptrsv(int upper, int unit, int64_t n, const int64_t *indptr, const int32_t *indices,
               const double *val, const double *b, double *x, double *S)
{
    for (int64_t i = 0; i < n; ++i) {
        int has_d = 0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            if (indices[p] == i) has_d = 1;
            if (upper ? indices[p] < i : indices[p] > i) return -2;
        }
        if (!has_d && !unit) return -3;
    }
    for (int64_t t = 0; t < n; ++t) {
        const int64_t i = upper ? n - 1 - t : t;
        acc_t s = (acc_t)b[i];
        acc_t d = 1;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            if (indices[p] == i) { if (!unit) d = (acc_t)val[p]; continue; }
            s -= (acc_t)val[p] * (acc_t)x[indices[p]];
        }
        x[i] = (double)(s / d);
    }
    if (S) {
        for (int64_t t = 0; t < n; ++t) {
            const int64_t i = upper ? n - 1 - t : t;
            acc_t tx = 0, off = 0, d = 1;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                const int32_t j = indices[p];
                if (j == i) { if (!unit) d = fabsl((acc_t)val[p]); continue; }
                tx += fabsl((acc_t)val[p] * (acc_t)x[j]);
                off += fabsl((acc_t)val[p]) * (acc_t)S[j];
            }
            tx += d * fabsl((acc_t)x[i]);
            S[i] = (double)((tx + off) / d);
        }
    }
    return 0;
}

/* VJP (Table 1 SpSolve row P:290-293 applied to a triangular T):
 *   db = T^{-T} v   "we first find L^{-T} v with our existing forward triangular solve routine":
 *                   T^T (the oracle's own counting-sort transpose, stored values kept) is
 *                   triangular on the other side, solved by orc_sptrsv with !upper;
 *   dT = -(db) x^T (.) mask(T)   "the masked outer-product ... in parallel over the nonzero
 *                   entries": dT[p] = -(db_i x_j), one IEEE double multiply; with unit != 0 a
 *                   stored diagonal is unused, so its gradient is 0.
 * dT, db nullable; S_db as in orc_sptrsv (for T^T).  Returns orc_sptrsv's codes. */
int orc_sptrsv_bwd(int upper, int unit, int64_t n, const int64_t *indptr, const int32_t *indices,
                   const double *val, const double *x, const double *v,
                   double *dT, double *db, double *S_db)
{
    const int64_t nnz = indptr[n];
    int64_t *Tp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int32_t *Ti = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    double *Tv = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    double *w = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    orc_csr_transpose(n, n, indptr, indices, val, Tp, Ti, Tv, NULL);
    int rc = orc_sptrsv(!upper, unit, n, Tp, Ti, Tv, v, w, S_db);
    if (rc == 0) {
        if (db) memcpy(db, w, sizeof(double) * (size_t)n);
        if (dT)
            for (int64_t i = 0; i < n; ++i)
                for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
                    dT[p] = (unit && indices[p] == i) ? 0.0 : -(w[i] * x[indices[p]]);
    }
    free(Tp); free(Ti); free(Tv); free(w);
    return rc;
}
