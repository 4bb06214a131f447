/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithms for the hot path
 * (autosparse, /root/reference/pkg/src/autosparse).  Nothing in the product
 * (paper_1805_03380_b200/) links, imports or calls this file: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker or as the timed CPU baseline.
 *
 * Types follow the reference's at-rest representation: int64 indices,
 * float64 values (csc.py:63-67).  Compiled with -ffp-contract=off because the
 * reference's numba kernels never contract a*b+c into an FMA.
 *
 * Each function cites the reference lines it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define DUP_SUM 0
#define DUP_LAST 1
#define DUP_SEQ 2 /* sequential left fold (not used by canonicalize; for tests) */

/* ---------------------------------------------------------------------- */
/* numpy's pairwise summation, as np.add.reduceat uses it for one segment:
 * result = v[0] + pairwise(v[1:]).  numpy/_core/src/umath/loops_utils.h
 * (pairwise_sum_DOUBLE): <8 -> sequential from -0.0; <=128 -> 8 accumulators
 * then a fixed tree then the tail; else split at n/2 rounded down to a
 * multiple of 8.  Verified bit-exact against numpy 2.3.5 (tests/golden).  */
static double pw_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
    }
}

double orc_segment_sum(const double *v, int64_t m) {
    /* np.add.reduceat over one segment of length m >= 1 (csc.py:179) */
    if (m == 1) return v[0];
    return v[0] + pw_sum(v + 1, m - 1);
}

/* ---------------------------------------------------------------------- */
/* canonicalize (csc.py:148-193): stable column-major sort, combine
 * duplicates (Sum via reduceat or LastWins), prune exact zeros,
 * bincount+cumsum col_offsets.  Returns nnz.  Outputs sized >= n.      */
int64_t orc_canonicalize(int64_t n_rows, int64_t n_cols, int64_t n, const int64_t *rows,
                         const int64_t *cols, const double *vals, int dup, int64_t *out_offs,
                         int64_t *out_rows, double *out_vals) {
    for (int64_t c = 0; c <= n_cols; c++) out_offs[c] = 0;
    if (n == 0) return 0;
    uint64_t *k = (uint64_t *)malloc(sizeof(uint64_t) * n * 2);
    int64_t *ix = (int64_t *)malloc(sizeof(int64_t) * n * 2);
    double *sv = (double *)malloc(sizeof(double) * n);
    uint64_t *k0 = k, *k1 = k + n;
    int64_t *i0 = ix, *i1 = ix + n;
    for (int64_t i = 0; i < n; i++) {
        k0[i] = (uint64_t)cols[i] * (uint64_t)n_rows + (uint64_t)rows[i];
        i0[i] = i;
    }
    /* bottom-up merge sort with explicit ping-pong tracking */
    int flip = 0;
    for (int64_t w = 1; w < n; w *= 2) {
        uint64_t *sk = flip ? k1 : k0, *dk = flip ? k0 : k1;
        int64_t *si = flip ? i1 : i0, *di = flip ? i0 : i1;
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n;
            int64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            int64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (sk[b] < sk[a]) { dk[o] = sk[b]; di[o++] = si[b++]; }
                else { dk[o] = sk[a]; di[o++] = si[a++]; }
            }
            while (a < mid) { dk[o] = sk[a]; di[o++] = si[a++]; }
            while (b < hi) { dk[o] = sk[b]; di[o++] = si[b++]; }
        }
        flip ^= 1;
    }
    uint64_t *sk = flip ? k1 : k0;
    int64_t *si = flip ? i1 : i0;
    for (int64_t i = 0; i < n; i++) sv[i] = vals[si[i]];
    int64_t nnz = 0;
    int64_t s = 0;
    while (s < n) {
        int64_t e = s + 1;
        while (e < n && sk[e] == sk[s]) e++;
        double v;
        if (dup == DUP_LAST) v = sv[e - 1];
        else if (dup == DUP_SEQ) { v = sv[s]; for (int64_t t = s + 1; t < e; t++) v += sv[t]; }
        else v = orc_segment_sum(sv + s, e - s);
        if (v != 0.0) {
            int64_t idx = si[s];
            out_rows[nnz] = rows[idx];
            out_vals[nnz] = v;
            out_offs[cols[idx] + 1] += 1;
            nnz++;
        }
        s = e;
    }
    for (int64_t c = 0; c < n_cols; c++) out_offs[c + 1] += out_offs[c];
    free(k); free(ix); free(sv);
    return nnz;
}

/* _kernels.transpose (_kernels.py:130-150): histogram rows, prefix sum,
 * stable scatter in column order.                                        */
void orc_transpose(int64_t n_rows, int64_t n_cols, const double *vals, const int64_t *rows,
                   const int64_t *offs, double *t_vals, int64_t *t_rows, int64_t *t_offs) {
    int64_t nnz = offs[n_cols];
    for (int64_t i = 0; i <= n_rows; i++) t_offs[i] = 0;
    for (int64_t k = 0; k < nnz; k++) t_offs[rows[k] + 1] += 1;
    for (int64_t i = 0; i < n_rows; i++) t_offs[i + 1] += t_offs[i];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (n_rows > 0 ? n_rows : 1));
    memcpy(cursor, t_offs, sizeof(int64_t) * n_rows);
    for (int64_t j = 0; j < n_cols; j++)
        for (int64_t k = offs[j]; k < offs[j + 1]; k++) {
            int64_t i = rows[k];
            int64_t pos = cursor[i]++;
            t_rows[pos] = j;
            t_vals[pos] = vals[k];
        }
    free(cursor);
}

/* _kernels.linear_combine (_kernels.py:12-48): alpha*A + beta*B by a
 * two-pointer row merge per column; exact zeros pruned.  Outputs sized
 * >= nnzA + nnzB.  Returns nnz.                                          */
int64_t orc_linear_combine(int64_t n_cols, const double *a_vals, const int64_t *a_rows,
                           const int64_t *a_offs, const double *b_vals, const int64_t *b_rows,
                           const int64_t *b_offs, double alpha, double beta, double *out_vals,
                           int64_t *out_rows, int64_t *out_offs) {
    int64_t k = 0;
    out_offs[0] = 0;
    for (int64_t j = 0; j < n_cols; j++) {
        int64_t ia = a_offs[j], ib = b_offs[j], ea = a_offs[j + 1], eb = b_offs[j + 1];
        while (ia < ea || ib < eb) {
            double v;
            int64_t r;
            if (ib >= eb || (ia < ea && a_rows[ia] < b_rows[ib])) {
                v = alpha * a_vals[ia]; r = a_rows[ia]; ia++;
            } else if (ia >= ea || b_rows[ib] < a_rows[ia]) {
                v = beta * b_vals[ib]; r = b_rows[ib]; ib++;
            } else {
                v = alpha * a_vals[ia] + beta * b_vals[ib]; r = a_rows[ia]; ia++; ib++;
            }
            if (v != 0.0) { out_vals[k] = v; out_rows[k] = r; k++; }
        }
        out_offs[j + 1] = k;
    }
    return k;
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* symbolic pass of _kernels.spgemm (_kernels.py:58-70): returns the total
 * number of distinct (row, col) output slots before pruning.             */
int64_t orc_spgemm_symbolic(int64_t n_rows_a, const int64_t *a_rows, const int64_t *a_offs,
                            const int64_t *b_rows, const int64_t *b_offs, int64_t n_cols_b) {
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * (n_rows_a > 0 ? n_rows_a : 1));
    for (int64_t i = 0; i < n_rows_a; i++) stamp[i] = -1;
    int64_t total = 0;
    for (int64_t j = 0; j < n_cols_b; j++)
        for (int64_t kk = b_offs[j]; kk < b_offs[j + 1]; kk++) {
            int64_t k = b_rows[kk];
            for (int64_t ii = a_offs[k]; ii < a_offs[k + 1]; ii++) {
                int64_t i = a_rows[ii];
                if (stamp[i] != j) { stamp[i] = j; total++; }
            }
        }
    free(stamp);
    return total;
}

/* numeric pass of _kernels.spgemm (_kernels.py:72-103): dense accumulator
 * with generation stamps (first product assigns, later ones +=, in B then
 * A order), per-column sort of touched rows, exact-zero prune.  Outputs
 * sized >= the symbolic total.  Returns nnz.                             */
int64_t orc_spgemm_numeric(int64_t n_rows_a, const double *a_vals, const int64_t *a_rows,
                           const int64_t *a_offs, const double *b_vals, const int64_t *b_rows,
                           const int64_t *b_offs, int64_t n_cols_b, double *out_vals,
                           int64_t *out_rows, int64_t *out_offs) {
    int64_t na = n_rows_a > 0 ? n_rows_a : 1;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * na);
    double *acc = (double *)calloc(na, sizeof(double));
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * na);
    for (int64_t i = 0; i < n_rows_a; i++) stamp[i] = -1;
    int64_t nnz = 0;
    out_offs[0] = 0;
    for (int64_t j = 0; j < n_cols_b; j++) {
        int64_t touched = 0;
        for (int64_t kk = b_offs[j]; kk < b_offs[j + 1]; kk++) {
            int64_t k = b_rows[kk];
            double bv = b_vals[kk];
            for (int64_t ii = a_offs[k]; ii < a_offs[k + 1]; ii++) {
                int64_t i = a_rows[ii];
                if (stamp[i] != j) { stamp[i] = j; acc[i] = a_vals[ii] * bv; tmp[touched++] = i; }
                else acc[i] += a_vals[ii] * bv;
            }
        }
        qsort(tmp, touched, sizeof(int64_t), cmp_i64);
        for (int64_t t = 0; t < touched; t++) {
            int64_t r = tmp[t];
            double v = acc[r];
            if (v != 0.0) { out_rows[nnz] = r; out_vals[nnz] = v; nnz++; }
        }
        out_offs[j + 1] = nnz;
    }
    free(stamp); free(acc); free(tmp);
    return nnz;
}

/* _kernels.vec_times_mat (_kernels.py:106-115) */
void orc_vec_times_mat(const double *v, const double *vals, const int64_t *rows,
                       const int64_t *offs, int64_t n_cols, double *w) {
    for (int64_t j = 0; j < n_cols; j++) {
        double s = 0.0;
        for (int64_t k = offs[j]; k < offs[j + 1]; k++) s += v[rows[k]] * vals[k];
        w[j] = s;
    }
}

/* _kernels.mat_times_vec (_kernels.py:118-127): column scatter, j ascending,
 * columns with x[j] == 0 skipped.  x is read with stride incx.           */
void orc_mat_times_vec(const double *vals, const int64_t *rows, const int64_t *offs,
                       const double *x, int64_t incx, int64_t n_rows, int64_t n_cols, double *y,
                       int64_t incy) {
    for (int64_t r = 0; r < n_rows; r++) y[r * incy] = 0.0;
    for (int64_t j = 0; j < n_cols; j++) {
        double xj = x[j * incx];
        if (xj != 0.0)
            for (int64_t k = offs[j]; k < offs[j + 1]; k++) y[rows[k] * incy] += vals[k] * xj;
    }
}

/* SpMM oracle: one mat_times_vec per dense column of a
 * column-major B (ldb) into a column-major C (ldc).  Columns are
 * independent, so they may run on several threads with identical results. */
typedef struct {
    const double *vals; const int64_t *rows, *offs; const double *B; int64_t ldb, n_rows, n_cols, k;
    double *C; int64_t ldc; int tid, nthreads;
} spmm_job;

static void *spmm_worker(void *p) {
    spmm_job *j = (spmm_job *)p;
    for (int64_t c = j->tid; c < j->k; c += j->nthreads)
        orc_mat_times_vec(j->vals, j->rows, j->offs, j->B + c * j->ldb, 1, j->n_rows, j->n_cols,
                          j->C + c * j->ldc, 1);
    return NULL;
}

void orc_spmm(const double *vals, const int64_t *rows, const int64_t *offs, const double *B,
              int64_t ldb, int64_t n_rows, int64_t n_cols, int64_t k, double *C, int64_t ldc,
              int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    spmm_job jobs[256];
    for (int t = 0; t < nthreads; t++) {
        spmm_job j = {vals, rows, offs, B, ldb, n_rows, n_cols, k, C, ldc, t, nthreads};
        jobs[t] = j;
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, spmm_worker, &jobs[t]);
    spmm_worker(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* _kernels.fused_trace (_kernels.py:153-175): per-column two-pointer
 * intersection, sequential left fold in column order.                    */
double orc_fused_trace(int64_t n_cols, const double *a_vals, const int64_t *a_rows,
                       const int64_t *a_offs, const double *b_vals, const int64_t *b_rows,
                       const int64_t *b_offs) {
    double total = 0.0;
    for (int64_t j = 0; j < n_cols; j++) {
        int64_t ia = a_offs[j], ib = b_offs[j], ea = a_offs[j + 1], eb = b_offs[j + 1];
        while (ia < ea && ib < eb) {
            int64_t ra = a_rows[ia], rb = b_rows[ib];
            if (ra == rb) { total += a_vals[ia] * b_vals[ib]; ia++; ib++; }
            else if (ra < rb) ia++;
            else ib++;
        }
    }
    return total;
}
