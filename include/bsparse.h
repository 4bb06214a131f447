/*
 * bsparse.h -- C ABI of libbsparse.so, the B200 (sm_100a) back end for the
 * hot path of the hybrid sparse matrix of arXiv 1805.03380 (reference:
 * autosparse, /root/reference/pkg/src/autosparse).
 *
 * Conventions:
 *  - every pointer argument is a DEVICE pointer unless marked (host);
 *  - indices on device are int32, col_ptr int32[n_cols+1]; values float64 (_f64)
 *    or float32 (_f32);
 *  - outputs are caller-allocated; outputs whose size is data dependent take
 *    a capacity upper bound and report the realised size in info[0] (device);
 *  - scratch comes from the caller (`ws`, `ws_bytes`, sized by the matching
 *    *_workspace_bytes function); the library never allocates or frees;
 *  - all work is enqueued on `stream` (a cudaStream_t); no call synchronises
 *    except where stated;
 *  - every function returns an as_status code; as_last_error() describes the
 *    last failure of the calling thread.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef BSPARSE_H_
#define BSPARSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum as_status {
  AS_OK = 0,
  AS_ERR_SHAPE = 1,   /* errors.ShapeError            (errors.py:14-21) */
  AS_ERR_COORD = 2,   /* errors.CoordinateError       (errors.py:7-8)   */
  AS_ERR_CORRUPT = 3, /* errors.CorruptionError       (errors.py:10-11) */
  AS_ERR_CUDA = 4,    /* CUDA runtime failure; see as_last_error()       */
  AS_ERR_ARG = 5      /* bad argument (null pointer, workspace too small, size limits) */
};

enum as_dup { AS_DUP_SUM = 0, AS_DUP_LAST = 1 }; /* csc.DUP_SUM / DUP_LAST (csc.py:20-21) */

const char *as_last_error(void);
int as_abi_version(void);
/* Construction / transpose engine selection (tests and measurements only):
 * 0 = automatic (single-launch kernel up to its envelope, then the
 * large-input pipeline, then the general bucket kernel), 1 = the large-input
 * pipeline whenever it applies, 2 = the general bucket kernel.  Process-wide. */
int as_set_engine(int engine);

/* ---------------------------------------------------------------------------
 * COO triplets -> canonical CSC.
 * Replaces csc.canonicalize (csc.py:148-193) and, with the range check,
 * csc.from_triplets (csc.py:208-222) / coo.to_csc (coo.py:51-62).
 * rows/cols are int32 (idx_bytes == 4) or int64 (idx_bytes == 8).  Outputs
 * are sized for n (nnz <= n).  info[0] = nnz, info[1] = index of the first
 * out-of-range triplet or a value >= n when all are in range (the kernels
 * skip bad triplets; the caller raises CoordinateError naming info[1]).
 */
size_t as_build_workspace_bytes(int64_t n, int64_t n_cols);
int as_coo_to_csc_f64(int64_t n_rows, int64_t n_cols, int64_t n, const void *rows, const void *cols,
                      int idx_bytes, const double *vals, int dup, int32_t *col_ptr, int32_t *row_idx,
                      double *out_vals, int64_t *info, void *ws, size_t ws_bytes, void *stream);
int as_coo_to_csc_f32(int64_t n_rows, int64_t n_cols, int64_t n, const void *rows, const void *cols,
                      int idx_bytes, const float *vals, int dup, int32_t *col_ptr, int32_t *row_idx,
                      float *out_vals, int64_t *info, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Host side of the end-to-end construction (csrc/upload.cu, host code).
 * Moves int64 host triplets (csc.py:63-67 index type) to the device as
 * int32 indices: the values' copy is enqueued first, host threads narrow
 * rows / cols into pinned staging (n_chunks pieces, each copied as soon as it
 * is narrowed) -- 16 instead of 24 bytes per triplet over PCIe.  An index
 * outside [0, 2^31) becomes -1, which as_coo_to_csc_* then reports as the
 * first out-of-range triplet.  Synchronous on the host for the narrowing,
 * asynchronous on `stream` for the copies; the staging must not be reused
 * before they complete.  vals == NULL: only the indices are moved.
 */
int as_upload_coo_i64(const int64_t *rows, const int64_t *cols, const void *vals, int64_t n, int64_t val_bytes,
                      int32_t *stage_rows, int32_t *stage_cols, int32_t *d_rows, int32_t *d_cols, void *d_vals,
                      int n_threads, int n_chunks, void *stream);

/* Same, for shapes whose row and column bit widths fit 31 bits together
 * (e.g. 10k x 10k: 14 + 14): host threads pack each triplet's indices into
 * one 32-bit key (col << row_bits | row) -- 12 instead of 16 bytes per
 * triplet over PCIe -- and a device kernel unpacks every copied chunk into
 * d_rows / d_cols.  Coordinates outside the shape arrive as -1 (the same
 * first-bad-triplet report).  d_keys: device scratch of n uint32.
 * *first_bad (nullable, host): the index of the first triplet outside the
 * shape, or -1 -- the packers see every coordinate, so a caller can raise
 * CoordinateError (csc.py:215-221) without waiting for the device.  Returns
 * AS_ERR_SHAPE when the bit widths do not fit (use as_upload_coo_i64).
 */
int as_upload_coo_packed(const int64_t *rows, const int64_t *cols, const void *vals, int64_t n,
                         int64_t val_bytes, int64_t n_rows, int64_t n_cols, uint32_t *stage_keys,
                         uint32_t *d_keys, int32_t *d_rows, int32_t *d_cols, void *d_vals, int n_threads,
                         int n_chunks, int64_t *first_bad, void *stream);

/* Read-back of a CSC's row indices at half width (host side of
 * CscData.to_host when every row is < 65536): d_rows -> uint16 on the device
 * (d_scratch, n uint16) -> pinned h_stage, asynchronous on `stream`; then
 * as_widen_u16 (host threads) once the copy has landed. */
int as_rows_to_host_u16(const int32_t *d_rows, int64_t n, uint16_t *d_scratch, uint16_t *h_stage, void *stream);
int as_widen_u16(const uint16_t *src, int32_t *dst, int64_t n, int n_threads);

/* ---------------------------------------------------------------------------
 * Insertion-cache flush: base CSC + element-write log -> canonical CSC.
 * Replaces rbt.to_csc (rbt.py:444-458) of the tree that RbtStore.insert
 * (rbt.py:371-387: overwrite; 0.0 erases, :374-376) built on top of
 * rbt.from_csc(base) (rbt.py:461-476).  Last write wins, exact zeros erase.
 * Outputs sized for nnz_base + n_log.  info[0] = nnz, info[1] as above.
 */
size_t as_flush_workspace_bytes(int64_t nnz_base, int64_t n_log, int64_t n_cols);
int as_flush_log_f64(int64_t n_rows, int64_t n_cols, int64_t nnz_base, const int32_t *base_col_ptr,
                     const int32_t *base_row_idx, const double *base_vals, int64_t n_log,
                     const int32_t *log_rows, const int32_t *log_cols, const double *log_vals,
                     int32_t *col_ptr, int32_t *row_idx, double *out_vals, int64_t *info, void *ws,
                     size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * CSC transpose.  Replaces _kernels.transpose (_kernels.py:130-150) via
 * ops.transpose (ops.py:123-128).  Output: CSC of A^T, n_rows+1 offsets,
 * nnz entries, rows sorted within each column (stable order of the reference).
 */
size_t as_transpose_workspace_bytes(int64_t nnz, int64_t n_rows);
int as_csc_transpose_f64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *col_ptr,
                         const int32_t *row_idx, const double *vals, int32_t *t_col_ptr,
                         int32_t *t_row_idx, double *t_vals, void *ws, size_t ws_bytes, void *stream);
int as_csc_transpose_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *col_ptr,
                         const int32_t *row_idx, const float *vals, int32_t *t_col_ptr,
                         int32_t *t_row_idx, float *t_vals, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * alpha*A + beta*B.  Replaces _kernels.linear_combine (_kernels.py:12-48) via
 * ops._combine/add/subtract/scaled_sum (ops.py:50-73).  Products and the sum
 * are separately rounded (no FMA), exact zeros pruned.  nnz_a/nnz_b (host)
 * size the launch.  Outputs sized for nnz_a + nnz_b; info[0] = nnz.
 */
size_t as_add_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b);
int as_csc_add_f64(int64_t n_rows, int64_t n_cols, double alpha, double beta, const int32_t *a_col_ptr,
                   const int32_t *a_row_idx, const double *a_vals, const int32_t *b_col_ptr,
                   const int32_t *b_row_idx, const double *b_vals, int64_t nnz_a, int64_t nnz_b,
                   int32_t *col_ptr, int32_t *row_idx, double *out_vals, int64_t *info, void *ws,
                   size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * SpGEMM C = A @ B (Gustavson, bit-exact accumulation order).  Replaces
 * _kernels.spgemm (_kernels.py:51-103) via ops.matmul (ops.py:110-120).
 * Two phases: as_spgemm_products writes prod_ptr (int64[n_cols_b+1], the
 * per-column product counts' prefix sum) and info[0] = total products, an
 * upper bound of nnz(C); as_spgemm_f64 then fills outputs sized for that
 * bound, info[0] = nnz.  prod_ptr must be kept between the calls.
 */
size_t as_spgemm_products_workspace_bytes(int64_t n_cols_b);
int as_spgemm_products(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t *a_col_ptr,
                       const int32_t *b_col_ptr, const int32_t *b_row_idx, int64_t *prod_ptr, int64_t *info,
                       void *ws, size_t ws_bytes, void *stream);
size_t as_spgemm_workspace_bytes(int64_t n_cols_b, int64_t nnz_b, int64_t total_products);
int as_spgemm_f64(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t *a_col_ptr,
                  const int32_t *a_row_idx, const double *a_vals, const int32_t *b_col_ptr,
                  const int32_t *b_row_idx, const double *b_vals, int64_t nnz_b, const int64_t *prod_ptr,
                  int64_t total_products, int32_t *col_ptr, int32_t *row_idx, double *out_vals,
                  int64_t *info, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * SpMM C = A @ B with dense column-major B (n_cols x k, ldb) and C
 * (n_rows x k, ldc).  A is given in CSR form, i.e. the CSC arrays of A^T
 * (row_ptr[n_rows+1], col_idx, vals), which the hybrid handle caches.  The
 * reference API has only the k = 1 case, _kernels.mat_times_vec
 * (_kernels.py:118-127) via ops.mat_times_vec (ops.py:97-107); its oracle
 * for k > 1 is k such calls.
 *  exact != 0: per output entry a float64 left fold in column order with
 *              separately rounded products, columns with B[j,c] == 0 skipped
 *              -- bit-identical to the reference for float64 data;
 *  exact == 0: float32 FMA accumulation (tolerance 1e-5, float32 only).
 * ws: as_spmm_workspace_bytes (one row-major chunk of B).
 */
size_t as_spmm_workspace_bytes(int64_t n_cols, int64_t k, int dtype_bytes);
int as_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t *row_ptr,
                    const int32_t *col_idx, const float *vals, const float *B, int64_t ldb, float *C,
                    int64_t ldc, int exact, void *ws, size_t ws_bytes, void *stream);
int as_spmm_csr_f64(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t *row_ptr,
                    const int32_t *col_idx, const double *vals, const double *B, int64_t ldb, double *C,
                    int64_t ldc, void *ws, size_t ws_bytes, void *stream);

/* SpMM C = A @ B straight over the CSC of A (col_ptr[n_cols+1], row_idx,
 * vals; nnz entries), no CSR: the column-merge variant, in the reference's
 * own loop order (_kernels.mat_times_vec, _kernels.py:118-127: for each
 * column, y[row] += val * x[col]).  Float32, additions in arrival order
 * (tolerance 1e-5; not bit-reproducible run to run).  Used for the first
 * product on a fresh CSC, when no CSR is cached (ops.mat_times_vec,
 * ops.py:97-107).  ws: as_spmm_csc_workspace_bytes (a row-major n_rows x 16
 * float32 accumulator and the tile table). */
size_t as_spmm_csc_workspace_bytes(int64_t n_rows, int64_t nnz);
int as_spmm_csc_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t k, const int32_t *col_ptr,
                    const int32_t *row_idx, const float *vals, const float *B, int64_t ldb, float *C,
                    int64_t ldc, void *ws, size_t ws_bytes, void *stream);

/* w = v^T A.  Replaces _kernels.vec_times_mat (_kernels.py:106-115). */
int as_vecmat_csc_f64(int64_t n_rows, int64_t n_cols, const int32_t *col_ptr, const int32_t *row_idx,
                      const double *vals, const double *v, double *w, void *stream);

/* ---------------------------------------------------------------------------
 * trace(A^T B) without forming the product: sum over coincident nonzeros.
 * Replaces _kernels.fused_trace (_kernels.py:153-175) via
 * expr.fused_trace_at_b (expr.py:197-209).
 * nnz_a/nnz_b (host) size the launch.  out[0] = the sum, out[1] = its
 * double-double residual (partials of column slices combine exactly, used by
 * the multi-GPU path).  Deterministic.  ws: as_trace_workspace_bytes.
 */
size_t as_trace_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b);
int as_trace_atb_f64(int64_t n_rows, int64_t n_cols, const int32_t *a_col_ptr, const int32_t *a_row_idx,
                     const double *a_vals, const int32_t *b_col_ptr, const int32_t *b_row_idx,
                     const double *b_vals, int64_t nnz_a, int64_t nnz_b, double *out, void *ws,
                     size_t ws_bytes, void *stream);
/* Trace kernel selection (tests and measurements only): 0 = automatic (the
 * tile kernel: column-pair tiles staged by bulk copies, lanes merging list
 * segments; falls back when the row arrays are not 16-byte aligned), 1 = the
 * warp-per-column kernel.  Process-wide. */
int as_set_trace_engine(int engine);

/* ---------------------------------------------------------------------------
 * Multi-GPU (no reference counterpart): one process per GPU.
 * The caller creates the NCCL communicator (ncclCommInitRank, or the one its
 * framework owns) and hands it over; NCCL's entry points are resolved at run
 * time from the libnccl the process has loaded (`nccl_library`: a path to try
 * first, or NULL for libnccl.so.2), so the library has no link-time
 * dependency on NCCL.  Each as_mg_* op is the rank-local kernel followed by
 * its collective on the caller's stream; paper_1805_03380_b200/dist.py is the
 * torch.distributed twin (it also gathers SpGEMM slices onto one rank, whose
 * variable-size exchange needs host-side sizing).
 *
 * as_mg_trace_atb_f64: trace(A^T B) over this rank's columns [c0, c1) (full
 *   A and B on every rank; dist.trace_shard balances the ranges), then an
 *   all-gather of the ranks' (sum, residual) pairs combined in rank order with
 *   TwoSum carries: every rank gets the same out[0..1], independent of the
 *   reduction tree.  ws: as_mg_trace_workspace_bytes.
 * as_mg_spmm_csr_f32: C = A @ B with A's CSR replicated and the k dense
 *   columns split evenly (k % world == 0, ldc == n_rows): rank r multiplies
 *   columns [r k / world, (r + 1) k / world) and the blocks are all-gathered
 *   in place into every rank's C.  ws: as_spmm_workspace_bytes.
 * as_mg_spgemm_f64: as_spgemm_f64 on this rank's standalone column slice of B
 *   (dist.spgemm_shard: ranges of equal Gustavson products; A replicated),
 *   then one all-gather of the slices' nnz: slice_nnz[world] (device) and
 *   slice_offset[0] = this slice's first element in the concatenation of all
 *   slices.  C stays distributed (dist.DistCsc); nothing is read on the host.
 */
int as_mg_init(void *nccl_comm, int rank, int world, const char *nccl_library);
int as_mg_shutdown(void);
int as_mg_rank(void);
int as_mg_world(void);
size_t as_mg_trace_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b, int world);
int as_mg_trace_atb_f64(int64_t n_rows, int64_t n_cols, const int32_t *a_col_ptr, const int32_t *a_row_idx,
                        const double *a_vals, const int32_t *b_col_ptr, const int32_t *b_row_idx,
                        const double *b_vals, int64_t nnz_a, int64_t nnz_b, int64_t c0, int64_t c1, double *out,
                        void *ws, size_t ws_bytes, void *stream);
int as_mg_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t *row_ptr, const int32_t *col_idx,
                       const float *vals, const float *B, int64_t ldb, float *C, int64_t ldc, void *ws,
                       size_t ws_bytes, void *stream);
int as_mg_spgemm_f64(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t *a_col_ptr,
                     const int32_t *a_row_idx, const double *a_vals, const int32_t *b_col_ptr,
                     const int32_t *b_row_idx, const double *b_vals, int64_t nnz_b, const int64_t *prod_ptr,
                     int64_t total_products, int32_t *col_ptr, int32_t *row_idx, double *out_vals,
                     int64_t *info, void *ws, size_t ws_bytes, int64_t *slice_nnz, int64_t *slice_offset,
                     void *stream);

/* ---------------------------------------------------------------------------
 * construction-funnelled ops and segmented reductions of the
 * reference's ops module (csrc/funnel.cu).
 *
 * as_expand_cols: column index of every CSC element (CscData.expand_cols).
 * as_kron_triplets_f64 / as_repmat_triplets_f64: the triplets ops.kron
 *   (ops.py:131-143) / ops.repmat (ops.py:146-163) hand to canonicalize, in
 *   the same order; the caller funnels them through as_coo_to_csc_f64.
 * as_segment_reduce_f64: per segment (CSC column, or CSR row) kind 0 = the
 *   sequential fold of np.add.at (ops.py:182-185), 1 / 2 = min / max with the
 *   implicit zero of a non-dense slice (ops.py:186-193), 3 = max of an
 *   empty-safe |x| (norms); xf transforms each value first (0 x, 1 |x|,
 *   2 x*x, 3 |x|**p).  full = the slice length (rows for columns).
 * as_pairwise_sum_f64: np.sum's pairwise summation of (transformed) x in its
 *   exact association order (trace, norms: ops.py:209-248); out[0].
 * as_csc_window_f64: ops.submat (ops.py:277-298) rows [r0,r1] x cols [c0,c1];
 *   outputs sized for the window's nnz bound, info[0] = nnz.
 * as_csc_diag_f64: ops.diag (ops.py:345-355), diagonal k as a dense vector.
 * as_scale_by_label_f64: out = vals / norms[labels] (0 norms count as 1),
 *   ops.normalise (ops.py:251-274) before its re-canonicalisation.
 */
int as_expand_cols(int64_t n_cols, const int32_t *col_ptr, int32_t *cols, void *stream);
int as_kron_triplets_f64(int64_t nnz_a, const int32_t *a_rows, const int32_t *a_cols, const double *a_vals,
                         int64_t nnz_b, const int32_t *b_rows, const int32_t *b_cols, const double *b_vals,
                         int64_t b_n_rows, int64_t b_n_cols, int32_t *rows, int32_t *cols, double *vals,
                         void *stream);
int as_repmat_triplets_f64(int64_t nnz, const int32_t *a_rows, const int32_t *a_cols, const double *a_vals,
                           int64_t n_rows, int64_t n_cols, int64_t reps_r, int64_t reps_c, int32_t *rows,
                           int32_t *cols, double *vals, void *stream);
int as_segment_reduce_f64(int64_t n_seg, const int32_t *seg_ptr, const double *vals, int kind, int xf, double p,
                          int64_t full, double *out, void *stream);
size_t as_pairwise_workspace_bytes(void);
int as_pairwise_sum_f64(int64_t n, const double *x, int xf, double p, double *out, void *ws, size_t ws_bytes,
                        void *stream);
size_t as_window_workspace_bytes(int64_t n_out_cols);
int as_csc_window_f64(int64_t n_rows, int64_t n_cols, const int32_t *col_ptr, const int32_t *row_idx,
                      const double *vals, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int32_t *out_col_ptr,
                      int32_t *out_rows, double *out_vals, int64_t *info, void *ws, size_t ws_bytes, void *stream);
int as_csc_diag_f64(int64_t n_rows, int64_t n_cols, const int32_t *col_ptr, const int32_t *row_idx,
                    const double *vals, int64_t k, int64_t length, double *out, void *stream);
int as_scale_by_label_f64(int64_t nnz, const int32_t *labels, const double *vals, const double *norms, double *out,
                          void *stream);

/* ---------------------------------------------------------------------------
 * Matrix Market coordinate I/O (io.py:33-132), HOST functions
 * (csrc/mmio.cu), multi-threaded; the triplets then go to as_coo_to_csc_f64.
 * as_mm_header: header + size line; as_mm_entries: the entries as 0-based
 *   int64 rows / cols and float64 values, validated in the reference's order
 *   (AS_ERR_ARG = MatrixMarketError, AS_ERR_CORRUPT = CorruptionError, with
 *   *err_line the reference's 1-based line number, as_last_error() the bare
 *   message); as_mm_format: "%d %d %.17g" lines after the header, returns
 *   the byte count (cap >= 64 + 72 * nnz suffices) or -1.
 */
int as_mm_header(const char *buf, int64_t len, int64_t *n_rows, int64_t *n_cols, int64_t *nnz, int64_t *entries_off,
                 int64_t *entries_line, int64_t *err_line);
int as_mm_entries(const char *buf, int64_t len, int64_t entries_off, int64_t entries_line, int64_t n_rows,
                  int64_t n_cols, int64_t nnz, int64_t *rows, int64_t *cols, double *vals, int n_threads,
                  int64_t *err_line);
int64_t as_mm_format(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t *rows, const int64_t *cols,
                     const double *vals, char *out, int64_t cap, int n_threads);

#ifdef __cplusplus
}
#endif

#endif /* BSPARSE_H_ */
