/*
 * sketchcu: C ABI of the B200 (sm_100a) hot path of preconditioned data
 * sparsification (arXiv 1511.00152).
 *
 * This is the drop-in boundary. Every entry point replaces one call of the reference
 * package `sketchpipe` (/root/reference/pkg/src/sketchpipe). Each one cites its
 * reference file:line. The reference has no FFI of its own because it is pure Python,
 * so these entry points are what its ctypes binding would call; see INTEGRATION.md.
 *
 * Conventions:
 *  - Plain device pointers and sizes. No framework types appear in any signature.
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy default stream.
 *    Every call is stream-ordered and asynchronous unless stated otherwise.
 *  - Samples are rows. X is (n, p) row-major with row stride `ld` elements, which is
 *    the reference's (p, n) column matrix in Fortran order. Sketch indices/values are
 *    (n, m) row-major, the same as SparseSketch.indices/.values (sketch.py:64-77).
 *  - Centres are (p_pad, K) row-major fp64, the same as CenterSet.centers (cluster.py:28-32).
 *  - Return value: SKC_OK, or an error code with a message from skc_last_error().
 *    SKC_EDIM maps to the reference's DimensionError and SKC_EPARAM to ParameterError
 *    (errors.py:4-9). Validation runs before any work is enqueued.
 *  - Outputs marked "+=" accumulate, so partials from several calls, chunks or ranks
 *    add up. Outputs marked "=" are overwritten.
 */
#ifndef SKETCHCU_H
#define SKETCHCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SKC_OK = 0, SKC_EDIM = 1, SKC_EPARAM = 2, SKC_ECUDA = 3, SKC_ENCCL = 4 };
/* transform kinds, transform.py:20-23 (DCT is outside the GPU hot path: SKC_EPARAM) */
enum { SKC_KIND_HADAMARD = 0, SKC_KIND_DCT = 1, SKC_KIND_NONE = 2 };
enum { SKC_F32 = 0, SKC_F64 = 1 };

/* Thread-local message for the last non-OK return on this thread. */
const char *skc_last_error(void);
int skc_abi_version(void);
/* Largest p_pad the kernels are instantiated for (4096). */
int32_t skc_max_p_pad(void);
/* Number of kernels this library has launched in the process (for launch accounting). */
uint64_t skc_launch_count(void);
/* Add kernels a replayed CUDA graph ran (skc_kmeans_lloyd) to skc_launch_count. */
void skc_count_launches(uint64_t kernels);

/* --- L0/L1: signs and transform -------------------------------------------------- */

/* D diagonal as fp64 +-1 (all ones for kind NONE) = PreconditionSpec.signs(),
 * transform.py:71-82 -> _hash.sign_array, _hash.py:38-43. out: device[p_pad] (=). */
int skc_signs(uint64_t sign_seed, int32_t p_pad, int32_t kind, double *out, void *stream);

/* precondition_columns, transform.py:180-189, for n rows: Y = H D pad(X). Y: (n, p_pad)
 * fp64 (=). fp64 arithmetic in the reference's butterfly order, so it is bit-exact. */
int skc_precondition(const void *X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                     int32_t kind, uint64_t sign_seed, double *Y, void *stream);

/* unprecondition_columns, transform.py:192-200: X = D^T H^T Y, keeping the first p_out
 * columns (the [:p] truncation of estimators.py:45/129 and cluster.py:388). Y: (n, p_pad)
 * fp64, X: (n, p_out) fp64 (=). Bit-exact. */
int skc_unprecondition(const double *Y, int64_t n, int32_t p_pad, int32_t kind, uint64_t sign_seed, int32_t p_out,
                       double *X, void *stream);

/* Normalised WHT of n rows of length p_pad (fwht_inplace / _fwht_axis0,
 * transform.py:92-122), fp64 in the reference stage order: bit-exact. X may alias Y. */
int skc_fwht(const double *Y, int64_t n, int32_t p_pad, double *X, void *stream);

/* --- L2: sampling plan and the fused single-pass sketch ------------------------------ */

/* SamplingPlan.indices_block(col0, col0+n), sketch.py:48-56. The m smallest splitmix64
 * keys of each column, sorted ascending (=). Bit-exact. */
int skc_indices(uint64_t master_seed, int64_t col0, int64_t n, int32_t p_pad, int32_t m, int32_t *idx_out,
                void *stream);

/* sketch_stream body, sketch.py:196-223, for rows [0, n) of X, which are global columns
 * [col0, col0+n). One pass: zero-pad, signs, normalised WHT, m-of-p_pad selection,
 * gather. compute_dtype SKC_F64 reproduces the reference values bit for bit;
 * SKC_F32 is the fast path (about 1e-7 relative). Indices are bit-exact in both.
 * idx_out: (n, m) int32, val_out: (n, m) of val_dtype (=). */
int skc_sketch(const void *X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
               uint64_t sign_seed, uint64_t master_seed, int64_t col0, int32_t m, int32_t compute_dtype,
               int32_t *idx_out, void *val_out, int32_t val_dtype, void *stream);

/* --- L3a: estimators ------------------------------------------------------------------ */

/* Mean accumulation of estimate_mean, estimators.py:39-43: acc[j] += sum of values with
 * index j (fp64, deterministic order). Also stats[0] += sum of squared values,
 * stats[1] = max(stats[1], max |value|), and stats[2] += n, which feed
 * skc_cov_accumulate's fixed-point scale. acc: device[p_pad], stats: device[3]. */
size_t skc_moments_workspace(int64_t n, int32_t m, int32_t p_pad);
int skc_moments(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                double *acc, double *stats, void *workspace, size_t ws_bytes, void *stream);

/* estimate_mean tail, estimators.py:44-45: mean = unprecondition((p_pad/m)*acc/n_total)[:p]
 * mean: device[p] (=). */
int skc_mean_finalize(const double *acc, int32_t p, int32_t p_pad, int32_t m, int64_t n_total, int32_t kind,
                      uint64_t sign_seed, double *mean, void *stream);

/* Raw second moment of estimate_covariance, estimators.py:59-61: the W W^T upper
 * triangle, packed row-major (entry (a,b), a<=b, at a*p_pad - a*(a-1)/2 + (b-a)), +=
 * into tri[p_pad*(p_pad+1)/2] fp64. Each product w_a*w_b is formed in fp32 from the
 * fp32-rounded values (relative error <= 2^-23 per product, also in f64 mode), scaled by
 * 2^S (S from stats, skc_moments) and added as an integer: int32 fixed-point shared-memory
 * accumulators through native ATOMS.ADD with carries to int64. Values above 8x the rms, or a
 * scale outside the float range, take exact fp64 products. Integer sums make the result
 * deterministic and order-independent. Measured relative Frobenius error against the
 * reference's fp64: 2.5e-9 (C3, n=2^24) to 1.2e-7 (C4, n=2^21), tests/test_full_configs.py;
 * the north_star bound is 1e-5.
 * For launches of 2^20 rows or more the shared-memory kernel keeps a small per-process table of
 * band boundaries per (device, p_pad, m, val_dtype) and tunes it over the first three launches from
 * per-band cycle counts read back asynchronously (pinned memory, no synchronisation); the result
 * does not depend on it. SKC_COV_ADAPT=0 disables the tuning. */
size_t skc_cov_workspace(int64_t n, int32_t m, int32_t p_pad);
int skc_cov_accumulate(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                       int32_t p_pad, const double *stats, double *tri, void *workspace, size_t ws_bytes,
                       void *stream);

/* estimate_covariance tail, estimators.py:62-65: scale by (p(p-1)/(m(m-1)))/n_total,
 * symmetrise, debias the diagonal. C: device[p_pad*p_pad] fp64 (=). */
int skc_cov_finalize(const double *tri, int32_t p_pad, int32_t m, int64_t n_total, double *C, void *stream);

/* --- L3b: sparsified K-means ---------------------------------------------------------- */

/* _SparseOps.init_centers, cluster.py:175-179: mu[:,k] = sparse column chosen[k] (=). */
int skc_kmeans_init(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                    const int64_t *chosen, int32_t K, int32_t p_pad, double *mu, void *stream);

/* _SparseOps.assign, cluster.py:181-187, in the reference's fp64 operation order
 * (CSR x dense axpy order, numpy pairwise row norm), so labels and d2min are bit-exact.
 * labels (n) int32, d2min (n) fp64 (=). If prev_labels is non-NULL, out[0] = number of
 * labels that differ from prev_labels. out[1] = first index of max d2min, which is the
 * reseed point of cluster.py:213. d2max[0] = that max value. */
size_t skc_kmeans_assign_workspace(int64_t n, int32_t p_pad, int32_t K);
int skc_kmeans_assign(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                      const double *mu, int32_t p_pad, int32_t K, const int32_t *prev_labels, int32_t *labels,
                      double *d2min, int64_t *out, double *d2max, void *workspace, size_t ws_bytes,
                      void *stream);

/* skc_kmeans_assign with the tensor-core filter (K5t, kmeans_tc.cu): identical results
 * (labels, d2min, out, d2max bit-identical to skc_kmeans_assign). The sketch is prepared
 * once (compact bf16 entries + numpy-order row norms) into prep with skc_kmeans_tc_prepare;
 * each call builds the bf16 table of [-2 mu ; mu*mu], filters on tcgen05 and verifies the
 * candidates in fp64. Applies when skc_kmeans_tc_supported(p_pad, K, m): p_pad % 32 == 0,
 * K <= 128. Replaces _SparseOps.assign, cluster.py:181-187 (the same contract as above). */
int skc_kmeans_tc_supported(int32_t p_pad, int32_t K, int32_t m);
size_t skc_kmeans_tc_prepare_workspace(int64_t n, int32_t m, int32_t p_pad);
int skc_kmeans_tc_prepare(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                          void *prep, size_t prep_bytes, void *stream);
size_t skc_kmeans_assign_tc_workspace(int64_t n, int32_t p_pad, int32_t K);
int skc_kmeans_assign_tc(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                         const double *mu, int32_t p_pad, int32_t K, const int32_t *prev_labels, int32_t *labels,
                         double *d2min, int64_t *out, double *d2max, const void *prep, void *workspace,
                         size_t ws_bytes, void *stream);

/* numpy pairwise summation of x[0..n) (objective = d2min.sum(), cluster.py:233). Bit-exact
 * to ndarray.sum. out: device[1] (=). */
size_t skc_pairwise_sum_workspace(int64_t n);
int skc_pairwise_sum(const double *x, int64_t n, double *out, void *workspace, size_t ws_bytes, void *stream);

/* _SparseOps.update partial sums, cluster.py:189-208: per (j,k) value sums (fp64) and
 * sampling counts (int64), plus cluster sizes n_k (int64). Points are grouped by label
 * with a stable counting sort and summed in fixed chunks, so the result is deterministic.
 * sums/counts: (p_pad, K), sizes: (K) (=). */
size_t skc_kmeans_partials_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K);
int skc_kmeans_partials(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                        const int32_t *labels, int32_t p_pad, int32_t K, double *sums, int64_t *counts,
                        int64_t *sizes, void *workspace, size_t ws_bytes, void *stream);

/* cluster.py:196-210: mu_out[j,k] = sums/counts where counts > 0, else mu_prev. An empty
 * cluster (sizes[k]==0) keeps mu_prev[:,k] and sets empty[k]=1. mu_out (=), empty (K) int32 (=). */
int skc_kmeans_centers(const double *sums, const int64_t *counts, const int64_t *sizes, const double *mu_prev,
                       int32_t p_pad, int32_t K, double *mu_out, int32_t *empty, void *stream);

/* _SparseOps.reseed, cluster.py:212-215, for every k with empty[k]: mu[:,k] = 0 except
 * the m sampled coordinates of the reseed point (idx_c, val_c: one sketch row). */
int skc_kmeans_reseed(const int32_t *idx_c, const void *val_c, int32_t val_dtype, int32_t m, const int32_t *empty,
                      int32_t p_pad, int32_t K, double *mu, void *stream);

/* The same partial sums through a transposed sketch that is built once and reused every
 * iteration: per-coordinate lists ascending in point index (a stable counting sort by
 * coordinate). skc_kmeans_partials_csc then sums each (coordinate, cluster) chain
 * sequentially in point order, exactly np.bincount's order in cluster.py:203-205, so sums
 * are bit-identical to the reference. csc: skc_kmeans_csc_workspace bytes (device), kept
 * alive between the calls; skc_kmeans_partials runs both steps in one call. Per
 * iteration each coordinate's list is split into segments, labels are counted per
 * segment, a scan makes every (coordinate, cluster) chain contiguous, values are scattered
 * stably, and one thread adds each chain in order. */
size_t skc_kmeans_csc_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t val_dtype);
int skc_kmeans_build_csc(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                         void *csc, size_t csc_bytes, void *stream);
/* seg: skc_kmeans_seg_workspace bytes of per-iteration scratch (labels per entry, the
 * values in chain order, segment offsets). K <= 256. sizes may be NULL when the caller does not
 * need the cluster sizes (they follow from the counts: sum_j counts[j][k] = m * n_k, SPEC.md:297;
 * skc_kmeans_lloyd's finish kernel uses that). */
size_t skc_kmeans_seg_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K, int32_t val_dtype);
int skc_kmeans_partials_csc(const void *csc, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                            const int32_t *labels, int32_t K, double *sums, int64_t *counts, int64_t *sizes, void *seg,
                            size_t seg_bytes, void *stream);

/* skc_kmeans_reseed with the point given on the device: row = max(*row, 0) (the argmax that
 * skc_kmeans_assign writes to out[1]), so a Lloyd iteration can be enqueued before the host
 * reads its convergence flag. idx/val are the whole (n, m) sketch. */
int skc_kmeans_reseed_at(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                         const int64_t *row, const int32_t *empty, int32_t p_pad, int32_t K, double *mu, void *stream);

/* The whole Lloyd loop of _lloyd_iterate (cluster.py:230-241) from centres mu0, device-resident:
 * ONE CUDA graph with a conditional WHILE node runs the iterations (assign, numpy-order objective,
 * convergence test on the device, partial sums through csc, centres, reseed) with no host round
 * trip; it is built once per argument set and relaunched. The assignment, objective-leaf and
 * partial-sum kernels are those of the host-driven loop; the objective's combine + check and the
 * centres + reseed + commit step are each one kernel (the latter takes "cluster empty" from the
 * counts), with the same arithmetic, so labels, mu and the objective trajectory are bit-identical
 * to the host-driven loop.
 * csc: from skc_kmeans_build_csc (required). tc_prep: from skc_kmeans_tc_prepare, or NULL (then
 * every assignment uses skc_kmeans_assign; otherwise iterations 2.. use the tensor-core filter).
 * ws: skc_kmeans_lloyd_workspace bytes. Outputs (device, =): labels (n) int32 of the last
 * assignment, mu (p_pad, K) the centres it used (updated when max_iter ends the loop), traj
 * (max_iter) fp64 objectives of the executed iterations, iters[0] their count. Asynchronous. */
size_t skc_kmeans_lloyd_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K, int32_t val_dtype, int32_t use_tc);
int skc_kmeans_lloyd(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                     int32_t K, const double *mu0, int32_t max_iter, const void *csc, const void *tc_prep, void *ws,
                     size_t ws_bytes, int32_t *labels, double *mu, double *traj, int32_t *iters, void *stream);
/* sparsified_assign, cluster.py:306-311, for ONE sketch column (idx_row, val_row: m entries,
 * device): argmin_k of (diff * diff).sum(axis=0) with diff = val[:, None] - mu[idx, :], in the
 * reference's own order (a sequential fp64 sum over the m coordinates, np.argmin ties to the
 * lowest k). label_out[0] (=), d2_out[0] (=, may be NULL). */
int skc_kmeans_assign_one(const int32_t *idx_row, const void *val_row, int32_t val_dtype, int32_t m, const double *mu,
                          int32_t p_pad, int32_t K, int32_t *label_out, double *d2_out, void *stream);
/* Kernels in the last skc_kmeans_lloyd graph of this thread: a run launches prologue + (iters - 1) * body. */
void skc_kmeans_lloyd_graph_kernels(int32_t *prologue, int32_t *body);

/* Row norms ||v_i||^2 of the sketch in numpy's pairwise order (the colsq of
 * cluster.py:148). out: (n) fp64 (=). */
int skc_row_sqnorms(const void *val, int32_t val_dtype, int64_t n, int32_t m, double *out, void *stream);

/* _SparseOps.d2_to_point, cluster.py:169-173: out[i] = (p_pad/m) * max(0, colsq[i] +
 * colsq[c] - 2 <w_i, w_c>). The inner product runs over shared coordinates in the row's
 * index order, as scipy's sparse product does. dense: device[p_pad] scratch. out: (n)
 * fp64 (=). */
int skc_kmeans_d2_to_point(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                           int32_t p_pad, int64_t c, const double *colsq, double *dense, double *out, void *stream);

/* skc_kmeans_d2_to_point for a point c held by ANOTHER shard (sharded K-means++ seeding):
 * the caller supplies W[:, c] densified (dense: device[p_pad], e.g. from the allreduced
 * init_centers column) and colsq[c] (dense_sq: device[1]). Same arithmetic, so the global
 * D^2 vector equals the unsharded one bit for bit. out: (n) fp64 (=). */
int skc_kmeans_d2_to_dense(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                           int32_t p_pad, const double *dense, const double *dense_sq, const double *colsq,
                           double *out, void *stream);

/* ---- Philox sampler and supplied-index sketching -----------------------------------
 * north_star's counter-based alternative to the reference hash (not reference-identical;
 * restated bit for bit by oracle/sketch_oracle.c:orc_philox_indices). Column g = col0 + i
 * draws m of p_pad coordinates without replacement with Floyd's algorithm on a
 * Philox4x32-10 stream keyed by mix64(master_seed ^ 0x50484C58); idx_out (n, m) int32,
 * ascending per row. Same role as skc_indices (sketch.py:48-56). */
int skc_indices_philox(uint64_t master_seed, int64_t col0, int64_t n, int32_t p_pad, int32_t m, int32_t *idx_out,
                       void *stream);
/* Sketch values at supplied indices: val_out[i][t] = precondition(x_i)[idx_in[i][t]].
 * idx_in is (n, m) int32, each row strictly increasing (from skc_indices,
 * skc_indices_philox, or the reference in oracle mode). Arguments as skc_sketch. */
int skc_sketch_given(const void *X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
                     uint64_t sign_seed, int32_t m, int32_t compute_dtype, const int32_t *idx_in, void *val_out,
                     int32_t val_dtype, void *stream);

/* ---- native streaming runtime ---------------------------------------------------------
 * sketch_stream + estimators.py:30-66 over host rows without keeping the sketch (the loop of
 * stream_moments, in C++). host_X: (n, p) rows, row stride ld, fp32 or fp64; pinned host
 * memory gives asynchronous copies. Chunks of chunk_rows are copied on a private stream into
 * two device buffers while the previous chunk's sketch, moments and covariance run on
 * `stream`; events gate buffer reuse. acc / stats / tri accumulate (+=) as in skc_moments /
 * skc_cov_accumulate; tri may be NULL (mean only). sampler: 0 oracle, 1 philox.
 * ws: skc_stream_workspace bytes (device). */
size_t skc_stream_workspace(int64_t chunk_rows, int32_t p, int32_t p_pad, int32_t m, int32_t x_dtype,
                            int32_t compute_dtype, int32_t covariance);
int skc_stream_moments(const void *host_X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                       int32_t kind, uint64_t sign_seed, uint64_t master_seed, int64_t col0, int32_t m,
                       int32_t compute_dtype, int32_t sampler, int64_t chunk_rows, double *acc, double *stats,
                       double *tri, void *ws, size_t ws_bytes, void *stream);

/* ---- SKCH1 file records (io.py:84-136) ---------------------------------------------
 * A record is the sample's m u32 indices followed by its m f64 values, 12 m bytes, no
 * padding; the file is a 61-byte header then n records. pack: (idx, val) -> out_words
 * (n * 3m u32, device); fp32 values widen exactly to f64. unpack: the inverse into int32
 * indices and f64 values. Replaces the numpy structured-dtype copies of write_sketch /
 * read_sketch (io.py:88-136). */
int skc_sketch_pack_records(const int32_t *idx, const void *val, int32_t val_dtype, int64_t n, int32_t m,
                            uint32_t *out_words, void *stream);
int skc_sketch_unpack_records(const uint32_t *words, int64_t n, int32_t m, int32_t *idx_out, double *val_out,
                              void *stream);

/* ---- Two-pass K-means, second pass (cluster.py:407-456) ------------------------------
 * Rows X (n, p) with leading dimension ld, fp32 or fp64; centres mu (K, p) fp64 row-major
 * (original domain, the first pass's mu_hat transposed).
 * skc_dense_assign: labels[i] = first argmin_k (|x_i|^2 - 2 <x_i, mu_k>) + |mu_k|^2 and
 *   d2min[i] = max(that minimum, 0) (cluster.py:437-440); ws: skc_dense_assign_workspace bytes
 *   (centre norms and a transposed, padded copy of mu).
 * skc_dense_sums: sums[k] += sum of rows with labels[i] == k, counts[k] += their number
 *   (cluster.py:434-436, 445); fp64 in a fixed order. ws: skc_dense_sums_workspace bytes. */
size_t skc_dense_assign_workspace(int32_t p, int32_t K);
int skc_dense_assign(const void *X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, const double *mu, int32_t K,
                     void *ws, int32_t *labels, double *d2min, void *stream);
size_t skc_dense_sums_workspace(int64_t n, int32_t p, int32_t K);
int skc_dense_sums(const void *X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, const int32_t *labels, int32_t K,
                   double *sums, int64_t *counts, void *ws, void *stream);

/* ---- device top-k eigensolve --------------------------------------
 * top_eigenvectors(C, k), estimators.py:69-81, on the device: the k largest eigenpairs of
 * 0.5 * (C + C^T) (C: p x p fp64, device) by cuSOLVER syevdx over the index range [p-k+1, p]
 * (only k eigenvectors are formed). V: (p, k) row-major, columns in descending eigenvalue order
 * (the reference's V[:, ::-1][:, :k]); w: (k) descending eigenvalues, may be NULL (=).
 * Eigenvector signs are arbitrary, as in LAPACK. ws: skc_top_eigenvectors_workspace bytes. */
size_t skc_top_eigenvectors_workspace(int32_t p, int32_t k);
int skc_top_eigenvectors(const double *C, int32_t p, int32_t k, double *V, double *w, void *ws, size_t ws_bytes,
                         void *stream);

/* ---- sample-sharded exchange (SURVEY 8(e); SPEC.md:212, :352 ordered combine of partials) ----
 * Rank r holds global columns [col0, col0 + n) and runs every entry point above on its shard
 * with that col0. Per pass, ONE fp64 SUM allreduce of the packed moments buffer
 * [acc (p_pad) | stats (3) | triangle] (skc_moments_packed_len; stats[1] becomes the sum of the
 * ranks' maxima, an upper bound that is all a later K3t scale needs). Per Lloyd iteration, ONE
 * allreduce of the packed K-means exchange (skc_kmeans_pack_exchange: the partials of
 * skc_kmeans_partials*, the changed count and objective, and per rank its max d2min with the
 * global row of its first argmax, from which every rank picks the reseed point), then
 * skc_kmeans_unpack_exchange -> skc_kmeans_centers. NCCL is dlopen'ed ("libnccl.so.2"); comm is
 * an ncclComm_t (void*); NCCL failures return SKC_ENCCL. */
int skc_nccl_get_unique_id(void *id_out /* 128 bytes: ncclUniqueId */);
int skc_nccl_comm_init_rank(void **comm_out, int32_t nranks, const void *id, int32_t rank);
int skc_nccl_comm_destroy(void *comm);
/* In-place fp64 SUM allreduce on `stream` (ncclAllReduce). */
int skc_allreduce_sum_f64(double *buf, size_t count, void *comm, void *stream);
size_t skc_moments_packed_len(int32_t p_pad, int32_t covariance);
size_t skc_kmeans_exchange_len(int32_t p_pad, int32_t K, int32_t world);
/* buf (skc_kmeans_exchange_len doubles, =): sums, counts (as exact fp64), sizes, out[0]
 * (changed), *objective, and this rank's slot (d2max[0], col0 + out[1]); other slots zero. */
int skc_kmeans_pack_exchange(const double *sums, const int64_t *counts, const int64_t *sizes, const int64_t *out,
                             const double *d2max, const double *objective, int32_t p_pad, int32_t K, int32_t rank,
                             int32_t world, int64_t col0, double *buf, void *stream);
int skc_kmeans_unpack_exchange(const double *buf, int32_t p_pad, int32_t K, double *sums, int64_t *counts,
                               int64_t *sizes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SKETCHCU_H */
