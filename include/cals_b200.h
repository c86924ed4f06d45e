/*
 * cals_b200.h -- C ABI of the B200-native CALS (Concurrent ALS, arXiv
 * 2010.04678) hot path.  Plain C types only: device pointers are `double*`,
 * streams are `cudaStream_t` passed as `void*` (0 = legacy default stream).
 *
 * The reference (arxiv/paper_2010_04678, pure-Python package `cals`) has no
 * native ABI of its own; its hot path calls numpy/scipy -> OpenBLAS/LAPACK.
 * Each entry point below names the reference interface it replaces
 * (file:line into pkg/src/cals).  Python binding: paper_2010_04678_b200/_native.py
 * (ctypes); other bindings: INTEGRATION.md.
 *
 * Conventions
 *   - every function returns 0 on success or a negative error code
 *     (-1 invalid argument, -2 CUDA failure, -3 capacity, -4 unsupported);
 *     cals_last_error() returns a thread-local message;
 *   - no exceptions cross the ABI; no allocation inside cals_mttkrp /
 *     cals_update_factor / cals_engine_run's iteration loop;
 *   - all calls are stream-ordered; one engine per device, not thread-safe
 *     per handle (the reference's orchestrator is single-threaded too,
 *     SPEC.md:453);
 *   - factor / output buffers are ROW-major [I_n][ld] with ld even, so one
 *     factor row of every concurrent model is contiguous.  The reference's
 *     multi-matrices are Fortran (I_n, R*) (multimatrix.py:41); the host
 *     layer transposes at admission / retirement only.
 */
#ifndef CALS_B200_H_
#define CALS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CALS_B200_ABI_VERSION 1

typedef struct cals_tensor cals_tensor;
typedef struct cals_engine cals_engine;

int cals_abi_version(void);
const char* cals_last_error(void);

/* ---- dense tensor (replaces tensor.py:15-89 DenseTensor storage) -------
 * Exactly one of host_data / device_data is non-null.  Data is mode-0
 * fastest (tensor.py:1-5).  The device copy pads I0 to an even extent (zero
 * fill) so every TMA stride is 16-byte aligned; an already aligned device
 * buffer with even I0 is borrowed, not copied. */
int cals_tensor_create(int order, const int64_t* dims, const double* host_data,
                       const double* device_data, void* stream, cals_tensor** out);
int cals_tensor_destroy(cals_tensor* t);
/* ||T||^2 on the device, computed once (tensor.py:77-82 `sqnorm`). */
int cals_tensor_sqnorm(cals_tensor* t, void* stream, double* out);
int cals_tensor_data(cals_tensor* t, double** data, int64_t* padded_i0);

/* ---- fused MTTKRP (replaces mttkrp.py:157-209 `_mttkrp_core`, called via
 * mttkrp.py:212-231 `mttkrp` and mttkrp.py:234-256 `fused_mttkrp`) --------
 * out[i][c] = sum over the other modes' indices of T * prod_{m != mode}
 * factors[m][i_m][c]  for i < I_mode, c < width   (T_(n) @ KRP, descending
 * mode order as in mttkrp.py:117-118).  factors[mode] is ignored (may be
 * null).  ldf, ldo even, >= width.  variant < 0 picks the tile shape. */
int cals_mttkrp_workspace_bytes(cals_tensor* t, int mode, int64_t capacity, size_t* bytes);
int cals_mttkrp(cals_tensor* t, int mode, int width, const double* const* factors, int64_t ldf,
                double* out, int64_t ldo, double* workspace, size_t workspace_bytes, int variant,
                void* stream);
int cals_mttkrp_variants(int* count);
/* Which kernel the MTTKRP of `mode` runs on at `width` (0 = FP64 DMMA,
 * 1 = Ozaki-sliced INT8 tcgen05) and the tensor-core operations one launch
 * executes on it (FP64 flops incl. tile padding, or INT8 ops incl. the 28
 * slice products and padding) -- for roofline accounting. */
int cals_mttkrp_kernel_info(cals_tensor* t, int mode, int64_t width, int32_t* kernel,
                            double* tensor_ops);

/* ---- factor update (replaces als.py:74-96 `update_factor`) -------------
 * a = m h^{-1} for one rows x rank block (row-major m, a; h rank x rank):
 * upper Cholesky + triangular solves, eigen-pinv fallback with cutoff
 * 1e-12 * max(lambda_max, 0).  *status (device int) = 1 when m or h held
 * non-finite values (the reference raises ValueError), else 0.
 * scratch: cals_update_scratch_bytes(rank) bytes of device memory. */
int cals_update_factor(int rows, int rank, const double* m, int64_t ldm, const double* h,
                       double* a, int64_t lda, double* scratch, int* status, void* stream);
size_t cals_update_scratch_bytes(int rank);

/* ---- device-resident CALS driver (replaces driver.py:185-307 `_run_cals`)
 * ranks[k] for the queued models in FIFO order; r_star = column capacity
 * (multimatrix.py:19, 123-167).  The starting factors live in the engine's
 * pool: per model k, per mode n, a COLUMN-major I_n x ranks[k] block (the
 * reference's Fortran factor, model.py:26-39, byte for byte), models in
 * queue order, modes ascending (cals_engine_pool gives the device pointer;
 * cals_engine_load_pool copies from host or device).  Results are written
 * back into the same pool; the engine transposes to its row-major
 * multi-matrices only at admission / retirement. */
int cals_engine_create(cals_tensor* t, int r_star, int n_models, const int32_t* ranks,
                       int trace_capacity, cals_engine** out);
int cals_engine_destroy(cals_engine* e);
/* Re-bind an engine (and its device workspaces) to another tensor of the same
 * shape, so repeated sweeps reuse every allocation. */
int cals_engine_set_tensor(cals_engine* e, cals_tensor* t);
/* Enqueue the once-per-tensor preparation of the engine's INT8 tensor-core
 * views (tensor slicing) on `stream` without waiting: lets it overlap host
 * work before cals_engine_run (which finishes and checks it). */
int cals_engine_prepare(cals_engine* e, void* stream);
int cals_engine_pool(cals_engine* e, double** pool, int64_t* elems);
int cals_engine_load_pool(cals_engine* e, const double* src, int src_is_device, void* stream);
/* Runs until every model has retired (ConvergenceConfig semantics,
 * als.py:24-37: tol <= 0 disables the fit test).  sqnorm = ||T||^2 as used
 * by the fast error.  *iterations = driver iterations executed. */
int cals_engine_run(cals_engine* e, double tol, int max_iterations, double sqnorm, int use_graph,
                    void* stream, int* iterations);
/* Host outputs (any may be null): status (0 pending, 1 active, 2 converged,
 * 3 iteration_cap, 4 failed -- model.py:13-18), iterations_done, error, fit,
 * retirement sequence number (the reference's output-queue order,
 * driver.py:274-275), seconds active, and per-column lambdas
 * (prod_n ||A_n[:, r]||, the CP weights of the normalised model). */
int cals_engine_results(cals_engine* e, double* pool, int32_t* status, int32_t* iterations,
                        double* error, double* fit, int32_t* retire_seq, double* seconds_active,
                        double* lambdas, void* stream);
/* Stream-ordered copy of the retired models' factors (the pool: per model,
 * per mode, the Fortran (I_n, R_k) block -- the reference's copy-out on
 * retirement, multimatrix.py:97-101) into host memory, without waiting: the
 * caller synchronises the stream before reading it (run() builds the
 * returned Model objects while the copy is in flight). */
int cals_engine_pool_download(cals_engine* e, double* host_pool, void* stream);
/* Kernel launches of the last cals_engine_run (graph path): kernel nodes of
 * the captured driver-iteration graph x graph launches, plus the reset,
 * initial plan and move kernels.  Measurement only -- the reference has no
 * counterpart (its driver loop, driver.py:185-285, is host code). */
int cals_engine_last_launches(cals_engine* e, long long* launches);
/* One record per driver iteration (driver.py:278-284 SegmentTrace meta). */
int cals_engine_trace(cals_engine* e, int32_t* widths, int32_t* n_active, double* seconds,
                      int capacity, int* count);
int cals_engine_variant(cals_engine* e, int mode, int* variant, int* bm, int* bn, int* splits);

/* Line search (replaces als.py:127-144 extrapolate_factors as called from
 * driver.py:250-259, 272-273): after every iteration each model holding a
 * snapshot of its previous iterate is extrapolated to prev + alpha (curr -
 * prev) (alpha <= 0 selects alpha = iteration^(1/3), als.py:56-59); ONE fused
 * last-mode MTTKRP evaluates every candidate; a candidate with a lower error
 * replaces the iterate.  Takes effect at the next cals_engine_run. */
int cals_engine_set_line_search(cals_engine* e, int enabled, double alpha);

/* Non-negative updates (replaces als.py:185-278 nnls_solve_row /
 * nnls_update as called from driver.py:226-227): every factor row is fitted
 * by a warm-started Lawson-Hanson active-set search (one warp per row, ranks
 * <= 32), the active sets persisting per model / mode / row across
 * iterations.  cals_engine_nnls_warnings reports per model whether a row hit
 * the 3R iteration cap (NonConvergedNnlsWarning, als.py:70-71). */
int cals_engine_set_nonneg(cals_engine* e, int enabled);
/* Operator level (replaces als.py:185-278 for one block): x[i] = argmin
 * x^T h x - 2 m[i]^T x, x >= 0, warm-started from active[i] (bit a set =
 * variable a pinned to zero; updated in place); converged[i] = 0 when the
 * max_iter cap (< 0: 3 * rank) was hit.  rank <= 32. */
int cals_nnls_rows(int rows, int rank, const double* m, int64_t ldm, const double* h,
                   uint32_t* active, double* x, int64_t ldx, int32_t* converged, int max_iter,
                   void* stream);
int cals_engine_nnls_warnings(cals_engine* e, int32_t* flags);
/* Per model: 1 when a factor update raised in the reference's terms
 * (update_factor / nnls_update on non-finite input -> ValueError,
 * als.py:84-85; caught as a numerical failure, driver.py:229-231 for CALS,
 * driver.py:148-160 _fit_or_fail for SEQUENTIAL / PARALLEL).  The sequential
 * drivers use it to return the reference's failure record (starting factors,
 * iterations_done 0, error nan); run_single_als re-raises ValueError.
 * Blocking copy; call after the run. */
int cals_engine_update_failures(cals_engine* e, int32_t* flags);

/* Step-wise driving of the same loop (what cals_engine_run replays as a CUDA
 * graph), for host-orchestrated runs that interleave collectives: the
 * mode-0-sharded configuration all-reduces the partial MTTKRP of modes >= 1
 * (between _mttkrp and _update) and the mode-0 Gramians (after _update(0)).
 * One driver iteration = for n: enqueue_mttkrp(n), enqueue_update(n); then
 * enqueue_plan.  cals_engine_done reads the mapped flag the plan kernel sets.
 * cals_engine_buffers exposes the device MTTKRP output ([max I][ld]), the
 * Gramians ([order][gram_stride], per-model R_k x R_k blocks) and the factor
 * buffers ([I_n][ld] each). */
int cals_engine_begin(cals_engine* e, double tol, int max_iterations, double sqnorm,
                      void* stream);
int cals_engine_enqueue_mttkrp(cals_engine* e, int mode, void* stream);
int cals_engine_enqueue_update(cals_engine* e, int mode, void* stream);
int cals_engine_enqueue_plan(cals_engine* e, void* stream);
int cals_engine_done(cals_engine* e, int* done);
int cals_engine_buffers(cals_engine* e, double** mttkrp_out, double** grams, int64_t* ld,
                        int64_t* gram_stride, double** factors);

/* ---- diagnostics (no reference counterpart) ------------------------------
 * Live FP64 tensor-core peak (DMMA.8x8x4 on every SM, TFLOP/s): the
 * roofline denominator for the fused MTTKRP. */
int cals_fp64_peak_probe(void* stream, double* tflops);

/* Live INT8 tensor-core peak (tcgen05.mma kind::i8, M=128 N=256 K=32 on every
 * SM, TOPS): the roofline denominator of the Ozaki-sliced INT8 MTTKRP. */
int cals_int8_peak_probe(void* stream, double* tops);

#ifdef __cplusplus
}
#endif

#endif /* CALS_B200_H_ */
