/*
 * fastgauss_b200.h -- C ABI of the B200-native Gaussian-summation engine.
 *
 * Drop-in boundary for the reference package `fastgauss`
 * (/root/reference/pkg/src/fastgauss/, cited below as `file.py:line`).
 * The reference has no FFI of its own (it is pure Python/NumPy); each entry
 * point here replaces the Python function named in its comment, and the
 * Python shim `paper_1206_6857_b200` binds them with ctypes (INTEGRATION.md
 * shows the binding).  Plain pointers and sizes only; no torch types.
 *
 * Pointers marked "host or device" are classified with
 * cudaPointerGetAttributes: device/managed memory is used in place, host
 * memory is staged through the engine's device buffers.  All work of a host
 * thread is issued on that thread's stream (fg_set_stream; default: the
 * per-thread default stream) and every call returns when its results are
 * available to the caller (fg_moments_refresh is stream-ordered instead).
 *
 * Ownership and threading: a tree handle owns its
 * device buffers and its per-tree state; one traversal owns a query tree at a
 * time, and the reference side is read-only after its refresh.  Concurrent
 * calls from different host threads on distinct query trees are safe: every
 * engine scratch buffer belongs to one (host thread, device), each thread
 * issues on its own stream, and work queued on a tree (moments) is fenced by
 * the tree's event before any other stream uses it.  A tree's calls run on
 * the device it was built on.
 *
 * Status codes (every function returns one):
 *   FG_OK 0, FG_EINVAL 1 (-> ValueError), FG_ESTALE 2 (stale moments ->
 *   RuntimeError, summation_engine.py:433-441), FG_ECUDA 3 (CUDA/NCCL error),
 *   FG_EUNSUPPORTED 4 (a size this build does not support -> ValueError).
 * fg_last_error() returns a thread-local message for the last failure.
 */
#ifndef FASTGAUSS_B200_H
#define FASTGAUSS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_OK 0
#define FG_EINVAL 1
#define FG_ESTALE 2
#define FG_ECUDA 3
#define FG_EUNSUPPORTED 4

/* algorithms: summation_engine.py:458-480 */
#define FG_DFD 1
#define FG_DFDO 2
#define FG_DITO 3

/* TraversalCounters (summation_engine.py:81-104) plus exact pair count */
typedef struct {
    int64_t pair_visits;
    int64_t base_cases;
    int64_t fd_prunes;
    int64_t hermite_prunes;
    int64_t local_prunes;
    int64_t h2l_prunes;
    int64_t exact_pairs; /* query x reference pairs evaluated exactly in FP64 */
    int64_t fp32_pairs;  /* pairs evaluated in FP32 with their error bound charged
                            through the token rule (see fg_set_engine_params) */
    int64_t hermite_evals; /* (Hermite item, query) evaluations of EVALM: the far-field
                              leg of the traversal kernel's roofline */
    int64_t hermite_terms; /* sum over those evaluations of K_p (coefficients used) */
    int64_t local_evals;   /* queries evaluated against a local expansion (EVALL) */
} fg_counters;

typedef struct fg_tree fg_tree; /* device-resident kd-tree (KdTree, spatial_index.py:144) */

/* one audit-ledger event (ResultVector.audit, summation_engine.py:107-119;
 * recorded at :250, :350, :394-398): kind 0 base case, 1 FD prune, 2 Hermite,
 * 3 direct local, 4 H2L; the query block (see fg_query_block_ranges), the
 * traversal step and item lane (ordering within the block); W_R, the error
 * bound charged through the token rule, G_min at the decision, token flow
 * (required tokens: negative = credit). */
typedef struct {
    int32_t kind, qblock, seq, lane;
    double w_ref, bound, mass_lo, token_flow;
} fg_audit_event;

int fg_version(void);
const char *fg_last_error(void);
/* diagnostics: number of kernels this library has launched so far, and
 * measured FP64 FMA throughput (TFLOP/s) on the current device */
int fg_launch_count(int64_t *count);
int fg_fp64_peak(double *tflops);
/* measured ex2.approx.f32 (SFU) throughput, Gop/s: the FP32 base case's
 * per-pair limit (one ex2 per pair) */
int fg_ex2_peak(double *gops);
/* the calling thread's stream: a cudaStream_t on the current device (NULL =
 * the per-thread default stream).  Switching drains the previous stream. */
int fg_set_stream(void *stream);
int fg_get_stream(void **stream);
int fg_set_device(int device);
int fg_synchronize(void);

/* ---- exhaustive sums: naive_sum (summation_engine.py:122-154) ---------
 * queries (m x dim) and references (n x dim) row-major, weights (n,), all
 * host or device; out (m,) host or device.  nh bandwidths -> out is
 * (nh x m).  exact_pairs (nullable) receives m*n*nh. */
int fg_naive_sum(const double *queries, int64_t m, const double *references,
                 const double *weights, int64_t n, int32_t dim, const double *bandwidths,
                 int32_t nh, double *out);

/* ---- trees: PointStore (spatial_index.py:47-80) + build_tree (:231-276) --
 * points (n x dim) host or device; weights NULL -> all ones; rejects n < 1,
 * dim < 1, non-positive weights, leaf_threshold < 1 (FG_EINVAL).  The
 * device build reproduces the reference permutation and node ranges. */
int fg_tree_build(const double *points, const double *weights, int64_t n, int32_t dim,
                  int32_t leaf_threshold, fg_tree **out);
int fg_tree_free(fg_tree *tree);
/* n, dim, number of nodes, sum of weights, number of levels */
int fg_tree_info(const fg_tree *tree, int64_t *n, int32_t *dim, int64_t *nnodes,
                 double *total_weight, int32_t *levels);
/* Node arrays in the reference's PREORDER numbering (Node.index), host
 * pointers, each nullable: perm (n), start/end/left/right (nnodes, -1 for
 * no child), lo/hi/center (nnodes x dim), weight/inf_radius (nnodes). */
int fg_tree_export(const fg_tree *tree, int64_t *perm, int64_t *start, int64_t *end,
                   double *lo, double *hi, double *center, double *weight,
                   double *inf_radius, int64_t *left, int64_t *right);
/* points (n x dim) and weights (n) in tree order, host or device */
int fg_tree_points(const fg_tree *tree, double *points, double *weights);

/* ---- moments: KdTree.refresh_moments (spatial_index.py:171-197) -------- */
int fg_moments_refresh(fg_tree *tree, double h, int32_t plimit);
/* (nnodes x K) in preorder numbering; K = C(dim+plimit-1, dim) */
int fg_moments_export(const fg_tree *tree, double *out, int32_t *K, double *h,
                      int32_t *order);

/* ---- runs: dfd_run / dfdo_run / dito_run (summation_engine.py:431-480) --
 * qtree may equal rtree (monochromatic).  values (m,) host or device, in
 * ORIGINAL query order.  plimit <= 0 -> default_plimit(dim).  Requires
 * fresh moments for FG_DITO (else FG_ESTALE).  seconds = device time of the
 * run (reset + traverse + post, like summation_engine.py:447-452). */
int fg_run(fg_tree *qtree, fg_tree *rtree, double h, double eps, int32_t mode,
           int32_t plimit, double *values, fg_counters *counters, double *seconds);
/* Bandwidth sweep (the loop of run_sweep, cli_harness.py:246-283, for one
 * algorithm): for each of the nh bandwidths (host or device array), refresh
 * rtree's moments (FG_DITO) and run, all stream-ordered with a single
 * synchronisation at the end.  values (nh x m) host or device, row j in
 * original query order; counters and seconds (nh each, nullable).  rtree's
 * moments are left at the last bandwidth. */
/* plimit <= 0 in a sweep -> the engine's own series order cap for the
 * dimension (fg_engine_plimit: 10 at D = 3, where this engine's evaluators run
 * every order's exact coefficient count; default_plimit(dim) elsewhere).  The
 * order bounds of error_bounds.py:107-145 hold for any order, so the eps
 * contract is unchanged; an explicit plimit is honoured as given. */
int fg_engine_plimit(int32_t dim);
int fg_run_sweep(fg_tree *qtree, fg_tree *rtree, const double *bandwidths, int32_t nh,
                 double eps, int32_t mode, int32_t plimit, double *values, fg_counters *counters,
                 double *seconds);
/* the sweep on query blocks block_begin, +block_stride, ... (< block_end)
 * only; other entries of values are kept */
int fg_run_sweep_range(fg_tree *qtree, fg_tree *rtree, const double *bandwidths, int32_t nh,
                       double eps, int32_t mode, int32_t plimit, int64_t block_begin,
                       int64_t block_end, int64_t block_stride, double *values,
                       fg_counters *counters, double *seconds);
/* Query-sharded run: only query blocks block_begin,
 * block_begin + block_stride, ... (< block_end) of qtree are processed;
 * values is written only at those blocks' queries (original order).  A
 * query block is <= 64 consecutive tree-order points (a maximal tree node);
 * fg_query_blocks reports
 * the block count. */
int fg_query_blocks(fg_tree *qtree, int64_t *nblocks);
/* tree-order start and point count of every query block (host arrays) */
int fg_query_block_ranges(fg_tree *qtree, int32_t *starts, int32_t *counts);
/* fg_run with the audit ledger (the reference's audit=True): up to capacity
 * events copied to `events` (host), *nevents = events recorded (re-run with a
 * larger capacity when it exceeds capacity; pair_visits always suffices). */
int fg_run_audit(fg_tree *qtree, fg_tree *rtree, double h, double eps, int32_t mode,
                 int32_t plimit, double *values, fg_counters *counters, double *seconds,
                 fg_audit_event *events, int64_t capacity, int64_t *nevents);
int fg_run_range(fg_tree *qtree, fg_tree *rtree, double h, double eps, int32_t mode,
                 int32_t plimit, int64_t block_begin, int64_t block_end, int64_t block_stride,
                 double *values, fg_counters *counters, double *seconds);
/* engine knobs: ref_leaf = reference-side base-item size (> 0 fixes it, 0
 * keeps the current setting, -1 restores the default choice by bandwidth);
 * stack_cap = per-warp frontier capacity (0 keeps); fp32_base (-1 keeps, 0
 * off, 1 on, default on) lets the traversal evaluate leaf pairs in FP32 when
 * the rigorous error bound of that evaluation fits a reserved share of eps
 * (eps = 0 always uses FP64).  Not part of the
 * reference API. */
int fg_set_engine_params(int32_t ref_leaf, int32_t stack_cap, int32_t fp32_base);
/* device bounds-check violations counted since the last call (and reset);
 * -1 when the library was built without -DFG_CHECKS=1 */
int fg_check_failures(int64_t *count);

/* ---- series algebra (series_expansion.py), batched over `batch` items ---
 * All arrays host or device, row-major per item.  Used by the Python mirror
 * of the reference's series functions and by the parity tests. */
/* accumulate_far_field (:76-92) / accumulate_local_direct (:110-126):
 * item b owns points [offsets[b], offsets[b+1]) of pts (npts x dim) and w. */
int fg_series_accumulate(int32_t kind /*0 far, 1 local*/, const double *pts, const double *w,
                         const int64_t *offsets, int32_t batch, int32_t dim,
                         const double *centers, int32_t order, double h, double *coeffs);
/* eval_far_field (:95-107) / eval_local (:129-136): evaluates item b's
 * expansion (coeffs b x K_stored, prefix `order`) at its points */
int fg_series_eval(int32_t kind /*0 far, 1 local*/, const double *coeffs, int32_t k_stored,
                   const double *centers, int32_t batch, int32_t dim, int32_t order,
                   double h, const double *x, const int64_t *offsets, double *out);
/* translate_h2h (:139-157) kind 0, translate_l2l (:197-217) kind 1,
 * translate_h2l (:167-194) kind 2 (src_order = order_src, dest = order) */
int fg_series_translate(int32_t kind, const double *coeffs, int32_t k_stored,
                        const double *src_centers, const double *dst_centers, int32_t batch,
                        int32_t dim, int32_t order_src, int32_t order, double h,
                        double *out);
/* The graded-lex index set |alpha| < order (kernel_math.py:111-209) the
 * kernels use, exported from the same host tables (no GPU needed): K, digits
 * (K x dim), degrees (K), alpha! (K), prefix counts (order + 1), and the shift
 * pairs (a, b, s) with digits_a + digits_b = digits_s, degree < order
 * (npairs x 3).  Every output pointer is nullable (query K / npairs first). */
int fg_iset_export(int32_t dim, int32_t order, int32_t *K, int32_t *digits, int32_t *degrees,
                   double *fact, int32_t *prefix, int32_t *npairs, int32_t *pairs);
/* best_method (error_bounds.py:168-230) on `batch` geometries:
 * geom rows = (min_sq, max_sq, r_ref, r_query, w_ref, n_query, n_ref, h, maxerr);
 * out rows = (method 0/2/3/4, order, bound, cost) as doubles. */
int fg_best_method(const double *geom, int32_t batch, int32_t dim, int32_t plimit,
                   double *out);

#ifdef __cplusplus
}
#endif
#endif
