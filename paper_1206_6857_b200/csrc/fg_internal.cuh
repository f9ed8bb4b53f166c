// fg_internal.cuh -- shared host/device definitions of the B200 engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/fastgauss_b200.h"

namespace fg {

constexpr int kMaxDim = 8;      // index-set digit rows (series tables) hold 8 dimensions
// Kernel dimensions: 1..8 natively; 9..12 and 13..16 run as 12 and 16 with the
// extra coordinates zero (distances, boxes, the split rule and therefore the
// tree, and every sum are unchanged; the series bounds use the user dimension)
constexpr int kMaxUserDim = 16;
inline int kernel_dim(int dim) { return dim <= 8 ? dim : dim <= 12 ? 12 : dim <= 16 ? 16 : -1; }
constexpr int kDimSlots = 17;  // per-dimension caches indexed by kernel dimension
#ifndef FG_MAX_ORDER
#define FG_MAX_ORDER 12
#endif
constexpr int kMaxOrder = FG_MAX_ORDER;   // series order cap on the device
constexpr int kMaxK = 384;      // coefficient-count cap per expansion (K = 364 at D = 3, order 12)
// local expansions (direct local, H2L, L2L) are held per warp in shared memory:
// their order is capped lower (any feasible method keeps the error guarantee)
constexpr int kLocOrder = 10;
constexpr int kLocK = 256;
constexpr double kSqrt2 = 1.4142135623730951;

// the reference's series order cap per dimension (spatial_index.py:39-44)
__host__ __device__ constexpr int default_plimit_c(int D) {
    return D == 1 ? 8 : D == 2 ? 8 : D == 3 ? 6 : D == 4 ? 4 : D == 5 ? 4 : D == 6 ? 2 : 1;
}

// The engine's own Hermite order cap per dimension: the order its evaluators are
// compiled for.  At D = 3 it exceeds the reference's default_plimit (6): on a
// GPU the exhaustive-vs-series crossover sits at higher orders (a K_p-term
// FP64 dot against N_R FP32 pairs), and every order's bound
// (error_bounds.py:107-117) holds for any p.  Sweeps use it when the caller
// leaves RunConfig.plimit unset.
#ifndef FG_ORDER3
#define FG_ORDER3 12
#endif
__host__ __device__ constexpr int engine_order_c(int D) {
    return D == 3 ? (FG_ORDER3 <= kMaxOrder ? FG_ORDER3 : kMaxOrder) : default_plimit_c(D);
}


// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
struct Status {
    int code;
};

#define FG_CUDA_TRY(expr)                                                        \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            ::fg::set_error(std::string(#expr) + " (" + __FILE__ + ":" +        \
                            std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
            return FG_ECUDA;                                                     \
        }                                                                        \
    } while (0)

#define FG_TRY(expr)                  \
    do {                              \
        int _s = (expr);              \
        if (_s != FG_OK) return _s;   \
    } while (0)

#define FG_REQUIRE(cond, code, msg)   \
    do {                              \
        if (!(cond)) {                \
            ::fg::set_error(msg);     \
            return code;              \
        }                             \
    } while (0)

// The calling host thread's engine stream (fg_set_stream; default: the
// per-thread default stream).  Every call of one thread is ordered on it.
cudaStream_t stream();
// keep freed pool memory cached (release threshold = max) on the current device
void pool_init();
// every kernel launch of the library bumps this (fg_launch_count)
void count_launch();

// ------------------------------------------------------- device buffers
struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() { release(); }
    // Stream-ordered allocation from the device's memory pool (kept warm, see
    // pool_init), so per-sweep trees and scratch cost no cudaMalloc/cudaFree.
    void release() {
        if (p && cudaFreeAsync(p, stream()) != cudaSuccess) {
            cudaGetLastError();  // e.g. the stream is gone (thread exit): free synchronously
            cudaFree(p);
            cudaGetLastError();
        }
        p = nullptr;
        bytes = 0;
    }
    // grow-only (re)allocation; contents are not preserved
    int reserve(size_t nbytes) {
        if (nbytes <= bytes) return FG_OK;
        release();
        pool_init();
        size_t nb = nbytes < 256 ? 256 : nbytes;
        cudaError_t e = cudaMallocAsync(&p, nb, stream());
        if (e != cudaSuccess) {
            set_error(std::string("cudaMalloc(") + std::to_string(nb) + "): " +
                      cudaGetErrorString(e));
            p = nullptr;
            return FG_ECUDA;
        }
        bytes = nb;
        return FG_OK;
    }
    template <class T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

// Scratch owned by one (host thread, device): engine calls from different host
// threads, or on different devices, never share a buffer (SPEC.md:487 --
// concurrent traversals own distinct query trees).  `Tag` names
// the use site; T is default-constructed on first use.
template <class T>
struct PerDevice {
    std::vector<std::unique_ptr<T>> v;
    T &get() {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) {
            cudaGetLastError();
            dev = 0;
        }
        if ((int)v.size() <= dev) v.resize(dev + 1);
        if (!v[dev]) v[dev].reset(new T());
        return *v[dev];
    }
};
template <class Tag, class T = DBuf>
T &scratch() {
    static thread_local PerDevice<T> m;
    return m.get();
}

// true when ptr is device (or managed) memory usable by kernels
bool is_device_ptr(const void *ptr);

// Make `src` (count elements) available on the device: returns src itself
// when it is device memory, otherwise copies into `stage`.
int to_device(const void *src, size_t bytes, DBuf &stage, const void **dptr);
// Copy device data to a destination that may be host or device.
int from_device(void *dst, const void *dsrc, size_t bytes);

// ------------------------------------------------------- series tables
// Graded-lex multi-index tables for (dim, order) (kernel_math.py:111-209),
// resident on the device.  Cached per (dim, order).
struct SeriesTables {
    int dim = 0, order = 0, K = 0, npairs = 0;
    std::vector<uint8_t> h_digits;     // K x dim
    std::vector<int> h_degrees;        // K
    std::vector<double> h_fact;        // K
    std::vector<int> h_prefix;         // order + 1
    std::vector<int> h_pair_a, h_pair_b, h_pair_s;
    // device copies
    DBuf digits;     // uint8 K x kMaxDim (padded)
    DBuf inv_fact;   // double K
    DBuf fact;       // double K
    DBuf degrees;    // int K
    DBuf h2h_off;    // int K+1: CSR of shift pairs by s
    DBuf h2h_ab;     // int2 npairs: (a, b) sorted by s
    DBuf l2l_off;    // int K+1: CSR of shift pairs by a
    DBuf l2l_bs;     // int2 npairs: (b, s) sorted by a
};
const SeriesTables *series_tables(int dim, int order, int *status);

// tail tables (error_bounds.py:73-92): ct[p] = count/denom, cross[p]
void tail_tables(int dim, int plimit, double *ct, double *cross, double *floor_c);
int default_plimit(int dim);  // spatial_index.py:39-44
int engine_plimit(int dim);   // the engine's own order cap (sweeps with plimit <= 0)
int iset_count(int dim, int order);

// -------------------------------------------------------------- the tree
// Node numbering on the device is BFS (level by level); `pre_of_bfs` maps
// to the reference's preorder numbering for export.
struct TreeDev {
    int device = 0;       // the tree's buffers live on this device
    // per-handle ordering: work queued on one host thread's stream that later
    // calls (possibly from another thread/stream) must wait for
    cudaEvent_t ready = nullptr;
    bool pending = false;
    ~TreeDev() {
        if (ready) cudaEventDestroy(ready);
    }
    int64_t n = 0;
    int dim = 0, leaf = 25, stride = 0;  // stride: doubles per packed point; dim = kernel dim
    int dim_user = 0;                    // the caller's dimension (<= dim, see kernel_dim)
    int64_t nnodes = 0;
    int levels = 0;
    double total_w = 0.0;
    std::vector<int64_t> level_begin;  // BFS node id range per level
    DBuf level_begin_dev;              // the same, int, on the device
    DBuf pw;       // n x stride: coords then weight (tree order), padded
    DBuf perm;     // int64 n: tree position -> original index
    DBuf node_i;   // int4 nnodes: start, count, left, right (BFS ids, -1 = leaf)
    DBuf node_box; // double nnodes x 2*dim: lo[dim], hi[dim]
    DBuf node_c;   // double nnodes x dim: centroid
    DBuf node_wr;  // double2 nnodes: weight, inf_radius
    // moments (bandwidth-dependent), K per node, BFS numbering
    DBuf mom, mom0;
    // direct-moment work items (node, chunk): bandwidth-independent
    bool mom_items_valid = false;
    int mom_nitems = 0;
    DBuf mom_items, mom_off;
    int mom_order = 0, mom_K = 0;
    double mom_h = 0.0, mom0_h = 0.0;
    bool mom_valid = false, mom0_valid = false;
    // query blocks (bandwidth-independent): ranges of <= 32 tree-order points
    bool qb_valid = false;
    bool fp32_ok = true;  // coordinates and weights fit the FP32 base case's range
    // FP32 records for the traversal's FP32 base case (fp32_pack, fg_traverse.cu)
    bool pf_valid = false;
    // per node (|weighted mean offset from the centre|, weighted mean squared
    // offset): the traversal's Jensen mass bound (node_stats_js, fg_traverse.cu)
    bool js_valid = false;
    DBuf node_js;
    DBuf pf;      // float n x fstride: coords about the anchor centre, then weight
    DBuf anchor;  // int n: the point's maximal node with <= 32 points (BFS id)
    int64_t nqb = 0;
    double qb_rad_median = 0.0;  // median query-block inf-radius (base-item size rule)
    DBuf qb_range;  // int2 (start, count)
    DBuf qb_box;    // double nqb x 2*dim
    DBuf qb_c;      // double nqb x dim
    DBuf qb_rad;    // double nqb
    DBuf qb_wmin;   // double nqb: smallest weight among the block's points
    // super-nodes: the maximal nodes the blocks are cut from (the far-field
    // pass settles reference nodes for a whole super-node, fg_far_kernel.cuh)
    int64_t nsn = 0;
    DBuf qb_node;   // int nqb: BFS id of the block's super-node
    DBuf qb_super;  // int nqb: the block's super-node index
    DBuf sn_node;   // int nsn: BFS node id
    DBuf sn_first;  // int nsn + 1: first block of each super-node
    DBuf sn_wmin;   // double nsn: smallest point weight
    DBuf qb_wsum;   // double nqb: total weight of the block's points
    // heaviest-first visiting order from the previous full run's block costs
    bool qb_order_valid = false;
    DBuf qb_cost;   // uint64 nqb: cycles per block in the last full run
    DBuf qb_order;  // int nqb
    DBuf qb_keys, qb_sort_tmp, qb_iota;
};

// Make the calling thread's stream wait for asynchronous work queued on the
// tree by earlier calls (tree_use), and mark such work (tree_mark).
int tree_use(TreeDev &t);
int tree_mark(TreeDev &t);

// Selects a tree's device for the duration of a call, restoring the caller's.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace fg

struct fg_tree {
    fg::TreeDev t;
};

namespace fg {
// implemented in fg_tree.cu / fg_moments.cu / fg_traverse.cu / fg_naive.cu
int tree_build(const double *d_points, const double *d_weights, int64_t n, int dim, int leaf,
               TreeDev &t);
int tree_export(const TreeDev &t, int64_t *perm, int64_t *start, int64_t *end, double *lo,
                double *hi, double *center, double *weight, double *inf_radius,
                int64_t *left, int64_t *right);
int moments_refresh(TreeDev &t, double h, int plimit);
int mom_items(TreeDev &t);  // (node, chunk) work items, shared with node_js
int node_js(TreeDev &t);    // Jensen statistics per node (fg_moments.cu)
int moments_multi(TreeDev &t, const double *hs, int nh, int plimit, DBuf &dst);
int moments_export(const TreeDev &t, double *out);
int query_blocks(TreeDev &t);
// optional audit ledger of a single run (device buffers)
struct AuditSink {
    void *events;                 // AuditEvent[cap] (fg_audit_event layout)
    unsigned long long *count;    // events recorded (may exceed cap)
    long long cap;
};
int run_traversal(TreeDev &q, TreeDev &r, double h, double eps, int mode, int plimit,
                  int64_t b0, int64_t b1, int64_t stride, double *d_values, fg_counters *counters,
                  double *seconds, const AuditSink *audit = nullptr);
// all bandwidths of a sweep through shared launches (values: nh x m, device)
int run_sweep(TreeDev &q, TreeDev &r, const double *hs, int nh, double eps, int mode, int plimit,
              double *d_values, fg_counters *counters, double *seconds, int64_t b0 = 0,
              int64_t b1 = -1, int64_t stride = 1);
int preorder_map(const TreeDev &t, std::vector<int64_t> &pre);
int naive_sum(const double *d_q, int64_t m, const double *d_r, const double *d_w, int64_t n,
              int dim, const double *hs, int nh, double *d_out);
extern int g_ref_leaf;
extern int g_qblock_mode;
extern int g_stack_cap;
extern int g_fp32_base;
}  // namespace fg
