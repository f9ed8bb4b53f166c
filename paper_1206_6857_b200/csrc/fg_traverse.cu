// fg_traverse.cu -- K2 + K6..K11 fused: the dual-tree traversal with token
// error control, series prunes and exhaustive leaf-pair base cases
// (replaces _traverse/visit, dito_base and dito_post:
//  summation_engine.py:157-455; best_method, error_bounds.py:168-230).
//
// Work decomposition:
//  * The query side is cut into blocks of <= 64 consecutive tree-order points
//    (a query "node" with a tight box, centroid and inf-radius).  One warp owns
//    one block at a time; lane j holds query point j in registers.  Warps pull
//    blocks from an atomic counter (persistent kernel), so every block is
//    processed start-to-finish by one warp: results are deterministic.
//  * The warp walks the reference tree with a private stack of frontier
//    entries (node, K_lo, K_hi, min_sq) and processes up to 32 entries per
//    step, one per lane: box bounds and both kernel bounds are computed in
//    parallel, then the token rule (summation_engine.py:157-188) is applied in
//    lane order (a warp-serial scan over the candidates that can possibly be
//    admitted).
//  * The mass lower bound used by every decision is
//        G_min = min_j exact_j + settled + sum_{frontier} W_R K_lo(Q, R)
//    i.e. the exact base-case sums of each point, the bounds of every settled
//    prune, and the K_lo bound of every not-yet-settled frontier entry.  The
//    settled set plus the frontier partitions the references, so this is a
//    valid lower bound on G(x) for every x in the block at every step
//    (Theorem 2).
//  * Base cases (leaf x leaf) run eagerly inside the same warp: all 32 lanes
//    stream the reference leaf's points (broadcast loads) through the FP64
//    pipe -- this is the roofline-critical inner loop.
//  * Series prunes: Hermite (EVALM per lane), direct local and H2L (lanes own
//    local coefficients in shared memory); the post pass is one EVALL per lane.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fg_device.cuh"
#include "fg_exp.cuh"
#include "fg_internal.cuh"
#include "fg_series.cuh"
#include "fg_traverse_kernel.cuh"
#include "fg_far_kernel.cuh"

namespace fg {

// reference-side base-item size: 0 = by bandwidth (ref_leaf_for), else fixed
int g_ref_leaf = 0;
#ifndef FG_BIG_ITEM_RATIO
#define FG_BIG_ITEM_RATIO 1.0
#endif
static constexpr double kBigItemRatio = FG_BIG_ITEM_RATIO;  // h / r_b above which items reach kAnchorMax

// Base-item granularity by bandwidth relative to the query blocks' median
// inf-radius r_b (D >= 5: 32-point items win below ~0.05 r_b, 48 below
// ~0.4 r_b, then larger).
// At D >= 5 the direct FP32 stream takes items of any size: at h >~ 0.4 r_b,
// where nearly every pair is exact, bigger items save traversal steps (C4
// single runs: 128 points -2 % at 0.44 r_b, 256 points -8..-14 % from 0.6 r_b;
// C3 -6..-14 % at 1-11 r_b).
static int ref_leaf_for(const TreeDev &q, double h) {
    if (g_ref_leaf > 0) return g_ref_leaf;
    const double rb = q.qb_rad_median;
    if (!(rb > 0.0)) return 48;
    // single-run scans per bandwidth with the Jensen bound and run-based query
    // blocks (C3, C4, C5; r_b = median block inf-radius): small items where
    // pruning still bites, bigger ones where nearly every pair is exact
    // anchored FP32 items: <= kAnchorMax (336) points; 256-point items above
    // r_b measured C5 -2.3 % against 128 (and 128 between r_b and 1.5 r_b: no
    // gain), C2 neutral
    if (q.dim <= 4) {
        // re-scanned with the order-12 far field (C5 -3.1 %, C2 -5 % against
        // 0.2 / 1.0 / 1.0: the series now take the mid-size nodes, so larger
        // items pay earlier)
        double t0 = 0.05, t1 = 0.3, t2 = 0.5 * kBigItemRatio;
        if (const char *env = getenv("FG_LEAF_T0")) t0 = atof(env);  // experiment knobs
        if (const char *env = getenv("FG_LEAF_T1")) t1 = atof(env);
        if (const char *env = getenv("FG_LEAF_T2")) t2 = atof(env);
        if (h < t0 * rb) return 32;
        if (h < t1 * rb) return kStageMax;
        if (kAnchorMax > 128 && h < t2 * rb) return 128;
        return kAnchorMax;
    }
    if (h < 0.1 * rb) return 32;
    if (h < 0.25 * rb) return 64;
    if (h < 0.6 * rb) return 128;
    return 256;
}
int g_stack_cap = 4096;
// h / (median query-block radius) at which a bandwidth's tasks cost most
// (C2 sweep per-block cycles: the heaviest groups sit at h / r_b ~ 1.5-20)
static constexpr double kHeavyRatio = 5.0;
int g_fp32_base = 1;
static constexpr double kFp32Share = 0.1;  // measured: C5 0.02: +97%, 0.05: +5%, 0.2: +4%
#ifndef FG_TRAV_MINB
#define FG_TRAV_MINB 4  // resident 128-thread CTAs per SM the traversal is compiled for
#endif

// ---------------------------------------------------------- query blocks
// A query block is a run of <= kQBlock (64) consecutive tree-order points owned
// by one warp (lane l holds points l and l + 32).  Mode 0 (default): the
// maximal kd-tree nodes with <= kQBlock points (tight node boxes; larger
// leaves -- duplicate points -- are cut into runs).  Mode 1: fixed runs
// regardless of node boundaries.
int g_qblock_mode = 0;
// Query blocks: maximal nodes with <= kQBlockNode points (at most n / 16), cut
// into even runs of <= kQBlock consecutive tree-order points.  Depth-first
// order keeps a run spatially compact, and runs fill a warp's 64 query slots:
// against maximal <= 64-point nodes (41 points on average on C2) the sweeps
// run C2 -10 %, C3 -32 %, C4 -35 %, C5 -22 % (4096; 16384 >= C2's n / 8 loses)
static constexpr int kQBlockNode = 4096;

template <int D>
__global__ void query_blocks_kernel(int64_t nqb, const double *__restrict__ pw,
                                    const int2 *__restrict__ range, double *__restrict__ box,
                                    double *__restrict__ ctr, double *__restrict__ rad,
                                    double *__restrict__ wmin, double *__restrict__ wsum) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (b >= nqb) return;
    const int2 rg = range[b];
    const int cnt = rg.y;
    bool v[kQPL];
    double x[kQPL][D], wl = CUDART_INF, ws = 0.0;
#pragma unroll
    for (int qi = 0; qi < kQPL; qi++) {
        v[qi] = lane + 32 * qi < cnt;
        if (v[qi]) {
            double w;
            load_point_w<D>(pw + ((int64_t)rg.x + lane + 32 * qi) * S, x[qi], w);
            wl = fmin(wl, w);
            ws += w;
        }
    }
    wl = warp_min(wl);
    ws = warp_sum(ws);
    if (lane == 0) {
        wmin[b] = wl;
        wsum[b] = ws;
    }
    double c[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        double lo = CUDART_INF, hi = -CUDART_INF, sm = 0.0;
#pragma unroll
        for (int qi = 0; qi < kQPL; qi++) {
            if (v[qi]) {
                lo = fmin(lo, x[qi][d]);
                hi = fmax(hi, x[qi][d]);
                sm += x[qi][d];
            }
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        sm = warp_sum(sm);
        c[d] = sm / cnt;
        if (lane == 0) {
            box[b * 2 * D + d] = lo;
            box[b * 2 * D + D + d] = hi;
            ctr[b * D + d] = c[d];
        }
    }
    double r = 0.0;
#pragma unroll
    for (int qi = 0; qi < kQPL; qi++) {
        if (v[qi]) {
#pragma unroll
            for (int d = 0; d < D; d++) r = fmax(r, fabs(x[qi][d] - c[d]));
        }
    }
    r = warp_max(r);
    if (lane == 0) rad[b] = r;
}

static void block_ranges(const TreeDev &t, std::vector<int2> &out) {
    out.clear();
    const char *env = getenv("FG_QBLOCK_MODE");
    const int mode = env ? atoi(env) : g_qblock_mode;
    // experiment knob: smaller query blocks
    const char *lenv = getenv("FG_QBLOCK_LIMIT");
    const int lim = lenv ? std::max(1, std::min(kQBlock, atoi(lenv))) : kQBlock;
    if (mode == 1) {
        for (int64_t s = 0; s < t.n; s += lim)
            out.push_back(make_int2((int)s, (int)std::min<int64_t>(lim, t.n - s)));
        return;
    }
    std::vector<int4> ni(t.nnodes);
    cudaMemcpy(ni.data(), t.node_i.p, sizeof(int4) * t.nnodes, cudaMemcpyDeviceToHost);
    std::vector<int> stack(1, 0);
    while (!stack.empty()) {  // preorder, left first: blocks come out in tree order
        const int v = stack.back();
        stack.pop_back();
        const int4 e = ni[v];
        if (e.y <= lim || e.z < 0) {
            for (int s = 0; s < e.y; s += lim) out.push_back(make_int2(e.x + s, std::min(lim, e.y - s)));
        } else {
            stack.push_back(e.w);
            stack.push_back(e.z);
        }
    }
}

// Block starts on the device (default mode): every maximal node with <= lim
// points (or leaf) is cut into even runs of <= kQBlock points; every node with
// > lim points marks its qualifying children, and a run marks its start with
// its length in a per-point array.  Runs tile the tree order, so an exclusive
// scan over the marks numbers them in tree order.
__global__ void block_marks_kernel(int64_t nnodes, const int4 *__restrict__ ni, int lim,
                                   int *__restrict__ len, int *__restrict__ own) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nnodes) return;
    const int4 e = ni[v];
    // a node of <= lim points is cut into runs of <= kQBlock consecutive points;
    // each run start records the node (its super-node)
    auto emit = [&](const int4 c, int node) {
        const int nr = (c.y + kQBlock - 1) / kQBlock;  // runs, as even as possible
        for (int r = 0; r < nr; r++) {
            const int s0 = (int)((int64_t)c.y * r / nr), s1 = (int)((int64_t)c.y * (r + 1) / nr);
            len[c.x + s0] = s1 - s0;
            own[c.x + s0] = node;
        }
    };
    if (v == 0 && (e.y <= lim || e.z < 0)) emit(e, 0);
    if (e.y <= lim || e.z < 0) return;
    for (int k = 0; k < 2; k++) {
        const int ch = k == 0 ? e.z : e.w;
        const int4 c = ni[ch];
        if (c.y <= lim || c.z < 0) emit(c, ch);
    }
}

__global__ void block_flags_kernel(int64_t n, const int *__restrict__ len, int *__restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = len[i] > 0 ? 1 : 0;
}

__global__ void block_ranges_kernel(int64_t n, const int *__restrict__ len,
                                    const int *__restrict__ idx, const int *__restrict__ own,
                                    int2 *__restrict__ range, int *__restrict__ qb_node) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && len[i] > 0) {
        range[idx[i]] = make_int2((int)i, len[i]);
        qb_node[idx[i]] = own[i];
    }
}

// super-node numbering: consecutive blocks of one maximal node form a
// super-node (blocks are in tree order, so each node's blocks are contiguous)
__global__ void sn_flags_kernel(int64_t nqb, const int *__restrict__ qb_node, int *__restrict__ flag) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b < nqb) flag[b] = (b == 0 || qb_node[b] != qb_node[b - 1]) ? 1 : 0;
}

__global__ void sn_fill_kernel(int64_t nqb, const int *__restrict__ flag,
                               const int *__restrict__ incl, const int *__restrict__ qb_node,
                               int *__restrict__ qb_super, int *__restrict__ sn_node,
                               int *__restrict__ sn_first) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nqb) return;
    const int k = incl[b] - 1;
    qb_super[b] = k;
    if (flag[b]) {
        sn_node[k] = qb_node[b];
        sn_first[k] = (int)b;
    }
    if (b == nqb - 1) sn_first[k + 1] = (int)nqb;
}

__global__ void sn_stats_kernel(int64_t nsn, const int *__restrict__ sn_first,
                                const double *__restrict__ qb_wmin, double *__restrict__ sn_wmin) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nsn) return;
    double m = CUDART_INF;
    for (int b = sn_first[k]; b < sn_first[k + 1]; b++) m = fmin(m, qb_wmin[b]);
    sn_wmin[k] = m;
}

static int device_block_ranges(TreeDev &t, int64_t &nqb) {
    struct BlockScr {
        DBuf len, flag, idx, tmp, own;
    };
    BlockScr &bs = scratch<BlockScr, BlockScr>();
    DBuf &s_len = bs.len, &s_flag = bs.flag, &s_idx = bs.idx, &s_tmp = bs.tmp, &s_own = bs.own;
    const int64_t n = t.n;
    FG_TRY(s_own.reserve(sizeof(int) * (n + 1)));
    FG_TRY(s_len.reserve(sizeof(int) * (n + 1)));
    FG_TRY(s_flag.reserve(sizeof(int) * (n + 1)));
    FG_TRY(s_idx.reserve(sizeof(int) * (n + 1)));
    FG_CUDA_TRY(cudaMemsetAsync(s_len.p, 0, sizeof(int) * (n + 1), stream()));
    count_launch();
    const char *lenv = getenv("FG_QBLOCK_NODE");  // experiment knob
    const int lim = lenv ? std::max(kQBlock, atoi(lenv))
                         : (int)std::max<int64_t>(kQBlock, std::min<int64_t>(kQBlockNode, n / 16));
    block_marks_kernel<<<(unsigned)((t.nnodes + 255) / 256), 256, 0, stream()>>>(
        t.nnodes, t.node_i.as<int4>(), lim, s_len.as<int>(), s_own.as<int>());
    count_launch();
    block_flags_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, stream()>>>(n + 1, s_len.as<int>(),
                                                                              s_flag.as<int>());
    FG_CUDA_TRY(cudaGetLastError());
    size_t tmp = 0;
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, s_flag.as<int>(), s_idx.as<int>(),
                                              (int)(n + 1), stream()));
    FG_TRY(s_tmp.reserve(tmp + 16));
    count_launch();
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(s_tmp.p, tmp, s_flag.as<int>(), s_idx.as<int>(),
                                              (int)(n + 1), stream()));
    static thread_local int *h_cnt = nullptr;
    if (!h_cnt) FG_CUDA_TRY(cudaMallocHost(&h_cnt, sizeof(int)));
    FG_CUDA_TRY(cudaMemcpyAsync(h_cnt, s_idx.as<int>() + n, sizeof(int), cudaMemcpyDeviceToHost,
                                stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    nqb = *h_cnt;
    FG_TRY(t.qb_range.reserve(sizeof(int2) * (nqb > 0 ? nqb : 1)));
    FG_TRY(t.qb_node.reserve(sizeof(int) * (nqb > 0 ? nqb : 1)));
    count_launch();
    block_ranges_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        n, s_len.as<int>(), s_idx.as<int>(), s_own.as<int>(), t.qb_range.as<int2>(),
        t.qb_node.as<int>());
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

// Super-nodes of the device blocks (after device_block_ranges): numbering,
// first block, smallest weight; the count is read back with the median.
static int super_nodes(TreeDev &t, int *h_nsn) {
    struct SnScr {
        DBuf flag, incl, tmp;
    };
    SnScr &ss = scratch<SnScr, SnScr>();
    const int64_t nqb = t.nqb;
    FG_TRY(ss.flag.reserve(sizeof(int) * nqb));
    FG_TRY(ss.incl.reserve(sizeof(int) * nqb));
    FG_TRY(t.qb_super.reserve(sizeof(int) * nqb));
    FG_TRY(t.sn_node.reserve(sizeof(int) * nqb));
    FG_TRY(t.sn_first.reserve(sizeof(int) * (nqb + 1)));
    FG_TRY(t.sn_wmin.reserve(sizeof(double) * nqb));
    const unsigned g = (unsigned)((nqb + 255) / 256);
    count_launch();
    sn_flags_kernel<<<g, 256, 0, stream()>>>(nqb, t.qb_node.as<int>(), ss.flag.as<int>());
    size_t tmp = 0;
    FG_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp, ss.flag.as<int>(), ss.incl.as<int>(),
                                              (int)nqb, stream()));
    FG_TRY(ss.tmp.reserve(tmp + 16));
    count_launch();
    FG_CUDA_TRY(cub::DeviceScan::InclusiveSum(ss.tmp.p, tmp, ss.flag.as<int>(), ss.incl.as<int>(),
                                              (int)nqb, stream()));
    count_launch();
    sn_fill_kernel<<<g, 256, 0, stream()>>>(nqb, ss.flag.as<int>(), ss.incl.as<int>(),
                                            t.qb_node.as<int>(), t.qb_super.as<int>(),
                                            t.sn_node.as<int>(), t.sn_first.as<int>());
    FG_CUDA_TRY(cudaGetLastError());
    FG_CUDA_TRY(cudaMemcpyAsync(h_nsn, ss.incl.as<int>() + nqb - 1, sizeof(int),
                                cudaMemcpyDeviceToHost, stream()));
    return FG_OK;
}

int query_blocks(TreeDev &t) {
    if (t.qb_valid) return FG_OK;
    int64_t nqb = 0;
    // super-nodes come with the device block cut (the experiment knobs' host
    // walks have none: the far-field pass is then off)
    bool sn_ok = false;
    if (getenv("FG_QBLOCK_MODE") || getenv("FG_QBLOCK_LIMIT")) {
        // experiment knobs (fixed runs / smaller blocks): the host walk
        std::vector<int2> ranges;
        block_ranges(t, ranges);
        nqb = (int64_t)ranges.size();
        FG_TRY(t.qb_range.reserve(sizeof(int2) * nqb));
        FG_CUDA_TRY(cudaMemcpyAsync(t.qb_range.p, ranges.data(), sizeof(int2) * nqb,
                                    cudaMemcpyHostToDevice, stream()));
    } else {
        FG_TRY(device_block_ranges(t, nqb));
        sn_ok = true;
    }
    t.nsn = 0;
    const int D = t.dim;
    FG_TRY(t.qb_box.reserve(sizeof(double) * nqb * 2 * D));
    FG_TRY(t.qb_c.reserve(sizeof(double) * nqb * D));
    FG_TRY(t.qb_rad.reserve(sizeof(double) * nqb));
    FG_TRY(t.qb_wmin.reserve(sizeof(double) * nqb));
    FG_TRY(t.qb_wsum.reserve(sizeof(double) * nqb));
    const unsigned blocks = (unsigned)((nqb * 32 + 255) / 256);
#define FG_QB(DD)                                                                           \
    case DD:                                                                                \
        count_launch();                                                                     \
        query_blocks_kernel<DD><<<blocks, 256, 0, stream()>>>(                              \
            nqb, t.pw.as<double>(), t.qb_range.as<int2>(), t.qb_box.as<double>(),           \
            t.qb_c.as<double>(), t.qb_rad.as<double>(), t.qb_wmin.as<double>(),             \
            t.qb_wsum.as<double>());                                                        \
        break;
    switch (D) {
        FG_QB(1) FG_QB(2) FG_QB(3) FG_QB(4) FG_QB(5) FG_QB(6) FG_QB(7) FG_QB(8) FG_QB(12)
        FG_QB(16)
        default: return FG_EUNSUPPORTED;
    }
#undef FG_QB
    FG_CUDA_TRY(cudaGetLastError());
    {
        // median block radius: device sort on the high 32 bits (radii are
        // non-negative doubles, so their bit patterns sort like the values; the
        // low bits only reorder radii within 2^-20 of each other -- the median
        // drives heuristics only), one pinned read-back
        struct MedScr {
            DBuf sorted, tmp;
        };
        MedScr &ms = scratch<MedScr, MedScr>();
        DBuf &s_sorted = ms.sorted, &s_tmp = ms.tmp;
        static thread_local double *h_med = nullptr;
        if (!h_med) FG_CUDA_TRY(cudaMallocHost(&h_med, sizeof(double)));
        FG_TRY(s_sorted.reserve(sizeof(double) * (nqb > 0 ? nqb : 1)));
        const auto *keys = reinterpret_cast<const unsigned long long *>(t.qb_rad.p);
        auto *sorted = s_sorted.as<unsigned long long>();
        size_t tmp = 0;
        FG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, sorted, (int)nqb, 32, 64,
                                                   stream()));
        FG_TRY(s_tmp.reserve(tmp + 16));
        count_launch();
        FG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(s_tmp.p, tmp, keys, sorted, (int)nqb, 32, 64,
                                                   stream()));
        *h_med = 0.0;
        if (nqb > 0)
            FG_CUDA_TRY(cudaMemcpyAsync(h_med, s_sorted.as<double>() + nqb / 2, sizeof(double),
                                        cudaMemcpyDeviceToHost, stream()));
        static thread_local int *h_nsn = nullptr;
        if (!h_nsn) FG_CUDA_TRY(cudaMallocHost(&h_nsn, sizeof(int)));
        *h_nsn = 0;
        t.nqb = nqb;
        if (sn_ok && nqb > 0) FG_TRY(super_nodes(t, h_nsn));
        FG_CUDA_TRY(cudaStreamSynchronize(stream()));
        t.qb_rad_median = *h_med;
        t.nsn = *h_nsn;
        if (t.nsn > 0) {
            count_launch();
            sn_stats_kernel<<<(unsigned)((t.nsn + 255) / 256), 256, 0, stream()>>>(
                t.nsn, t.sn_first.as<int>(), t.qb_wmin.as<double>(), t.sn_wmin.as<double>());
            FG_CUDA_TRY(cudaGetLastError());
        }
    }
    t.nqb = nqb;
    t.qb_valid = true;
    t.qb_order_valid = false;
    return FG_OK;
}

// ------------------------------------------------------------ FP32 records
// Anchor of a point = its maximal tree node with <= kAnchorMax points (every
// FP32 base item lies inside one).  One thread per node: an internal node with
// > kAnchorMax points labels the points of each child that has <= kAnchorMax.
__global__ void anchor_kernel(int64_t nnodes, const int4 *__restrict__ ni, int *__restrict__ anchor) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nnodes) return;
    const int4 e = ni[v];
    if (v == 0 && e.y <= kAnchorMax) {
        for (int i = 0; i < e.y; i++) anchor[e.x + i] = 0;
        return;
    }
    if (e.y <= kAnchorMax || e.z < 0) return;
    for (int c = 0; c < 2; c++) {
        const int ch = c == 0 ? e.z : e.w;
        const int4 ce = ni[ch];
        if (ce.y <= kAnchorMax)
            for (int i = 0; i < ce.y; i++) anchor[ce.x + i] = ch;
    }
}

// FP32 record of each point: coordinates about its anchor's centre (rounded
// from the FP64 difference) and the weight.  Points of leaves with > 32
// points have no anchor and are never evaluated in FP32 (zero records).
template <int D>
__global__ void fp32_pack_kernel(int64_t n, const double *__restrict__ pw,
                                 const double *__restrict__ ctr, const int *__restrict__ anchor,
                                 float *__restrict__ pf) {
    constexpr int S = packed_stride(D);
    constexpr int F = fstride<D>();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = anchor[i];
    float rec[F];
#pragma unroll
    for (int k = 0; k < F; k++) rec[k] = 0.f;
    if (a >= 0) {
#pragma unroll
        for (int d = 0; d < D; d++) rec[d] = (float)(pw[i * S + d] - ctr[(int64_t)a * D + d]);
        rec[D] = (float)pw[i * S + D];
    }
#pragma unroll
    for (int k = 0; k < F; k += 4)
        *reinterpret_cast<float4 *>(pf + i * F + k) = make_float4(rec[k], rec[k + 1], rec[k + 2], rec[k + 3]);
}

#if FG_PAIR_DOT
// Dot-form record PAIRS (points 2k and 2k + 1 interleaved, so every f32x2
// operand of the batch loop comes straight from one 8-byte load): per pair
// {Y_0a, Y_0b, ..., Y_{D-1}a, Y_{D-1}b, B_a, B_b, W_a, W_b, pad} with
// Y = fl(y - c_a) about the point's own anchor centre, B = fl(|Y|^2) (from the
// rounded Y, in FP64) and W = fl(w).  Points without an anchor get zeros.
template <int D>
__global__ void fp32_pair_pack_kernel(int64_t n, const double *__restrict__ pw,
                                      const double *__restrict__ ctr,
                                      const int *__restrict__ anchor, float *__restrict__ pd) {
    constexpr int S = packed_stride(D);
    constexpr int P = pstride<D>();
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (2 * k >= n) return;
    float rec[P];
#pragma unroll
    for (int i = 0; i < P; i++) rec[i] = 0.f;
#pragma unroll
    for (int hf = 0; hf < 2; hf++) {
        const int64_t i = 2 * k + hf;
        if (i >= n) break;
        const int a = anchor[i];
        if (a < 0) continue;
        double b = 0.0;
#pragma unroll
        for (int d = 0; d < D; d++) {
            const float y = (float)(pw[i * S + d] - ctr[(int64_t)a * D + d]);
            rec[2 * d + hf] = y;
            b = fma((double)y, (double)y, b);
        }
        rec[2 * D + hf] = (float)b;
        rec[2 * D + 2 + hf] = (float)pw[i * S + D];
    }
#pragma unroll
    for (int i = 0; i < P; i += 4)
        *reinterpret_cast<float4 *>(pd + k * P + i) = make_float4(rec[i], rec[i + 1], rec[i + 2], rec[i + 3]);
}
#endif

static int fp32_pack(TreeDev &t) {
    if (t.pf_valid) return FG_OK;
    const int D = t.dim;
#if FG_PAIR_DOT
    const int P = (2 * (D + 2) + 3) & ~3;
    const int64_t npair = (t.n + 1) / 2;
    FG_TRY(t.anchor.reserve(sizeof(int) * t.n));
    FG_TRY(t.pf.reserve(sizeof(float) * npair * P));
#else
    const int F = (D + 1 + 3) & ~3;
    FG_TRY(t.anchor.reserve(sizeof(int) * t.n));
    FG_TRY(t.pf.reserve(sizeof(float) * t.n * F));
#endif
    FG_CUDA_TRY(cudaMemsetAsync(t.anchor.p, 0xff, sizeof(int) * t.n, stream()));
    count_launch();
    anchor_kernel<<<(unsigned)((t.nnodes + 255) / 256), 256, 0, stream()>>>(
        t.nnodes, t.node_i.as<int4>(), t.anchor.as<int>());
    FG_CUDA_TRY(cudaGetLastError());
#if FG_PAIR_DOT
    const unsigned blocks = (unsigned)((npair + 255) / 256);
#define FG_PF(DD)                                                                            \
    case DD:                                                                                 \
        count_launch();                                                                      \
        fp32_pair_pack_kernel<DD><<<blocks, 256, 0, stream()>>>(                             \
            t.n, t.pw.as<double>(), t.node_c.as<double>(), t.anchor.as<int>(), t.pf.as<float>()); \
        break;
#else
    const unsigned blocks = (unsigned)((t.n + 255) / 256);
#define FG_PF(DD)                                                                            \
    case DD:                                                                                 \
        count_launch();                                                                      \
        fp32_pack_kernel<DD><<<blocks, 256, 0, stream()>>>(t.n, t.pw.as<double>(),           \
                                                            t.node_c.as<double>(),           \
                                                            t.anchor.as<int>(), t.pf.as<float>()); \
        break;
#endif
    switch (D) {
        FG_PF(1) FG_PF(2) FG_PF(3) FG_PF(4) FG_PF(5) FG_PF(6) FG_PF(7) FG_PF(8)
        default: return FG_EUNSUPPORTED;
    }
#undef FG_PF
    FG_CUDA_TRY(cudaGetLastError());
    t.pf_valid = true;
    return FG_OK;
}

// ---------------------------------------------------------------- launch
__global__ void iota_kernel(int *out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

struct TravScratch {
    DBuf st_node, st_f, ser, work, counters, dbg;
    int grid = 0, cap = 0;
};
// per (host thread, device): concurrent traversals never share scratch
static TravScratch &trav_scratch() { return scratch<TravScratch, TravScratch>(); }

// Launches with few tasks per resident warp are tail-bound: the last tasks run
// nearly alone, so per-warp latency (register-starved address rematerialisation,
// serialised record chains) matters more than warps per SM.  Those launches
// (D <= 4) use the 3-CTA instantiation (<= 168 registers): C2 sweep -4 %, but
// C5 (~600 tasks per warp) +10 %.
constexpr int64_t kFatTasksPerWarp = 16;

template <int D, bool AUDIT, int MB>
static int launch_traverse(TravArgs &A, size_t smem, int64_t nblocks) {
    // 4 resident CTAs of 128 threads per SM (<= 128 registers): measured best
    // for throughput; capping registers lower spills and runs slower
    auto kern = traverse_kernel<D, MB, AUDIT>;
    // resident-grid size, cached per (kernel, shared memory size)
    static thread_local const void *c_kern = nullptr;
    static thread_local size_t c_smem = 0;
    static thread_local int c_dev = -1, c_full = 0;
    int dev = 0;
    FG_CUDA_TRY(cudaGetDevice(&dev));
    if (c_kern != (const void *)kern || c_smem != smem || c_dev != dev) {
        // (static + dynamic shared memory above 48 KB needs the opt-in)
        FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        int sms = 0, occ = 0;
        FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        FG_CUDA_TRY(
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTravThreads, smem));
        c_full = sms * (occ < 1 ? 1 : occ);
        c_kern = (const void *)kern;
        c_smem = smem;
        c_dev = dev;
    }
    int64_t grid = c_full;
    const int64_t need = (nblocks + kTravWarps - 1) / kTravWarps;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    const int cap = A.stack_cap;
    TravScratch &g_scr = trav_scratch();
    if (g_scr.grid < grid || g_scr.cap != cap) {
        const int64_t warps = grid * kTravWarps;
        FG_TRY(g_scr.st_node.reserve(sizeof(int) * warps * cap));
        FG_TRY(g_scr.st_f.reserve(sizeof(double) * warps * cap * 3));
        FG_TRY(g_scr.ser.reserve(sizeof(int2) * warps * cap));
        g_scr.grid = (int)grid;
        g_scr.cap = cap;
    }
    A.st_node = g_scr.st_node.as<int>();
    A.st_f = g_scr.st_f.as<double>();
    A.ser_list = g_scr.ser.as<int2>();
    FG_CUDA_TRY(cudaMemsetAsync(A.work, 0, sizeof(unsigned long long), stream()));
    count_launch();
    kern<<<(unsigned)grid, kTravThreads, smem, stream()>>>(A);
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

template <bool AUDIT>
static int launch_dispatch_t(int D, TravArgs &A, size_t smem, int64_t nb) {
    constexpr int M = FG_TRAV_MINB;
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const char *env = getenv("FG_FAT_TASKS");  // experiment knob: tasks-per-warp threshold
    const int64_t thr = env ? atoll(env) : kFatTasksPerWarp;
    const bool fat = !AUDIT && nb <= thr * (int64_t)sms * M * kTravWarps;
    switch (D) {
        case 1: return fat ? launch_traverse<1, AUDIT, 3>(A, smem, nb) : launch_traverse<1, AUDIT, M>(A, smem, nb);
        case 2: return fat ? launch_traverse<2, AUDIT, 3>(A, smem, nb) : launch_traverse<2, AUDIT, M>(A, smem, nb);
        case 3: return fat ? launch_traverse<3, AUDIT, 3>(A, smem, nb) : launch_traverse<3, AUDIT, M>(A, smem, nb);
        case 4: return fat ? launch_traverse<4, AUDIT, 3>(A, smem, nb) : launch_traverse<4, AUDIT, M>(A, smem, nb);
        case 5: return launch_traverse<5, AUDIT, M>(A, smem, nb);
        case 6: return launch_traverse<6, AUDIT, M>(A, smem, nb);
        case 7: return launch_traverse<7, AUDIT, M>(A, smem, nb);
        case 8: return launch_traverse<8, AUDIT, M>(A, smem, nb);
        case 12: return launch_traverse<12, AUDIT, M>(A, smem, nb);
        case 16: return launch_traverse<16, AUDIT, M>(A, smem, nb);
        default: return FG_EUNSUPPORTED;
    }
}

static int launch_dispatch(int D, TravArgs &A, size_t smem, int64_t nb) {
    return A.audit ? launch_dispatch_t<true>(D, A, smem, nb) : launch_dispatch_t<false>(D, A, smem, nb);
}

// ------------------------------------------------------- far-field pass
// (fg_far_kernel.cuh) outputs per (bandwidth in launch, super-node) and the
// far kernel's per-warp scratch; per (host thread, device) like all scratch
struct FarScratch {
    DBuf work, st_node, st_f, ser, flag, tokens, settled, est, loc, rcnt, res;
    int grid = 0, cap = 0;
};

template <int D>
static int launch_far_t(TravArgs &A, int64_t ntask) {
    auto kern = far_kernel<D>;
    const size_t smem = sizeof(double) * (((3 * D + 1) & ~1) + ((A.K_loc + 1) & ~1)) * kFarWarps;
    int dev = 0, sms = 0, occ = 0;
    FG_CUDA_TRY(cudaGetDevice(&dev));
    FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFarThreads, smem));
    const int64_t full = (int64_t)sms * (occ < 1 ? 1 : occ);
    int64_t grid = std::min<int64_t>(full, (ntask + kFarWarps - 1) / kFarWarps);
    if (grid < 1) grid = 1;
    FarScratch &F = scratch<FarScratch, FarScratch>();
    const int cap = A.stack_cap;
    if (F.grid < grid || F.cap != cap) {
        const int64_t warps = grid * kFarWarps;
        FG_TRY(F.st_node.reserve(sizeof(int) * warps * cap));
        FG_TRY(F.st_f.reserve(sizeof(double) * warps * cap * 3));
        FG_TRY(F.ser.reserve(sizeof(int2) * warps * cap));
        F.grid = (int)grid;
        F.cap = cap;
    }
    A.far_st_node = F.st_node.as<int>();
    A.far_st_f = F.st_f.as<double>();
    A.far_ser = F.ser.as<int2>();
    FG_CUDA_TRY(cudaMemsetAsync(A.far_work, 0, sizeof(unsigned long long), stream()));
    count_launch();
    kern<<<(unsigned)grid, kFarThreads, smem, stream()>>>(A);
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

// Queue the far-field pass for the launch described by A (nh bandwidths).
static int queue_far(TreeDev &q, TravArgs &A) {
    const int64_t ntask = (int64_t)A.nh * q.nsn;
    FarScratch &F = scratch<FarScratch, FarScratch>();
    FG_TRY(F.work.reserve(sizeof(unsigned long long)));
    FG_TRY(F.flag.reserve(sizeof(int) * ntask));
    FG_TRY(F.tokens.reserve(sizeof(double) * ntask));
    FG_TRY(F.settled.reserve(sizeof(double) * ntask));
    FG_TRY(F.est.reserve(sizeof(double) * ntask));
    FG_TRY(F.rcnt.reserve(sizeof(int) * ntask));
    FG_TRY(F.res.reserve(sizeof(int) * ntask * kFarResCap));
    FG_TRY(F.loc.reserve(sizeof(double) * ntask * std::max(A.K_loc, 1)));
    A.q_ni = q.node_i.as<int4>();
    A.q_box = q.node_box.as<double>();
    A.q_c = q.node_c.as<double>();
    A.q_wr = q.node_wr.as<double2>();
    A.nsn = q.nsn;
    A.sn_node = q.sn_node.as<int>();
    A.sn_wmin = q.sn_wmin.as<double>();
    A.qb_super = q.qb_super.as<int>();
    A.far_work = F.work.as<unsigned long long>();
    A.far_flag = F.flag.as<int>();
    A.far_tokens = F.tokens.as<double>();
    A.far_settled = F.settled.as<double>();
    A.far_est = F.est.as<double>();
    A.far_loc = F.loc.as<double>();
    A.far_rcnt = F.rcnt.as<int>();
    A.far_res = F.res.as<int>();
    switch (q.dim) {
        case 1: return launch_far_t<1>(A, ntask);
        case 2: return launch_far_t<2>(A, ntask);
        case 3: return launch_far_t<3>(A, ntask);
        case 4: return launch_far_t<4>(A, ntask);
        case 5: return launch_far_t<5>(A, ntask);
        case 6: return launch_far_t<6>(A, ntask);
        case 7: return launch_far_t<7>(A, ntask);
        case 8: return launch_far_t<8>(A, ntask);
        case 12: return launch_far_t<12>(A, ntask);
        case 16: return launch_far_t<16>(A, ntask);
        default: return FG_EUNSUPPORTED;
    }
}

// The far-field pass is off by default: measured on C5's heaviest bandwidth
// (h = 0.153, ncu launch list) it costs 433 ms to save ~10 ms of the blocks'
// 946 ms -- at eps = 0.001 the reference's H2L bound (the (sqrt2 r_R)^p
// cross[p] term, 448x Hermite's at p = 6) almost never admits a super-node
// level translation, so S-level work is FD prunes and a few direct locals
// (DESIGN.md "Far-field pass").  FG_FAR=1 / fg_set_far_pass(1) turn it on.
int g_far_pass = 0;
static constexpr int64_t kFarMinBlocks = 4;  // blocks per super-node on average

// FP32 base cases for these bandwidths?
static int fp32_enabled(const TreeDev &q, const TreeDev &r, const double *hs, int nh, double eps) {
    int fp32 = g_fp32_base;
    if (const char *env = getenv("FG_FP32_BASE")) fp32 = atoi(env);
    if (!q.fp32_ok || !r.fp32_ok || !(eps > 0.0)) fp32 = 0;
    for (int j = 0; j < nh; j++)
        if (!(fabs(-1.4426950408889634 / (2.0 * hs[j] * hs[j])) < 1e30)) fp32 = 0;
    return fp32;
}

// Per-tree preparation the traversal needs (each computed once per tree and
// cached): query blocks, the Jensen node statistics, the anchored FP32 records.
// Queued before a launch's timing window so that window holds the traversal.
static int prepare_traversal(TreeDev &q, TreeDev &r, const double *hs, int nh, double eps) {
    FG_TRY(query_blocks(q));
    if (!getenv("FG_NO_JENSEN")) FG_TRY(node_js(r));
    if (fp32_enabled(q, r, hs, nh, eps) && q.dim < 5) FG_TRY(fp32_pack(r));
    return FG_OK;
}

// Queue one traversal launch over nh bandwidths (tasks = (bandwidth, query
// block) pairs, bandwidth-major), without synchronising.  moms[j] are the
// reference moments for hs[j] (DITO), outs[j] the value vectors, dcnt the
// nh x kCounters device counter block (zeroed here).  order/cost: LPT order
// and per-block cost capture (single full runs only).
static int queue_traversal(TreeDev &q, TreeDev &r, int nh, const double *hs,
                           const double *const *moms, double eps, int mode, int plimit,
                           int64_t b0, int64_t b1, int64_t stride, double *const *outs,
                           unsigned long long *dcnt, bool lpt, const AuditSink *audit = nullptr) {
    FG_REQUIRE(nh >= 1 && nh <= kMaxSweep, FG_EINVAL, "bad bandwidth count");
    FG_REQUIRE(eps >= 0.0, FG_EINVAL, "epsilon must be non-negative");
    FG_REQUIRE(mode >= FG_DFD && mode <= FG_DITO, FG_EINVAL, "unknown algorithm");
    FG_REQUIRE(q.dim == r.dim && q.dim_user == r.dim_user, FG_EINVAL,
               "query and reference dimensions differ");
    for (int j = 0; j < nh; j++) FG_REQUIRE(hs[j] > 0.0, FG_EINVAL, "bandwidth must be positive");
    const int D = q.dim;
    const bool series = mode == FG_DITO;
    FG_TRY(query_blocks(q));
    if (b1 < 0 || b1 > q.nqb) b1 = q.nqb;
    if (b0 < 0) b0 = 0;
    TravArgs A;
    memset(&A, 0, sizeof(A));
    A.r_pw = r.pw.as<double>();
    A.r_ni = r.node_i.as<int4>();
    A.r_box = r.node_box.as<double>();
    A.r_c = r.node_c.as<double>();
    A.r_wr = r.node_wr.as<double2>();
    if (!getenv("FG_NO_JENSEN")) {  // experiment knob: K_lo-only mass bounds
        FG_TRY(node_js(r));
        A.r_js = r.node_js.as<double2>();
    }
    A.q_pw = q.pw.as<double>();
    A.qb_range = q.qb_range.as<int2>();
    A.qb_box = q.qb_box.as<double>();
    A.qb_c = q.qb_c.as<double>();
    A.qb_rad = q.qb_rad.as<double>();
    // monochromatic: every query is also a reference point, so G(x_q) >= w_q
    // (its own term, K(0) = 1) -- a lower bound available from the first step
    A.qb_wmin = &q == &r ? q.qb_wmin.as<double>() : nullptr;
    A.qb_wsum = q.qb_wsum.as<double>();
    A.q_perm = q.perm.as<int64_t>();
    A.b0 = b0;
    A.b1 = b1;
    A.stride = stride < 1 ? 1 : stride;
    A.nbl = b1 > b0 ? (b1 - b0 + A.stride - 1) / A.stride : 0;
    A.total_w = r.total_w;
    A.use_tokens = mode >= FG_DFDO;
    A.use_series = series;
    A.plimit = plimit;
    A.stack_cap = g_stack_cap;
    {
        const char *env = getenv("FG_BFS_CAP");
        A.bfs_cap = env ? atoi(env) : g_stack_cap / 16;  // (256: C5 -1.9 % against 1024)
    }
    if (series) {
        int st = FG_OK;
        const SeriesTables *T = series_tables(D, plimit, &st);
        FG_TRY(st);
        A.K = T->K;
        A.digits = T->digits.as<uint8_t>();
        A.inv_fact = T->inv_fact.as<double>();
        A.degrees = T->degrees.as<int>();
        A.mom_K = r.mom_K;
        double ct[kMaxOrder + 1], cross[kMaxOrder + 1], floor_c;
        // the caller's dimension: padded coordinates add nothing to the bounds
        tail_tables(q.dim_user > 0 ? q.dim_user : D, plimit, ct, cross, &floor_c);
        for (int p = 0; p <= plimit; p++) {
            A.ct[p] = ct[p];
            A.cross[p] = cross[p];
            A.kp[p] = T->h_prefix[p];
        }
        A.floor_c = floor_c;
        // local expansions live in shared memory per warp: capped order
        A.plimit_loc = std::min(plimit, kLocOrder);
        while (A.plimit_loc > 1 && T->h_prefix[A.plimit_loc] > kLocK) A.plimit_loc--;
        A.K_loc = T->h_prefix[A.plimit_loc];
    }
    // per warp: query box + centroid + local coefficients, 2 x 32 staged FP64
    // points, the FP32 batch
    size_t smem;
    {
        static const int fixd[kDimSlots] = {0,
                                    warp_fixed_doubles<1>(), warp_fixed_doubles<2>(),
                                    warp_fixed_doubles<3>(), warp_fixed_doubles<4>(),
                                    warp_fixed_doubles<5>(), warp_fixed_doubles<6>(),
                                    warp_fixed_doubles<7>(), warp_fixed_doubles<8>(), 0, 0, 0,
                                    warp_fixed_doubles<12>(), 0, 0, 0, warp_fixed_doubles<16>()};
        smem = sizeof(double) * (fixd[D] + ((A.K_loc + 1) & ~1)) *kTravWarps;
    }
    TravScratch &g_scr = trav_scratch();
    FG_TRY(g_scr.work.reserve(sizeof(unsigned long long)));
    A.work = g_scr.work.as<unsigned long long>();
    FG_CUDA_TRY(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * kCounters * nh, stream()));
    // FP32 base cases: a share kFp32Share of eps
    // is reserved for their rounding error, the rest drives the traversal
    const int fp32 = fp32_enabled(q, r, hs, nh, eps);
    if (fp32 && D < 5) {  // anchored FP32 records (the direct stream at D >= 5 needs none)
        FG_TRY(fp32_pack(r));
        A.r_pf = r.pf.as<float>();
        A.r_anchor = r.anchor.as<int>();
    }
    A.nh = nh;
    // D <= 4 (record-pair batches): 0.2 measured C5 -2.3 %, C2 -4 % against 0.1
    double phi = D <= 4 ? 2.0 * kFp32Share : kFp32Share;
    if (const char *env = getenv("FG_FP32_SHARE")) phi = atof(env);  // experiment knob
    for (int j = 0; j < nh; j++) {
        TravH &H = A.hp[j];
        const double h = hs[j];
        H.h = h;
        H.neg_inv = -0.5 / (h * h);
        H.inv_h = 1.0 / h;
        H.sc = kSqrt2 * h;
        H.inv_sc = 1.0 / H.sc;
        H.fp32_rho = fp32 ? phi * eps : 0.0;
        H.eps = fp32 ? (1.0 - phi) * eps : eps;
        H.ex2_scale = (float)(-1.4426950408889634 / (2.0 * h * h));
        H.r_mom = series ? moms[j] : nullptr;
        H.out = outs[j];
        H.counters = dcnt + (size_t)kCounters * j;
        H.ref_leaf = ref_leaf_for(q, h);
        {
            // leaves mostly run as packed FP32 when that path is on: the measured
            // best exhaustive-vs-series balance is ~(3D + 8) / 6 per pair column
            // (C5: 2.5-3.5 beat 5 by 10-18 %, 8.5 by 25 %), against 2D + 20 in FP64
            double c = fp32 ? (3.0 * D + 8.0) / 6.0 : 2.0 * D + 20.0;
            if (const char *env = getenv("FG_PAIR_COST")) c = atof(env);  // experiment knob
            H.pair_cost = c;
            // Hermite evaluation per query slot: c0 + c1 K_p.  D = 3 runs the row
            // machine (fg_series.cuh: one FMA and half a shared-memory load per
            // coefficient and slot; C5 scan: (40, 2) beats (96, 4) by 1.8 %)
            H.herm_c0 = D == 3 ? 40.0 : 32.0 * D;
            H.herm_c1 = D == 3 ? 2.0 : D + 1.0;
            if (const char *env = getenv("FG_HERM_C0")) H.herm_c0 = atof(env);  // experiment knobs
            if (const char *env = getenv("FG_HERM_C1")) H.herm_c1 = atof(env);
        }
    }
    // Bandwidth groups run heaviest-first: a (bandwidth, block) task costs most
    // when h is a few times the query block's radius (the block can neither be
    // pruned whole nor use a cheap series, and the exact region is wide).
    // Starting those groups first leaves the cheap ones to fill the launch's
    // tail (C2 sweep: tasks' summed cycles / launch time 0.67 -> see DESIGN.md
    // "Task order").  Order only: every task's result is unchanged.
    {
        const double rb = q.qb_rad_median > 0.0 ? q.qb_rad_median : 1.0;
        double key[kMaxSweep];
        for (int j = 0; j < nh; j++) {
            key[j] = fabs(log(hs[j] / rb) - log(kHeavyRatio));
            A.jord[j] = j;
        }
        if (getenv("FG_SWEEP_NATURAL") == nullptr)
            std::stable_sort(A.jord, A.jord + nh, [&](int a, int b) { return key[a] < key[b]; });
    }
    if (audit) {
        FG_REQUIRE(nh == 1, FG_EINVAL, "the audit ledger records single runs");
        A.audit = reinterpret_cast<AuditEvent *>(audit->events);
        A.audit_count = audit->count;
        A.audit_cap = audit->cap;
        FG_CUDA_TRY(cudaMemsetAsync(audit->count, 0, sizeof(unsigned long long), stream()));
    }
    if (getenv("FG_DEBUG_BLOCKS") && nh == 1) {
        FG_TRY(g_scr.dbg.reserve(sizeof(unsigned long long) * kDbgFields * q.nqb));
        FG_CUDA_TRY(cudaMemsetAsync(g_scr.dbg.p, 0, sizeof(unsigned long long) * kDbgFields * q.nqb, stream()));
        A.dbg = g_scr.dbg.as<unsigned long long>();
    }
    const bool full = b0 == 0 && b1 == q.nqb && A.stride == 1 && nh == 1 && lpt;
    if (full && A.nbl > 1) {
        FG_TRY(q.qb_cost.reserve(sizeof(unsigned long long) * q.nqb));
        A.cost = q.qb_cost.as<unsigned long long>();
        if (q.qb_order_valid) A.order = q.qb_order.as<int>();
    }
    {
        int far = g_far_pass;
        if (const char *env = getenv("FG_FAR")) far = atoi(env);  // experiment knob
        if (far && !audit && A.nbl > 0 && q.nsn > 0 && q.nqb >= kFarMinBlocks * q.nsn)
            FG_TRY(queue_far(q, A));
    }
    if (A.nbl > 0) FG_TRY(launch_dispatch(D, A, smem, A.nbl * nh));
    if (A.cost) {
        // the next single run on this tree visits blocks heaviest-first (LPT
        // order); keys are cycle counts, so bits 8..40 order them well enough
        const int nq = (int)q.nqb;
        size_t tmp_bytes = 0;
        FG_TRY(q.qb_iota.reserve(sizeof(int) * nq));
        const int *iota = q.qb_iota.as<int>();
        count_launch();
        iota_kernel<<<(nq + 255) / 256, 256, 0, stream()>>>(q.qb_iota.as<int>(), nq);
        cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(
            nullptr, tmp_bytes, A.cost, (unsigned long long *)nullptr, iota, (int *)nullptr, nq,
            8, 40, stream());
        if (e == cudaSuccess) {
            FG_TRY(q.qb_sort_tmp.reserve(tmp_bytes + 16));
            FG_TRY(q.qb_keys.reserve(sizeof(unsigned long long) * nq));
            FG_TRY(q.qb_order.reserve(sizeof(int) * nq));
            e = cub::DeviceRadixSort::SortPairsDescending(
                q.qb_sort_tmp.p, tmp_bytes, A.cost, q.qb_keys.as<unsigned long long>(), iota,
                q.qb_order.as<int>(), nq, 8, 40, stream());
        }
        if (e != cudaSuccess) {
            set_error(std::string("block order sort: ") + cudaGetErrorString(e));
            return FG_ECUDA;
        }
        count_launch();
        q.qb_order_valid = true;
    }
    return FG_OK;
}

static void fill_counters(const unsigned long long *c, fg_counters *o) {
    o->pair_visits = (int64_t)c[0];
    o->base_cases = (int64_t)c[1];
    o->fd_prunes = (int64_t)c[2];
    o->hermite_prunes = (int64_t)c[3];
    o->local_prunes = (int64_t)c[4];
    o->h2l_prunes = (int64_t)c[5];
    o->exact_pairs = (int64_t)c[6];
    o->fp32_pairs = (int64_t)c[7];
    o->hermite_evals = (int64_t)c[9];
    o->hermite_terms = (int64_t)c[11];
    o->local_evals = (int64_t)c[10];
}

int run_traversal(TreeDev &q, TreeDev &r, double h, double eps, int mode, int plimit,
                  int64_t b0, int64_t b1, int64_t stride, double *d_values, fg_counters *counters,
                  double *seconds, const AuditSink *audit) {
    FG_REQUIRE(h > 0.0, FG_EINVAL, "bandwidth must be positive");
    const int D = q.dim;
    if (plimit <= 0) plimit = default_plimit(D);
    if (mode == FG_DITO) {
        FG_REQUIRE(plimit <= kMaxOrder, FG_EUNSUPPORTED, "plimit above the device order cap (12) is not supported");
        FG_REQUIRE(r.mom_valid && r.mom_h == h && r.mom_order >= plimit, FG_ESTALE,
                   "reference moments missing or stale; call refresh_moments for this "
                   "bandwidth first");
    }
    // timing events and the pinned counter buffer are created once per thread
    static thread_local cudaEvent_t e0 = nullptr, e1 = nullptr;
    static thread_local unsigned long long *cnt = nullptr;
    if (!e0) {
        FG_CUDA_TRY(cudaEventCreate(&e0));
        FG_CUDA_TRY(cudaEventCreate(&e1));
        FG_CUDA_TRY(cudaMallocHost(&cnt, sizeof(unsigned long long) * kCounters));
    }
    TravScratch &g_scr = trav_scratch();
    FG_TRY(g_scr.counters.reserve(sizeof(unsigned long long) * kCounters));
    const double *mom = r.mom.as<double>();
    FG_TRY(prepare_traversal(q, r, &h, 1, eps));
    FG_CUDA_TRY(cudaEventRecord(e0, stream()));
    FG_TRY(queue_traversal(q, r, 1, &h, &mom, eps, mode, plimit, b0, b1, stride, &d_values,
                           g_scr.counters.as<unsigned long long>(), !audit, audit));
    FG_CUDA_TRY(cudaEventRecord(e1, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(cnt, g_scr.counters.p, sizeof(unsigned long long) * kCounters,
                                cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    if (seconds) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *seconds = ms * 1e-3;
    }
    if (const char *dbg_path = getenv("FG_DEBUG_BLOCKS")) {
        std::vector<unsigned long long> hd(kDbgFields * q.nqb);
        cudaMemcpy(hd.data(), g_scr.dbg.p, sizeof(unsigned long long) * kDbgFields * q.nqb,
                   cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(dbg_path, "ab")) {
            fwrite(hd.data(), sizeof(unsigned long long), hd.size(), f);
            fclose(f);
        }
    }
    if (counters) fill_counters(cnt, counters);
    return FG_OK;
}

int run_sweep(TreeDev &q, TreeDev &r, const double *hs, int nh, double eps, int mode, int plimit,
              double *d_values, fg_counters *counters, double *seconds, int64_t b0, int64_t b1,
              int64_t stride) {
    const int D = q.dim;
    // the engine's own order cap unless the caller fixes one (padded
    // dimensions: the caller's dimension decides, as for the bounds)
    if (plimit <= 0) {
        const int du = q.dim_user > 0 ? q.dim_user : D;
        plimit = engine_plimit(du);
        // The engine's own cap must not outgrow the device: a chunk of the sweep
        // keeps one moment set per bandwidth (nodes x K doubles each, plus the
        // base set and the partial sums).  Fall back towards the reference's
        // cap while they would take more than 40 % of the free memory.
        if (mode == FG_DITO) {
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
                const double sets = (double)std::min(nh, kMaxSweep) + 3.0;
                while (plimit > default_plimit(du) &&
                       sets * (double)r.nnodes * iset_count(du, plimit) * 8.0 > 0.4 * (double)fr)
                    plimit--;
            } else {
                cudaGetLastError();
            }
        }
    }
    FG_REQUIRE(nh >= 1, FG_EINVAL, "need at least one bandwidth");
    for (int j = 0; j < nh; j++) FG_REQUIRE(hs[j] > 0.0, FG_EINVAL, "bandwidth must be positive");
    const bool series = mode == FG_DITO;
    struct SweepScr {
        DBuf mom, cnt;
    };
    SweepScr &ss = scratch<SweepScr, SweepScr>();
    DBuf &s_mom = ss.mom, &s_cnt = ss.cnt;
    static thread_local std::vector<cudaEvent_t> evs;
    const int nchunk = (nh + kMaxSweep - 1) / kMaxSweep;
    while ((int)evs.size() < 2 * nchunk) {
        cudaEvent_t e;
        FG_CUDA_TRY(cudaEventCreate(&e));
        evs.push_back(e);
    }
    FG_TRY(s_cnt.reserve(sizeof(unsigned long long) * kCounters * nh));
    FG_TRY(query_blocks(q));
    const int64_t m = q.n;
    for (int c = 0; c < nchunk; c++) {
        const int j0 = c * kMaxSweep, nj = std::min(kMaxSweep, nh - j0);
        std::vector<const double *> moms(nj, nullptr);
        std::vector<double *> outs(nj);
        for (int j = 0; j < nj; j++) outs[j] = d_values + m * (j0 + j);
        if (series) {
            // every bandwidth's moments by the exact rescaling law from the
            // tree's base moments (moments_refresh), materialised side by side
            FG_TRY(moments_multi(r, hs + j0, nj, plimit, s_mom));
            for (int j = 0; j < nj; j++)
                moms[j] = s_mom.as<double>() + (size_t)j * r.nnodes * r.mom_K;
        }
        // the event window holds the traversal launch alone (the moment
        // rescaling above and the per-tree preparation are outside it)
        FG_TRY(prepare_traversal(q, r, hs + j0, nj, eps));
        FG_CUDA_TRY(cudaEventRecord(evs[2 * c], stream()));
        FG_TRY(queue_traversal(q, r, nj, hs + j0, moms.data(), eps, mode, plimit, b0, b1, stride,
                               outs.data(), s_cnt.as<unsigned long long>() + kCounters * j0, false));
        FG_CUDA_TRY(cudaEventRecord(evs[2 * c + 1], stream()));
    }
    std::vector<unsigned long long> hc((size_t)kCounters * nh);
    FG_CUDA_TRY(cudaMemcpyAsync(hc.data(), s_cnt.p, sizeof(unsigned long long) * kCounters * nh,
                                cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    for (int c = 0; c < nchunk; c++) {
        const int j0 = c * kMaxSweep, nj = std::min(kMaxSweep, nh - j0);
        float ms = 0.f;
        FG_CUDA_TRY(cudaEventElapsedTime(&ms, evs[2 * c], evs[2 * c + 1]));
        // one launch serves nj bandwidths: split its time by their summed
        // per-block cycles
        double cyc = 0.0;
        for (int j = 0; j < nj; j++) cyc += (double)hc[(size_t)kCounters * (j0 + j) + 8];
        if (getenv("FG_DEBUG_SWEEP"))
            fprintf(stderr, "sweep chunk %d: %.3f ms, task cycles %.4e (= %.3f ms over %d warps at 1.965 GHz)\n",
                    c, ms, cyc, cyc / (1.965e6 * 148 * 16), 148 * 16);
        for (int j = 0; j < nj; j++) {
            const double share = cyc > 0.0 ? hc[(size_t)kCounters * (j0 + j) + 8] / cyc : 1.0 / nj;
            if (seconds) seconds[j0 + j] = ms * 1e-3 * share;
            if (counters) fill_counters(hc.data() + (size_t)kCounters * (j0 + j), counters + j0 + j);
        }
    }
    if (series) {
        // leave the tree's moments at the last bandwidth (refresh semantics)
        FG_TRY(moments_refresh(r, hs[nh - 1], plimit));
    }
    return FG_OK;
}

}  // namespace fg

extern "C" int fg_check_failures(int64_t *count) {
    FG_REQUIRE(count, FG_EINVAL, "null argument");
#if FG_CHECKS
    unsigned long long v = 0, z = 0;
    FG_CUDA_TRY(cudaMemcpyFromSymbol(&v, fg::g_fg_check_fail, sizeof(v)));
    FG_CUDA_TRY(cudaMemcpyToSymbol(fg::g_fg_check_fail, &z, sizeof(z)));
    *count = (int64_t)v;
#else
    *count = -1;  // this build has no device checks
#endif
    return FG_OK;
}
