// fg_tree.cu -- K3/K4: level-synchronous kd-tree build on the device
// (replaces build_tree, spatial_index.py:231-276).
//
// Every level processes all active nodes at once.  A node's contiguous range
// is cut into chunks of kChunk points; per-chunk partial statistics are
// combined per node in a fixed order (deterministic).  The split rule is the
// reference's: widest bounding-box dimension (first on ties), midpoint of the
// points' range, `x[dim] < mid` goes left with order preserved, and a node is
// a leaf when count <= leaf_threshold, its box has zero width, or the split is
// one-sided.  The stable per-chunk partition therefore reproduces the
// reference's permutation and node ranges exactly.
//
// The whole build is ONE cooperative launch: a resident grid walks all levels,
// separating the phases of a level (chunk statistics, node combine, radius and
// left counts, split decision, grid-wide scans, stable scatter, child
// allocation) with grid-wide barriers.  No host round trip per level.
//
// Points live as SoA coordinate planes (ping-pong) during the build; a node's
// points are copied to the final tree-order arrays when it becomes a leaf.
// Node ids are allocated level by level (BFS), so each level is a contiguous
// id range, which the bottom-up moment pass uses.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "fg_device.cuh"
#include "fg_internal.cuh"

namespace cg = cooperative_groups;

namespace fg {

// A chunk is processed by one warp (8 points per lane): deep levels hold many
// tiny nodes, and warp-level reductions need no block barriers.
#ifndef FG_BUILD_CHUNK
#define FG_BUILD_CHUNK 256
#endif
constexpr int kChunk = FG_BUILD_CHUNK;
constexpr int kBuildThreads = 256;
constexpr int kPerThread = kChunk / kBuildThreads;  // 8
constexpr int kMaxLevels = 1024;

// control block (device): level state written by one thread between barriers
enum { kNa = 0, kNchunks = 1, kNextBase = 2, kLevels = 3, kOverflow = 4, kSplit0 = 5, kCtl = 8 };
// kSplit0..kSplit0+2: per-level split counters of the small-node phase (by level % 3)

struct BuildBufs {
    DBuf x[2], w[2], idx[2];   // SoA coords (dim planes of n), weights, original index
    DBuf xf, wf, idxf;         // final (tree order)
    DBuf act[2];               // active node ids per level
    DBuf nch, choff;           // chunks per active slot, exclusive offsets (2 halves)
    DBuf chunk_slot, chunk_begin;
    DBuf part;                 // per-chunk partial stats (3*dim+1 doubles)
    DBuf part2;                // per-chunk radius partial
    DBuf lcnt, loff;           // per-chunk left counts / left offsets within node
    DBuf split_dim, split_mid, nleft, sval;
    DBuf done;                 // last-done counters, 2 per slot, by level parity
    DBuf lb_flag, lb_agg, lb_incl;  // per-CTA look-back state of the slot scan
    DBuf ctl, level_begin;
    DBuf bad;                  // validation flag
};

struct BuildArgs {
    int64_t n, nmax;
    int leaf;
    double *x[2], *w[2];
    int *idx[2];
    double *xf, *wf;
    int *idxf;
    int *act[2];
    int *nch, *choff;  // each 2 * nmax (halves by level parity)
    int *chunk_slot, *chunk_begin;
    double *part, *part2;
    int *lcnt, *loff;
    int *split_dim;
    double *split_mid;
    int *nleft;
    unsigned long long *sval;
    int *done, *lb_flag;
    unsigned long long *lb_agg, *lb_incl;
    int *ctl, *level_begin;
    int4 *node_i;
    double *node_box, *node_c;
    double2 *node_wr;
};

// -------------------------------------------------------------- kernels
__global__ void init_soa_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                int64_t n, int dim, double *__restrict__ x,
                                double *__restrict__ wo, int *__restrict__ idx,
                                int *__restrict__ bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int d = 0; d < dim; d++) {
        double v = pts[i * dim + d];
        x[(int64_t)d * n + i] = v;
        if (!(v == v) || v == CUDART_INF || v == -CUDART_INF) atomicOr(bad, 2);
        else if (fabs(v) > 0x1.0p60) atomicOr(bad, 4);
    }
    double wi = w ? w[i] : 1.0;
    if (!(wi > 0.0)) atomicOr(bad, 1);
    // FP32 base cases need weights well inside the FP32 normal range
    else if (wi < 0x1.0p-60 || wi > 0x1.0p60) atomicOr(bad, 4);
    wo[i] = wi;
    idx[i] = (int)i;
}

template <int D>
__device__ __forceinline__ void block_reduce_stats(double (&lo)[D], double (&hi)[D],
                                                   double (&sm)[D], double &ws,
                                                   double *sh /* [8 warps][3D+1] */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = warp_min(lo[d]);
        hi[d] = warp_max(hi[d]);
        sm[d] = warp_sum(sm[d]);
    }
    ws = warp_sum(ws);
    constexpr int F = 3 * D + 1;
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; d++) {
            sh[wid * F + d] = lo[d];
            sh[wid * F + D + d] = hi[d];
            sh[wid * F + 2 * D + d] = sm[d];
        }
        sh[wid * F + 3 * D] = ws;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = kBuildThreads / 32;
#pragma unroll
        for (int d = 0; d < D; d++) {
            lo[d] = lane < nw ? sh[lane * F + d] : CUDART_INF;
            hi[d] = lane < nw ? sh[lane * F + D + d] : -CUDART_INF;
            sm[d] = lane < nw ? sh[lane * F + 2 * D + d] : 0.0;
        }
        ws = lane < nw ? sh[lane * F + 3 * D] : 0.0;
#pragma unroll
        for (int d = 0; d < D; d++) {
            lo[d] = warp_min(lo[d]);
            hi[d] = warp_max(hi[d]);
            sm[d] = warp_sum(sm[d]);
        }
        ws = warp_sum(ws);
    }
    __syncthreads();
}

#include "fg_tree_coop.cuh"

template <int D>
__global__ void pack_tree_kernel(int64_t n, const double *__restrict__ xf,
                                 const double *__restrict__ wf, const int *__restrict__ idxf,
                                 double *__restrict__ pw, int64_t *__restrict__ perm) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    constexpr int S = packed_stride(D);
    double *o = pw + i * S;
#pragma unroll
    for (int d = 0; d < D; d++) o[d] = xf[(int64_t)d * n + i];
    o[D] = wf[i];
#pragma unroll
    for (int d = D + 1; d < S; d++) o[d] = 0.0;
    perm[i] = idxf[i];
}

// ------------------------------------------------------------- host side
__global__ void build_init_kernel(int4 *node_i, int *ctl, int *act0, int *nch, int *choff,
                                  int *level_begin, int *lb_flag, int grid, int *done,
                                  int64_t nmax, int n, int root_nch) {
    const int i = threadIdx.x;
    for (int k = i; k < grid; k += blockDim.x) lb_flag[k] = 0;
    if (i < kCtl) ctl[i] = i == kNa ? 1 : i == kNchunks ? root_nch : i == kNextBase ? 1 : 0;
    if (i == 0) {
        node_i[0] = make_int4(0, n, -1, -1);
        act0[0] = 0;
        nch[0] = root_nch;
        choff[0] = 0;
        level_begin[0] = 0;  // level 0 = {root}, level 1 starts at id 1
        level_begin[1] = 1;
        // level 0's slot (the root); later slots are zeroed when allocated
        done[0] = 0;
        done[nmax] = 0;
    }
}

template <int D>
static int build_levels(int64_t n, int leaf, BuildBufs &B, TreeDev &t) {
    const int64_t nmax = std::max<int64_t>(2 * n, 2);
    BuildArgs A;
    A.n = n;
    A.nmax = nmax;
    A.leaf = leaf;
    for (int k = 0; k < 2; k++) {
        A.x[k] = B.x[k].as<double>();
        A.w[k] = B.w[k].as<double>();
        A.idx[k] = B.idx[k].as<int>();
        A.act[k] = B.act[k].as<int>();
    }
    A.xf = B.xf.as<double>();
    A.wf = B.wf.as<double>();
    A.idxf = B.idxf.as<int>();
    A.nch = B.nch.as<int>();
    A.choff = B.choff.as<int>();
    A.chunk_slot = B.chunk_slot.as<int>();
    A.chunk_begin = B.chunk_begin.as<int>();
    A.part = B.part.as<double>();
    A.part2 = B.part2.as<double>();
    A.lcnt = B.lcnt.as<int>();
    A.loff = B.loff.as<int>();
    A.split_dim = B.split_dim.as<int>();
    A.split_mid = B.split_mid.as<double>();
    A.nleft = B.nleft.as<int>();
    A.sval = B.sval.as<unsigned long long>();
    A.ctl = B.ctl.as<int>();
    A.level_begin = B.level_begin.as<int>();
    A.node_i = t.node_i.as<int4>();
    A.node_box = t.node_box.as<double>();
    A.node_c = t.node_c.as<double>();
    A.node_wr = t.node_wr.as<double2>();

    // level 0: the root owns every point (one tiny kernel instead of a string
    // of host->device copies and memsets)
    const int root_nch = (int)((n + kChunk - 1) / kChunk);

    // resident grid for the cooperative launch (cached per dimension)
    struct GridCache {
        int g[kDimSlots] = {0};
    };
    auto &grid_cache = scratch<GridCache, GridCache>().g;  // per device
    int dev = 0;
    FG_CUDA_TRY(cudaGetDevice(&dev));
    if (!grid_cache[D]) {
        int sms = 0, occ = 0;
        FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, build_coop_kernel<D>,
                                                                  kBuildThreads, 0));
        const char *env = getenv("FG_BUILD_OCC");
        const int cap = env ? atoi(env) : 2;  // more CTAs only make the grid barriers dearer
        grid_cache[D] = sms * std::max(1, std::min(occ, cap));
    }
    const int grid = grid_cache[D];
    FG_TRY(B.lb_flag.reserve(sizeof(int) * grid));
    FG_TRY(B.lb_agg.reserve(sizeof(unsigned long long) * grid));
    FG_TRY(B.lb_incl.reserve(sizeof(unsigned long long) * grid));
    count_launch();
    build_init_kernel<<<1, 256, 0, stream()>>>(A.node_i, A.ctl, A.act[0], A.nch, A.choff,
                                               A.level_begin, B.lb_flag.as<int>(), grid,
                                               B.done.as<int>(), nmax, (int)n, root_nch);
    FG_CUDA_TRY(cudaGetLastError());
    A.lb_flag = B.lb_flag.as<int>();
    A.lb_agg = B.lb_agg.as<unsigned long long>();
    A.lb_incl = B.lb_incl.as<unsigned long long>();
    A.done = B.done.as<int>();
    void *args[] = {(void *)&A};
    count_launch();
    FG_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)build_coop_kernel<D>, grid,
                                            kBuildThreads, args, 0, stream()));
    // final packing (needs nothing from the host)
    FG_TRY(t.pw.reserve(sizeof(double) * n * packed_stride(D)));
    FG_TRY(t.perm.reserve(sizeof(int64_t) * n));
    count_launch();
    pack_tree_kernel<D><<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        n, B.xf.as<double>(), B.wf.as<double>(), B.idxf.as<int>(), t.pw.as<double>(),
        t.perm.as<int64_t>());
    FG_CUDA_TRY(cudaGetLastError());
    // one pinned read-back and one synchronisation: control block, validation
    // flags, root statistics, level starts
    struct Readback {
        int ctl[kCtl];
        int bad;
        double2 rootwr;
        int lb[kMaxLevels + 2];
    };
    static thread_local Readback *rb = nullptr;
    if (!rb) FG_CUDA_TRY(cudaMallocHost(&rb, sizeof(Readback)));
    FG_CUDA_TRY(cudaMemcpyAsync(rb->ctl, B.ctl.p, sizeof(rb->ctl), cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(&rb->bad, B.bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(&rb->rootwr, t.node_wr.p, sizeof(double2), cudaMemcpyDeviceToHost,
                                stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(rb->lb, B.level_begin.p, sizeof(rb->lb), cudaMemcpyDeviceToHost,
                                stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    FG_REQUIRE(!(rb->bad & 1), FG_EINVAL, "weights must be positive");
    FG_REQUIRE(!(rb->bad & 2), FG_EINVAL, "points must be finite");
    t.fp32_ok = !(rb->bad & 4);
    FG_REQUIRE(!rb->ctl[kOverflow] && rb->ctl[kNa] == 0, FG_ECUDA,
               "tree build: node capacity exceeded");
    const int levels = rb->ctl[kLevels];
    FG_TRY(t.level_begin_dev.reserve(sizeof(int) * (levels + 1)));
    FG_CUDA_TRY(cudaMemcpyAsync(t.level_begin_dev.p, B.level_begin.p, sizeof(int) * (levels + 1),
                                cudaMemcpyDeviceToDevice, stream()));
    t.levels = levels;
    t.nnodes = rb->ctl[kNextBase];
    t.level_begin.assign(rb->lb, rb->lb + levels + 1);
    t.total_w = rb->rootwr.x;
    return FG_OK;
}

int tree_build(const double *d_points, const double *d_weights, int64_t n, int dim, int leaf,
               TreeDev &t) {
    FG_REQUIRE(n >= 1, FG_EINVAL, "points must be a non-empty (N, D) array");
    FG_REQUIRE(dim >= 1, FG_EINVAL, "points must be a non-empty (N, D) array");
    FG_REQUIRE(leaf >= 1, FG_EINVAL, "leaf threshold must be at least 1");
    FG_REQUIRE(kernel_dim(dim) == dim, FG_EUNSUPPORTED, "kernel dimension must be 1..8, 12 or 16");
    FG_REQUIRE(n < (int64_t)1 << 30, FG_EUNSUPPORTED, "more than 2^30 points per tree");
    // build scratch is kept between builds (grow-only): a per-step tree costs
    // no allocation calls
    BuildBufs &B = scratch<BuildBufs, BuildBufs>();
    const int64_t nmax = std::max<int64_t>(2 * n, 2);
    const int64_t maxchunks = n / kChunk + nmax + 2;
    for (int k = 0; k < 2; k++) {
        FG_TRY(B.x[k].reserve(sizeof(double) * n * dim));
        FG_TRY(B.w[k].reserve(sizeof(double) * n));
        FG_TRY(B.idx[k].reserve(sizeof(int) * n));
        FG_TRY(B.act[k].reserve(sizeof(int) * nmax));
    }
    FG_TRY(B.xf.reserve(sizeof(double) * n * dim));
    FG_TRY(B.wf.reserve(sizeof(double) * n));
    FG_TRY(B.idxf.reserve(sizeof(int) * n));
    FG_TRY(B.nch.reserve(sizeof(int) * 2 * nmax));
    FG_TRY(B.choff.reserve(sizeof(int) * 2 * nmax));
    FG_TRY(B.chunk_slot.reserve(sizeof(int) * maxchunks));
    FG_TRY(B.chunk_begin.reserve(sizeof(int) * maxchunks));
    FG_TRY(B.part.reserve(sizeof(double) * maxchunks * (3 * dim + 1)));
    FG_TRY(B.part2.reserve(sizeof(double) * maxchunks));
    FG_TRY(B.lcnt.reserve(sizeof(int) * maxchunks));
    FG_TRY(B.loff.reserve(sizeof(int) * maxchunks));
    FG_TRY(B.split_dim.reserve(sizeof(int) * nmax));
    FG_TRY(B.split_mid.reserve(sizeof(double) * nmax));
    FG_TRY(B.nleft.reserve(sizeof(int) * nmax));
    FG_TRY(B.done.reserve(sizeof(int) * 4 * nmax));
    FG_TRY(B.sval.reserve(sizeof(unsigned long long) * nmax));
    FG_TRY(B.ctl.reserve(sizeof(int) * kCtl));
    FG_TRY(B.level_begin.reserve(sizeof(int) * (kMaxLevels + 2)));
    FG_TRY(B.bad.reserve(sizeof(int)));
    FG_TRY(t.node_i.reserve(sizeof(int4) * nmax));
    FG_TRY(t.node_box.reserve(sizeof(double) * nmax * 2 * dim));
    FG_TRY(t.node_c.reserve(sizeof(double) * nmax * dim));
    FG_TRY(t.node_wr.reserve(sizeof(double2) * nmax));
    FG_CUDA_TRY(cudaMemsetAsync(B.bad.p, 0, sizeof(int), stream()));
    count_launch();
    init_soa_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        d_points, d_weights, n, dim, B.x[0].as<double>(), B.w[0].as<double>(),
        B.idx[0].as<int>(), B.bad.as<int>());
    FG_CUDA_TRY(cudaGetLastError());
    // (validation flags are read back with the build's results: invalid
    // inputs still build a finite tree -- NaN compares false -- then raise)
    t.n = n;
    t.dim = dim;
    t.leaf = leaf;
    t.stride = packed_stride(dim);
    t.mom_valid = t.mom0_valid = false;
    t.qb_valid = false;
    t.pf_valid = false;
    t.js_valid = false;
    t.mom_items_valid = false;
    switch (dim) {
        case 1: return build_levels<1>(n, leaf, B, t);
        case 2: return build_levels<2>(n, leaf, B, t);
        case 3: return build_levels<3>(n, leaf, B, t);
        case 4: return build_levels<4>(n, leaf, B, t);
        case 5: return build_levels<5>(n, leaf, B, t);
        case 6: return build_levels<6>(n, leaf, B, t);
        case 7: return build_levels<7>(n, leaf, B, t);
        case 8: return build_levels<8>(n, leaf, B, t);
        case 12: return build_levels<12>(n, leaf, B, t);
        default: return build_levels<16>(n, leaf, B, t);
    }
}

// --------------------------------------------------- export (preorder)
// preorder numbering: depth-first, left before right (spatial_index.py:246-273)
static void preorder_numbering(const std::vector<int4> &ni, std::vector<int64_t> &pre) {
    pre.assign(ni.size(), -1);
    std::vector<int> stack;
    stack.reserve(128);
    stack.push_back(0);
    int64_t next = 0;
    while (!stack.empty()) {
        int v = stack.back();
        stack.pop_back();
        pre[v] = next++;
        if (ni[v].z >= 0) {
            stack.push_back(ni[v].w);
            stack.push_back(ni[v].z);
        }
    }
}

int preorder_map(const TreeDev &t, std::vector<int64_t> &pre) {
    std::vector<int4> ni(t.nnodes);
    FG_CUDA_TRY(cudaMemcpyAsync(ni.data(), t.node_i.p, sizeof(int4) * t.nnodes,
                                cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    preorder_numbering(ni, pre);
    return FG_OK;
}

int tree_export(const TreeDev &t, int64_t *perm, int64_t *start, int64_t *end, double *lo,
                double *hi, double *center, double *weight, double *inf_radius, int64_t *left,
                int64_t *right) {
    const int64_t nn = t.nnodes;
    const int D = t.dim, DU = t.dim_user > 0 ? t.dim_user : t.dim;
    std::vector<int4> ni(nn);
    std::vector<double> box(nn * 2 * D), ctr(nn * D);
    std::vector<double2> wr(nn);
    FG_CUDA_TRY(cudaMemcpyAsync(ni.data(), t.node_i.p, sizeof(int4) * nn, cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(box.data(), t.node_box.p, sizeof(double) * nn * 2 * D, cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(ctr.data(), t.node_c.p, sizeof(double) * nn * D, cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(wr.data(), t.node_wr.p, sizeof(double2) * nn, cudaMemcpyDeviceToHost, stream()));
    if (perm) FG_CUDA_TRY(cudaMemcpyAsync(perm, t.perm.p, sizeof(int64_t) * t.n, cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    std::vector<int64_t> pre;
    preorder_numbering(ni, pre);
    for (int64_t v = 0; v < nn; v++) {
        const int64_t p = pre[v];
        if (start) start[p] = ni[v].x;
        if (end) end[p] = (int64_t)ni[v].x + ni[v].y;
        if (left) left[p] = ni[v].z >= 0 ? pre[ni[v].z] : -1;
        if (right) right[p] = ni[v].w >= 0 ? pre[ni[v].w] : -1;
        for (int d = 0; d < DU; d++) {  // the caller's dimensions (padding dropped)
            if (lo) lo[p * DU + d] = box[v * 2 * D + d];
            if (hi) hi[p * DU + d] = box[v * 2 * D + D + d];
            if (center) center[p * DU + d] = ctr[v * D + d];
        }
        if (weight) weight[p] = wr[v].x;
        if (inf_radius) inf_radius[p] = wr[v].y;
    }
    return FG_OK;
}

}  // namespace fg
