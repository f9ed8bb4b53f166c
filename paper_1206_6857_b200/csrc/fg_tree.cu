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
// Points live as SoA coordinate planes (ping-pong) during the build; a node's
// points are copied to the final tree-order arrays when it becomes a leaf.
// Node ids are allocated level by level (BFS), so each level is a contiguous
// id range, which the bottom-up moment pass uses.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "fg_device.cuh"
#include "fg_internal.cuh"

namespace fg {

constexpr int kChunk = 2048;
constexpr int kBuildThreads = 256;
constexpr int kPerThread = kChunk / kBuildThreads;  // 8

struct BuildBufs {
    DBuf x[2], w[2], idx[2];   // SoA coords (dim planes of n), weights, original index
    DBuf xf, wf, idxf;         // final (tree order)
    DBuf act[2];               // active node ids per level
    DBuf nch, choff;           // chunks per active slot, exclusive offsets
    DBuf chunk_slot, chunk_begin;
    DBuf part;                 // per-chunk partial stats (3*dim+1 doubles)
    DBuf part2;                // per-chunk radius partial
    DBuf lcnt, loff;           // per-chunk left counts / left offsets within node
    DBuf split_dim, split_mid, nleft, flag, rank;
    DBuf totals;               // int2: (nsplit, nchunks_next)
    DBuf scan_tmp;
    DBuf bad;                  // validation flag
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
    }
    double wi = w ? w[i] : 1.0;
    if (!(wi > 0.0)) atomicOr(bad, 1);
    wo[i] = wi;
    idx[i] = (int)i;
}

// chunk list for the active slots
__global__ void fill_chunks_kernel(int na, const int *__restrict__ act,
                                   const int4 *__restrict__ node_i, const int *__restrict__ nch,
                                   const int *__restrict__ choff, int *__restrict__ chunk_slot,
                                   int *__restrict__ chunk_begin) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= na) return;
    int4 ni = node_i[act[s]];
    int o = choff[s];
    for (int k = 0; k < nch[s]; k++) {
        chunk_slot[o + k] = s;
        chunk_begin[o + k] = ni.x + k * kChunk;
    }
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
}

template <int D>
__global__ void __launch_bounds__(kBuildThreads)
stats_partial_kernel(int64_t n, const double *__restrict__ x, const double *__restrict__ w,
                     const int *__restrict__ act, const int4 *__restrict__ node_i,
                     const int *__restrict__ chunk_slot, const int *__restrict__ chunk_begin,
                     double *__restrict__ part) {
    __shared__ double sh[(kBuildThreads / 32) * (3 * D + 1)];
    const int c = blockIdx.x;
    const int4 ni = node_i[act[chunk_slot[c]]];
    const int cb = chunk_begin[c];
    const int ce = min(cb + kChunk, ni.x + ni.y);
    double lo[D], hi[D], sm[D], ws = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = CUDART_INF;
        hi[d] = -CUDART_INF;
        sm[d] = 0.0;
    }
    for (int i = cb + threadIdx.x; i < ce; i += kBuildThreads) {
#pragma unroll
        for (int d = 0; d < D; d++) {
            double v = x[(int64_t)d * n + i];
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
            sm[d] += v;
        }
        ws += w[i];
    }
    block_reduce_stats<D>(lo, hi, sm, ws, sh);
    if (threadIdx.x == 0) {
        double *p = part + (int64_t)c * (3 * D + 1);
#pragma unroll
        for (int d = 0; d < D; d++) {
            p[d] = lo[d];
            p[D + d] = hi[d];
            p[2 * D + d] = sm[d];
        }
        p[3 * D] = ws;
    }
}

// warp per active slot: combine chunk partials, choose the split
template <int D>
__global__ void node_stats_kernel(int na, int leaf, const int *__restrict__ act,
                                  int4 *__restrict__ node_i, const int *__restrict__ nch,
                                  const int *__restrict__ choff, const double *__restrict__ part,
                                  double *__restrict__ node_box, double *__restrict__ node_c,
                                  double2 *__restrict__ node_wr, int *__restrict__ split_dim,
                                  double *__restrict__ split_mid) {
    const int lane = threadIdx.x & 31;
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= na) return;
    const int node = act[s];
    const int4 ni = node_i[node];
    double lo[D], hi[D], sm[D], ws = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = CUDART_INF;
        hi[d] = -CUDART_INF;
        sm[d] = 0.0;
    }
    const int c0 = choff[s], c1 = c0 + nch[s];
    for (int c = c0 + lane; c < c1; c += 32) {
        const double *p = part + (int64_t)c * (3 * D + 1);
#pragma unroll
        for (int d = 0; d < D; d++) {
            lo[d] = fmin(lo[d], p[d]);
            hi[d] = fmax(hi[d], p[D + d]);
            sm[d] += p[2 * D + d];
        }
        ws += p[3 * D];
    }
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = warp_min(lo[d]);
        hi[d] = warp_max(hi[d]);
        sm[d] = warp_sum(sm[d]);
    }
    ws = warp_sum(ws);
    if (lane == 0) {
        const double cnt = (double)ni.y;
        int sd = 0;
        double best = hi[0] - lo[0];
#pragma unroll
        for (int d = 0; d < D; d++) {
            node_box[(int64_t)node * 2 * D + d] = lo[d];
            node_box[(int64_t)node * 2 * D + D + d] = hi[d];
            node_c[(int64_t)node * D + d] = sm[d] / cnt;
            double wd = hi[d] - lo[d];
            if (d > 0 && wd > best) {
                best = wd;
                sd = d;
            }
        }
        node_wr[node] = make_double2(ws, 0.0);
        const bool leafy = ni.y <= leaf || best == 0.0;
        split_dim[s] = leafy ? -1 : sd;
        split_mid[s] = 0.5 * (lo[sd] + hi[sd]);
    }
}

// per chunk: inf-norm radius partial and left count
template <int D>
__global__ void __launch_bounds__(kBuildThreads)
radius_count_kernel(int64_t n, const double *__restrict__ x, const int *__restrict__ act,
                    const int4 *__restrict__ node_i, const int *__restrict__ chunk_slot,
                    const int *__restrict__ chunk_begin, const double *__restrict__ node_c,
                    const int *__restrict__ split_dim, const double *__restrict__ split_mid,
                    double *__restrict__ part2, int *__restrict__ lcnt) {
    __shared__ double shr[kBuildThreads / 32];
    __shared__ int shc[kBuildThreads / 32];
    const int c = blockIdx.x;
    const int s = chunk_slot[c];
    const int node = act[s];
    const int4 ni = node_i[node];
    const int cb = chunk_begin[c];
    const int ce = min(cb + kChunk, ni.x + ni.y);
    const int sd = split_dim[s];
    const double mid = split_mid[s];
    double ctr[D];
#pragma unroll
    for (int d = 0; d < D; d++) ctr[d] = node_c[(int64_t)node * D + d];
    double rad = 0.0;
    int cnt = 0;
    for (int i = cb + threadIdx.x; i < ce; i += kBuildThreads) {
#pragma unroll
        for (int d = 0; d < D; d++) {
            double v = x[(int64_t)d * n + i];
            rad = fmax(rad, fabs(v - ctr[d]));
        }
        if (sd >= 0) cnt += x[(int64_t)sd * n + i] < mid ? 1 : 0;
    }
    rad = warp_max(rad);
    cnt = warp_sum(cnt);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        shr[wid] = rad;
        shc[wid] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        int t = 0;
        for (int k = 0; k < kBuildThreads / 32; k++) {
            r = fmax(r, shr[k]);
            t += shc[k];
        }
        part2[c] = r;
        lcnt[c] = t;
    }
}

// warp per slot: radius, left count, per-chunk left offsets, final leaf test
__global__ void node_decide_kernel(int na, const int *__restrict__ act,
                                   const int4 *__restrict__ node_i, const int *__restrict__ nch,
                                   const int *__restrict__ choff, const double *__restrict__ part2,
                                   const int *__restrict__ lcnt, int *__restrict__ loff,
                                   double2 *__restrict__ node_wr, int *__restrict__ split_dim,
                                   int *__restrict__ nleft, int *__restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= na) return;
    const int node = act[s];
    const int4 ni = node_i[node];
    const int c0 = choff[s], c1 = c0 + nch[s];
    double rad = 0.0;
    int run = 0;  // running left count (exclusive offsets)
    for (int base = c0; base < c1; base += 32) {
        int c = base + lane;
        int v = c < c1 ? lcnt[c] : 0;
        if (c < c1) rad = fmax(rad, part2[c]);
        // inclusive warp scan
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        if (c < c1) loff[c] = run + incl - v;
        run += __shfl_sync(kFull, incl, 31);
    }
    rad = warp_max(rad);
    if (lane == 0) {
        double2 wr = node_wr[node];
        wr.y = rad;
        node_wr[node] = wr;
        int sd = split_dim[s];
        bool split = sd >= 0 && run > 0 && run < ni.y;
        if (!split) split_dim[s] = -1;
        nleft[s] = run;
        flag[s] = split ? 1 : 0;
    }
}

// per chunk: leaves copy to the final arrays; split nodes partition stably
template <int D>
__global__ void __launch_bounds__(kBuildThreads)
scatter_kernel(int64_t n, const double *__restrict__ x, const double *__restrict__ w,
               const int *__restrict__ idx, double *__restrict__ xn, double *__restrict__ wn,
               int *__restrict__ idxn, double *__restrict__ xf, double *__restrict__ wf,
               int *__restrict__ idxf, const int *__restrict__ act,
               const int4 *__restrict__ node_i, const int *__restrict__ chunk_slot,
               const int *__restrict__ chunk_begin, const int *__restrict__ split_dim,
               const double *__restrict__ split_mid, const int *__restrict__ nleft,
               const int *__restrict__ loff) {
    typedef cub::BlockScan<int, kBuildThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int c = blockIdx.x;
    const int s = chunk_slot[c];
    const int4 ni = node_i[act[s]];
    const int cb = chunk_begin[c];
    const int ce = min(cb + kChunk, ni.x + ni.y);
    const int sd = split_dim[s];
    if (sd < 0) {
        for (int i = cb + threadIdx.x; i < ce; i += kBuildThreads) {
#pragma unroll
            for (int d = 0; d < D; d++) xf[(int64_t)d * n + i] = x[(int64_t)d * n + i];
            wf[i] = w[i];
            idxf[i] = idx[i];
        }
        return;
    }
    const double mid = split_mid[s];
    const int i0 = cb + threadIdx.x * kPerThread;
    unsigned mask = 0;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kPerThread; k++) {
        int i = i0 + k;
        if (i < ce && x[(int64_t)sd * n + i] < mid) {
            mask |= 1u << k;
            cnt++;
        }
    }
    int excl;
    Scan(tmp).ExclusiveSum(cnt, excl);
    const int left_base = ni.x + loff[c];
    // elements of this chunk before thread: threadIdx.x*kPerThread (if in range)
    const int before = threadIdx.x * kPerThread;
    const int right_base = ni.x + nleft[s] + (cb - ni.x - loff[c]);
    int lrank = excl, rrank = before - excl;
#pragma unroll
    for (int k = 0; k < kPerThread; k++) {
        int i = i0 + k;
        if (i >= ce) break;
        int dst;
        if (mask & (1u << k)) dst = left_base + lrank++;
        else dst = right_base + rrank++;
#pragma unroll
        for (int d = 0; d < D; d++) xn[(int64_t)d * n + dst] = x[(int64_t)d * n + i];
        wn[dst] = w[i];
        idxn[dst] = idx[i];
    }
}

__global__ void make_children_kernel(int na, int next_base, const int *__restrict__ act,
                                     int4 *__restrict__ node_i, const int *__restrict__ flag,
                                     const int *__restrict__ rank, const int *__restrict__ nleft,
                                     int *__restrict__ act_next, int *__restrict__ nch_next) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= na) return;
    if (!flag[s]) return;
    const int node = act[s];
    int4 ni = node_i[node];
    const int r = rank[s];
    const int L = next_base + 2 * r, R = L + 1;
    const int nl = nleft[s];
    node_i[L] = make_int4(ni.x, nl, -1, -1);
    node_i[R] = make_int4(ni.x + nl, ni.y - nl, -1, -1);
    ni.z = L;
    ni.w = R;
    node_i[node] = ni;
    act_next[2 * r] = L;
    act_next[2 * r + 1] = R;
    nch_next[2 * r] = (nl + kChunk - 1) / kChunk;
    nch_next[2 * r + 1] = (ni.y - nl + kChunk - 1) / kChunk;
}

__global__ void totals_kernel(int na, const int *__restrict__ flag, const int *__restrict__ rank,
                              const int *__restrict__ nch_next, const int *__restrict__ choff_next,
                              int *__restrict__ totals) {
    int nsplit = na > 0 ? rank[na - 1] + flag[na - 1] : 0;
    int nn = 2 * nsplit;
    totals[0] = nsplit;
    totals[1] = nn > 0 ? choff_next[nn - 1] + nch_next[nn - 1] : 0;
}

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
static int scan_ints(const int *in, int *out, int count, BuildBufs &B) {
    size_t bytes = 0;
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, stream()));
    FG_TRY(B.scan_tmp.reserve(bytes + 16));
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(B.scan_tmp.p, bytes, in, out, count, stream()));
    return FG_OK;
}

template <int D>
static int build_levels(int64_t n, int leaf, BuildBufs &B, TreeDev &t) {
    const int nmax = (int)std::max<int64_t>(2 * n, 2);
    // node 0 = root
    int4 root = make_int4(0, (int)n, -1, -1);
    FG_CUDA_TRY(cudaMemcpyAsync(t.node_i.p, &root, sizeof(int4), cudaMemcpyHostToDevice, stream()));
    int zero = 0;
    int root_nch = (int)((n + kChunk - 1) / kChunk);
    FG_CUDA_TRY(cudaMemcpyAsync(B.act[0].p, &zero, sizeof(int), cudaMemcpyHostToDevice, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(B.nch.p, &root_nch, sizeof(int), cudaMemcpyHostToDevice, stream()));
    FG_CUDA_TRY(cudaMemcpyAsync(B.choff.p, &zero, sizeof(int), cudaMemcpyHostToDevice, stream()));
    int na = 1, nchunks = root_nch, cur = 0, next_base = 1, level = 0;
    t.level_begin.assign(1, 0);
    int *h_tot = nullptr;
    FG_CUDA_TRY(cudaMallocHost(&h_tot, 2 * sizeof(int)));
    int status = FG_OK;
    while (na > 0) {
        int *act = B.act[cur & 1].as<int>();
        int *act_next = B.act[(cur + 1) & 1].as<int>();
        int *nch = B.nch.as<int>() + (cur & 1) * nmax;
        int *choff = B.choff.as<int>() + (cur & 1) * nmax;
        int *nch_next = B.nch.as<int>() + ((cur + 1) & 1) * nmax;
        int *choff_next = B.choff.as<int>() + ((cur + 1) & 1) * nmax;
        const double *x = B.x[cur & 1].as<double>();
        const double *w = B.w[cur & 1].as<double>();
        const int *idx = B.idx[cur & 1].as<int>();
        count_launch();
        fill_chunks_kernel<<<(na + 127) / 128, 128, 0, stream()>>>(
            na, act, t.node_i.as<int4>(), nch, choff, B.chunk_slot.as<int>(),
            B.chunk_begin.as<int>());
        count_launch();
        stats_partial_kernel<D><<<nchunks, kBuildThreads, 0, stream()>>>(
            n, x, w, act, t.node_i.as<int4>(), B.chunk_slot.as<int>(), B.chunk_begin.as<int>(),
            B.part.as<double>());
        const int wblocks = (na * 32 + 255) / 256;
        count_launch();
        node_stats_kernel<D><<<wblocks, 256, 0, stream()>>>(
            na, leaf, act, t.node_i.as<int4>(), nch, choff, B.part.as<double>(),
            t.node_box.as<double>(), t.node_c.as<double>(), t.node_wr.as<double2>(),
            B.split_dim.as<int>(), B.split_mid.as<double>());
        count_launch();
        radius_count_kernel<D><<<nchunks, kBuildThreads, 0, stream()>>>(
            n, x, act, t.node_i.as<int4>(), B.chunk_slot.as<int>(), B.chunk_begin.as<int>(),
            t.node_c.as<double>(), B.split_dim.as<int>(), B.split_mid.as<double>(),
            B.part2.as<double>(), B.lcnt.as<int>());
        count_launch();
        node_decide_kernel<<<wblocks, 256, 0, stream()>>>(
            na, act, t.node_i.as<int4>(), nch, choff, B.part2.as<double>(), B.lcnt.as<int>(),
            B.loff.as<int>(), t.node_wr.as<double2>(), B.split_dim.as<int>(),
            B.nleft.as<int>(), B.flag.as<int>());
        FG_CUDA_TRY(cudaGetLastError());
        FG_TRY(scan_ints(B.flag.as<int>(), B.rank.as<int>(), na, B));
        count_launch();
        scatter_kernel<D><<<nchunks, kBuildThreads, 0, stream()>>>(
            n, x, w, idx, B.x[(cur + 1) & 1].as<double>(), B.w[(cur + 1) & 1].as<double>(),
            B.idx[(cur + 1) & 1].as<int>(), B.xf.as<double>(), B.wf.as<double>(),
            B.idxf.as<int>(), act, t.node_i.as<int4>(), B.chunk_slot.as<int>(),
            B.chunk_begin.as<int>(), B.split_dim.as<int>(), B.split_mid.as<double>(),
            B.nleft.as<int>(), B.loff.as<int>());
        FG_CUDA_TRY(cudaMemsetAsync(nch_next, 0, sizeof(int) * 2 * na, stream()));
        count_launch();
        make_children_kernel<<<(na + 127) / 128, 128, 0, stream()>>>(
            na, next_base, act, t.node_i.as<int4>(), B.flag.as<int>(), B.rank.as<int>(),
            B.nleft.as<int>(), act_next, nch_next);
        FG_CUDA_TRY(cudaGetLastError());
        FG_TRY(scan_ints(nch_next, choff_next, 2 * na, B));
        count_launch();
        totals_kernel<<<1, 1, 0, stream()>>>(na, B.flag.as<int>(), B.rank.as<int>(), nch_next,
                                             choff_next, B.totals.as<int>());
        FG_CUDA_TRY(cudaMemcpyAsync(h_tot, B.totals.p, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                                    stream()));
        FG_CUDA_TRY(cudaStreamSynchronize(stream()));
        const int nsplit = h_tot[0];
        nchunks = h_tot[1];
        level++;
        if (nsplit > 0) t.level_begin.push_back(next_base);
        next_base += 2 * nsplit;
        na = 2 * nsplit;
        cur++;
        if (next_base > nmax) {
            set_error("tree build: node capacity exceeded");
            status = FG_ECUDA;
            break;
        }
    }
    cudaFreeHost(h_tot);
    FG_TRY(status);
    t.levels = level;
    t.nnodes = next_base;
    t.level_begin.push_back(next_base);
    // final packing
    FG_TRY(t.pw.reserve(sizeof(double) * n * packed_stride(D)));
    FG_TRY(t.perm.reserve(sizeof(int64_t) * n));
    count_launch();
    pack_tree_kernel<D><<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        n, B.xf.as<double>(), B.wf.as<double>(), B.idxf.as<int>(), t.pw.as<double>(),
        t.perm.as<int64_t>());
    FG_CUDA_TRY(cudaGetLastError());
    double2 rootwr;
    FG_CUDA_TRY(cudaMemcpyAsync(&rootwr, t.node_wr.p, sizeof(double2), cudaMemcpyDeviceToHost,
                                stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    t.total_w = rootwr.x;
    return FG_OK;
}

int tree_build(const double *d_points, const double *d_weights, int64_t n, int dim, int leaf,
               TreeDev &t) {
    FG_REQUIRE(n >= 1, FG_EINVAL, "points must be a non-empty (N, D) array");
    FG_REQUIRE(dim >= 1, FG_EINVAL, "points must be a non-empty (N, D) array");
    FG_REQUIRE(leaf >= 1, FG_EINVAL, "leaf threshold must be at least 1");
    FG_REQUIRE(dim <= kMaxDim, FG_EUNSUPPORTED, "dimension > 8 is not supported by this build");
    FG_REQUIRE(n < (int64_t)1 << 30, FG_EUNSUPPORTED, "more than 2^30 points per tree");
    BuildBufs B;
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
    FG_TRY(B.flag.reserve(sizeof(int) * nmax));
    FG_TRY(B.rank.reserve(sizeof(int) * nmax));
    FG_TRY(B.totals.reserve(sizeof(int) * 2));
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
    int bad = 0;
    FG_CUDA_TRY(cudaMemcpyAsync(&bad, B.bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    FG_REQUIRE(!(bad & 1), FG_EINVAL, "weights must be positive");
    FG_REQUIRE(!(bad & 2), FG_EINVAL, "points must be finite");
    t.n = n;
    t.dim = dim;
    t.leaf = leaf;
    t.stride = packed_stride(dim);
    t.mom_valid = t.mom0_valid = false;
    t.qb_valid = false;
    switch (dim) {
        case 1: return build_levels<1>(n, leaf, B, t);
        case 2: return build_levels<2>(n, leaf, B, t);
        case 3: return build_levels<3>(n, leaf, B, t);
        case 4: return build_levels<4>(n, leaf, B, t);
        case 5: return build_levels<5>(n, leaf, B, t);
        case 6: return build_levels<6>(n, leaf, B, t);
        case 7: return build_levels<7>(n, leaf, B, t);
        default: return build_levels<8>(n, leaf, B, t);
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
    const int D = t.dim;
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
        for (int d = 0; d < D; d++) {
            if (lo) lo[p * D + d] = box[v * 2 * D + d];
            if (hi) hi[p * D + d] = box[v * 2 * D + D + d];
            if (center) center[p * D + d] = ctr[v * D + d];
        }
        if (weight) weight[p] = wr[v].x;
        if (inf_radius) inf_radius[p] = wr[v].y;
    }
    return FG_OK;
}

}  // namespace fg
