// fg_moments.cu -- K5: far-field moments per reference node
// (replaces KdTree.refresh_moments, spatial_index.py:171-197).
//
// Direct chunked accumulation for every node (see moments_direct).  The first
// refresh for a given order is kept as a base
// (h0); later refreshes at other bandwidths apply the exact rescaling law
// A_a(h) = (h0/h)^{|a|} A_a(h0), pinned by the reference's
// tests/test_spatial_index.py:147-162, as one elementwise kernel.
#include <cmath>
#include <vector>

#include "fg_device.cuh"
#include <cub/cub.cuh>

#include <algorithm>

#include "fg_internal.cuh"
#include "fg_series.cuh"

namespace fg {


__global__ void rescale_factors_kernel(int K, double ratio, const int *__restrict__ degrees,
                                       double *__restrict__ fac) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) fac[k] = pow(ratio, (double)degrees[k]);
}

__global__ void moments_rescale_kernel(int64_t total, int K, const double *__restrict__ src,
                                       const double *__restrict__ fac, double *__restrict__ dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    dst[i] = src[i] * fac[i % K];
}

// ---- direct chunked moments ----------------------------------------------
// Every node's moments straight from its points, A_a = (1/a!) sum_r w_r u_r^a
// with u = (x_r - c)/(sqrt2 h) (accumulate_far_field, series_expansion.py:76-92,
// for every node; mathematically identical to the reference's leaf moments +
// translate_h2h bottom-up, spatial_index.py:171-197).  Work items are
// (node, chunk of kMomChunk points); a warp sums one item with lanes owning
// coefficients and per-point power tables staged in shared memory, and a
// second pass adds each node's chunk partials in chunk order (deterministic).
// No level-by-level dependency: two launches for the whole tree.
constexpr int kMomChunk = 256;
constexpr int kMomWarps = 8;
// power-table orders held per (lane, dimension): padded dimensions (> 8) only
// carry order-1 index sets, which keeps their shared memory small
template <int D>
constexpr int mom_ord() { return D > 8 ? 1 : kMaxOrder; }
constexpr int kMomKPLMax = kMaxK / 32;  // coefficients per lane (largest K)

__global__ void mom_items_count_kernel(int64_t nn, const int4 *__restrict__ node_i,
                                       int *__restrict__ cnt) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < nn) cnt[v] = (node_i[v].y + kMomChunk - 1) / kMomChunk;
}

__global__ void mom_items_fill_kernel(int64_t nn, const int4 *__restrict__ node_i,
                                      const int *__restrict__ off, int2 *__restrict__ items) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nn) return;
    const int c = (node_i[v].y + kMomChunk - 1) / kMomChunk;
    for (int j = 0; j < c; j++) items[off[v] + j] = make_int2((int)v, j);
}

// KPL: coefficient slots per lane, ceil(K / 32) rounded up to a power of two
// (a kernel sized for the expansion at hand keeps its registers -- and so its
// occupancy -- to what K needs)
template <int D, int kMomKPL>
__global__ void __launch_bounds__(32 * kMomWarps)
mom_partial_kernel(int nitems, const int2 *__restrict__ items, const int4 *__restrict__ node_i,
                   const double *__restrict__ node_c, const double *__restrict__ pw, int p,
                   int K, double sc, const uint8_t *__restrict__ digits,
                   double *__restrict__ partial, int small_only) {
    constexpr int S = packed_stride(D);
    extern __shared__ double sh[];  // per warp: 32 points x D x p powers (weight folded in d=0)
    const int lane = threadIdx.x & 31;
    const int P = p;
    double *tab = sh + (threadIdx.x >> 5) * 32 * D * mom_ord<D>();
    const int gwarps = gridDim.x * kMomWarps;
    // per owned coefficient: table offsets d * mom_ord<D>() + digit_d
    int toff[kMomKPL][D];
#pragma unroll
    for (int j = 0; j < kMomKPL; j++) {
        const int k = lane + 32 * j;
        const uint64_t dg = k < K ? digits_of(digits, k) : 0;
#pragma unroll
        for (int d = 0; d < D; d++) toff[j][d] = d * mom_ord<D>() + digit(dg, d);
    }
    for (int it = blockIdx.x * kMomWarps + (threadIdx.x >> 5); it < nitems; it += gwarps) {
        const int2 item = items[it];
        const int4 ni = node_i[item.x];
        // nodes of more than one chunk get their moments from their children
        // (mom_h2h_level_kernel) when small_only is set
        if (small_only && ni.y > kMomChunk && ni.z >= 0) continue;  // (large leaves stay direct)
        double c[D];
#pragma unroll
        for (int d = 0; d < D; d++) c[d] = node_c[(int64_t)item.x * D + d];
        const int b = ni.x + item.y * kMomChunk, e = min(b + kMomChunk, ni.x + ni.y);
        double acc[kMomKPL];
#pragma unroll
        for (int j = 0; j < kMomKPL; j++) acc[j] = 0.0;
        double yn[D], wn = 0.0;  // next batch's point, loaded one batch ahead
        if (b + lane < e) load_point_w<D>(pw + (int64_t)(b + lane) * S, yn, wn);
        for (int base = b; base < e; base += 32) {
            const int i = base + lane;
            double y[D], w = wn;
#pragma unroll
            for (int d = 0; d < D; d++) y[d] = yn[d];
            if (i + 32 < e) load_point_w<D>(pw + (int64_t)(i + 32) * S, yn, wn);
            if (i < e) {
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const double u = (y[d] - c[d]) / sc;
                    double v = d == 0 ? w : 1.0;
                    double *row = tab + (lane * D + d) * mom_ord<D>();
                    for (int k = 0; k < P; k++) {
                        row[k] = v;
                        v *= u;
                    }
                }
            }
            __syncwarp();
            const int nv = min(32, e - base);
            int q = 0;
            // two points per round: independent product chains
            for (; q + 1 < nv; q += 2) {
                const double *t0 = tab + q * D * mom_ord<D>(), *t1 = t0 + D * mom_ord<D>();
#pragma unroll
                for (int j = 0; j < kMomKPL; j++) {
                    if (32 * j < K) {
                        double v0 = t0[toff[j][0]], v1 = t1[toff[j][0]];
#pragma unroll
                        for (int d = 1; d < D; d++) {
                            v0 *= t0[toff[j][d]];
                            v1 *= t1[toff[j][d]];
                        }
                        acc[j] += v0 + v1;
                    }
                }
            }
            if (q < nv) {
                const double *t0 = tab + q * D * mom_ord<D>();
#pragma unroll
                for (int j = 0; j < kMomKPL; j++) {
                    if (32 * j < K) {
                        double v0 = t0[toff[j][0]];
#pragma unroll
                        for (int d = 1; d < D; d++) v0 *= t0[toff[j][d]];
                        acc[j] += v0;
                    }
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < kMomKPL; j++) {
            const int k = lane + 32 * j;
            if (k < K) partial[(int64_t)it * K + k] = acc[j];
        }
    }
}

// One CTA (8 warps) per node: warp w sums items w, w+8, ... of the node, then
// the 8 warp sums are added in warp order (deterministic).
__global__ void __launch_bounds__(256)
mom_combine_kernel(const int *__restrict__ off, const double *__restrict__ partial, int K,
                   const double *__restrict__ inv_fact, double *__restrict__ mom, int small_only,
                   const int4 *__restrict__ node_i) {
    __shared__ double sh[8][kMaxK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t v = blockIdx.x;
    const int i0 = off[v], i1 = off[v + 1];
    // more than one chunk and children: from the children (mom_h2h_level_kernel)
    if (small_only && i1 - i0 > 1 && node_i[v].z >= 0) return;
    if (i1 - i0 == 1) {  // single chunk: copy
        for (int k = threadIdx.x; k < K; k += 256)
            mom[v * K + k] = partial[(int64_t)i0 * K + k] * inv_fact[k];
        return;
    }
    for (int k = lane; k < K; k += 32) {
        double s = 0.0;
#pragma unroll 4
        for (int it = i0 + wid; it < i1; it += 8) s += partial[(int64_t)it * K + k];
        sh[wid][k] = s;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += 256) {
        double s = sh[0][k];
#pragma unroll
        for (int w = 1; w < 8; w++) s += sh[w][k];
        mom[v * K + k] = s * inv_fact[k];
    }
}

// Moments of the nodes of one tree level that span more than one chunk, from
// their children's by H2H (series_expansion.py:139-164, the reference's own
// upward pass): A'_s = sum over pairs (a, b) -> s of A_a u^b / b!,
// u = (c_child - c_node) / sc.  One warp per node; lanes own destination
// coefficients, the pairs come sorted by s (SeriesTables::h2h_ab), the sums run
// in a fixed order (deterministic).
template <int D>
__global__ void __launch_bounds__(128)
mom_h2h_level_kernel(int v0, int v1, const int4 *__restrict__ node_i,
                     const double *__restrict__ node_c, int p, int K, double sc,
                     const uint8_t *__restrict__ digits, const double *__restrict__ inv_fact,
                     const int *__restrict__ off, const int2 *__restrict__ pr,
                     double *__restrict__ mom) {
    extern __shared__ double tab[];  // K shift terms u^b / b!
    const int v = v0 + blockIdx.x;   // one CTA per node: threads own destination coefficients
    if (v >= v1) return;
    const int4 ni = node_i[v];
    if (ni.y <= kMomChunk || ni.z < 0) return;  // accumulated directly (uniform per CTA)
    constexpr int KPT = (kMaxK + 127) / 128;
    double acc[KPT];
#pragma unroll
    for (int j = 0; j < KPT; j++) acc[j] = 0.0;
#pragma unroll 1
    for (int c = 0; c < 2; c++) {
        const int ch = c == 0 ? ni.z : ni.w;
        double pwt[D][kMaxOrder];
#pragma unroll
        for (int d = 0; d < D; d++)
            power_ladder((node_c[(int64_t)ch * D + d] - node_c[(int64_t)v * D + d]) / sc, p - 1,
                         pwt[d]);
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += 128)
            tab[k] = product<D>(digits_of(digits, k), pwt) * inv_fact[k];
        __syncthreads();
        const double *A = mom + (int64_t)ch * K;
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const int t = threadIdx.x + 128 * j;
            if (t < K) {
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // fixed order: deterministic
                const int q1 = off[t + 1];
                int q = off[t];
                for (; q + 4 <= q1; q += 4) {
                    const int2 e0 = pr[q], e1 = pr[q + 1], e2 = pr[q + 2], e3 = pr[q + 3];
                    a0 = fma(A[e0.x], tab[e0.y], a0);
                    a1 = fma(A[e1.x], tab[e1.y], a1);
                    a2 = fma(A[e2.x], tab[e2.y], a2);
                    a3 = fma(A[e3.x], tab[e3.y], a3);
                }
                for (; q < q1; q++) {
                    const int2 e = pr[q];
                    a0 = fma(A[e.x], tab[e.y], a0);
                }
                acc[j] += (a0 + a1) + (a2 + a3);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        const int t = threadIdx.x + 128 * j;
        if (t < K) mom[(int64_t)v * K + t] = acc[j];
    }
}

// items of a tree (bandwidth-independent, built once per tree)
int mom_items(TreeDev &t) {
    if (t.mom_items_valid) return FG_OK;
    const int64_t nn = t.nnodes;
    FG_TRY(t.mom_off.reserve(sizeof(int) * (nn + 1)));
    int *off = t.mom_off.as<int>();
    FG_CUDA_TRY(cudaMemsetAsync(off + nn, 0, sizeof(int), stream()));
    const unsigned blocks = (unsigned)((nn + 255) / 256);
    count_launch();
    mom_items_count_kernel<<<blocks, 256, 0, stream()>>>(nn, t.node_i.as<int4>(), off);
    size_t tmp = 0;
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, off, off, (int)(nn + 1), stream()));
    struct MomItemsTmp;
    DBuf &s_tmp = scratch<MomItemsTmp>();
    FG_TRY(s_tmp.reserve(tmp + 16));
    count_launch();
    FG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(s_tmp.p, tmp, off, off, (int)(nn + 1), stream()));
    int total = 0;
    FG_CUDA_TRY(cudaMemcpyAsync(&total, off + nn, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    FG_TRY(t.mom_items.reserve(sizeof(int2) * std::max(total, 1)));
    count_launch();
    mom_items_fill_kernel<<<blocks, 256, 0, stream()>>>(nn, t.node_i.as<int4>(), off,
                                                        t.mom_items.as<int2>());
    FG_CUDA_TRY(cudaGetLastError());
    t.mom_nitems = total;
    t.mom_items_valid = true;
    return FG_OK;
}

template <int D>
static int moments_direct(TreeDev &t, const SeriesTables &T, double h, DBuf &dst) {
    const int K = T.K, p = T.order;
    const double sc = kSqrt2 * h;
    // Nodes of more than one 256-point chunk take their moments from their
    // children by H2H instead of from their points (C5, order 12: mom_partial
    // 24 ms -> see DESIGN.md); FG_MOM_DIRECT=1 keeps the direct accumulation.
    const int h2h = D <= kMaxDim && getenv("FG_MOM_DIRECT") == nullptr ? 1 : 0;
    FG_TRY(mom_items(t));
    struct MomPartial;
    DBuf &s_partial = scratch<MomPartial>();
    FG_TRY(s_partial.reserve(sizeof(double) * (size_t)t.mom_nitems * K));
    const size_t smem = sizeof(double) * 32 * D * mom_ord<D>() * kMomWarps;
    const int kpl = (K + 31) / 32;
    auto kern = kpl <= 1 ? mom_partial_kernel<D, 1>
                : kpl <= 2 ? mom_partial_kernel<D, 2>
                : kpl <= 4 ? mom_partial_kernel<D, 4>
                : kpl <= 8 ? mom_partial_kernel<D, 8>
                           : mom_partial_kernel<D, kMomKPLMax>;
    const int ki = kpl <= 1 ? 0 : kpl <= 2 ? 1 : kpl <= 4 ? 2 : kpl <= 8 ? 3 : 4;
    struct MomGrid {
        int g[kDimSlots][5] = {};
    };
    auto &c_grid = scratch<MomGrid, MomGrid>().g;  // per device
    if (!c_grid[D][ki]) {
        int dev = 0, sms = 0, occ = 0;
        FG_CUDA_TRY(cudaGetDevice(&dev));
        FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (smem > 48 * 1024)
            FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
        FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kMomWarps, smem));
        c_grid[D][ki] = sms * std::max(occ, 1);
    }
    const int grid = std::max(1, std::min(c_grid[D][ki], (t.mom_nitems + kMomWarps - 1) / kMomWarps));
    count_launch();
    kern<<<grid, 32 * kMomWarps, smem, stream()>>>(t.mom_nitems, t.mom_items.as<int2>(),
                                                  t.node_i.as<int4>(), t.node_c.as<double>(),
                                                  t.pw.as<double>(), p, K, sc,
                                                  T.digits.as<uint8_t>(), s_partial.as<double>(),
                                                  h2h);
    FG_CUDA_TRY(cudaGetLastError());
    const int64_t nn = t.nnodes;
    count_launch();
    mom_combine_kernel<<<(unsigned)nn, 256, 0, stream()>>>(
        t.mom_off.as<int>(), s_partial.as<double>(), K, T.inv_fact.as<double>(), dst.as<double>(),
        h2h, t.node_i.as<int4>());
    FG_CUDA_TRY(cudaGetLastError());
    if (h2h) {
        // upward pass over the levels that hold nodes of more than one chunk
        // (bottom-up: a node's children sit one level below it)
        const size_t smem2 = sizeof(double) * K;
        for (int L = t.levels - 2; L >= 0; L--) {
            const int v0 = (int)t.level_begin[L], v1 = (int)t.level_begin[L + 1];
            if (v1 <= v0) continue;
            count_launch();
            mom_h2h_level_kernel<D><<<(unsigned)(v1 - v0), 128, smem2, stream()>>>(
                v0, v1, t.node_i.as<int4>(), t.node_c.as<double>(), p, K, sc,
                T.digits.as<uint8_t>(), T.inv_fact.as<double>(), T.h2h_off.as<int>(),
                T.h2h_ab.as<int2>(), dst.as<double>());
        }
        FG_CUDA_TRY(cudaGetLastError());
    }
    return FG_OK;
}

// ---- Jensen node statistics (the traversal's mass bound, entry_bounds) ----
// Per (node, chunk) item: sum w, sum w u_d, sum w |u|^2 with u = r - c (c the
// node's centre); a warp per node then adds its items' partials (lanes strided
// over the items, a fixed-order warp reduction: deterministic) and stores
// (|m|, s2) = (|sum w u| / W, sum w |u|^2 / W).
template <int D>
__global__ void js_partial_kernel(int nitems, const int2 *__restrict__ items,
                                  const int4 *__restrict__ node_i, const double *__restrict__ node_c,
                                  const double *__restrict__ pw, double *__restrict__ partial) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    const int it = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (it >= nitems) return;
    const int2 item = items[it];
    const int4 ni = node_i[item.x];
    double c[D], m[D], ws = 0.0, s2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        c[d] = node_c[(int64_t)item.x * D + d];
        m[d] = 0.0;
    }
    const int b = ni.x + item.y * kMomChunk, e = min(b + kMomChunk, ni.x + ni.y);
    for (int i = b + lane; i < e; i += 32) {
        double y[D], w;
        load_point_w<D>(pw + (int64_t)i * S, y, w);
        ws += w;
#pragma unroll
        for (int d = 0; d < D; d++) {
            const double u = y[d] - c[d];
            m[d] = fma(w, u, m[d]);
            s2 = fma(w * u, u, s2);
        }
    }
    ws = warp_sum(ws);
    s2 = warp_sum(s2);
#pragma unroll
    for (int d = 0; d < D; d++) m[d] = warp_sum(m[d]);
    if (lane == 0) {
        double *o = partial + (int64_t)it * (D + 2);
        o[0] = ws;
        o[1] = s2;
#pragma unroll
        for (int d = 0; d < D; d++) o[2 + d] = m[d];
    }
}

template <int D>
__global__ void js_combine_kernel(int64_t nn, const int *__restrict__ off,
                                  const double *__restrict__ partial, double2 *__restrict__ js) {
    const int lane = threadIdx.x & 31;
    const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (v >= nn) return;
    double a[D + 2];
#pragma unroll
    for (int k = 0; k < D + 2; k++) a[k] = 0.0;
    for (int it = off[v] + lane; it < off[v + 1]; it += 32)
#pragma unroll
        for (int k = 0; k < D + 2; k++) a[k] += partial[(int64_t)it * (D + 2) + k];
#pragma unroll
    for (int k = 0; k < D + 2; k++) a[k] = warp_sum(a[k]);
    double mm = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double md = a[2 + d] / a[0];
        mm = fma(md, md, mm);
    }
    if (lane == 0) js[v] = make_double2(sqrt(mm), a[1] / a[0]);
}

template <int D>
static int node_js_t(TreeDev &t) {
    FG_TRY(mom_items(t));
    struct JsPart;
    DBuf &s_part = scratch<JsPart>();
    FG_TRY(s_part.reserve(sizeof(double) * (size_t)std::max(t.mom_nitems, 1) * (D + 2)));
    FG_TRY(t.node_js.reserve(sizeof(double2) * t.nnodes));
    count_launch();
    js_partial_kernel<D><<<(unsigned)(((int64_t)t.mom_nitems * 32 + 255) / 256), 256, 0, stream()>>>(
        t.mom_nitems, t.mom_items.as<int2>(), t.node_i.as<int4>(), t.node_c.as<double>(),
        t.pw.as<double>(), s_part.as<double>());
    count_launch();
    js_combine_kernel<D><<<(unsigned)((t.nnodes * 32 + 255) / 256), 256, 0, stream()>>>(
        t.nnodes, t.mom_off.as<int>(), s_part.as<double>(), t.node_js.as<double2>());
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

int node_js(TreeDev &t) {
    if (t.js_valid) return FG_OK;
    int st;
    switch (t.dim) {
        case 1: st = node_js_t<1>(t); break;
        case 2: st = node_js_t<2>(t); break;
        case 3: st = node_js_t<3>(t); break;
        case 4: st = node_js_t<4>(t); break;
        case 5: st = node_js_t<5>(t); break;
        case 6: st = node_js_t<6>(t); break;
        case 7: st = node_js_t<7>(t); break;
        case 8: st = node_js_t<8>(t); break;
        case 12: st = node_js_t<12>(t); break;
        default: st = node_js_t<16>(t); break;
    }
    FG_TRY(st);
    t.js_valid = true;
    return FG_OK;
}

struct RescaleFac;

int moments_refresh(TreeDev &t, double h, int plimit) {
    FG_REQUIRE(h > 0.0 && std::isfinite(h), FG_EINVAL, "bandwidth must be positive");
    FG_REQUIRE(plimit >= 1, FG_EINVAL, "truncation order must be at least 1");
    FG_REQUIRE(plimit <= kMaxOrder, FG_EUNSUPPORTED, "plimit above the device order cap (12) is not supported");
    int st = FG_OK;
    const SeriesTables *T = series_tables(t.dim, plimit, &st);
    FG_TRY(st);
    const int K = T->K;
    const int64_t total = t.nnodes * K;
    FG_TRY(t.mom.reserve(sizeof(double) * total));
    if (t.mom0_valid && t.mom_K == K && t.mom_order == plimit) {
        // exact rescaling from the base bandwidth: (h0/h)^{|a|} per coefficient
        DBuf &g_rescale_fac = scratch<RescaleFac>();
        FG_TRY(g_rescale_fac.reserve(sizeof(double) * K));
        count_launch();
        rescale_factors_kernel<<<1, 256, 0, stream()>>>(K, t.mom0_h / h, T->degrees.as<int>(),
                                                        g_rescale_fac.as<double>());
        count_launch();
        moments_rescale_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream()>>>(
            total, K, t.mom0.as<double>(), g_rescale_fac.as<double>(), t.mom.as<double>());
        FG_CUDA_TRY(cudaGetLastError());
    } else {
        FG_TRY(t.mom0.reserve(sizeof(double) * total));
        switch (t.dim) {
            case 1: st = moments_direct<1>(t, *T, h, t.mom0); break;
            case 2: st = moments_direct<2>(t, *T, h, t.mom0); break;
            case 3: st = moments_direct<3>(t, *T, h, t.mom0); break;
            case 4: st = moments_direct<4>(t, *T, h, t.mom0); break;
            case 5: st = moments_direct<5>(t, *T, h, t.mom0); break;
            case 6: st = moments_direct<6>(t, *T, h, t.mom0); break;
            case 7: st = moments_direct<7>(t, *T, h, t.mom0); break;
            case 8: st = moments_direct<8>(t, *T, h, t.mom0); break;
            case 12: st = moments_direct<12>(t, *T, h, t.mom0); break;
            default: st = moments_direct<16>(t, *T, h, t.mom0); break;
        }
        FG_TRY(st);
        FG_CUDA_TRY(cudaMemcpyAsync(t.mom.p, t.mom0.p, sizeof(double) * total,
                                    cudaMemcpyDeviceToDevice, stream()));
        t.mom0_valid = true;
        t.mom0_h = h;
    }
    t.mom_K = K;
    t.mom_order = plimit;
    t.mom_h = h;
    t.mom_valid = true;
    return FG_OK;
}

// Moments of several bandwidths side by side (sweeps): dst[j] = the moments
// moments_refresh(t, hs[j], plimit) would produce, by the same rescaling of
// the base moments (bit-identical to it).
struct RatioList {
    double r[32];
};
__global__ void rescale_factors_multi_kernel(int nh, int K, RatioList ratios,
                                             const int *__restrict__ degrees,
                                             double *__restrict__ fac) {
    for (int i = threadIdx.x; i < nh * K; i += blockDim.x)
        fac[i] = pow(ratios.r[i / K], (double)degrees[i % K]);
}

__global__ void moments_rescale_multi_kernel(int64_t total, int nh, int K,
                                             const double *__restrict__ src,
                                             const double *__restrict__ fac,
                                             double *__restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const double v = src[i];
    const int k = (int)(i % K);
    for (int j = 0; j < nh; j++) dst[(int64_t)j * total + i] = v * fac[j * K + k];
}

int moments_multi(TreeDev &t, const double *hs, int nh, int plimit, DBuf &dst) {
    FG_REQUIRE(nh >= 1 && nh <= 32, FG_EINVAL, "bad bandwidth count");
    int st = FG_OK;
    const SeriesTables *T = series_tables(t.dim, plimit, &st);
    FG_TRY(st);
    const int K = T->K;
    if (!(t.mom0_valid && t.mom_K == K && t.mom_order == plimit))
        FG_TRY(moments_refresh(t, hs[0], plimit));  // base moments at hs[0]
    const int64_t total = t.nnodes * K;
    FG_TRY(dst.reserve(sizeof(double) * total * nh));
    struct MultiFac;
    DBuf &fac = scratch<MultiFac>();
    FG_TRY(fac.reserve(sizeof(double) * K * nh));
    RatioList rl;
    for (int j = 0; j < nh; j++) {
        FG_REQUIRE(hs[j] > 0.0 && std::isfinite(hs[j]), FG_EINVAL, "bandwidth must be positive");
        rl.r[j] = t.mom0_h / hs[j];
    }
    count_launch();
    rescale_factors_multi_kernel<<<1, 256, 0, stream()>>>(nh, K, rl, T->degrees.as<int>(),
                                                          fac.as<double>());
    count_launch();
    moments_rescale_multi_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream()>>>(
        total, nh, K, t.mom0.as<double>(), fac.as<double>(), dst.as<double>());
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

int moments_export(const TreeDev &t, double *out) {
    FG_REQUIRE(t.mom_valid, FG_ESTALE, "no moments: call refresh_moments first");
    const int K = t.mom_K;
    std::vector<double> m((size_t)t.nnodes * K);
    FG_CUDA_TRY(cudaMemcpyAsync(m.data(), t.mom.p, sizeof(double) * m.size(),
                                cudaMemcpyDeviceToHost, stream()));
    FG_CUDA_TRY(cudaStreamSynchronize(stream()));
    std::vector<int64_t> pre;
    FG_TRY(preorder_map(t, pre));
    for (int64_t v = 0; v < t.nnodes; v++)
        for (int k = 0; k < K; k++) out[pre[v] * K + k] = m[v * K + k];
    return FG_OK;
}

}  // namespace fg
