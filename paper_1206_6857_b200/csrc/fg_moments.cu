// fg_moments.cu -- K5: far-field moments per reference node
// (replaces KdTree.refresh_moments, spatial_index.py:171-197).
//
// Direct accumulation at the leaves (accumulate_far_field,
// series_expansion.py:76-92) and exact H2H shifts bottom-up level by level
// (translate_h2h + add_far_field, :139-164), one warp per node with lanes
// owning coefficients.  The first refresh for a given order is kept as a base
// (h0); later refreshes at other bandwidths apply the exact rescaling law
// A_a(h) = (h0/h)^{|a|} A_a(h0), pinned by the reference's
// tests/test_spatial_index.py:147-162, as one elementwise kernel.
#include <cmath>
#include <vector>

#include "fg_device.cuh"
#include <cooperative_groups.h>

#include <algorithm>

#include "fg_internal.cuh"
#include "fg_series.cuh"

namespace fg {
namespace cg = cooperative_groups;
// internal nodes with at most this many points get their moments directly
// from their points, larger ones by H2H from their children (0: leaves only;
// direct accumulation re-reads every point once per level, which measured
// slower than H2H)
constexpr int kDirectMax = 0;


template <int D>
__global__ void moments_leaf_kernel(int64_t node_begin, int64_t node_end,
                                    const int4 *__restrict__ node_i,
                                    const double *__restrict__ node_c,
                                    const double *__restrict__ pw, int p, int K, double sc,
                                    const uint8_t *__restrict__ digits,
                                    const double *__restrict__ inv_fact,
                                    double *__restrict__ mom) {
    const int64_t node = node_begin + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (node >= node_end) return;
    const int4 ni = node_i[node];
    if (ni.z >= 0 && ni.y > kDirectMax) return;  // large internal: H2H pass
    double c[D];
#pragma unroll
    for (int d = 0; d < D; d++) c[d] = node_c[node * D + d];
    accumulate_warp<D>(0, pw, ni.x, (int64_t)ni.x + ni.y, c, p, K, sc, digits, inv_fact,
                       mom + node * K, true);
}

// Internal nodes (> kDirectMax points), all levels bottom-up in ONE
// cooperative launch (a grid barrier between levels): A = H2H(left) + H2H(right).
template <int D>
__global__ void moments_h2h_coop_kernel(const int *__restrict__ level_begin, int levels,
                                        const int4 *__restrict__ node_i,
                                        const double *__restrict__ node_c, int p, int K, double sc,
                                        const uint8_t *__restrict__ digits,
                                        const double *__restrict__ inv_fact,
                                        const int *__restrict__ off, const int2 *__restrict__ ab,
                                        double *__restrict__ mom) {
    cg::grid_group g = cg::this_grid();
    extern __shared__ double sh[];  // per warp: 2*K shift values
    const int lane = threadIdx.x & 31;
    const int gwarps = gridDim.x * (blockDim.x >> 5);
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    double *shift = sh + (threadIdx.x >> 5) * 2 * K;
    for (int lv = levels - 1; lv >= 0; lv--) {
        const int b = level_begin[lv], e = level_begin[lv + 1];
        for (int node = b + gwarp; node < e; node += gwarps) {
            const int4 ni = node_i[node];
            if (ni.z < 0 || ni.y <= kDirectMax) continue;
            for (int c = 0; c < 2; c++) {
                const int64_t ch = c == 0 ? ni.z : ni.w;
                double pwt[D][2 * kMaxOrder];
#pragma unroll
                for (int d = 0; d < D; d++)
                    power_ladder((node_c[ch * D + d] - node_c[(int64_t)node * D + d]) / sc, p - 1,
                                 pwt[d]);
                for (int k = lane; k < K; k += 32)
                    shift[c * K + k] = product<D>(digits_of(digits, k), pwt) * inv_fact[k];
            }
            __syncwarp();
            const double *Al = mom + (int64_t)ni.z * K;
            const double *Ar = mom + (int64_t)ni.w * K;
            for (int s = lane; s < K; s += 32) {
                double l = 0.0, r = 0.0;
                for (int q = off[s]; q < off[s + 1]; q++) {
                    const int2 pr = ab[q];
                    l += Al[pr.x] * shift[pr.y];
                }
                for (int q = off[s]; q < off[s + 1]; q++) {
                    const int2 pr = ab[q];
                    r += Ar[pr.x] * shift[K + pr.y];
                }
                mom[(int64_t)node * K + s] = l + r;
            }
            __syncwarp();
        }
        g.sync();
    }
}

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

template <int D>
static int moments_direct(TreeDev &t, const SeriesTables &T, double h, DBuf &dst) {
    const int K = T.K, p = T.order;
    const double sc = kSqrt2 * h;
    const int warps_per_block = 8;
    const int64_t nn = t.nnodes;
    {
        const unsigned blocks = (unsigned)((nn + warps_per_block - 1) / warps_per_block);
        count_launch();
        moments_leaf_kernel<D><<<blocks, 32 * warps_per_block, 0, stream()>>>(
            0, nn, t.node_i.as<int4>(), t.node_c.as<double>(), t.pw.as<double>(), p, K, sc,
            T.digits.as<uint8_t>(), T.inv_fact.as<double>(), dst.as<double>());
        FG_CUDA_TRY(cudaGetLastError());
    }
    {
        // one cooperative launch for the large internal nodes of every level
        auto kern = moments_h2h_coop_kernel<D>;
        const int threads = 32 * warps_per_block;
        const size_t smem = sizeof(double) * 2 * K * warps_per_block;
        static int c_grid[9] = {0};
        static size_t c_smem[9] = {0};
        if (c_grid[D] == 0 || c_smem[D] != smem) {
            int dev = 0, sms = 0, occ = 0;
            FG_CUDA_TRY(cudaGetDevice(&dev));
            FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            if (smem > 48 * 1024)
                FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
            FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
            c_grid[D] = sms * std::max(1, std::min(occ, 2));
            c_smem[D] = smem;
        }
        const int *lb = t.level_begin_dev.as<int>();
        int levels = t.levels;
        int p_ = p, K_ = K;
        double sc_ = sc;
        const int4 *ni = t.node_i.as<int4>();
        const double *nc = t.node_c.as<double>();
        const uint8_t *dg = T.digits.as<uint8_t>();
        const double *ifa = T.inv_fact.as<double>();
        const int *off = T.h2h_off.as<int>();
        const int2 *ab = T.h2h_ab.as<int2>();
        double *mom = dst.as<double>();
        void *args[] = {(void *)&lb, &levels, (void *)&ni, (void *)&nc, &p_, &K_, &sc_,
                        (void *)&dg, (void *)&ifa, (void *)&off, (void *)&ab, (void *)&mom};
        count_launch();
        FG_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)kern, c_grid[D], threads, args, smem,
                                                stream()));
    }
    return FG_OK;
}

static DBuf g_rescale_fac;

int moments_refresh(TreeDev &t, double h, int plimit) {
    FG_REQUIRE(h > 0.0 && std::isfinite(h), FG_EINVAL, "bandwidth must be positive");
    FG_REQUIRE(plimit >= 1, FG_EINVAL, "truncation order must be at least 1");
    FG_REQUIRE(plimit <= kMaxOrder, FG_EUNSUPPORTED, "plimit > 8 is not supported on the device");
    int st = FG_OK;
    const SeriesTables *T = series_tables(t.dim, plimit, &st);
    FG_TRY(st);
    const int K = T->K;
    const int64_t total = t.nnodes * K;
    FG_TRY(t.mom.reserve(sizeof(double) * total));
    if (t.mom0_valid && t.mom_K == K && t.mom_order == plimit) {
        // exact rescaling from the base bandwidth: (h0/h)^{|a|} per coefficient
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
            default: st = moments_direct<8>(t, *T, h, t.mom0); break;
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
    static DBuf fac;
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
