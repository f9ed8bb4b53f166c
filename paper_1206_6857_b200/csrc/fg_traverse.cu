// fg_traverse.cu -- K2 + K6..K11 fused: the dual-tree traversal with token
// error control, series prunes and exhaustive leaf-pair base cases
// (replaces _traverse/visit, dito_base and dito_post:
//  summation_engine.py:157-455; best_method, error_bounds.py:168-230).
//
// Work decomposition:
//  * The query side is cut into blocks of <= 32 consecutive tree-order points
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

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fg_device.cuh"
#include "fg_exp.cuh"
#include "fg_internal.cuh"
#include "fg_series.cuh"

namespace fg {

int g_ref_leaf = 32;
int g_stack_cap = 4096;

constexpr int kTravThreads = 128;
constexpr int kTravWarps = kTravThreads / 32;
// Relative safety margin on the running mass bound: the frontier sum is kept
// incrementally, so it carries <= (#updates) ulps of drift relative to G_min.
constexpr double kMassSafety = 1.0 - 1e-10;

struct TravArgs {
    // reference tree (BFS numbering)
    const double *r_pw;
    const int4 *r_ni;
    const double *r_box;
    const double *r_c;
    const double2 *r_wr;
    const double *r_mom;
    int mom_K;
    // query blocks
    const double *q_pw;
    const int2 *qb_range;
    const double *qb_box;
    const double *qb_c;
    const double *qb_rad;
    const int64_t *q_perm;
    long long b0, b1, stride;
    double *out;
    // scalars
    double h, neg_inv, inv_h, sc, eps, total_w, floor_c;
    int use_tokens, use_series, plimit, K, ref_leaf;
    double ct[kMaxOrder + 1], cross[kMaxOrder + 1];
    int kp[kMaxOrder + 1];  // coefficient count for order p
    const uint8_t *digits;
    const double *inv_fact;
    const int *degrees;
    // scratch
    int *st_node;
    double *st_f;
    int stack_cap;
    unsigned long long *work;
    unsigned long long *counters;  // 7 counters
};

// Admit candidates in lane order under the token rule.  Unconditional
// candidates (req <= 0) bank their surplus first; the rest are taken greedily
// in lane order while the balance covers them.  Never lets tokens go negative.
__device__ __forceinline__ unsigned admit(bool cand, double req, double &tokens) {
    const int lane = threadIdx.x & 31;
    const unsigned un = __ballot_sync(kFull, cand && req <= 0.0);
    tokens += warp_sum(((un >> lane) & 1u) ? -req : 0.0);
    unsigned pos = __ballot_sync(kFull, cand && req > 0.0 && req <= tokens);
    unsigned adm = un;
    while (pos) {
        const int i = __ffs(pos) - 1;
        pos &= pos - 1;
        const double ri = __shfl_sync(kFull, req, i);
        if (tokens >= ri) {
            tokens -= ri;
            adm |= 1u << i;
        }
    }
    return adm;
}

__device__ __forceinline__ double required_tokens(double wr, double err, double eps,
                                                  double gmin, double total_w) {
    if (err <= 0.0) return -wr;
    const double den = eps * gmin;
    return den > 0.0 ? total_w * err / den - wr : CUDART_INF;
}

template <int D>
__device__ __forceinline__ void entry_bounds(const TravArgs &A, const double (&qlo)[D],
                                             const double (&qhi)[D], int node, double &klo,
                                             double &khi, double &mn) {
    double mx;
    box_bounds<D>(qlo, qhi, A.r_box + (int64_t)node * 2 * D, mn, mx);
    khi = exp(mn * A.neg_inv);
    klo = exp(mx * A.neg_inv);
}

template <int D>
__global__ void __launch_bounds__(kTravThreads)
traverse_kernel(const TravArgs A) {
    constexpr int S = packed_stride(D);
    extern __shared__ double sh_local[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kTravWarps + wib;
    int *sn = A.st_node + gw * A.stack_cap;
    double *skl = A.st_f + gw * A.stack_cap * 3;
    double *skh = skl + A.stack_cap;
    double *smn = skh + A.stack_cap;
    double *loc = sh_local + wib * (A.K > 0 ? A.K : 1);
    const unsigned lt_mask = (1u << lane) - 1u;

    for (;;) {
        long long b = 0;
        if (lane == 0) b = (long long)atomicAdd(A.work, 1ULL) * A.stride + A.b0;
        b = __shfl_sync(kFull, b, 0);
        if (b >= A.b1) break;

        const int2 rg = A.qb_range[b];
        const int qs = rg.x, qn = rg.y;
        const bool valid = lane < qn;
        double qlo[D], qhi[D], qc[D], x[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            qlo[d] = A.qb_box[b * 2 * D + d];
            qhi[d] = A.qb_box[b * 2 * D + D + d];
            qc[d] = A.qb_c[b * D + d];
        }
        const double qrad = A.qb_rad[b];
        if (valid) load_point<D>(A.q_pw + (int64_t)(qs + lane) * S, x);
        else {
#pragma unroll
            for (int d = 0; d < D; d++) x[d] = qc[d];
        }
        double pt_est = 0.0, pt_mass = 0.0;                  // per point
        double node_est = 0.0, node_mass = 0.0, tokens = 0.0; // per block (uniform)
        bool local_used = false;
        unsigned c_vis = 0, c_base = 0, c_fd = 0, c_dh = 0, c_dl = 0, c_h2l = 0, c_pairs = 0;
        if (A.use_series)
            for (int k = lane; k < A.K; k += 32) loc[k] = 0.0;

        // root entry
        double fsum;  // sum over the frontier of W_R * K_lo
        int sp = 1;
        {
            double klo, khi, mn;
            entry_bounds<D>(A, qlo, qhi, 0, klo, khi, mn);
            if (lane == 0) {
                sn[0] = 0;
                skl[0] = klo;
                skh[0] = khi;
                smn[0] = mn;
            }
            fsum = A.r_wr[0].x * klo;
        }
        __syncwarp();

        while (sp > 0) {
            const int nb = min(sp, 32);
            const int base = sp - nb;
            sp = base;
            const bool act = lane < nb;
            int node = 0;
            double klo = 0.0, khi = 0.0, mn = 0.0;
            int4 ni = make_int4(0, 0, -1, -1);
            double2 wr = make_double2(0.0, 0.0);
            if (act) {
                node = sn[base + lane];
                klo = skl[base + lane];
                khi = skh[base + lane];
                mn = smn[base + lane];
                ni = A.r_ni[node];
                wr = A.r_wr[node];
            }
            __syncwarp();
            const double WR = wr.x;
            c_vis += nb;
            const double batch_sum = warp_sum(act ? WR * klo : 0.0);
            const double pmin = warp_min(valid ? pt_mass : CUDART_INF);
            const double gmin = (pmin + node_mass + fsum) * kMassSafety;

            // ---- finite-difference prune (summation_engine.py:327-351)
            const double fd_err = 0.5 * WR * (khi - klo);
            const double req = required_tokens(WR, fd_err, A.eps, gmin, A.total_w);
            unsigned fd_mask;
            if (A.use_tokens) fd_mask = admit(act, req, tokens);
            else fd_mask = __ballot_sync(kFull, act && req <= 0.0);
            const bool fd = (fd_mask >> lane) & 1u;
            c_fd += __popc(fd_mask);
            double settled = fd ? WR * klo : 0.0;
            double est_add = 0.0;
            if (fd) {
                const double dl = WR * klo, du = WR * khi - WR;
                est_add = 0.5 * (dl + du + WR);
            }

            // ---- series prunes (summation_engine.py:352-399)
            unsigned ser_mask = 0;
            int meth = 0, p = 0;
            if (A.use_series) {
                const bool cand0 = act && !fd;
                double bound = 0.0;
                if (cand0) {
                    const double maxerr = A.eps * (WR + tokens) * gmin / A.total_w;
                    const double r_ref = wr.y * A.inv_h;
                    const double r_qu = qrad * A.inv_h;
                    const double rmin = r_ref < r_qu ? r_ref : r_qu;
                    double possible = sqrt(khi) * WR * A.floor_c;
                    if (rmin < 1.0) {
                        double pw = 1.0;
                        for (int k = 0; k < A.plimit; k++) pw *= rmin;
                        possible *= pw;
                    }
                    if (possible <= maxerr) {
                        select_method_gpu(mn, r_ref, r_qu, WR, (double)ni.y, D, A.h, maxerr,
                                          A.plimit, A.ct, A.cross, A.kp, meth, p, bound);
                    }
                }
                const bool cand = cand0 && meth != 0;
                const double sreq = cand ? required_tokens(WR, bound, A.eps, gmin, A.total_w)
                                         : CUDART_INF;
                ser_mask = admit(cand, sreq, tokens);
                if ((ser_mask >> lane) & 1u) settled = WR * klo;
            }
            node_mass += warp_sum(settled);
            node_est += warp_sum(est_add);

            if (ser_mask) {
                const unsigned dh = __ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 2);
                const unsigned dl = __ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 3);
                const unsigned tl = __ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 4);
                c_dh += __popc(dh);
                c_dl += __popc(dl);
                c_h2l += __popc(tl);
                for (unsigned m = dh; m; m &= m - 1) {
                    const int i = __ffs(m) - 1;
                    const int nd = __shfl_sync(kFull, node, i);
                    const int pi = __shfl_sync(kFull, p, i);
                    const double v = eval_far_lane<D>(x, A.r_c + (int64_t)nd * D,
                                                      A.r_mom + (int64_t)nd * A.mom_K, pi,
                                                      A.kp[pi], A.sc, A.digits);
                    pt_est += v;
                }
                for (unsigned m = dl; m; m &= m - 1) {
                    const int i = __ffs(m) - 1;
                    const int rs = __shfl_sync(kFull, ni.x, i);
                    const int rc = __shfl_sync(kFull, ni.y, i);
                    const int pi = __shfl_sync(kFull, p, i);
                    accumulate_warp<D>(1, A.r_pw, rs, (int64_t)rs + rc, qc, pi, A.kp[pi], A.sc,
                                       A.digits, A.inv_fact, loc, false);
                    __syncwarp();
                }
                for (unsigned m = tl; m; m &= m - 1) {
                    const int i = __ffs(m) - 1;
                    const int nd = __shfl_sync(kFull, node, i);
                    const int pi = __shfl_sync(kFull, p, i);
                    h2l_warp_add<D>(A.r_mom + (int64_t)nd * A.mom_K, A.r_c + (int64_t)nd * D, qc,
                                    pi, A.kp[pi], pi, A.kp[pi], A.sc, A.digits, A.inv_fact,
                                    A.degrees, loc);
                    __syncwarp();
                }
                if (dl | tl) local_used = true;
            }

            // ---- descend or evaluate exactly (summation_engine.py:400-426)
            const bool rem = act && !fd && !((ser_mask >> lane) & 1u);
            const bool leafy = ni.z < 0 || ni.y <= A.ref_leaf;
            unsigned split_mask = __ballot_sync(kFull, rem && !leafy);
            unsigned base_mask = __ballot_sync(kFull, rem && leafy);
            const int nsplit = __popc(split_mask);
            if (sp + 2 * nsplit > A.stack_cap) {
                // frontier capacity reached: settle these exactly (always admissible)
                base_mask |= split_mask;
                split_mask = 0;
            }
            double child_sum = 0.0;
            if ((split_mask >> lane) & 1u) {
                const int pos = sp + 2 * __popc(split_mask & lt_mask);
                const int ch[2] = {ni.z, ni.w};
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    double cl, chh, cm;
                    entry_bounds<D>(A, qlo, qhi, ch[c], cl, chh, cm);
                    sn[pos + c] = ch[c];
                    skl[pos + c] = cl;
                    skh[pos + c] = chh;
                    smn[pos + c] = cm;
                    child_sum += A.r_wr[ch[c]].x * cl;
                }
            }
            sp += 2 * __popc(split_mask);
            fsum = fsum - batch_sum + warp_sum(child_sum);
            if (fsum < 0.0) fsum = 0.0;

            // ---- exhaustive base cases, eager (dito_base, :221-250)
            for (unsigned m = base_mask; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const int rs = __shfl_sync(kFull, ni.x, i);
                const int rc = __shfl_sync(kFull, ni.y, i);
                const double wri = __shfl_sync(kFull, WR, i);
                const double *rp = A.r_pw + (int64_t)rs * S;
                double acc0 = 0.0, acc1 = 0.0;
                int j = 0;
                for (; j + 1 < rc; j += 2) {
                    double y0[D], y1[D], w0, w1;
                    load_point_w<D>(rp + (int64_t)j * S, y0, w0);
                    load_point_w<D>(rp + (int64_t)(j + 1) * S, y1, w1);
                    double e0 = x[0] - y0[0], e1 = x[0] - y1[0];
                    double d0 = e0 * e0, d1 = e1 * e1;
#pragma unroll
                    for (int d = 1; d < D; d++) {
                        const double f0 = x[d] - y0[d], f1 = x[d] - y1[d];
                        d0 = fma(f0, f0, d0);
                        d1 = fma(f1, f1, d1);
                    }
                    acc0 = fma(fg_exp(d0 * A.neg_inv), w0, acc0);
                    acc1 = fma(fg_exp(d1 * A.neg_inv), w1, acc1);
                }
                if (j < rc) {
                    double y0[D], w0;
                    load_point_w<D>(rp + (int64_t)j * S, y0, w0);
                    double e0 = x[0] - y0[0];
                    double d0 = e0 * e0;
#pragma unroll
                    for (int d = 1; d < D; d++) {
                        const double f0 = x[d] - y0[d];
                        d0 = fma(f0, f0, d0);
                    }
                    acc0 = fma(fg_exp(d0 * A.neg_inv), w0, acc0);
                }
                const double contrib = acc0 + acc1;
                pt_est += contrib;
                pt_mass += contrib;
                if (A.use_tokens) tokens += wri;
                c_base++;
                c_pairs += (unsigned)(qn * rc);
            }
        }

        // ---- post pass for this block (dito_post, :253-281)
        double val = pt_est + node_est;
        if (local_used) {
            __syncwarp();
            val += eval_local_lane<D>(x, qc, loc, A.plimit, A.K, A.sc, A.digits);
        }
        if (valid) A.out[A.q_perm[qs + lane]] = val;
        if (lane == 0) {
            atomicAdd(A.counters + 0, (unsigned long long)c_vis);
            atomicAdd(A.counters + 1, (unsigned long long)c_base);
            atomicAdd(A.counters + 2, (unsigned long long)c_fd);
            atomicAdd(A.counters + 3, (unsigned long long)c_dh);
            atomicAdd(A.counters + 4, (unsigned long long)c_dl);
            atomicAdd(A.counters + 5, (unsigned long long)c_h2l);
            atomicAdd(A.counters + 6, (unsigned long long)c_pairs);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------- query blocks
template <int D>
__global__ void query_blocks_kernel(int64_t n, int64_t nqb, const double *__restrict__ pw,
                                    int2 *__restrict__ range, double *__restrict__ box,
                                    double *__restrict__ ctr, double *__restrict__ rad) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (b >= nqb) return;
    const int64_t s = b * 32;
    const int cnt = (int)min((int64_t)32, n - s);
    const bool v = lane < cnt;
    double x[D];
    if (v) load_point<D>(pw + (s + lane) * S, x);
    double c[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double lo = warp_min(v ? x[d] : CUDART_INF);
        const double hi = warp_max(v ? x[d] : -CUDART_INF);
        const double sm = warp_sum(v ? x[d] : 0.0);
        c[d] = sm / cnt;
        if (lane == 0) {
            box[b * 2 * D + d] = lo;
            box[b * 2 * D + D + d] = hi;
            ctr[b * D + d] = c[d];
        }
    }
    double r = 0.0;
    if (v) {
#pragma unroll
        for (int d = 0; d < D; d++) r = fmax(r, fabs(x[d] - c[d]));
    }
    r = warp_max(r);
    if (lane == 0) {
        rad[b] = r;
        range[b] = make_int2((int)s, cnt);
    }
}

int query_blocks(TreeDev &t) {
    if (t.qb_valid) return FG_OK;
    const int64_t nqb = (t.n + 31) / 32;
    const int D = t.dim;
    FG_TRY(t.qb_range.reserve(sizeof(int2) * nqb));
    FG_TRY(t.qb_box.reserve(sizeof(double) * nqb * 2 * D));
    FG_TRY(t.qb_c.reserve(sizeof(double) * nqb * D));
    FG_TRY(t.qb_rad.reserve(sizeof(double) * nqb));
    const unsigned blocks = (unsigned)((nqb * 32 + 255) / 256);
#define FG_QB(DD)                                                                           \
    case DD:                                                                                \
        count_launch();                                                                     \
        query_blocks_kernel<DD><<<blocks, 256, 0, stream()>>>(                              \
            t.n, nqb, t.pw.as<double>(), t.qb_range.as<int2>(), t.qb_box.as<double>(),      \
            t.qb_c.as<double>(), t.qb_rad.as<double>());                                    \
        break;
    switch (D) {
        FG_QB(1) FG_QB(2) FG_QB(3) FG_QB(4) FG_QB(5) FG_QB(6) FG_QB(7) FG_QB(8)
        default: return FG_EUNSUPPORTED;
    }
#undef FG_QB
    FG_CUDA_TRY(cudaGetLastError());
    t.nqb = nqb;
    t.qb_valid = true;
    return FG_OK;
}

// ---------------------------------------------------------------- launch
struct TravScratch {
    DBuf st_node, st_f, work, counters;
    int grid = 0, cap = 0;
};
static TravScratch g_scr;

template <int D>
static int launch_traverse(TravArgs &A, size_t smem, int64_t nblocks, cudaEvent_t e0,
                           cudaEvent_t e1) {
    auto kern = traverse_kernel<D>;
    if (smem > 48 * 1024)
        FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    int dev = 0, sms = 0, occ = 0;
    FG_CUDA_TRY(cudaGetDevice(&dev));
    FG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTravThreads, smem));
    if (occ < 1) occ = 1;
    int64_t grid = (int64_t)sms * occ;
    const int64_t need = (nblocks + kTravWarps - 1) / kTravWarps;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    const int cap = A.stack_cap;
    if (g_scr.grid < grid || g_scr.cap != cap) {
        const int64_t warps = grid * kTravWarps;
        FG_TRY(g_scr.st_node.reserve(sizeof(int) * warps * cap));
        FG_TRY(g_scr.st_f.reserve(sizeof(double) * warps * cap * 3));
        g_scr.grid = (int)grid;
        g_scr.cap = cap;
    }
    A.st_node = g_scr.st_node.as<int>();
    A.st_f = g_scr.st_f.as<double>();
    FG_CUDA_TRY(cudaEventRecord(e0, stream()));
    count_launch();
    kern<<<(unsigned)grid, kTravThreads, smem, stream()>>>(A);
    FG_CUDA_TRY(cudaGetLastError());
    FG_CUDA_TRY(cudaEventRecord(e1, stream()));
    return FG_OK;
}

int run_traversal(TreeDev &q, TreeDev &r, double h, double eps, int mode, int plimit,
                  int64_t b0, int64_t b1, int64_t stride, double *d_values, fg_counters *counters,
                  double *seconds) {
    FG_REQUIRE(h > 0.0, FG_EINVAL, "bandwidth must be positive");
    FG_REQUIRE(eps >= 0.0, FG_EINVAL, "epsilon must be non-negative");
    FG_REQUIRE(mode >= FG_DFD && mode <= FG_DITO, FG_EINVAL, "unknown algorithm");
    FG_REQUIRE(q.dim == r.dim, FG_EINVAL, "query and reference dimensions differ");
    const int D = q.dim;
    if (plimit <= 0) plimit = default_plimit(D);
    const bool series = mode == FG_DITO;
    if (series) {
        FG_REQUIRE(plimit <= kMaxOrder, FG_EUNSUPPORTED, "plimit > 8 is not supported on the device");
        FG_REQUIRE(r.mom_valid && r.mom_h == h && r.mom_order >= plimit, FG_ESTALE,
                   "reference moments missing or stale; call refresh_moments for this "
                   "bandwidth first");
    }
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
    A.q_pw = q.pw.as<double>();
    A.qb_range = q.qb_range.as<int2>();
    A.qb_box = q.qb_box.as<double>();
    A.qb_c = q.qb_c.as<double>();
    A.qb_rad = q.qb_rad.as<double>();
    A.q_perm = q.perm.as<int64_t>();
    A.b0 = b0;
    A.b1 = b1;
    A.stride = stride < 1 ? 1 : stride;
    A.out = d_values;
    A.h = h;
    A.neg_inv = -0.5 / (h * h);
    A.inv_h = 1.0 / h;
    A.sc = kSqrt2 * h;
    A.eps = eps;
    A.total_w = r.total_w;
    A.use_tokens = mode >= FG_DFDO;
    A.use_series = series;
    A.plimit = plimit;
    A.ref_leaf = g_ref_leaf;
    A.stack_cap = g_stack_cap;
    size_t smem = 0;
    if (series) {
        int st = FG_OK;
        const SeriesTables *T = series_tables(D, plimit, &st);
        FG_TRY(st);
        A.K = T->K;
        A.digits = T->digits.as<uint8_t>();
        A.inv_fact = T->inv_fact.as<double>();
        A.degrees = T->degrees.as<int>();
        A.r_mom = r.mom.as<double>();
        A.mom_K = r.mom_K;
        double ct[kMaxOrder + 1], cross[kMaxOrder + 1], floor_c;
        tail_tables(D, plimit, ct, cross, &floor_c);
        for (int p = 0; p <= plimit; p++) {
            A.ct[p] = ct[p];
            A.cross[p] = cross[p];
            A.kp[p] = T->h_prefix[p];
        }
        A.floor_c = floor_c;
        smem = sizeof(double) * A.K * kTravWarps;
    }
    FG_TRY(g_scr.work.reserve(sizeof(unsigned long long)));
    FG_TRY(g_scr.counters.reserve(sizeof(unsigned long long) * 8));
    FG_CUDA_TRY(cudaMemsetAsync(g_scr.work.p, 0, sizeof(unsigned long long), stream()));
    FG_CUDA_TRY(cudaMemsetAsync(g_scr.counters.p, 0, sizeof(unsigned long long) * 8, stream()));
    A.work = g_scr.work.as<unsigned long long>();
    A.counters = g_scr.counters.as<unsigned long long>();
    cudaEvent_t e0, e1;
    FG_CUDA_TRY(cudaEventCreate(&e0));
    FG_CUDA_TRY(cudaEventCreate(&e1));
    int st = FG_OK;
    const int64_t nb = b1 > b0 ? (b1 - b0 + A.stride - 1) / A.stride : 0;
    if (nb > 0) {
        switch (D) {
            case 1: st = launch_traverse<1>(A, smem, nb, e0, e1); break;
            case 2: st = launch_traverse<2>(A, smem, nb, e0, e1); break;
            case 3: st = launch_traverse<3>(A, smem, nb, e0, e1); break;
            case 4: st = launch_traverse<4>(A, smem, nb, e0, e1); break;
            case 5: st = launch_traverse<5>(A, smem, nb, e0, e1); break;
            case 6: st = launch_traverse<6>(A, smem, nb, e0, e1); break;
            case 7: st = launch_traverse<7>(A, smem, nb, e0, e1); break;
            case 8: st = launch_traverse<8>(A, smem, nb, e0, e1); break;
            default: st = FG_EUNSUPPORTED;
        }
    } else {
        cudaEventRecord(e0, stream());
        cudaEventRecord(e1, stream());
    }
    unsigned long long cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (st == FG_OK) {
        cudaError_t e = cudaMemcpyAsync(cnt, g_scr.counters.p, sizeof(cnt),
                                        cudaMemcpyDeviceToHost, stream());
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream());
        if (e != cudaSuccess) {
            set_error(std::string("traversal: ") + cudaGetErrorString(e));
            st = FG_ECUDA;
        }
    }
    if (st == FG_OK && seconds) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *seconds = ms * 1e-3;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    FG_TRY(st);
    if (counters) {
        counters->pair_visits = (int64_t)cnt[0];
        counters->base_cases = (int64_t)cnt[1];
        counters->fd_prunes = (int64_t)cnt[2];
        counters->hermite_prunes = (int64_t)cnt[3];
        counters->local_prunes = (int64_t)cnt[4];
        counters->h2l_prunes = (int64_t)cnt[5];
        counters->exact_pairs = (int64_t)cnt[6];
    }
    return FG_OK;
}

}  // namespace fg
