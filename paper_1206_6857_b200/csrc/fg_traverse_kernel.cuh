// fg_traverse_kernel.cuh -- the fused traversal kernel (see fg_traverse.cu for
// the design notes).  Kept in its own header so the launch code and the kernel
// body evolve separately.
#pragma once

#include <cuda_pipeline.h>

#include "fg_device.cuh"
#include "fg_exp.cuh"
#include "fg_internal.cuh"
#include "fg_series.cuh"

namespace fg {

// Device-side bounds checks (a -DFG_CHECKS=1 build; compute-sanitizer is not
// available on the GPU pool): every violated invariant bumps a counter that
// fg_check_failures reads back (tools/check_run.py runs the workloads).
#ifndef FG_CHECKS
#define FG_CHECKS 0
#endif
static __device__ unsigned long long g_fg_check_fail;
#define FG_CHECK(cond)                                                   \
    do {                                                                 \
        if (FG_CHECKS && !(cond)) atomicAdd(&::fg::g_fg_check_fail, 1ull); \
    } while (0)

constexpr int kTravThreads = 128;
// queries per lane: a query block has up to 32 * kQPL points (lane l holds
// queries l and l + 32)
constexpr int kQPL = 2;
constexpr int kQBlock = 32 * kQPL;
// largest anchored FP32 base item (and anchor) in points (D <= 4): with the
// Jensen mass bound 128-point items beat 64 (C2 sweep -4.7 %); 336 = what the
// pair staging holds (C5 -0.7 %, C2 -1 % against 256)
#ifndef FG_ANCHOR_MAX
#define FG_ANCHOR_MAX 336
#endif
constexpr int kAnchorMax = FG_ANCHOR_MAX;
// FP64 base items up to kStageMax points are staged in shared memory (two
// buffers of kStageMax records at D <= 5); larger ones read global memory
constexpr int kStageMax = 64;
constexpr int kTravWarps = kTravThreads / 32;
// Relative safety margin on the running mass bound: the frontier sum is kept
// incrementally, so it carries <= (#updates) ulps of drift relative to G_min.
constexpr double kMassSafety = 1.0 - 1e-10;

// Per-bandwidth parameters of one launch (a launch serves up to kMaxSweep
// bandwidths of a sweep; its tasks are (bandwidth, query block) pairs).
constexpr int kMaxSweep = 24;
constexpr int kDbgFields = 16;  // per-block debug record (FG_DEBUG_BLOCKS)
#ifndef FG_PHASE_PROF
#define FG_PHASE_PROF 0  // per-block phase cycle counters in the debug record
#endif
constexpr int kCounters = 16;  // per-bandwidth device counter slots (13 used)
constexpr int kFarResCapT = 2048;  // residual entries per far-field task (fg_far_kernel.cuh)
struct TravH {
    double h, neg_inv, inv_h, sc, inv_sc, eps;
    double fp32_rho;              // relative error allowed per FP32 leaf item (0: FP64 only)
    const double *r_mom;          // reference moments for this bandwidth
    double *out;                  // values (original query order)
    unsigned long long *counters; // kCounters slots: the 8 fg_counters fields, cycles
    float ex2_scale;              // -log2(e) / (2 h^2)
    int ref_leaf;                 // reference nodes with <= ref_leaf points are base items
    double pair_cost;             // selector's exhaustive cost per pair (FP32 or FP64 leaves)
    double herm_c0, herm_c1;      // selector's Hermite cost per query slot: c0 + c1 K_p
};

// One audit-ledger event (summation_engine.py:250, 350, 394-398): kind 0 base
// case, 1 FD prune, 2 Hermite, 3 direct local, 4 H2L; the query block, the
// step of its traversal and the lane (item) for ordering; W_R, the error
// bound charged through the token rule, G_min at the decision, token flow.
struct AuditEvent {
    int kind, qblock, seq, lane;
    double w_ref, bound, mass_lo, flow;
};

struct TravArgs {
    // reference tree (BFS numbering)
    const double *r_pw;
    const int4 *r_ni;
    const double *r_box;
    const double *r_c;
    const double2 *r_wr;
    const double2 *r_js;  // per node: |weighted mean offset from the centre|, weighted mean |r - c|^2
    int mom_K;
    // query blocks
    const double *q_pw;
    const int2 *qb_range;
    const double *qb_box;
    const double *qb_c;
    const double *qb_rad;
    const double *qb_wmin;  // monochromatic runs: per-block min weight (G floor), else null
    const double *qb_wsum;  // per-block total weight
    const int64_t *q_perm;
    long long b0, b1, stride;
    long long nbl;  // blocks per bandwidth in [b0, b1) at this stride
    // scalars
    double total_w, floor_c;
    int use_tokens, use_series, plimit, K;
    double ct[kMaxOrder + 1], cross[kMaxOrder + 1];
    int kp[kMaxOrder + 1];  // coefficient count for order p
    int plimit_loc, K_loc;  // order cap and coefficient count of the local expansions
    const uint8_t *digits;
    const double *inv_fact;
    const int *degrees;
    // per-warp scratch: frontier stack and deferred series list
    int *st_node;
    double *st_f;
    int2 *ser_list;
    int stack_cap;
    int bfs_cap;  // breadth-first while the frontier holds <= bfs_cap entries
    unsigned long long *work;
    unsigned long long *dbg;       // optional per-block kDbgFields: cycles, steps, visits,
                                   // radius bits, FP32 pairs, -, -, -, phase cycles x 8
    const int *order;              // block visiting order (single full runs) or null
    unsigned long long *cost;      // per-block cycles of this run (or null)
    const float *r_pf;             // FP32 records about each point's anchor (fp32_pack)
    const int *r_anchor;           // per point: its anchor node
    AuditEvent *audit;             // ledger (AUDIT kernels only)
    unsigned long long *audit_count;
    long long audit_cap;
    int nh;                        // bandwidths in this launch
    int jord[kMaxSweep];           // task group k runs bandwidth jord[k] (heaviest first)
    TravH hp[kMaxSweep];
    // far-field pass over super-nodes (fg_far_kernel.cuh); far_flag == null: off
    const int4 *q_ni;              // query tree nodes (BFS): start, count, left, right
    const double *q_box;
    const double *q_c;
    const double2 *q_wr;
    long long nsn;                 // super-nodes
    const int *sn_node;            // BFS node of each super-node
    const double *sn_wmin;         // smallest point weight per super-node (monochromatic)
    const int *qb_super;           // super-node of each block
    unsigned long long *far_work;
    int *far_st_node;              // far kernel per-warp frontier / series scratch
    double *far_st_f;
    int2 *far_ser;
    // per (bandwidth in launch, super-node) task t = j * nsn + k:
    int *far_flag;                 // 0: abandoned (blocks start at the root), bit 0 ok, bit 1 local
    double *far_tokens, *far_settled, *far_est, *far_loc;  // far_loc: K per task
    int *far_rcnt, *far_res;       // residual entries: kFarResCap per task
};

// Append the events of the lanes in `mask` (each lane passes its own fields).
__device__ __forceinline__ void audit_append(const TravArgs &A, unsigned mask, int kind, int qb,
                                             int seq, double wr, double bound, double mass_lo,
                                             double flow) {
    const int lane = threadIdx.x & 31;
    if (!mask) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(A.audit_count, (unsigned long long)__popc(mask));
    base = __shfl_sync(kFull, base, 0);
    if ((mask >> lane) & 1u) {
        const unsigned long long i = base + __popc(mask & ((1u << lane) - 1u));
        if ((long long)i < A.audit_cap) {
            AuditEvent e;
            e.kind = kind;
            e.qblock = qb;
            e.seq = seq;
            e.lane = lane;
            e.w_ref = wr;
            e.bound = bound;
            e.mass_lo = mass_lo;
            e.flow = flow;
            A.audit[i] = e;
        }
    }
}

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

// _required_tokens (summation_engine.py:157-173)
// scale = W / (eps G_min), or +inf when eps G_min <= 0 (no inexact prune)
__device__ __forceinline__ double required_tokens(double wr, double err, double scale) {
    if (err <= 0.0) return -wr;
    return scale < CUDART_INF ? err * scale - wr : CUDART_INF;
}

// Box bounds of (query block box in shared memory, reference node) and both
// kernel bounds (summation_engine.py:315-328), plus lb: the mass lower bound
// per unit weight used for G_min, max(K_lo, Jensen's bound).  Jensen: with the
// node's weights as probabilities, sum_r w_r K(x - r) >= W_R exp(-E|x - r|^2
// / 2h^2), and E|x - r|^2 = |x - c|^2 - 2 (x - c).m + s2 <= (|x - c| + |m|)^2
// - |m|^2 + s2 (c the node's centre, m the weighted mean offset from it, s2
// the weighted mean squared offset; node_js = (|m|, s2)) -- far tighter than
// K_lo (the farthest pair) for a wide node, so G_min, the token budget and
// the prunes it admits grow (Theorem 2 needs only a valid lower bound).
template <int D>
__device__ __forceinline__ void entry_bounds(const TravArgs &A, const double *sq, int node,
                                             double neg_inv, double &klo, double &khi, double &lb,
                                             const double *s_tab) {
    const double *rbox = A.r_box + (int64_t)node * 2 * D;
    const double *rc = A.r_c + (int64_t)node * D;
    double mx = 0.0, mn = 0.0, dq = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double qlo = sq[d], qhi = sq[D + d];
        const double rlo = __ldg(rbox + d), rhi = __ldg(rbox + D + d);
        const double a = qlo - rhi, b = rlo - qhi;
        const double g = a > b ? a : b;
        if (g > 0.0) mn += g * g;
        const double s1 = qhi - rlo, s2 = rhi - qlo;
        const double s = s1 > s2 ? s1 : s2;
        mx += s * s;
        const double c = __ldg(rc + d);
        const double e = fmax(fabs(qlo - c), fabs(qhi - c));
        dq += e * e;
    }
    khi = fg_exp_fast(mn * neg_inv, s_tab);
    klo = fg_exp_fast(mx * neg_inv, s_tab);
    lb = klo;
    if (A.r_js) {
        const double2 js = __ldg(A.r_js + node);
        const double r = sqrt(dq) * (1.0 + 0x1.0p-50) + js.x;
        // (1 + 2^-40) covers the roundings of the squared distances, the
        // square root and the stored statistics (all <= ~2^-50 relative)
        const double ex = (r * r - js.x * js.x + js.y) * (1.0 + 0x1.0p-40);
        if (ex < mx) lb = fmin(khi, fmax(klo, fg_exp_fast(ex * neg_inv, s_tab) * (1.0 - 0x1.0p-40)));
    }
}

// Exact contribution of reference points [rs, rs+rc) to this lane's query
// (_leaf_kernel_block, summation_engine.py:206-218): all lanes read the same
// record (broadcast), two independent exp chains per step.
// Copy the points of base item `i` (lanes' (ni_x, ni_y) = start, count <= 32)
// into a shared-memory buffer with cp.async; one commit group per call.
template <int D>
__device__ __forceinline__ void stage_points(const double *__restrict__ pw, int ni_x, int ni_y,
                                             int i, double *buf) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    const int rs = __shfl_sync(kFull, ni_x, i);
    const int rc = __shfl_sync(kFull, ni_y, i);
    FG_CHECK(rc >= 1 && rc <= kStageMax && rs >= 0);
    for (int l = lane; l < rc; l += 32) {
        const double *src = pw + (int64_t)(rs + l) * S;
        double *dst = buf + l * S;
#pragma unroll
        for (int q = 0; q < S / 2; q++) __pipeline_memcpy_async(dst + 2 * q, src + 2 * q, 16);
    }
    __pipeline_commit();
}

template <int D>
__device__ __forceinline__ void read_point_w(const double *rec, double (&x)[D], double &w) {
    constexpr int S = packed_stride(D);
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int k = 0; k < S / 2; k++) {
        const double2 v = r2[k];
        if (2 * k < D) x[2 * k] = v.x;
        else if (2 * k == D) w = v.x;
        if (2 * k + 1 < D) x[2 * k + 1] = v.y;
        else if (2 * k + 1 == D) w = v.y;
    }
}

template <int D, bool CHECKED>
__device__ __forceinline__ double base_case(const double (&x)[D],
                                            const double *__restrict__ rp, int rc,
                                            double neg_inv, const double *s_tab) {
    constexpr int S = packed_stride(D);
    constexpr int U = CHECKED ? 2 : 4;  // independent exp chains per step
    const ExpK K = exp_consts(s_tab);   // register-resident for the loop
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; u++) acc[u] = 0.0;
    int j = 0;
    for (; j + U - 1 < rc; j += U) {
        double y[U][D], w[U], d2[U];
#pragma unroll
        for (int u = 0; u < U; u++) read_point_w<D>(rp + (int64_t)(j + u) * S, y[u], w[u]);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const double e = x[0] - y[u][0];
            d2[u] = e * e;
        }
#pragma unroll
        for (int d = 1; d < D; d++)
#pragma unroll
            for (int u = 0; u < U; u++) {
                const double f = x[d] - y[u][d];
                d2[u] = fma(f, f, d2[u]);
            }
#pragma unroll
        for (int u = 0; u < U; u++)
            acc[u] = fma(CHECKED ? fg_exp_kc(d2[u] * neg_inv, K) : fg_exp_k(d2[u] * neg_inv, K),
                         w[u], acc[u]);
    }
#pragma unroll 1
    for (; j < rc; j++) {
        double y0[D], w0;
        read_point_w<D>(rp + (int64_t)j * S, y0, w0);
        const double e0 = x[0] - y0[0];
        double d0 = e0 * e0;
#pragma unroll
        for (int d = 1; d < D; d++) {
            const double f0 = x[d] - y0[d];
            d0 = fma(f0, f0, d0);
        }
        acc[0] = fma(CHECKED ? fg_exp_kc(d0 * neg_inv, K) : fg_exp_k(d0 * neg_inv, K), w0,
                     acc[0]);
    }
    double s = acc[0];
#pragma unroll
    for (int u = 1; u < U; u++) s += acc[u];
    return s;
}

// Both query slots of a lane against one staged item in a single pass over
// its points (two points x two queries = four independent exp chains).
template <int D, bool CHECKED>
__device__ __forceinline__ void base_case2(const double (&x)[kQPL][D],
                                           const double *__restrict__ rp, int rc, double neg_inv,
                                           const double *s_tab, double &out0, double &out1) {
    constexpr int S = packed_stride(D);
    const ExpK K = exp_consts(s_tab);
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;  // a<query><point>
    int j = 0;
    for (; j + 1 < rc; j += 2) {
        double y0[D], y1[D], w0, w1;
        read_point_w<D>(rp + (int64_t)j * S, y0, w0);
        read_point_w<D>(rp + (int64_t)(j + 1) * S, y1, w1);
        double d00, d01, d10, d11;
        {
            const double e00 = x[0][0] - y0[0], e01 = x[0][0] - y1[0];
            const double e10 = x[1][0] - y0[0], e11 = x[1][0] - y1[0];
            d00 = e00 * e00; d01 = e01 * e01; d10 = e10 * e10; d11 = e11 * e11;
        }
#pragma unroll
        for (int d = 1; d < D; d++) {
            const double f00 = x[0][d] - y0[d], f01 = x[0][d] - y1[d];
            const double f10 = x[1][d] - y0[d], f11 = x[1][d] - y1[d];
            d00 = fma(f00, f00, d00);
            d01 = fma(f01, f01, d01);
            d10 = fma(f10, f10, d10);
            d11 = fma(f11, f11, d11);
        }
        a00 = fma(CHECKED ? fg_exp_kc(d00 * neg_inv, K) : fg_exp_k(d00 * neg_inv, K), w0, a00);
        a01 = fma(CHECKED ? fg_exp_kc(d01 * neg_inv, K) : fg_exp_k(d01 * neg_inv, K), w1, a01);
        a10 = fma(CHECKED ? fg_exp_kc(d10 * neg_inv, K) : fg_exp_k(d10 * neg_inv, K), w0, a10);
        a11 = fma(CHECKED ? fg_exp_kc(d11 * neg_inv, K) : fg_exp_k(d11 * neg_inv, K), w1, a11);
    }
    if (j < rc) {
        double y0[D], w0;
        read_point_w<D>(rp + (int64_t)j * S, y0, w0);
        const double e0 = x[0][0] - y0[0], e1 = x[1][0] - y0[0];
        double d0 = e0 * e0, d1 = e1 * e1;
#pragma unroll
        for (int d = 1; d < D; d++) {
            const double f0 = x[0][d] - y0[d], f1 = x[1][d] - y0[d];
            d0 = fma(f0, f0, d0);
            d1 = fma(f1, f1, d1);
        }
        a00 = fma(CHECKED ? fg_exp_kc(d0 * neg_inv, K) : fg_exp_k(d0 * neg_inv, K), w0, a00);
        a10 = fma(CHECKED ? fg_exp_kc(d1 * neg_inv, K) : fg_exp_k(d1 * neg_inv, K), w0, a10);
    }
    out0 = a00 + a01;
    out1 = a10 + a11;
}

// ---- FP32 base case --------------------------------------------------------
// The reference tree keeps an FP32 copy of its points (fp32_pack,
// fg_traverse.cu): coordinates relative to the centre c_a of the point's
// anchor (its maximal tree node with <= 32 points) and the weight.  A base
// item of <= 32 points lies inside one anchor.  All FP32 items of a traversal
// step are evaluated as ONE batch: their records are staged back to back
// (each item padded to a multiple of 4 with zero records) in transposed
// layout, every group of 4 points carries its item's offset
// delta = fl(c_a - c_b) (c_b = the query block's centroid), and each lane
// streams the whole batch with its query xf = fl(x - c_b) shifted to
// xq = fl(xf - delta): packed FP32 pairs (FADD2/FFMA2/FMUL2), exp2 on the SFU
// (ex2.approx), four FP32 accumulators.
//
// The batch error is bounded by rho S + abs (fp32_item_bound; DESIGN.md
// "FP32 base case"), S the exact sum.  An item joins only when rho <=
// H.fp32_rho = phi * eps -- all FP32 items together then err by at most
// phi * eps * G(x_q) through their relative parts -- and when its own token
// share covers abs, which is charged through the token rule
// (summation_engine.py:157-188) like a prune's error.  The host runs the
// traversal's approximation rules with (1 - phi) * eps, so the total error
// stays within eps * G (Theorem 2).
template <int D>
constexpr int fstride() { return (D + 1 + 3) & ~3; }
// Anchored FP32 items (D <= 4) in dot form from record PAIRS (fp32_pair_pack,
// fg_traverse.cu): every f32x2 operand comes straight from shared memory, so
// the loop needs no register packing.
#ifndef FG_DEFER_CREDIT
#define FG_DEFER_CREDIT 0
#endif
#ifndef FG_PAIR_DOT
#define FG_PAIR_DOT 1
#endif
// items whose dot-form bound fails fall back to the difference form (else FP64)
#ifndef FG_PAIR_DIFF
#define FG_PAIR_DIFF 1
#endif
// per-item A = fl(-s |X|^2) and the fold of an item's partial sums in FP32
#ifndef FG_PAIR_F32_PROLOGUE
#define FG_PAIR_F32_PROLOGUE 1
#endif
// floats per record pair: {Y_d a/b} x D, {B a/b}, {W a/b}, padded to 16 bytes
template <int D>
constexpr int pstride() { return (2 * (D + 2) + 3) & ~3; }
// points per staged batch and floats per group offset record
template <int D>
constexpr int f32_cap() { return D <= 4 ? 256 : 128; }
template <int D>
constexpr int f32_fd() { return (D + 3) & ~3; }
// per-warp shared memory of the batch, in doubles: CAP AoS records of
// fstride floats, then the item table (32 x {offset, count, offset vector})
// D >= 5 streams FP32 records converted from the FP64 points instead (see
// "Direct FP32 stream" below): one window of f32_win converted records
template <int D>
constexpr bool f32_direct() { return D >= 5; }
// FP64 staging buffer in records: two kStageMax buffers (double-buffered FP64
// items) at D <= 4; one at D >= 5, where the query coordinates take the
// shared memory instead (registers are the scarcer resource there)
template <int D>
constexpr int stage_recs() { return D <= 5 ? 2 * kStageMax : kStageMax; }
template <int D>
constexpr bool stage_db() { return stage_recs<D>() >= 2 * kStageMax; }
// records per direct-stream window (two windows fill the staging buffer)
template <int D>
constexpr int f32_win() { return stage_recs<D>() / 2; }
#ifndef FG_DOT_FORM
#define FG_DOT_FORM 1
#endif
constexpr bool g_dot_form = FG_DOT_FORM;
// dot-form records of the direct stream: 2s(y - c_b), -s |y - c_b|^2, w
template <int D>
constexpr int dstride() { return (D + 2 + 3) & ~3; }
template <int D>
constexpr int f32_smem_doubles() {
    return f32_direct<D>() ? f32_win<D>() * dstride<D>() / 2
                           : (f32_cap<D>() * fstride<D>() + 32 * (2 + f32_fd<D>())) / 2;
}

// per-warp shared memory before the local coefficients (K doubles): query
// box and centroid, the FP64 staging buffer, the FP32 batch / window
// At D <= 4 the block's query coordinates live in shared memory (xs_doubles)
// rather than in registers: the traversal kernel is register-bound, and the
// FP32 batch loop is scheduled tighter with the 4D registers back.
template <int D>
constexpr bool xs_smem() { return true; }
template <int D>
constexpr int xs_doubles() { return xs_smem<D>() ? kQBlock * D : 0; }
// one 8-byte mbarrier per warp (bulk copies of FP32 record pairs), padded
constexpr int kMbarDoubles = 2;
template <int D>
constexpr int warp_fixed_doubles() {
    return ((3 * D + 1) & ~1) + stage_recs<D>() * packed_stride(D) + f32_smem_doubles<D>() +
           kMbarDoubles + xs_doubles<D>();
}
// record pairs the anchored batch can stage: the FP64 staging buffer and the
// FP32 record area are contiguous and idle while a batch runs (the item table
// follows them)
template <int D>
constexpr int pair_cap() {
    return (stage_recs<D>() * packed_stride(D) * 8 + f32_cap<D>() * fstride<D>() * 4) /
           (pstride<D>() * 4);
}

// ---- bulk copies (cp.async.bulk + mbarrier) -------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) writes to the same bytes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ float ex2_approx(float v) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// Error bound |S_fp32 - S| <= rho S + abs for one item (query block box `sq`
// with centroid `sqc`, reference points inside anchor `anc`, weight wr), for
// every query of the block.  With M bounding |x - c_b|, |c_a - c_b|,
// |x - c_a| and |y - c_a| per coordinate, each coordinate difference carries
// at most 4 u M of rounding (u = 2^-24) before its own rounding, so a term
// with exponent a has an exponent error (= relative error) of at most
//   da(a) = C1 sqrt(a) + C2 a,  C1 = 2^-21 sqrt(D) M / (sqrt2 h),  C2 = (4+D) u
// (the FP32 difference, squared distance and scaling), plus 2^-17 for
// ex2.approx (measured <= 2^-22.7 by tools/ex2_accuracy.cu), weight rounding
// and <= 63 additions per FP32 accumulator (four per query slot); rho doubles that
// for safety.  The relative part is only claimed up to a cut a_c: the largest
// exponent with rho(a_c) <= rho_max, capped at 80 and at a_max = -ln K_lo,
// the item's largest pair exponent.  Terms beyond a_c (ex2 may flush them)
// are worth at most w e^-a_c, and so are their computed values up to the
// factor e^{da(a_c)} (a - da(a) grows with a): abs = 2.03 wr e^-a_c when
// a_max > a_c, plus 2^-140 for subnormal rounding in the accumulation.
// Returns rho, or +inf when no cut fits.
template <int D>
__device__ __forceinline__ double fp32_item_bound(const TravArgs &A, const double *sq, int anc,
                                                  double inv_h, double klo, double wr,
                                                  double rho_max, double &abs_err) {
    // an upper bound on a_max = -ln K_lo (MUFU lg2: <= 2^-21 relative plus the
    // FP32 rounding of K_lo, covered by the margins; +inf below FLT_MIN)
    const float kf = (float)klo;
    const double a_max = kf >= 1.17549435e-38f ? (double)(-__logf(kf)) * (1.0 + 0x1.0p-18) + 0x1.0p-18
                                               : CUDART_INF;
    const double *abox = A.r_box + (int64_t)anc * 2 * D;
    const double *ac = A.r_c + (int64_t)anc * D;
    double M = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double c = __ldg(ac + d), cb = sq[2 * D + d];
        const double qlo = sq[d], qhi = sq[D + d];
        M = fmax(M, fmax(fmax(fabs(__ldg(abox + d) - c), fabs(__ldg(abox + D + d) - c)),
                         fmax(fabs(qlo - c), fabs(qhi - c))));
        M = fmax(M, fmax(fabs(c - cb), fmax(fabs(qlo - cb), fabs(qhi - cb))));
    }
    const double c1 = 0x1.0p-21 * sqrt((double)D) * M * inv_h * 0.7071067811865476;
    const double c2 = (4.0 + D) * 0x1.0p-24;
    const double room = 0.5 * rho_max - 0x1.0p-17;
    abs_err = CUDART_INF;
    if (!(room > 0.0)) return CUDART_INF;
    // largest s = sqrt(a) with c2 s^2 + c1 s <= room
    const double sfit = 2.0 * room / (c1 + sqrt(c1 * c1 + 4.0 * c2 * room));
    const double a_c = fmin(fmin(a_max, 80.0), sfit * sfit * (1.0 - 0x1.0p-40));
    abs_err = 0x1.0p-140;
    if (a_max > a_c)
        abs_err += 2.03 * wr * (double)ex2_approx((float)(-a_c * 1.4426950408889634)) * 1.0001;
    return 2.0 * (c1 * sqrt(a_c) + c2 * a_c + 0x1.0p-17);
}

// packed FP32 pairs (sm_100 FADD2 / FFMA2 / FMUL2, round-to-nearest per lane)
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    return (unsigned long long)__float_as_uint(lo) |
           ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float f2_hi(unsigned long long v) {
    return __uint_as_float((unsigned)(v >> 32));
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// acc += a * b in place (ties the accumulator register to the FFMA2 output)
__device__ __forceinline__ void f2_fma_acc(unsigned long long &acc, unsigned long long a,
                                           unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ unsigned long long f2_ex2(unsigned long long v) {
    return f2_pack(ex2_approx(f2_lo(v)), ex2_approx(f2_hi(v)));
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// 2^t on the FMA pipe (t <= 0, both halves): t is clamped at -125, split as
// n + f with n = rint(t) (the 1.5 * 2^23 trick) and f in [-0.5, 0.5], 2^f by a
// degree-5 polynomial (fitted to relative error 2^-23.7; evaluated in FP32
// Horner form: <= 2^-22.2 over 2e6 points, against ex2.approx's measured
// 2^-22.7 -- both inside the 2^-17 share fp32_item_bound / fp32_pair_bound
// reserve for the exponential, weight rounding and accumulation), then n is
// added to the exponent bits.  Results below 2^-125 come out as ~2^-125:
// such terms have exponent a > 86 > a_c, inside the bounds' absolute part.
// It relieves the SFU (one ex2 per pair, the FP32 base case's bound) for a
// share of the pairs (the FA4 offload).
__device__ __forceinline__ unsigned long long f2_ex2_poly(unsigned long long t) {
    const float lo = fmaxf(f2_lo(t), -125.f), hi = fmaxf(f2_hi(t), -125.f);
    const unsigned long long tc = f2_pack(lo, hi);
    const unsigned long long M = f2_pack(12582912.f, 12582912.f);
    const unsigned long long r = f2_add(tc, M);
    const unsigned long long f = f2_sub(tc, f2_sub(r, M));
    unsigned long long p = f2_fma(f2_pack(0.00132748f, 0.00132748f), f,
                                  f2_pack(0.00967553f, 0.00967553f));
    p = f2_fma(p, f, f2_pack(0.05550718f, 0.05550718f));
    p = f2_fma(p, f, f2_pack(0.2402212f, 0.2402212f));
    p = f2_fma(p, f, f2_pack(0.69314694f, 0.69314694f));
    p = f2_fma(p, f, f2_pack(1.0000001f, 1.0000001f));
    const unsigned plo = (unsigned)p + ((unsigned)r << 23);
    const unsigned phi = (unsigned)(p >> 32) + ((unsigned)(r >> 32) << 23);
    return (unsigned long long)plo | ((unsigned long long)phi << 32);
}

// Stream one staged batch: nitems items, item t with `cnt` AoS records
// (fstride floats: coordinates about its anchor, weight) at record offset
// `off`, and its offset vector dl = fl(c_a - c_b).  The two query slots of the
// lane form the packed FP32 pair, so every record is loaded once for both
// (the reference coordinate and weight enter as broadcast operands); four
// records per iteration, each with its own accumulator pair.
template <int D>
__device__ __forceinline__ void batch_f32(const unsigned long long (&xf2)[D], const float *fst,
                                          const int *ioff, const int *icnt, const float *idl,
                                          int nitems, float ex2s, double &sum0, double &sum1) {
    constexpr int F = fstride<D>(), FD = f32_fd<D>();
    const unsigned long long s2 = f2_pack(ex2s, ex2s);
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll 1
    for (int it = 0; it < nitems; it++) {
        const int off = ioff[it], cnt = icnt[it];
        unsigned long long q2[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            const float dv = idl[it * FD + d];
            q2[d] = f2_sub(xf2[d], f2_pack(dv, dv));
        }
        const float *rec = fst + off * F;
        int j = 0;
        for (; j + 4 <= cnt; j += 4) {
            // four records, dimension-major: four independent FFMA2 chains
            // interleaved, so a lone warp (the launch's tail) still issues
            // back to back instead of waiting on each chain's latency
            float y[4][F];
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int k = 0; k < F; k += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(rec + (j + u) * F + k);
                    y[u][k] = v.x; y[u][k + 1] = v.y; y[u][k + 2] = v.z; y[u][k + 3] = v.w;
                }
            unsigned long long dd[4];
#pragma unroll
            for (int d = 0; d < D; d++)
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const unsigned long long f = f2_sub(q2[d], f2_pack(y[u][d], y[u][d]));
                    dd[u] = d == 0 ? f2_mul(f, f) : f2_fma(f, f, dd[u]);
                }
#pragma unroll
            for (int u = 0; u < 4; u++) dd[u] = f2_ex2(f2_mul(dd[u], s2));
#pragma unroll
            for (int u = 0; u < 4; u++) f2_fma_acc(acc[u], dd[u], f2_pack(y[u][D], y[u][D]));
        }
        for (; j < cnt; j++) {
            const float *r = rec + j * F;
            float y[F];
#pragma unroll
            for (int k = 0; k < F; k += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(r + k);
                y[k] = v.x; y[k + 1] = v.y; y[k + 2] = v.z; y[k + 3] = v.w;
            }
            unsigned long long dd = 0ull;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const unsigned long long f = f2_sub(q2[d], f2_pack(y[d], y[d]));
                dd = d == 0 ? f2_mul(f, f) : f2_fma(f, f, dd);
            }
            f2_fma_acc(acc[j & 3], f2_ex2(f2_mul(dd, s2)), f2_pack(y[D], y[D]));
        }
    }
    sum0 = ((double)f2_lo(acc[0]) + (double)f2_lo(acc[1])) +
           ((double)f2_lo(acc[2]) + (double)f2_lo(acc[3]));
    sum1 = ((double)f2_hi(acc[0]) + (double)f2_hi(acc[1])) +
           ((double)f2_hi(acc[2]) + (double)f2_hi(acc[3]));
}

// ---- Anchored dot-form batches from record pairs (D <= 4, FG_PAIR_DOT) -----
// The exponent (log2 units, s = log2(e) / 2h^2) of query x and record y of an
// item inside anchor a (centre c_a) is evaluated as
//     t = A + (-s) B + sum_d X'_d Y_d,  A = fl(-s |X|^2), X' = fl(2 s X),
// X = fl(fl(x - c_b) - fl(c_a - c_b)) (as in batch_f32), Y and B = fl(|Y|^2)
// from the record pair: D + 2 FFMA2 and two ex2 per record pair and query
// slot, no operand packing.
//
// Error bound (fp32_pair_bound): the coordinate roundings are those of
// fp32_item_bound (<= 4 u M per coordinate difference: the C1 sqrt(a) term).
// The dot form adds roundings that are absolute in t: A and B one rounding
// each, fl(-s) and X' one relative rounding each, and the D + 1 chained FFMA
// roundings; every partial sum is bounded by s (|X| + |Y|)^2, so in natural-log
// units E = (D + 4) u (R_q + R_r)^2 / 2h^2 (one spare term), with R_q, R_r
// the largest 2-norm offsets of the query box and of the item's node box from
// c_a (inflated for the coordinate roundings).  rho = 2 (C1 sqrt(a_c) + E +
// 2^-17), cut at a_c as in fp32_item_bound; the per-item FP32 sums are folded
// into FP64 after each item, so no FP32 accumulator adds more than 84 terms
// (336-point items: 168 pairs over two accumulator pairs; with ex2, weight and
// FMA roundings <= 91 u of the 128 u = 2^-17 the bound reserves).
template <int D>
__device__ __forceinline__ double fp32_pair_bound(const TravArgs &A, const double *sq, int anc,
                                                  int node, double inv_h, double klo, double wr,
                                                  double rho_max, double &abs_err) {
    const float kf = (float)klo;
    const double a_max = kf >= 1.17549435e-38f ? (double)(-__logf(kf)) * (1.0 + 0x1.0p-18) + 0x1.0p-18
                                               : CUDART_INF;
    const double *abox = A.r_box + (int64_t)anc * 2 * D;
    const double *nbox = A.r_box + (int64_t)node * 2 * D;
    const double *ac = A.r_c + (int64_t)anc * D;
    double M = 0.0, rq2 = 0.0, rr2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double c = __ldg(ac + d), cb = sq[2 * D + d];
        const double qlo = sq[d], qhi = sq[D + d];
        const double mq = fmax(fabs(qlo - c), fabs(qhi - c));
        const double mr = fmax(fabs(__ldg(nbox + d) - c), fabs(__ldg(nbox + D + d) - c));
        M = fmax(M, fmax(fmax(fabs(__ldg(abox + d) - c), fabs(__ldg(abox + D + d) - c)), mq));
        M = fmax(M, fmax(fabs(c - cb), fmax(fabs(qlo - cb), fabs(qhi - cb))));
        rq2 += mq * mq;
        rr2 += mr * mr;
    }
    const double c1 = 0x1.0p-21 * sqrt((double)D) * M * inv_h * 0.7071067811865476;
    const double rs = (sqrt(rq2) + sqrt(rr2)) * (1.0 + 0x1.0p-20) * inv_h;
    const double e = (D + 4.0 + (FG_PAIR_F32_PROLOGUE ? D : 0)) * 0x1.0p-24 * 0.5 * rs * rs * 1.01;
    const double room = 0.5 * rho_max - 0x1.0p-17 - e;
    abs_err = CUDART_INF;
    if (!(room > 0.0)) return CUDART_INF;
    const double sf = c1 > 0.0 ? room / c1 : CUDART_INF;
    const double a_c = fmin(fmin(a_max, 80.0), sf * sf * (1.0 - 0x1.0p-40));
    abs_err = 0x1.0p-140;
    if (a_max > a_c)
        abs_err += 2.03 * wr * (double)ex2_approx((float)(-a_c * 1.4426950408889634)) * 1.0001;
    return 2.0 * (c1 * sqrt(a_c) + e + 0x1.0p-17);
}

// Stream one staged batch of record pairs: item t has icnt[t] pairs at pair
// offset ioff[t] and the offset vector idl[t] = fl(c_a - c_b); xs holds the
// lane's two query slots about c_b (FP32).  Per item the slots' A and X' are
// formed once, then two record pairs per iteration (four independent chains
// per slot pair); each item's FP32 sums are folded into FP64.
// Items whose dot-form bound does not fit (wide items at small h: the dot
// form's rounding grows with (R_q + R_r)^2 / h^2) but whose difference-form
// bound does (fp32_item_bound) are flagged kPairDiff in icnt and streamed in
// the difference form from the same record pairs:
//     t = -s |X - Y|^2  (D FADD2, D FFMA2/FMUL2, one FMUL2 by -s).
constexpr int kPairDiff = 1 << 30;
// One difference-form item (out of line: rare, and it keeps the dot-form
// loop's register allocation intact).
// (query offsets by value and sums returned by value: reference parameters of an
// out-of-line function would pin the caller's copies to local memory)
template <int D>
struct SlotOffsets {
    float v[kQPL][D];
};
template <int D>
__device__ __noinline__ double2 item_pairs_diff(SlotOffsets<D> xsv, const float *pitem, int np,
                                                const float *dli, unsigned long long nss) {
    const float (&xs)[kQPL][D] = xsv.v;
    constexpr int P = pstride<D>(), P2 = P / 2;
    unsigned long long xq[kQPL][D];
#pragma unroll
    for (int q = 0; q < kQPL; q++)
#pragma unroll
        for (int d = 0; d < D; d++) {
            const float X = xs[q][d] - dli[d];
            xq[q][d] = f2_pack(X, X);
        }
    const unsigned long long *rec = reinterpret_cast<const unsigned long long *>(pitem);
    unsigned long long acc[kQPL][2] = {{0ull, 0ull}, {0ull, 0ull}};
#pragma unroll 1
    for (int j = 0; j < np; j += 2) {
        const int nu = j + 1 < np ? 2 : 1;
        unsigned long long r[2][P2];
#pragma unroll
        for (int u = 0; u < 2; u++)
#pragma unroll
            for (int k = 0; k < P2; k += 2) {
                // a lone last pair re-reads itself; its second copy is not accumulated
                const ulonglong2 v =
                    *reinterpret_cast<const ulonglong2 *>(rec + (j + (u < nu ? u : 0)) * P2 + k);
                r[u][k] = v.x;
                r[u][k + 1] = v.y;
            }
#pragma unroll
        for (int q = 0; q < kQPL; q++)
#pragma unroll
            for (int u = 0; u < 2; u++) {
                unsigned long long f = f2_sub(xq[q][0], r[u][0]);
                unsigned long long dd = f2_mul(f, f);
#pragma unroll
                for (int d = 1; d < D; d++) {
                    f = f2_sub(xq[q][d], r[u][d]);
                    f2_fma_acc(dd, f, f);
                }
                const unsigned long long e = f2_ex2(f2_mul(dd, nss));
                if (u < nu) f2_fma_acc(acc[q][u], e, r[u][D + 1]);
            }
    }
    return make_double2(((double)f2_lo(acc[0][0]) + (double)f2_hi(acc[0][0])) +
                            ((double)f2_lo(acc[0][1]) + (double)f2_hi(acc[0][1])),
                        ((double)f2_lo(acc[1][0]) + (double)f2_hi(acc[1][0])) +
                            ((double)f2_lo(acc[1][1]) + (double)f2_hi(acc[1][1])));
}

template <int D>
__device__ __forceinline__ void batch_pairs(const float (&xs)[kQPL][D], const float *pbuf,
                                            const int *ioff, const int *icnt, const float *idl,
                                            int nitems, double s, double &sum0, double &sum1) {
    constexpr int P = pstride<D>(), FD = f32_fd<D>(), P2 = P / 2;
    const float sf = (float)s, s2f = (float)(2.0 * s);
    const unsigned long long nss = f2_pack(-sf, -sf);
#pragma unroll 1
    for (int it = 0; it < nitems; it++) {
        const int off = ioff[it], np = icnt[it] & (kPairDiff - 1);
        if (icnt[it] & kPairDiff) {
            SlotOffsets<D> xsv;
#pragma unroll
            for (int q = 0; q < kQPL; q++)
#pragma unroll
                for (int d = 0; d < D; d++) xsv.v[q][d] = xs[q][d];
            const double2 r = item_pairs_diff<D>(xsv, pbuf + off * P, np, idl + it * FD, nss);
            sum0 += r.x;
            sum1 += r.y;
            continue;
        }
        unsigned long long xx[kQPL][D], aa[kQPL];
#pragma unroll
        for (int q = 0; q < kQPL; q++) {
#if FG_PAIR_F32_PROLOGUE
            // A = fl(-s |X|^2) in FP32: D + 1 roundings instead of one (the D
            // extra are covered by fp32_pair_bound's E, see there); no FP64 <->
            // FP32 conversions (they share the SFU with ex2) per item
            float a = 0.f;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const float X = xs[q][d] - idl[it * FD + d];
                const float Xp = s2f * X;
                xx[q][d] = f2_pack(Xp, Xp);
                a = fmaf(X, X, a);
            }
            const float av = -sf * a;
#else
            double a = 0.0;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const float X = xs[q][d] - idl[it * FD + d];
                const float Xp = s2f * X;
                xx[q][d] = f2_pack(Xp, Xp);
                a = fma((double)X, (double)X, a);
            }
            const float av = (float)(-s * a);
#endif
            aa[q] = f2_pack(av, av);
        }
        const unsigned long long *rec = reinterpret_cast<const unsigned long long *>(pbuf + off * P);
        unsigned long long acc[kQPL][2] = {{0ull, 0ull}, {0ull, 0ull}};
        int j = 0;
#ifndef FG_PAIR_UNROLL
#define FG_PAIR_UNROLL 4
#endif
        constexpr int PU = FG_PAIR_UNROLL;  // record pairs per iteration (PU x 2 chains)
#ifndef FG_POLY_CHAINS
#define FG_POLY_CHAINS 0
#endif
        // chains (slot q, pair u) per iteration whose 2^t runs on the FMA pipe
        constexpr int NPOLY = FG_POLY_CHAINS;
        for (; j + PU <= np; j += PU) {
            unsigned long long r[PU][P2];
#pragma unroll
            for (int u = 0; u < PU; u++)
#pragma unroll
                for (int k = 0; k < P2; k += 2) {
                    const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(rec + (j + u) * P2 + k);
                    r[u][k] = v.x;
                    r[u][k + 1] = v.y;
                }
#pragma unroll
            for (int q = 0; q < kQPL; q++)
#pragma unroll
                for (int u = 0; u < PU; u++) {
                    unsigned long long t = f2_fma(r[u][D], nss, aa[q]);
#pragma unroll
                    for (int d = 0; d < D; d++) f2_fma_acc(t, xx[q][d], r[u][d]);
                    const bool poly = u == PU - 1 && (NPOLY >= 2 || (NPOLY == 1 && q == 1));
                    f2_fma_acc(acc[q][u & 1], poly ? f2_ex2_poly(t) : f2_ex2(t), r[u][D + 1]);
                }
        }
        for (; j + 2 <= np; j += 2) {
            unsigned long long r[2][P2];
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int k = 0; k < P2; k += 2) {
                    const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(rec + (j + u) * P2 + k);
                    r[u][k] = v.x;
                    r[u][k + 1] = v.y;
                }
#pragma unroll
            for (int q = 0; q < kQPL; q++)
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    unsigned long long t = f2_fma(r[u][D], nss, aa[q]);
#pragma unroll
                    for (int d = 0; d < D; d++) f2_fma_acc(t, xx[q][d], r[u][d]);
                    f2_fma_acc(acc[q][u], f2_ex2(t), r[u][D + 1]);
                }
        }
        if (j < np) {
            unsigned long long r[P2];
#pragma unroll
            for (int k = 0; k < P2; k += 2) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(rec + j * P2 + k);
                r[k] = v.x;
                r[k + 1] = v.y;
            }
#pragma unroll
            for (int q = 0; q < kQPL; q++) {
                unsigned long long t = f2_fma(r[D], nss, aa[q]);
#pragma unroll
                for (int d = 0; d < D; d++) f2_fma_acc(t, xx[q][d], r[d]);
                f2_fma_acc(acc[q][0], f2_ex2(t), r[D + 1]);
            }
        }
#if FG_PAIR_F32_PROLOGUE
        // the four partial sums of a slot are added in FP32 (two more roundings
        // on accumulators of <= 84 terms each: inside the bounds' 2^-17 reserve)
        sum0 += (double)((f2_lo(acc[0][0]) + f2_hi(acc[0][0])) +
                         (f2_lo(acc[0][1]) + f2_hi(acc[0][1])));
        sum1 += (double)((f2_lo(acc[1][0]) + f2_hi(acc[1][0])) +
                         (f2_lo(acc[1][1]) + f2_hi(acc[1][1])));
#else
        sum0 += ((double)f2_lo(acc[0][0]) + (double)f2_hi(acc[0][0])) +
                ((double)f2_lo(acc[0][1]) + (double)f2_hi(acc[0][1]));
        sum1 += ((double)f2_lo(acc[1][0]) + (double)f2_hi(acc[1][0])) +
                ((double)f2_lo(acc[1][1]) + (double)f2_hi(acc[1][1]));
#endif
    }
}

// ---- Direct FP32 stream (D >= 5) ------------------------------------------
// At D >= 5 the per-item loop of batch_f32 (each item re-centres the query,
// then a short record loop with a ragged tail) costs more than converting the
// records: the items' FP64 points are copied (cp.async) window by window into
// the FP64 staging buffer -- the next window's copy in flight while the
// current one computes -- converted by the lanes to FP32 records about the
// query block's centroid, y' = fl(y - c_b) with fl(w), and streamed in one
// flat loop.  Records are item-independent, so windows cut items anywhere and
// items may exceed an anchor (measured: C3 -11 %, C4 -9 % vs anchored batches;
// at D = 3 the conversion costs more than it saves, +3 %).
//
// Error bound of an item (query block box `sq` with centroid c_b, node
// `node`): with M bounding |x - c_b| over the query box and |y - c_b| over the
// node's box per coordinate, each coordinate difference fl(xf - y') carries at
// most 2 u M of rounding (xf and y' one rounding each) before its own
// rounding, so C1 = 2^-22 sqrt(D) M / (sqrt2 h) in fp32_item_bound's model;
// everything else is as there (<= 16 additions per accumulator per window).
//
// Dot form.  The stream may instead expand the exponent (log2 units,
// s = log2(e) / 2h^2) as  t = (A_q + B_r) + sum_d X_d C_d  with per-query
// A_q = fl(-s |X|^2) (X = the FP32 query offsets), per-record
// B_r = fl(-s |Y|^2), C_d = fl(2 s Y_d) (Y = y - c_b in FP64): one FFMA2 per
// coordinate instead of FADD2 + FFMA2.  Every rounding is absolute in t:
// u (|A| + |B| + sum |X_d C_d|) for the stored values and u |t_k| for the
// D + 1 chain steps, each <= u s (|X| + |Y|)^2, so in natural-log units
// E = (D + 2) u (R_q + R_r)^2 / 2h^2 with R_q, R_r the largest 2-norm
// offsets of the query box and the node box from c_b; the query rounding
// adds C1 / 2 sqrt(a) as above (the record side is exact before its own
// rounding).  rho_dot = 2 (C1 / 2 sqrt(a) + E + 2^-17), cut as above.
template <int D>
__device__ __forceinline__ double fp32_node_bound(const TravArgs &A, const double *sq, int node,
                                                  double inv_h, double klo, double wr,
                                                  double rho_max, double &abs_err,
                                                  double &rho_dot, double &abs_dot) {
    const float kf = (float)klo;
    const double a_max = kf >= 1.17549435e-38f ? (double)(-__logf(kf)) * (1.0 + 0x1.0p-18) + 0x1.0p-18
                                               : CUDART_INF;
    const double *rbox = A.r_box + (int64_t)node * 2 * D;
    double M = 0.0, Mq = 0.0, rq2 = 0.0, rr2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double cb = sq[2 * D + d];
        const double mr = fmax(fabs(__ldg(rbox + d) - cb), fabs(__ldg(rbox + D + d) - cb));
        const double mq = fmax(fabs(sq[d] - cb), fabs(sq[D + d] - cb));
        M = fmax(M, fmax(mr, mq));
        Mq = fmax(Mq, mq);
        rq2 += mq * mq;
        rr2 += mr * mr;
    }
    // 2^-22 (1 + 2^-4): the FP64 differences x - c_b, y - c_b before their
    // FP32 rounding carry 2^-53 relative, covered by the margin
    const double c1 = 0x1.1p-22 * sqrt((double)D) * M * inv_h * 0.7071067811865476;
    const double c2 = (4.0 + D) * 0x1.0p-24;
    const double room = 0.5 * rho_max - 0x1.0p-17;
    abs_err = abs_dot = CUDART_INF;
    rho_dot = CUDART_INF;
    if (!(room > 0.0)) return CUDART_INF;
    {
        const double c1q = 0x1.1p-23 * sqrt((double)D) * Mq * inv_h * 0.7071067811865476;
        const double rs = (sqrt(rq2) + sqrt(rr2)) * inv_h;
        const double e = (D + 2.0) * 0x1.0p-24 * 0.5 * rs * rs * 1.01;
        const double rm = room - e;
        if (rm > 0.0) {
            const double sf = c1q > 0.0 ? rm / c1q : CUDART_INF;
            const double ac = fmin(fmin(a_max, 80.0), sf * sf * (1.0 - 0x1.0p-40));
            abs_dot = 0x1.0p-140;
            if (a_max > ac)
                abs_dot += 2.03 * wr * (double)ex2_approx((float)(-ac * 1.4426950408889634)) * 1.0001;
            rho_dot = 2.0 * (c1q * sqrt(ac) + e + 0x1.0p-17);
        }
    }
    const double sfit = 2.0 * room / (c1 + sqrt(c1 * c1 + 4.0 * c2 * room));
    const double a_c = fmin(fmin(a_max, 80.0), sfit * sfit * (1.0 - 0x1.0p-40));
    abs_err = 0x1.0p-140;
    if (a_max > a_c)
        abs_err += 2.03 * wr * (double)ex2_approx((float)(-a_c * 1.4426950408889634)) * 1.0001;
    return 2.0 * (c1 * sqrt(a_c) + c2 * a_c + 0x1.0p-17);
}

// Stream one converted window of n records (n a multiple of 4): the lane's two
// query slots form the packed pair, four records per iteration.
template <int D>
__device__ __forceinline__ void window_f32(const unsigned long long (&xf2)[D], const float *fst,
                                           int n, unsigned long long s2, double &sum0,
                                           double &sum1) {
    constexpr int F = fstride<D>();
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll 1
    for (int j = 0; j < n; j += 4) {
        float y[4][F];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int k = 0; k < F; k += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(fst + (j + u) * F + k);
                y[u][k] = v.x; y[u][k + 1] = v.y; y[u][k + 2] = v.z; y[u][k + 3] = v.w;
            }
        unsigned long long dd[4];
#pragma unroll
        for (int d = 0; d < D; d++)
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const unsigned long long f = f2_sub(xf2[d], f2_pack(y[u][d], y[u][d]));
                dd[u] = d == 0 ? f2_mul(f, f) : f2_fma(f, f, dd[u]);
            }
#pragma unroll
        for (int u = 0; u < 4; u++) dd[u] = f2_ex2(f2_mul(dd[u], s2));
#pragma unroll
        for (int u = 0; u < 4; u++) f2_fma_acc(acc[u], dd[u], f2_pack(y[u][D], y[u][D]));
    }
    sum0 = ((double)f2_lo(acc[0]) + (double)f2_lo(acc[1])) +
           ((double)f2_lo(acc[2]) + (double)f2_lo(acc[3]));
    sum1 = ((double)f2_hi(acc[0]) + (double)f2_hi(acc[1])) +
           ((double)f2_hi(acc[2]) + (double)f2_hi(acc[3]));
}

// cp.async the FP64 points of stream window [w0, w0 + f32_win) into `dst`:
// item t of the stream (lanes of `items`, in lane order) covers stream
// positions [off, off + cnt) and tree positions [start, start + cnt).
template <int D>
__device__ __forceinline__ void stage_window(const double *__restrict__ pw, unsigned items, int off,
                                             int cnt, int start, int w0, double *dst) {
    constexpr int S = packed_stride(D), W = f32_win<D>();
    const int lane = threadIdx.x & 31;
    const unsigned ov = __ballot_sync(kFull, ((items >> lane) & 1u) && off < w0 + W &&
                                                 off + cnt > w0);
    for (unsigned m = ov; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const int o = __shfl_sync(kFull, off, i);
        const int c = __shfl_sync(kFull, cnt, i);
        const int st = __shfl_sync(kFull, start, i);
        const int p0 = max(o, w0), p1 = min(o + c, w0 + W);
        for (int p = p0 + lane; p < p1; p += 32) {
            const double *src = pw + (int64_t)(st + p - o) * S;
            double *d = dst + (p - w0) * S;
#pragma unroll
            for (int q = 0; q < S / 2; q++) __pipeline_memcpy_async(d + 2 * q, src + 2 * q, 16);
        }
    }
    __pipeline_commit();
}

// FP64 window records -> FP32 records about c_b (y' = fl(y - c_b), fl(w)),
// one record per lane per pass; records [n, n4) become zero-weight padding.
template <int D>
__device__ __forceinline__ void convert_window(const double *raw, int n, int n4, const double *sqc,
                                               float *fst) {
    constexpr int S = packed_stride(D), F = fstride<D>();
    const int lane = threadIdx.x & 31;
    for (int r = lane; r < n4; r += 32) {
        float rec[F];
#pragma unroll
        for (int k = 0; k < F; k++) rec[k] = 0.f;
        if (r < n) {
            double y[D], w;
            read_point_w<D>(raw + r * S, y, w);
#pragma unroll
            for (int d = 0; d < D; d++) rec[d] = (float)(y[d] - sqc[d]);
            rec[D] = (float)w;
        }
#pragma unroll
        for (int k = 0; k < F; k += 4)
            *reinterpret_cast<float4 *>(fst + r * F + k) =
                make_float4(rec[k], rec[k + 1], rec[k + 2], rec[k + 3]);
    }
}

// Dot-form window: records {C_0..C_{D-1}, B, w} (dstride floats), lane
// query X (packed, both slots) and A_q (packed): t = (A_q + B) + sum X_d C_d.
template <int D>
__device__ __forceinline__ void window_dot(const unsigned long long (&xf2)[D],
                                           unsigned long long aq2, const float *fst, int n,
                                           double &sum0, double &sum1) {
    constexpr int F = dstride<D>();
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll 1
    for (int j = 0; j < n; j += 4) {
        float y[4][F];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int k = 0; k < F; k += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(fst + (j + u) * F + k);
                y[u][k] = v.x; y[u][k + 1] = v.y; y[u][k + 2] = v.z; y[u][k + 3] = v.w;
            }
        unsigned long long t[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            unsigned long long b2 = f2_pack(y[u][D], y[u][D]);
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t[u]) : "l"(aq2), "l"(b2));
        }
#pragma unroll
        for (int d = 0; d < D; d++)
#pragma unroll
            for (int u = 0; u < 4; u++) f2_fma_acc(t[u], xf2[d], f2_pack(y[u][d], y[u][d]));
#pragma unroll
        for (int u = 0; u < 4; u++) t[u] = f2_ex2(t[u]);
#pragma unroll
        for (int u = 0; u < 4; u++) f2_fma_acc(acc[u], t[u], f2_pack(y[u][D + 1], y[u][D + 1]));
    }
    sum0 = ((double)f2_lo(acc[0]) + (double)f2_lo(acc[1])) +
           ((double)f2_lo(acc[2]) + (double)f2_lo(acc[3]));
    sum1 = ((double)f2_hi(acc[0]) + (double)f2_hi(acc[1])) +
           ((double)f2_hi(acc[2]) + (double)f2_hi(acc[3]));
}

// FP64 window records -> dot-form records about c_b (s = log2(e) / 2h^2).
template <int D>
__device__ __forceinline__ void convert_window_dot(const double *raw, int n, int n4,
                                                   const double *sqc, double s, float *fst) {
    constexpr int S = packed_stride(D), F = dstride<D>();
    const int lane = threadIdx.x & 31;
    for (int r = lane; r < n4; r += 32) {
        float rec[F];
#pragma unroll
        for (int k = 0; k < F; k++) rec[k] = 0.f;
        if (r < n) {
            double y[D], w, q = 0.0;
            read_point_w<D>(raw + r * S, y, w);
#pragma unroll
            for (int d = 0; d < D; d++) {
                const double e = y[d] - sqc[d];
                q = fma(e, e, q);
                rec[d] = (float)(2.0 * s * e);
            }
            rec[D] = (float)(-s * q);
            rec[D + 1] = (float)w;
        }
#pragma unroll
        for (int k = 0; k < F; k += 4)
            *reinterpret_cast<float4 *>(fst + r * F + k) =
                make_float4(rec[k], rec[k + 1], rec[k + 2], rec[k + 3]);
    }
}

// query slot qi of a lane without dynamic register indexing (keeps the
// per-lane arrays out of local memory inside non-unrolled loops)
template <int D>
__device__ __forceinline__ void pick_query(const double (&x)[kQPL][D], int qi, double (&xq)[D]) {
#pragma unroll
    for (int d = 0; d < D; d++) xq[d] = qi ? x[1][d] : x[0][d];
}
__device__ __forceinline__ void add_slot(double (&acc)[kQPL], int qi, double v) {
    if (qi) acc[1] += v;
    else acc[0] += v;
}

__device__ __forceinline__ int warp_excl_scan(int v) {
    const int lane = threadIdx.x & 31;
    int s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, s, o);
        if (lane >= o) s += t;
    }
    return s - v;
}

static __constant__ Nest3Perm<engine_order_c(3)> c_nest3 = Nest3Perm<engine_order_c(3)>();

template <int D, int MINB, bool AUDIT>
__global__ void __launch_bounds__(kTravThreads, MINB)
traverse_kernel(const TravArgs A) {
    constexpr int S = packed_stride(D);
    extern __shared__ double smem[];
    __shared__ double s_tab[kExpTab];
    // staging permutation of the D = 3 Hermite items (graded-lex -> nested)
    __shared__ unsigned short s_nest[D == 3 ? ((Nest3Perm<engine_order_c(3)>::kTotal + 7) & ~7) : 8];
    exp_table_init(s_tab);
    if constexpr (D == 3)
        for (int i = threadIdx.x; i < Nest3Perm<engine_order_c(3)>::kTotal; i += blockDim.x)
            s_nest[i] = c_nest3.pos[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kTravWarps + wib;
    // per-warp shared memory: query box (lo, hi), centroid, local coefficients,
    // a double buffer of 2 x 32 staged FP64 reference points, then the FP32
    // batch (transposed records and per-group offsets)
    // (fixed-size parts first: every pointer below is sq + a compile-time
    // offset, so the kernel keeps one shared-memory base register)
    double *sq = smem + wib * (warp_fixed_doubles<D>() + ((A.K_loc + 1) & ~1));
    double *sqc = sq + 2 * D;
    double *sbuf = sq + ((3 * D + 1) & ~1);
    float *fst = reinterpret_cast<float *>(sbuf + stage_recs<D>() * S);
    int *itab = reinterpret_cast<int *>(fst + f32_cap<D>() * fstride<D>());  // offsets, counts
    float *idl = reinterpret_cast<float *>(itab + 64);                       // 32 x FD
    double *loc = sq + warp_fixed_doubles<D>();
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(
        sbuf + stage_recs<D>() * S + f32_smem_doubles<D>());
    unsigned mphase = 0;
    if (lane == 0) mbar_init(mbar, 1);
    __syncwarp();
    // query coordinates (D <= 4): sx[(d * kQPL + qi) * 32 + lane]
    double *sx = loc - xs_doubles<D>();
    int *sn = A.st_node + gw * A.stack_cap;
    double *skl = A.st_f + gw * A.stack_cap * 3;
    double *skh = skl + A.stack_cap;
    double *slb = skh + A.stack_cap;  // mass lower bound per unit weight (entry_bounds' lb)
    int2 *sl = A.ser_list + gw * A.stack_cap;
    const unsigned lt_mask = (1u << lane) - 1u;

    for (;;) {
        // task = (bandwidth j, query block b), bandwidth-major: a warp that
        // finishes early moves on to the next bandwidth's blocks, so only the
        // launch's last tasks form a tail
        long long t = 0;
        if (lane == 0) t = (long long)atomicAdd(A.work, 1ULL);
        t = __shfl_sync(kFull, t, 0);
        if (t >= A.nbl * A.nh) break;
        const int g = (int)(t / A.nbl);
        const int j = A.jord[g];
        long long b = (t - (long long)g * A.nbl) * A.stride + A.b0;
        // single full runs visit blocks in the given order (heaviest first,
        // from the previous run's measured costs): shortens the tail
        if (A.order) b = __ldg(A.order + b);
        const TravH &H = A.hp[j];

        const long long t_start = clock64();
#if FG_PHASE_PROF
        unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long ph_t = t_start;
#define PH_MARK(k)                           \
    do {                                     \
        const long long ph_n = clock64();    \
        ph[k] += (unsigned long long)(ph_n - ph_t); \
        ph_t = ph_n;                         \
    } while (0)
#else
#define PH_MARK(k) \
    do {           \
    } while (0)
#endif
        unsigned steps = 0;
        const int2 rg = A.qb_range[b];
        const int qs = rg.x, qn = rg.y;
        FG_CHECK(qn >= 1 && qn <= kQBlock && qs >= 0);
        const int nq = qn > 32 ? 2 : 1;  // query slots in use (warp-uniform)
        bool valid[kQPL];
        if (lane < 2 * D) sq[lane] = A.qb_box[b * 2 * D + lane];
        if (lane < D) sqc[lane] = A.qb_c[b * D + lane];
        if (A.use_series)
            for (int k = lane; k < A.K_loc; k += 32) loc[k] = 0.0;
        __syncwarp();
        double xr[xs_smem<D>() ? 1 : kQPL][D];  // query coordinates in registers (D >= 5)
#pragma unroll
        for (int qi = 0; qi < kQPL; qi++) {
            valid[qi] = lane + 32 * qi < qn;
            double xq[D];
            if (valid[qi]) load_point<D>(A.q_pw + (int64_t)(qs + lane + 32 * qi) * S, xq);
            else {
#pragma unroll
                for (int d = 0; d < D; d++) xq[d] = sqc[d];
            }
#pragma unroll
            for (int d = 0; d < D; d++) {
                if constexpr (xs_smem<D>()) sx[(d * kQPL + qi) * 32 + lane] = xq[d];
                else xr[qi][d] = xq[d];
            }
        }
        // the lane's query coordinates, wherever they live
        auto get_x = [&](double (&xx)[kQPL][D]) {
#pragma unroll
            for (int qi = 0; qi < kQPL; qi++)
#pragma unroll
                for (int d = 0; d < D; d++) {
                    if constexpr (xs_smem<D>()) xx[qi][d] = sx[(d * kQPL + qi) * 32 + lane];
                    else xx[qi][d] = xr[xs_smem<D>() ? 0 : qi][d];
                }
        };
        double pt_est[kQPL], pt_mass[kQPL];  // per point
#pragma unroll
        for (int qi = 0; qi < kQPL; qi++) pt_est[qi] = pt_mass[qi] = 0.0;
        double lane_est = 0.0;  // this lane's share of the node-level estimates
        // lower bound on G for every query of the block known up front: in a
        // monochromatic run each query's own term (w_q K(0) = w_q)
        // and the block's own points: G(x_q) >= W_block exp(-diam^2 / 2h^2)
        double gfloor = 0.0;
        if (A.qb_wmin) {
            double dsq = 0.0;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const double e = sq[D + d] - sq[d];
                dsq += e * e;
            }
            gfloor = fmax(A.qb_wmin[b],
                          A.qb_wsum[b] * fg_exp_fast(dsq * H.neg_inv, s_tab) * (1.0 - 1e-12));
        }
        double tokens = 0.0;    // per block (uniform)
        unsigned c_vis = 0, c_base = 0, c_fd = 0;
        unsigned long long c_pairs = 0, c_f32 = 0;  // up to 64 x N_ref per task
        int nh = 0, no = 0;  // deferred series items: Hermite from the front, others from the back

        // root entry
        // mass = settled lower bounds + sum over the frontier of W_R * K_lo (uniform)
        double mass;
        // Frontier: circular buffer [head, head + cnt) of capacity stack_cap.
        // Breadth-first (pop the oldest entries) while it holds fewer than
        // bfs_cap entries, so the frontier's K_lo bound tightens everywhere
        // before any region is explored to the leaves; depth-first (pop the
        // newest) beyond that, which bounds its size.
        int head = 0, cnt = 1;
        const int cap = A.stack_cap;
        // far-field pass results of the block's super-node (fg_far_kernel.cuh)
        int far = 0;
        long long ft = 0;
        double far_est = 0.0;
        if (A.far_flag) {
            ft = (long long)j * A.nsn + __ldg(A.qb_super + b);
            far = A.far_flag[ft];
        }
        if (far) {
            // inherit S's leftover tokens, settled mass and node-level estimate;
            // start from S's residual entries, bounded against this block's box
            tokens = A.far_tokens[ft];
            far_est = A.far_est[ft];
            const int nr = A.far_rcnt[ft];
            FG_CHECK(nr >= 0 && nr <= kFarResCapT && nr <= cap);
            const int *res = A.far_res + ft * kFarResCapT;
            double lm = 0.0;
            for (int i = lane; i < nr; i += 32) {
                const int nd = __ldg(res + i);
                double klo, khi, lb;
                entry_bounds<D>(A, sq, nd, H.neg_inv, klo, khi, lb, s_tab);
                sn[i] = nd;
                skl[i] = klo;
                skh[i] = khi;
                slb[i] = lb;
                lm += A.r_wr[nd].x * lb;
            }
            cnt = nr;
            mass = A.far_settled[ft] + warp_sum(lm);
        } else {
            double klo, khi, lb;
            entry_bounds<D>(A, sq, 0, H.neg_inv, klo, khi, lb, s_tab);
            if (lane == 0) {
                sn[0] = 0;
                skl[0] = klo;
                skh[0] = khi;
                slb[0] = lb;
            }
            mass = A.r_wr[0].x * lb;
        }
        __syncwarp();

        PH_MARK(7);
        while (cnt > 0) {
            const int nb = min(cnt, 32);
            steps++;
            int base;
            if (cnt <= A.bfs_cap) {
                base = head;
                head = head + nb >= cap ? head + nb - cap : head + nb;
            } else {
                base = head + cnt - nb;
                if (base >= cap) base -= cap;
            }
            cnt -= nb;
            const bool act = lane < nb;
            int node = 0;
            double klo = 0.0, khi = 0.0, lb = 0.0;
            int4 ni = make_int4(0, 0, -1, -1);
            double2 wr = make_double2(0.0, 0.0);
            if (act) {
                int slot = base + lane;
                if (slot >= cap) slot -= cap;
                FG_CHECK(slot >= 0 && slot < cap);
                node = sn[slot];
                klo = skl[slot];
                khi = skh[slot];
                lb = slb[slot];
                ni = A.r_ni[node];
                wr = A.r_wr[node];
            }
            __syncwarp();
            const double WR = wr.x;
            c_vis += nb;
            const double pmin = warp_min(fmin(valid[0] ? pt_mass[0] : CUDART_INF,
                                              valid[1] ? pt_mass[1] : CUDART_INF));
            const double gmin = fmax((pmin + mass) * kMassSafety, gfloor);

            // ---- finite-difference prune (summation_engine.py:327-351)
            // finite difference over [lb, K_hi] (lb >= K_lo: the Jensen bound of
            // entry_bounds; every query's contribution lies in W_R [lb, K_hi])
            const double fd_err = 0.5 * WR * (khi - lb);
            // W / (eps G_min): one uniform division per step instead of one per entry
            const double den = H.eps * gmin;
            const double tok_scale = den > 0.0 ? A.total_w / den : CUDART_INF;
            const double err_scale = den / A.total_w;  // eps G_min / W
            const double req = required_tokens(WR, fd_err, tok_scale);
            unsigned fd_mask;
            if (A.use_tokens) fd_mask = admit(act, req, tokens);
            else fd_mask = __ballot_sync(kFull, act && req <= 0.0);
            const bool fd = (fd_mask >> lane) & 1u;
            c_fd += __popc(fd_mask);
            if constexpr (AUDIT)
                audit_append(A, fd_mask, 1, (int)b, (int)steps, WR, fd_err, gmin, req);
            double settled = 0.0, est_add = 0.0;
            if (fd) {
                settled = WR * lb;
                est_add = 0.5 * WR * (lb + khi);
            }

            PH_MARK(0);
            // ---- series prunes (summation_engine.py:352-399); the evaluation
            // itself is deferred to the end of the block (it never feeds a bound)
            unsigned ser_mask = 0;
            if (A.use_series && nh + no + 32 <= A.stack_cap) {
                int meth = 0, p = 0;
                double bound = 0.0;
                if (act && !fd) {
                    const double maxerr = (WR + tokens) * err_scale;
                    const double r_ref = wr.y * H.inv_h;
                    const double r_qu = A.qb_rad[b] * H.inv_h;
                    const double rmin = r_ref < r_qu ? r_ref : r_qu;
                    // W_R exp(-min_sq / 4h^2) = W_R sqrt(K_hi), bounded above from
                    // this engine's K_hi (<= 2.4e-14 relative error when normal,
                    // <= 2^-1074 absolute when subnormal)
                    const double base = WR * sqrt(khi + 0x1.0p-1073) * (1.0 + 0x1.0p-40);
                    double possible = base * A.floor_c;
                    if (rmin < 1.0) {
                        double pw = 1.0;
                        for (int k = 0; k < A.plimit; k++) pw *= rmin;
                        possible *= pw;
                    }
                    if (possible <= maxerr)
                        select_method_gpu(base, r_ref, r_qu, (double)ni.y, D, maxerr, A.plimit,
                                          A.plimit_loc, A.ct, A.cross, A.kp, (double)nq, H.pair_cost, H.herm_c0, H.herm_c1, meth, p,
                                          bound);
                }
                const bool cand = meth != 0;
                const double sreq = cand ? required_tokens(WR, bound, tok_scale)
                                         : CUDART_INF;
                ser_mask = admit(cand, sreq, tokens);
                if constexpr (AUDIT)
                    audit_append(A, ser_mask, meth, (int)b, (int)steps, WR, bound, gmin, sreq);
                const unsigned hm = __ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 2);
                const unsigned om = ser_mask & ~hm;
                if ((ser_mask >> lane) & 1u) {
                    settled = WR * lb;
                    const int slot = meth == 2 ? nh + __popc(hm & lt_mask)
                                               : A.stack_cap - 1 - no - __popc(om & lt_mask);
                    FG_CHECK(slot >= nh && slot < A.stack_cap && nh + no + 32 <= A.stack_cap);
                    sl[slot] = make_int2(node, p | (meth << 8));
                }
                nh += __popc(hm);
                no += __popc(om);
            }
            lane_est += est_add;

            PH_MARK(1);
            // ---- descend or evaluate exactly (summation_engine.py:400-426)
            const bool rem = act && !fd && !((ser_mask >> lane) & 1u);
#ifndef FG_EDGE_SPLIT
#define FG_EDGE_SPLIT 64
#endif
#ifndef FG_EDGE_MIN
#define FG_EDGE_MIN 32
#endif
            bool leafy = ni.z < 0 || ni.y <= H.ref_leaf;
            // an item whose finite-difference error is within a small factor of
            // what its own weight pays straddles the kernel's cut-off: its
            // children are likely prunable, so it is split instead of evaluated
            // (D <= 4, measured: C5 -1.0 % at factor 64; at D >= 5 it costs 4-10 %)
            if (FG_EDGE_SPLIT > 0 && !f32_direct<D>() && leafy && ni.z >= 0 && ni.y > FG_EDGE_MIN &&
                fd_err * tok_scale <= (double)FG_EDGE_SPLIT * WR)
                leafy = false;
            unsigned split_mask = __ballot_sync(kFull, rem && !leafy);
            unsigned base_mask = __ballot_sync(kFull, rem && leafy);
            if (cnt + 2 * __popc(split_mask) > cap) {
                // frontier capacity reached: settle these exactly (always admissible)
                base_mask |= split_mask;
                split_mask = 0;
            }
            double child_sum = 0.0;
            if ((split_mask >> lane) & 1u) {
                const int pos = head + cnt + 2 * __popc(split_mask & lt_mask);
#pragma unroll 1
                for (int c = 0; c < 2; c++) {
                    const int ch = c == 0 ? ni.z : ni.w;
                    double cl, chh, cm;
                    entry_bounds<D>(A, sq, ch, H.neg_inv, cl, chh, cm, s_tab);
                    int slot = pos + c;
                    if (slot >= cap) slot -= cap;
                    if (slot >= cap) slot -= cap;
                    FG_CHECK(slot >= 0 && slot < cap && cnt + 2 * __popc(split_mask) <= cap);
                    sn[slot] = ch;
                    skl[slot] = cl;
                    skh[slot] = chh;
                    slb[slot] = cm;
                    child_sum += A.r_wr[ch].x * cm;
                }
            }
            cnt += 2 * __popc(split_mask);
            // one reduction per step: popped entries leave the frontier, settled
            // ones and pushed children enter the mass bound (base cases move
            // into the per-point exact sums)
#if FG_DEFER_CREDIT
            // experiment: base items credit only their W_R lb (as a deferred
            // evaluation would); their exact sums do not feed G_min
            if ((base_mask >> lane) & 1u) settled = WR * lb;
#endif
            mass += warp_sum(settled + child_sum - (act ? WR * lb : 0.0));
            if (mass < 0.0) mass = 0.0;

            PH_MARK(2);
            // ---- exhaustive base cases, eager (dito_base, :221-250).  Items whose
            // FP32 error bound fits (decided lane-parallel, one item per lane) run
            // as one FP32 batch; the rest (FP64) are staged one by one into shared
            // memory with cp.async, double-buffered so the next item's points load
            // while this one computes (leaves of > 64 points read global memory).
            // anchored batches take items inside one anchor; the direct stream any item
            const unsigned small_mask =
                f32_direct<D>() ? base_mask : __ballot_sync(kFull, ni.y <= kAnchorMax) & base_mask;
            unsigned f32_mask = 0;
            int anc = 0;
            bool pdiff = false;  // anchored item streamed in the difference form
            double abs32 = 0.0;
            bool dot_step = false;
            if (H.fp32_rho > 0.0 && small_mask && tok_scale < CUDART_INF) {
                bool use = false, use_dot = false;
                double abs_dot_l = 0.0;
                if ((small_mask >> lane) & 1u) {
                    double rho;
                    if constexpr (f32_direct<D>()) {
                        double rho_dot, abs_dot;
                        rho = fp32_node_bound<D>(A, sq, node, H.inv_h, klo, WR, H.fp32_rho, abs32,
                                                 rho_dot, abs_dot);
                        use_dot = rho_dot <= H.fp32_rho && abs_dot * tok_scale <= WR &&
                                  g_dot_form;
                        if (use_dot) abs_dot_l = abs_dot;
                    } else {
                        anc = __ldg(A.r_anchor + ni.x);
#if FG_PAIR_DOT
                        rho = fp32_pair_bound<D>(A, sq, anc, node, H.inv_h, klo, WR, H.fp32_rho,
                                                 abs32);
                        if (FG_PAIR_DIFF && !(rho <= H.fp32_rho && abs32 * tok_scale <= WR)) {
                            // the difference form from the same records
                            rho = fp32_item_bound<D>(A, sq, anc, H.inv_h, klo, WR, H.fp32_rho,
                                                     abs32);
                            pdiff = true;
                        }
#else
                        rho = fp32_item_bound<D>(A, sq, anc, H.inv_h, klo, WR, H.fp32_rho, abs32);
#endif
                    }
                    use = rho <= H.fp32_rho && abs32 * tok_scale <= WR;
                }
                f32_mask = __ballot_sync(kFull, use);
                if constexpr (f32_direct<D>()) {
                    // the dot form when every eligible item admits it
                    const unsigned dm = __ballot_sync(kFull, use_dot);
                    dot_step = dm != 0u && (dm | f32_mask) == dm;
                    if (dot_step) {
                        f32_mask = dm;
                        abs32 = abs_dot_l;
                    }
                }
            }
            if constexpr (AUDIT) {
                // FP32 items charge their absolute error part to the tokens
                audit_append(A, f32_mask, 0, (int)b, (int)steps, WR, abs32, gmin,
                             abs32 * tok_scale - WR);
                audit_append(A, base_mask & ~f32_mask, 0, (int)b, (int)steps, WR, 0.0, gmin, -WR);
            }
            PH_MARK(3);
            if (f32_direct<D>() && f32_mask) {
                const bool mine = (f32_mask >> lane) & 1u;
                const int rcm = mine ? ni.y : 0;
                const int off = warp_excl_scan(rcm);
                const int total = __shfl_sync(kFull, off + rcm, 31);
                // the first window's copy is in flight during the bookkeeping
                stage_window<D>(A.r_pw, f32_mask, off, rcm, ni.x, 0, sbuf);
                if (A.use_tokens) tokens += warp_sum(mine ? WR - abs32 * tok_scale : 0.0);
                const double abs_sum = warp_sum(mine ? abs32 : 0.0);
                c_f32 += (unsigned long long)qn * (unsigned)total;
                c_base += __popc(f32_mask);
                // both query slots about the block centroid, packed (slot 0, slot 1)
                unsigned long long xf2[D];
                {
                    double x[kQPL][D];
                    get_x(x);
#pragma unroll
                    for (int d = 0; d < D; d++)
                        xf2[d] = f2_pack((float)(x[0][d] - sqc[d]), (float)(x[1][d] - sqc[d]));
                }
                const unsigned long long s2 = f2_pack(H.ex2_scale, H.ex2_scale);
                // dot form: per-slot A_q = fl(-s |X|^2) from the FP32 offsets X
                const double sdot = -H.neg_inv * 1.4426950408889634;
                unsigned long long aq2 = 0ull;
                if (dot_step) {
                    double q0 = 0.0, q1 = 0.0;
#pragma unroll
                    for (int d = 0; d < D; d++) {
                        const double e0 = f2_lo(xf2[d]), e1 = f2_hi(xf2[d]);
                        q0 = fma(e0, e0, q0);
                        q1 = fma(e1, e1, q1);
                    }
                    aq2 = f2_pack((float)(-sdot * q0), (float)(-sdot * q1));
                }
                double sum32[kQPL] = {0.0, 0.0};
                int wb = 0;
                constexpr int W = f32_win<D>();
                for (int w0 = 0; w0 < total; w0 += W) {
                    // the next window's copy overlaps this window's conversion + math
                    if (w0 + W < total)
                        stage_window<D>(A.r_pw, f32_mask, off, rcm, ni.x, w0 + W,
                                        sbuf + (wb ^ 1) * W * S);
                    else
                        __pipeline_commit();
                    __pipeline_wait_prior(1);
                    __syncwarp();
                    const int n = min(W, total - w0), n4 = (n + 3) & ~3;
                    double s0, s1;
                    if (dot_step) {
                        convert_window_dot<D>(sbuf + wb * W * S, n, n4, sqc, sdot, fst);
                        __syncwarp();
                        window_dot<D>(xf2, aq2, fst, n4, s0, s1);
                    } else {
                        convert_window<D>(sbuf + wb * W * S, n, n4, sqc, fst);
                        __syncwarp();
                        window_f32<D>(xf2, fst, n4, s2, s0, s1);
                    }
                    sum32[0] += s0;
                    sum32[1] += s1;
                    __syncwarp();
                    wb ^= 1;
                }
#pragma unroll
                for (int qi = 0; qi < kQPL; qi++) {
                    pt_est[qi] += sum32[qi];
                    if (!FG_DEFER_CREDIT) pt_mass[qi] += fmax(sum32[qi] * (1.0 - H.fp32_rho) - abs_sum, 0.0);
                }
            }
#if FG_PAIR_DOT
            if (!f32_direct<D>() && f32_mask) {
                // anchored dot-form batch from record pairs: each item's pair range
                // lands in shared memory with ONE bulk copy issued by its own lane
                constexpr int CAPP = pair_cap<D>(), FD = f32_fd<D>(), P = pstride<D>();
                static_assert(f32_direct<D>() || CAPP >= kAnchorMax / 2 + 1,
                              "one item must fit the pair staging");
                const bool mine = (f32_mask >> lane) & 1u;
                const int p0 = ni.x >> 1, p1 = (ni.x + ni.y + 1) >> 1;
                const int np = mine ? p1 - p0 : 0;
                const int off = warp_excl_scan(np);
                float dl[D];
                if (mine) {
#pragma unroll
                    for (int d = 0; d < D; d++)
                        dl[d] = (float)(__ldg(A.r_c + (int64_t)anc * D + d) - sqc[d]);
                }
                if (A.use_tokens) tokens += warp_sum(mine ? WR - abs32 * tok_scale : 0.0);
                const double abs_sum = warp_sum(mine ? abs32 : 0.0);
                c_f32 += (unsigned long long)qn * (unsigned)warp_sum(mine ? ni.y : 0);
                c_base += __popc(f32_mask);
                float xs[kQPL][D];
                {
                    double x[kQPL][D];
                    get_x(x);
#pragma unroll
                    for (int q = 0; q < kQPL; q++)
#pragma unroll
                        for (int d = 0; d < D; d++) xs[q][d] = (float)(x[q][d] - sqc[d]);
                }
                float *pbuf = reinterpret_cast<float *>(sbuf);
                const double sdot = -H.neg_inv * 1.4426950408889634;
                double sum32[kQPL] = {0.0, 0.0};
                unsigned todo = f32_mask;
                while (todo) {
                    // the next run of whole items that fits the staging area
                    const int base = __shfl_sync(kFull, off, __ffs(todo) - 1);
                    const bool in = ((todo >> lane) & 1u) && off - base + np <= CAPP;
                    const unsigned batch = __ballot_sync(kFull, in);
                    todo &= ~batch;
                    const int bytes = warp_sum(in ? np * P * 4 : 0);
                    if (in) {
                        const int t = __popc(batch & lt_mask);
                        itab[t] = off - base;
                        itab[32 + t] = np | (pdiff ? kPairDiff : 0);
#pragma unroll
                        for (int d = 0; d < D; d++) idl[t * FD + d] = dl[d];
                    }
                    // earlier generic accesses of the staging bytes before the
                    // async-proxy writes; lane 0 arms the warp's barrier
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_expect_tx(mbar, (unsigned)bytes);
                    __syncwarp();
                    FG_CHECK(!in || (off - base >= 0 && off - base + np <= CAPP && np >= 1 &&
                                     np <= kAnchorMax / 2 + 1));
                    if (in)
                        bulk_g2s(pbuf + (off - base) * P, A.r_pf + (int64_t)p0 * P,
                                 (unsigned)(np * P * 4), mbar);
                    mbar_wait(mbar, mphase);
                    mphase ^= 1u;
                    // the foreign half of a first / last pair carries weight 0
                    if (in) {
                        if (ni.x & 1) pbuf[(off - base) * P + 2 * D + 2] = 0.f;
                        if ((ni.x + ni.y) & 1) pbuf[(off - base + np - 1) * P + 2 * D + 3] = 0.f;
                    }
                    __syncwarp();
                    batch_pairs<D>(xs, pbuf, itab, itab + 32, idl, __popc(batch), sdot, sum32[0],
                                   sum32[1]);
                    __syncwarp();
                }
#pragma unroll
                for (int qi = 0; qi < kQPL; qi++) {
                    pt_est[qi] += sum32[qi];
                    // |sum32 - S| <= rho S + sum(abs) with rho <= fp32_rho
                    if (!FG_DEFER_CREDIT) pt_mass[qi] += fmax(sum32[qi] * (1.0 - H.fp32_rho) - abs_sum, 0.0);
                }
            }
#else
            if (!f32_direct<D>() && f32_mask) {
                constexpr int CAP = f32_cap<D>(), FD = f32_fd<D>(), F = fstride<D>();
                const bool mine = (f32_mask >> lane) & 1u;
                const int rcm = mine ? ni.y : 0;
                const int off = warp_excl_scan(rcm);
                float dl[D];
                if (mine) {
#pragma unroll
                    for (int d = 0; d < D; d++)
                        dl[d] = (float)(__ldg(A.r_c + (int64_t)anc * D + d) - sqc[d]);
                }
                if (A.use_tokens) tokens += warp_sum(mine ? WR - abs32 * tok_scale : 0.0);
                const double abs_sum = warp_sum(mine ? abs32 : 0.0);
                c_f32 += (unsigned long long)qn * (unsigned)warp_sum(rcm);
                c_base += __popc(f32_mask);
                // both query slots about the block centroid, packed (slot 0, slot 1)
                unsigned long long xf2[D];
                {
                    double x[kQPL][D];
                    get_x(x);
#pragma unroll
                    for (int d = 0; d < D; d++)
                        xf2[d] = f2_pack((float)(x[0][d] - sqc[d]), (float)(x[1][d] - sqc[d]));
                }
                double sum32[kQPL] = {0.0, 0.0};
                unsigned todo = f32_mask;
                while (todo) {
                    // the next run of whole items that fits the staging area
                    const int base = __shfl_sync(kFull, off, __ffs(todo) - 1);
                    const unsigned batch =
                        __ballot_sync(kFull, ((todo >> lane) & 1u) && off - base + rcm <= CAP);
                    todo &= ~batch;
                    if ((batch >> lane) & 1u) {
                        const int t = __popc(batch & lt_mask);
                        itab[t] = off - base;
                        itab[32 + t] = rcm;
#pragma unroll
                        for (int d = 0; d < D; d++) idl[t * FD + d] = dl[d];
                    }
                    for (unsigned m = batch; m; m &= m - 1) {
                        const int i = __ffs(m) - 1;
                        const int rs = __shfl_sync(kFull, ni.x, i);
                        const int rc = __shfl_sync(kFull, ni.y, i);
                        const int o = __shfl_sync(kFull, off, i) - base;
                        for (int l = lane; l < rc; l += 32) {
                            const float *src = A.r_pf + (int64_t)(rs + l) * F;
                            float *dst = fst + (o + l) * F;
#pragma unroll
                            for (int k = 0; k < F; k += 4) __pipeline_memcpy_async(dst + k, src + k, 16);
                        }
                    }
                    __pipeline_commit();
                    __pipeline_wait_prior(0);
                    __syncwarp();
                    double s0, s1;
                    batch_f32<D>(xf2, fst, itab, itab + 32, idl, __popc(batch), H.ex2_scale, s0, s1);
                    sum32[0] += s0;
                    sum32[1] += s1;
                    __syncwarp();
                }
#pragma unroll
                for (int qi = 0; qi < kQPL; qi++) {
                    pt_est[qi] += sum32[qi];
                    // |sum32 - S| <= rho S + sum(abs) with rho <= fp32_rho, so
                    // sum32 (1 - fp32_rho) - sum(abs) <= S
                    if (!FG_DEFER_CREDIT) pt_mass[qi] += fmax(sum32[qi] * (1.0 - H.fp32_rho) - abs_sum, 0.0);
                }
            }
#endif
            PH_MARK(4);
            const unsigned base64 = base_mask & ~f32_mask;
            const unsigned small64 = __ballot_sync(kFull, ni.y <= kStageMax) & base_mask & ~f32_mask;
            int bi = 0;
            if (small64) stage_points<D>(A.r_pw, ni.x, ni.y, __ffs(small64) - 1, sbuf);
            for (unsigned m = base64; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const int rs = __shfl_sync(kFull, ni.x, i);
                const int rc = __shfl_sync(kFull, ni.y, i);
                const double wri = __shfl_sync(kFull, WR, i);
                // every pair of this item has K >= K_lo: skip the exp range test
                // when K_lo is a normal number
                const double kli = __shfl_sync(kFull, klo, i);
                double contrib[kQPL] = {0.0, 0.0};
                if ((small64 >> i) & 1u) {
                    const unsigned rest = small64 & ~((2u << i) - 1u);
                    if (stage_db<D>() && rest) {
                        stage_points<D>(A.r_pw, ni.x, ni.y, __ffs(rest) - 1,
                                        sbuf + (bi ^ 1) * kStageMax * S);
                        __pipeline_wait_prior(1);
                    } else {
                        __pipeline_wait_prior(0);
                    }
                    __syncwarp();
                    const double *bp = sbuf + bi * kStageMax * S;
                    double x[kQPL][D];
                    get_x(x);
                    if (nq == 2) {
                        if (kli >= 2.3e-308)
                            base_case2<D, false>(x, bp, rc, H.neg_inv, s_tab, contrib[0], contrib[1]);
                        else
                            base_case2<D, true>(x, bp, rc, H.neg_inv, s_tab, contrib[0], contrib[1]);
                    } else {
                        contrib[0] = kli >= 2.3e-308 ? base_case<D, false>(x[0], bp, rc, H.neg_inv, s_tab)
                                                     : base_case<D, true>(x[0], bp, rc, H.neg_inv, s_tab);
                    }
                    __syncwarp();
                    if constexpr (stage_db<D>()) {
                        bi ^= 1;
                    } else if (rest) {  // single buffer: stage the next item now
                        stage_points<D>(A.r_pw, ni.x, ni.y, __ffs(rest) - 1, sbuf);
                    }
                } else {
                    const double *rp = A.r_pw + (int64_t)rs * S;
                    double x[kQPL][D];
                    get_x(x);
#pragma unroll 1
                    for (int qi = 0; qi < nq; qi++) {
                        double xq[D];
                        pick_query<D>(x, qi, xq);
                        add_slot(contrib, qi, base_case<D, true>(xq, rp, rc, H.neg_inv, s_tab));
                    }
                }
#pragma unroll
                for (int qi = 0; qi < kQPL; qi++) {
                    pt_est[qi] += contrib[qi];
                    if (!FG_DEFER_CREDIT) pt_mass[qi] += contrib[qi];
                }
                if (A.use_tokens) tokens += wri;
                c_base++;
                c_pairs += (unsigned long long)(qn * rc);
            }
            PH_MARK(5);
        }

        // ---- deferred series contributions, then the post pass (dito_post, :253-281)
        unsigned c_dh = 0, c_dl = 0, c_h2l = 0;
        unsigned long long c_hq = 0, c_lq = 0, c_ht = 0;
        bool local_used = false;
        if (far & 2) {
            // S.local pushed down to this block's centre (translate_l2l,
            // series_expansion.py:197-217), the block's own local terms added below
            l2l_warp_add<D>(A.far_loc + ft * A.K_loc,
                            A.q_c + (int64_t)__ldg(A.sn_node + __ldg(A.qb_super + b)) * D, sqc,
                            A.plimit_loc, A.K_loc, H.sc, A.digits, loc);
            __syncwarp();
            local_used = true;
        }
        if (nh + no > 0 || local_used) {
            double x[kQPL][D];
            get_x(x);
            double qc[D];
#pragma unroll
            for (int d = 0; d < D; d++) qc[d] = sqc[d];
            // Hermite items (EVALM): each item's moments and centre are staged
            // through a cp.async ring in the (now idle) FP64 staging buffer,
            // kRing - 1 items ahead of the one being evaluated
            constexpr int PF = engine_order_c(D);
            // D = 3: items are staged in the nested layout of their own order
            // (fg_series.cuh, the row machine: 16-byte coefficient loads); other
            // dimensions keep the graded-lex prefix
            const int slot = D == 3 ? nest3_slot(A.plimit) : (A.K + D + 1) & ~1;
            const int coff = D == 3 ? slot - 4 : A.K;  // the centre inside a slot
            // ring depth: 4 items, 2 for the 512-double slots of orders 11, 12
            const int kRing = D == 3 && slot > 256 ? 2 : 4;
            // the ring may run over the FP32 record area behind the FP64 staging
            // buffer (contiguous at D <= 4, idle after the traversal loop)
            constexpr int kRingDoubles =
                stage_recs<D>() * S + (f32_direct<D>() ? 0 : f32_cap<D>() * fstride<D>() / 2);
            const bool ring = A.plimit <= PF && kRing * slot <= kRingDoubles;
            auto stage_item = [&](int k) {
                const int2 e = sl[k];
                const int node = e.x, po = e.y & 0xff, kc = A.kp[po];  // the item's own order
                double *dst = sbuf + (k & (kRing - 1)) * slot;
                const double *mom = H.r_mom + (int64_t)node * A.mom_K;
                if constexpr (D == 3) {
                    const unsigned short *perm = s_nest + c_nest3.off[po];
                    // four positions per round: the permutation loads overlap
                    for (int q = lane; q < kc; q += 128) {
                        int pos[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) pos[u] = q + 32 * u < kc ? perm[q + 32 * u] : -1;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            FG_CHECK(po >= 1 && po <= PF && pos[u] < coff && kc <= A.mom_K);
                            if (pos[u] >= 0)
                                __pipeline_memcpy_async(dst + pos[u], mom + q + 32 * u, 8);
                        }
                    }
                } else {
                    for (int q = lane; q < kc; q += 32) __pipeline_memcpy_async(dst + q, mom + q, 8);
                }
                if (lane < D) __pipeline_memcpy_async(dst + coff + lane, A.r_c + (int64_t)node * D + lane, 8);
            };
            if (ring) {
#pragma unroll 1
                for (int k = 0; k < kRing - 1; k++) {
                    if (k < nh) stage_item(k);
                    __pipeline_commit();
                }
            }
            int p_next = nh > 0 ? sl[0].y & 0xff : 0;
            for (int i = 0; i < nh; i++) {
                const int p = p_next;
                // (the next entry's order is loaded one evaluation ahead)
                if (i + 1 < nh) p_next = sl[i + 1].y & 0xff;
                c_ht += (unsigned long long)A.kp[p] * qn;
                if (ring) {
                    if (i + kRing - 1 < nh) stage_item(i + kRing - 1);
                    __pipeline_commit();
                    if (kRing == 4) __pipeline_wait_prior(3);
                    else __pipeline_wait_prior(1);
                    __syncwarp();
                    const double *buf = sbuf + (i & (kRing - 1)) * slot;
                    if constexpr (D == 3) {
                        // the item's own order, both query slots from one pass
                        // over the coefficients (an unused slot holds the centroid)
                        double ta[3], tb[3], qa = 0.0, qb = 0.0;
#pragma unroll
                        for (int d = 0; d < 3; d++) {
                            const double c = buf[coff + d];
                            ta[d] = (x[0][d] - c) * H.inv_sc;
                            tb[d] = (x[1][d] - c) * H.inv_sc;
                            qa = fma(ta[d], ta[d], qa);
                            qb = fma(tb[d], tb[d], qb);
                        }
                        const double ga = fg_exp_fast(-qa, s_tab), gb = fg_exp_fast(-qb, s_tab);
                        double2 v;
#ifndef FG_FAR3_CALL
#define FG_FAR3_CALL 1
#endif
                        if constexpr (FG_FAR3_CALL)
                            v = far3_rows_cl_call<PF>(p, ta[0], ta[1], ta[2], tb[0], tb[1], tb[2],
                                                      (int)(buf - smem));
                        else
                            far3_rows_cl<PF>(p, ta, tb, buf, v.x, v.y);
                        // (no inf * 0 for absurdly distant centres)
                        pt_est[0] += ga == 0.0 ? 0.0 : v.x * ga;
                        pt_est[1] += gb == 0.0 ? 0.0 : v.y * gb;
                    } else {
#pragma unroll 1
                        for (int qi = 0; qi < nq; qi++) {
                            double xq[D];
                            pick_query<D>(x, qi, xq);
                            add_slot(pt_est, qi,
                                     eval_far_fixed<D, PF>(xq, buf + A.K, buf, p, H.inv_sc,
                                                           [&](double v) { return fg_exp_fast(v, s_tab); }));
                        }
                    }
                    __syncwarp();
                } else {
                    const int node = sl[i].x;
#pragma unroll 1
                    for (int qi = 0; qi < nq; qi++) {
                        double xq[D];
                        pick_query<D>(x, qi, xq);
                        add_slot(pt_est, qi,
                                 eval_far_lane<D>(xq, A.r_c + (int64_t)node * D,
                                                  H.r_mom + (int64_t)node * A.mom_K, p, A.kp[p],
                                                  H.sc, A.digits));
                    }
                }
            }
            c_dh += nh;
            c_hq += (unsigned long long)nh * qn;
            // direct-local and H2L items accumulate into the block's local expansion
            for (int k = 0; k < no; k++) {
                const int2 e = sl[A.stack_cap - 1 - k];
                const int meth = e.y >> 8, p = e.y & 0xff;
                if (meth == 3) {
                    const int4 ni = A.r_ni[e.x];
                    accumulate_warp<D, kLocK / 32>(1, A.r_pw, ni.x, (int64_t)ni.x + ni.y, qc, p, A.kp[p], H.sc,
                                       A.digits, A.inv_fact, loc, false);
                    c_dl++;
                } else {
                    h2l_warp_add<D>(H.r_mom + (int64_t)e.x * A.mom_K, A.r_c + (int64_t)e.x * D, qc,
                                    p, A.kp[p], p, A.kp[p], H.sc, A.digits, A.inv_fact, A.degrees,
                                    loc);
                    c_h2l++;
                }
                local_used = true;
                __syncwarp();
            }
            if (local_used) {
                c_lq += qn;
#pragma unroll 1
                for (int qi = 0; qi < nq; qi++) {
                    double xq[D];
                    pick_query<D>(x, qi, xq);
                    add_slot(pt_est, qi, eval_local_lane<D>(xq, qc, loc, A.plimit_loc, A.K_loc, H.sc, A.digits));
                }
            }
        }
        PH_MARK(6);
        const double node_est = warp_sum(lane_est) + far_est;
#pragma unroll
        for (int qi = 0; qi < kQPL; qi++)
            if (valid[qi]) H.out[A.q_perm[qs + lane + 32 * qi]] = pt_est[qi] + node_est;
        const unsigned long long cyc = (unsigned long long)(clock64() - t_start);
        if (lane == 0 && A.cost) A.cost[b] = cyc;
        if (lane == 0 && A.dbg) {
            A.dbg[kDbgFields * b + 0] = cyc;
            A.dbg[kDbgFields * b + 1] = steps;
            A.dbg[kDbgFields * b + 2] = c_vis;
            A.dbg[kDbgFields * b + 3] = (unsigned long long)__double_as_longlong(A.qb_rad[b]);
            A.dbg[kDbgFields * b + 4] = c_f32;
#if FG_PHASE_PROF
            for (int k = 0; k < 8; k++) A.dbg[kDbgFields * b + 8 + k] = ph[k];
#endif
        }
        if (lane == 0) {
            unsigned long long *cn = H.counters;
            atomicAdd(cn + 0, (unsigned long long)c_vis);
            atomicAdd(cn + 1, (unsigned long long)c_base);
            atomicAdd(cn + 2, (unsigned long long)c_fd);
            atomicAdd(cn + 3, (unsigned long long)c_dh);
            atomicAdd(cn + 4, (unsigned long long)c_dl);
            atomicAdd(cn + 5, (unsigned long long)c_h2l);
            atomicAdd(cn + 6, c_pairs);
            atomicAdd(cn + 7, c_f32);
            atomicAdd(cn + 8, cyc);
            if (c_hq) atomicAdd(cn + 9, c_hq);
            if (c_lq) atomicAdd(cn + 10, c_lq);
            if (c_ht) atomicAdd(cn + 11, c_ht);
        }
        __syncwarp();
    }
}

}  // namespace fg
