// fg_far_kernel.cuh -- the far-field pass over super-nodes (the query-side
// hierarchy above the <= 64-point blocks).
//
// The reference settles far-field work once at a coarse query node: an H2L
// translation into Q.local (summation_engine.py:388-392, series_expansion.py:
// 167-194) or a direct local accumulation (:376-386, :110-126), pushed down to
// the points by dito_post's L2L (summation_engine.py:253-281,
// series_expansion.py:197-217); a finite-difference prune at a coarse node
// likewise covers all of its points (:327-351).  The block traversal alone
// cannot share that work between its 64-point blocks, so each block
// re-evaluated the same far field (Hermite items per block).
//
// A super-node S is a maximal tree node the blocks are cut from (<= 4096
// points).  One warp per (bandwidth, S) walks the reference tree against S's
// box with the same token rule and mass bound as the block kernel:
//   * FD prune (admitted under the token rule against G_min(S), a lower bound
//     on G(x) for every x in S) -> a node-level estimate for all of S;
//   * direct local / H2L when feasible for S and cheaper than leaving the node
//     to S's blocks (select_method_gpu with S's query count) -> S.local;
//   * otherwise a node larger than S is split, a smaller one becomes a
//     RESIDUAL entry: the blocks of S start their own traversal from the
//     residual list instead of the root.
// Each block of S inherits S's leftover tokens (A.6: a node that settles no
// further pairs may push its leftover tokens to every child -- the query sets
// are disjoint), the settled mass (a valid lower bound for every x in S) and
// the node-level estimate; it seeds its local expansion with L2L(S.local,
// c_S -> c_b) and evaluates it once per query (EVALL) after its own traversal.
// For every query x in block b of S the settled references (S-level and
// b-level) partition the reference set and every bound was charged against a
// lower bound on G(x) through one chain of token accounts, so Theorem 2
// holds as for a single traversal.
#pragma once

#include "fg_traverse_kernel.cuh"

namespace fg {

constexpr int kFarThreads = 128;
constexpr int kFarWarps = kFarThreads / 32;
// residual entries one super-node may hand to its blocks (a task that would
// exceed it is abandoned: its blocks then traverse from the root)
constexpr int kFarResCap = kFarResCapT;
// largest reference node a super-node accumulates directly (DIRECTL)
constexpr int kFarDLMax = 256;

template <int D>
__global__ void __launch_bounds__(kFarThreads) far_kernel(const TravArgs A) {
    extern __shared__ double smem[];
    __shared__ double s_tab[kExpTab];
    exp_table_init(s_tab);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kFarWarps + wib;
    constexpr int kFix = (3 * D + 1) & ~1;
    double *sq = smem + wib * (kFix + ((A.K_loc + 1) & ~1));  // box lo, hi, centre
    double *sqc = sq + 2 * D;
    double *loc = sq + kFix;
    const int cap = A.stack_cap;
    int *sn = A.far_st_node + gw * cap;
    double *skl = A.far_st_f + gw * cap * 3;
    double *skh = skl + cap;
    double *slb = skh + cap;
    int2 *sl = A.far_ser + gw * cap;
    const unsigned lt_mask = (1u << lane) - 1u;
    const long long ntask = (long long)A.nh * A.nsn;

    for (;;) {
        long long t = 0;
        if (lane == 0) t = (long long)atomicAdd(A.far_work, 1ULL);
        t = __shfl_sync(kFull, t, 0);
        if (t >= ntask) break;
        const int j = (int)(t / A.nsn);
        const int k = (int)(t - (long long)j * A.nsn);
        const TravH &H = A.hp[j];
        const int snode = __ldg(A.sn_node + k);
        if (lane < 2 * D) sq[lane] = A.q_box[(int64_t)snode * 2 * D + lane];
        if (lane < D) sqc[lane] = A.q_c[(int64_t)snode * D + lane];
        if (A.use_series)
            for (int c = lane; c < A.K_loc; c += 32) loc[c] = 0.0;
        __syncwarp();
        const double2 swr = A.q_wr[snode];  // (weight, inf_radius) of S
        const int s_cnt = A.q_ni[snode].y;
        // G(x) >= w_x (monochromatic: x's own term) and >= W_S exp(-diam^2/2h^2)
        double gfloor = 0.0;
        if (A.qb_wmin) {
            double dsq = 0.0;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const double e = sq[D + d] - sq[d];
                dsq += e * e;
            }
            gfloor = fmax(A.sn_wmin[k], swr.x * fg_exp_fast(dsq * H.neg_inv, s_tab) * (1.0 - 1e-12));
        }
        double tokens = 0.0, settled_sum = 0.0, lane_est = 0.0;
        unsigned c_vis = 0, c_fd = 0, c_dl = 0, c_h2l = 0;
        int nser = 0, nres = 0;
        bool overflow = false;
        int *res = A.far_res + t * kFarResCap;
        double mass;
        int head = 0, cnt = 1;
        {
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
        while (cnt > 0) {
            const int nb = min(cnt, 32);
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
            const double gmin = fmax(mass * kMassSafety, gfloor);
            // ---- finite-difference prune for all of S (summation_engine.py:327-351)
            const double fd_err = 0.5 * WR * (khi - lb);
            const double den = H.eps * gmin;
            const double tok_scale = den > 0.0 ? A.total_w / den : CUDART_INF;
            const double err_scale = den / A.total_w;
            const double req = required_tokens(WR, fd_err, tok_scale);
            unsigned fd_mask;
            if (A.use_tokens) fd_mask = admit(act, req, tokens);
            else fd_mask = __ballot_sync(kFull, act && req <= 0.0);
            const bool fd = (fd_mask >> lane) & 1u;
            c_fd += __popc(fd_mask);
            double settled = 0.0;
            if (fd) {
                settled = WR * lb;
                lane_est += 0.5 * WR * (lb + khi);
            }
            // ---- direct local / H2L into S.local (summation_engine.py:352-399)
            unsigned ser_mask = 0;
            bool dh_ok = false;  // Hermite-feasible for S, hence for each of its blocks
            if (A.use_series && nser + 32 <= cap) {
                int meth = 0, p = 0;
                double bound = 0.0;
                if (act && !fd) {
                    const double maxerr = (WR + tokens) * err_scale;
                    const double r_ref = wr.y * H.inv_h;
                    const double r_qu = swr.y * H.inv_h;
                    const double rmin = r_ref < r_qu ? r_ref : r_qu;
                    const double bse = WR * sqrt(khi + 0x1.0p-1073) * (1.0 + 0x1.0p-40);
                    double possible = bse * A.floor_c;
                    if (rmin < 1.0) {
                        double pw = 1.0;
                        for (int q = 0; q < A.plimit; q++) pw *= rmin;
                        possible *= pw;
                    }
                    if (possible <= maxerr) {
                        select_method_gpu(bse, r_ref, r_qu, (double)ni.y, D, maxerr, A.plimit, A.plimit_loc,
                                          A.ct, A.cross, A.kp, (double)s_cnt / 32.0, H.pair_cost, H.herm_c0, H.herm_c1,
                                          meth, p, bound);
                        int p_h, p_l, p_t;
                        double e_h, e_l, e_t;
                        feasible_orders(bse, r_ref, r_qu, maxerr, A.plimit, A.plimit_loc, A.ct, A.cross, p_h,
                                        p_l, p_t, e_h, e_l, e_t);
                        dh_ok = p_h != 0;
                    }
                    // S-level work must beat leaving the node to S's blocks:
                    // a Hermite or exhaustive choice stays with the blocks, and
                    // a direct local accumulation (one warp streams all N_R
                    // points) only pays for small nodes
                    if (meth != 3 && meth != 4) meth = 0;
                    if (meth == 3 && ni.y > kFarDLMax) meth = 0;
                }
                const bool cand = meth != 0;
                const double sreq = cand ? required_tokens(WR, bound, tok_scale) : CUDART_INF;
                ser_mask = admit(cand, sreq, tokens);
                if ((ser_mask >> lane) & 1u) {
                    settled = WR * lb;
                    sl[nser + __popc(ser_mask & lt_mask)] = make_int2(node, p | (meth << 8));
                }
                nser += __popc(ser_mask);
                c_dl += __popc(__ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 3));
                c_h2l += __popc(__ballot_sync(kFull, ((ser_mask >> lane) & 1u) && meth == 4));
            }
            // ---- split nodes larger than S unless every block of S can take them
            // whole (Hermite-feasible against S's box: a block's box is inside
            // it, so its min distance and margin are no worse); the rest go
            // to S's blocks as residual entries
            const bool rem = act && !fd && !((ser_mask >> lane) & 1u);
            const bool big = ni.z >= 0 && wr.y > swr.y && !dh_ok;
            unsigned split_mask = __ballot_sync(kFull, rem && big);
            const unsigned res_mask = __ballot_sync(kFull, rem && !big) |
                                      (cnt + 2 * __popc(split_mask) > cap ? split_mask : 0u);
            if (cnt + 2 * __popc(split_mask) > cap) split_mask = 0;
            if (nres + __popc(res_mask) > kFarResCap) {
                overflow = true;
                break;
            }
            FG_CHECK(nres + __popc(res_mask) <= kFarResCap);
            if ((res_mask >> lane) & 1u) res[nres + __popc(res_mask & lt_mask)] = node;
            nres += __popc(res_mask);
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
                    sn[slot] = ch;
                    skl[slot] = cl;
                    skh[slot] = chh;
                    slb[slot] = cm;
                    child_sum += A.r_wr[ch].x * cm;
                }
            }
            cnt += 2 * __popc(split_mask);
            // residual entries keep their W_R lb in the mass bound (they stay
            // unsettled); settled ones move to settled_sum
            const bool keep = (res_mask >> lane) & 1u;
            mass += warp_sum(settled + child_sum - (act && !keep ? WR * lb : 0.0));
            if (mass < 0.0) mass = 0.0;
            settled_sum += warp_sum(settled);
            __syncwarp();
        }
        overflow = __any_sync(kFull, overflow);
        bool local_used = false;
        if (!overflow && nser > 0) {
            // the S-level series work: S.local += DIRECTL / H2L (lanes own coefficients)
            double qc[D];
#pragma unroll
            for (int d = 0; d < D; d++) qc[d] = sqc[d];
            for (int i = 0; i < nser; i++) {
                const int2 e = sl[i];
                const int meth = e.y >> 8, p = e.y & 0xff;
                if (meth == 3) {
                    const int4 ni = A.r_ni[e.x];
                    accumulate_warp<D, kLocK / 32>(1, A.r_pw, ni.x, (int64_t)ni.x + ni.y, qc, p, A.kp[p], H.sc,
                                       A.digits, A.inv_fact, loc, false);
                } else {
                    h2l_warp_add<D>(H.r_mom + (int64_t)e.x * A.mom_K, A.r_c + (int64_t)e.x * D, qc,
                                    p, A.kp[p], p, A.kp[p], H.sc, A.digits, A.inv_fact, A.degrees,
                                    loc);
                }
                __syncwarp();
            }
            local_used = true;
        }
        const double est = warp_sum(lane_est);
        if (!overflow && local_used)
            for (int c = lane; c < A.K_loc; c += 32) A.far_loc[t * A.K_loc + c] = loc[c];
        if (lane == 0) {
            A.far_flag[t] = overflow ? 0 : (1 | (local_used ? 2 : 0));
            A.far_tokens[t] = tokens;
            A.far_settled[t] = settled_sum;
            A.far_est[t] = est;
            A.far_rcnt[t] = overflow ? 0 : nres;
            unsigned long long *cn = H.counters;
            atomicAdd(cn + 0, (unsigned long long)c_vis);
            if (!overflow) {
                atomicAdd(cn + 2, (unsigned long long)c_fd);
                atomicAdd(cn + 4, (unsigned long long)c_dl);
                atomicAdd(cn + 5, (unsigned long long)c_h2l);
                atomicAdd(cn + 12, 1ULL);  // super-nodes settled at S level
            }
        }
        __syncwarp();
    }
}

}  // namespace fg
