// fg_tree_coop.cuh -- the single-launch cooperative kd-tree build kernel
// (included by fg_tree.cu).  Three grid-wide barriers per level:
//   A: chunk statistics; the warp that completes a node's last chunk (atomic
//      count) combines the partials in chunk order and picks the split |
//   B: chunk radius partials and left counts; the last warp of a node
//      combines them, writes per-chunk left offsets and decides the split |
//   C: scan over the slots with a decoupled look-back + child allocation,
//      then the stable scatter.
// A chunk finds its slot by binary search over the slots' chunk offsets, and
// one 64-bit scan over the slots yields both the children's BFS ranks and
// their chunk offsets.
//
// Once every active node fits one chunk (<= kChunk points), the rest of the
// tree is built in the small-node phase: one warp owns a node for the whole
// level (statistics, radius, split, stable partition) and allocates its
// children with an atomic rank, so a level costs ONE grid barrier.  Ids stay
// level-contiguous (BFS levels); their order within a level is the order of
// allocation, which nothing downstream depends on (export maps to preorder
// through the structure).
#pragma once
// (included inside namespace fg)

typedef cub::BlockScan<int, kBuildThreads> BlockScanInt;
typedef cub::BlockScan<unsigned long long, kBuildThreads> BlockScanU64;

// slot owning chunk c: the last s with choff[s] <= c (offsets strictly increase)
__device__ __forceinline__ int chunk_slot_of(const int *choff, int na, int c) {
    int lo = 0, hi = na - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (choff[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Small-node phase (see the header comment): levels from `level` on, every
// active node has <= kChunk points and one warp processes it start to finish.
template <int D>
__device__ void build_small_levels(const BuildArgs &B, cg::grid_group &g, int level) {
    const int lane = threadIdx.x & 31;
    const int64_t n = B.n;
    const int gtid = blockIdx.x * kBuildThreads + threadIdx.x;
    const int gwarps = gridDim.x * kBuildThreads / 32;
    const int gwarp = gtid >> 5;
    const int nmax = (int)B.nmax;
    const unsigned lt = (1u << lane) - 1u;
    if (level >= kMaxLevels) return;
    int na = B.ctl[kNa];
    int next_base = B.ctl[kNextBase];
    if (gtid == 0) {
        B.ctl[kSplit0 + level % 3] = 0;
        B.ctl[kSplit0 + (level + 1) % 3] = 0;
    }
    g.sync();
    for (; level < kMaxLevels && na > 0; level++) {
        const int cur = level & 1;
        const int *act = B.act[cur];
        int *act_next = B.act[cur ^ 1];
        const double *x = B.x[cur];
        const double *w = B.w[cur];
        const int *idx = B.idx[cur];
        double *xn = B.x[cur ^ 1];
        double *wn = B.w[cur ^ 1];
        int *idxn = B.idx[cur ^ 1];
        int *split_ctr = B.ctl + kSplit0 + level % 3;
        // the counter of level + 1 was last read before the previous barrier
        if (gtid == 0) B.ctl[kSplit0 + (level + 1) % 3] = 0;
        for (int s = gwarp; s < na; s += gwarps) {
            const int node = act[s];
            int4 ni = B.node_i[node];
            const int b = ni.x, e = ni.x + ni.y;
            double lo[D], hi[D], sm[D], ws = 0.0;
#pragma unroll
            for (int d = 0; d < D; d++) {
                lo[d] = CUDART_INF;
                hi[d] = -CUDART_INF;
                sm[d] = 0.0;
            }
            #pragma unroll 4
            for (int i = b + lane; i < e; i += 32) {
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const double v = x[(int64_t)d * n + i];
                    lo[d] = fmin(lo[d], v);
                    hi[d] = fmax(hi[d], v);
                    sm[d] += v;
                }
                ws += w[i];
            }
            int sd = 0;
            double best = 0.0, ctr[D];
#pragma unroll
            for (int d = 0; d < D; d++) {
                lo[d] = warp_min(lo[d]);
                hi[d] = warp_max(hi[d]);
                sm[d] = warp_sum(sm[d]);
                ctr[d] = sm[d] / (double)ni.y;
                const double wd = hi[d] - lo[d];
                if (d == 0 || wd > best) {
                    best = wd;
                    sd = d;
                }
            }
            ws = warp_sum(ws);
            const bool leafy = ni.y <= B.leaf || best == 0.0;
            const double mid = 0.5 * (lo[sd] + hi[sd]);
            double rad = 0.0;
            int cnt = 0;
            #pragma unroll 4
            for (int i = b + lane; i < e; i += 32) {
#pragma unroll
                for (int d = 0; d < D; d++) rad = fmax(rad, fabs(x[(int64_t)d * n + i] - ctr[d]));
                if (!leafy) cnt += x[(int64_t)sd * n + i] < mid ? 1 : 0;
            }
            rad = warp_max(rad);
            const int nl = warp_sum(cnt);
            const bool split = !leafy && nl > 0 && nl < ni.y;
            if (lane < D) {
#pragma unroll
                for (int d = 0; d < D; d++) {
                    if (d == lane) {
                        B.node_box[(int64_t)node * 2 * D + d] = lo[d];
                        B.node_box[(int64_t)node * 2 * D + D + d] = hi[d];
                        B.node_c[(int64_t)node * D + d] = ctr[d];
                    }
                }
            }
            if (lane == 0) B.node_wr[node] = make_double2(ws, rad);
            if (!split) {
                #pragma unroll 4
            for (int i = b + lane; i < e; i += 32) {
#pragma unroll
                    for (int d = 0; d < D; d++) B.xf[(int64_t)d * n + i] = x[(int64_t)d * n + i];
                    B.wf[i] = w[i];
                    B.idxf[i] = idx[i];
                }
                continue;
            }
            // stable warp partition, 32 points per round, in order; the next
            // round's point is loaded while this round is scattered
            int cl = 0, cr = 0;
            double yc[D], wc = 0.0;
            int ic = 0;
            if (b + lane < e) {
#pragma unroll
                for (int d = 0; d < D; d++) yc[d] = x[(int64_t)d * n + b + lane];
                wc = w[b + lane];
                ic = idx[b + lane];
            }
            for (int base = b; base < e; base += 32) {
                const int i = base + lane;
                const bool in = i < e;
                double yv[D];
#pragma unroll
                for (int d = 0; d < D; d++) yv[d] = yc[d];
                const double wv = wc;
                const int iv = ic;
                if (i + 32 < e) {
#pragma unroll
                    for (int d = 0; d < D; d++) yc[d] = x[(int64_t)d * n + i + 32];
                    wc = w[i + 32];
                    ic = idx[i + 32];
                }
                double xs = yv[0];
#pragma unroll
                for (int d = 0; d < D; d++)
                    if (d == sd) xs = yv[d];
                const bool goes_left = in && xs < mid;
                const unsigned lm = __ballot_sync(kFull, goes_left);
                const unsigned rm = __ballot_sync(kFull, in && !goes_left);
                if (in) {
                    const int dst = goes_left ? b + cl + __popc(lm & lt) : b + nl + cr + __popc(rm & lt);
#pragma unroll
                    for (int d = 0; d < D; d++) xn[(int64_t)d * n + dst] = yv[d];
                    wn[dst] = wv;
                    idxn[dst] = iv;
                }
                cl += __popc(lm);
                cr += __popc(rm);
            }
            int r = 0;
            if (lane == 0) r = atomicAdd(split_ctr, 1);
            r = __shfl_sync(kFull, r, 0);
            const int L = next_base + 2 * r, R = L + 1;
            if (lane == 0) {
                if (R < nmax) {
                    B.node_i[L] = make_int4(b, nl, -1, -1);
                    B.node_i[R] = make_int4(b + nl, ni.y - nl, -1, -1);
                    ni.z = L;
                    ni.w = R;
                    B.node_i[node] = ni;
                    act_next[2 * r] = L;
                    act_next[2 * r + 1] = R;
                } else {
                    B.ctl[kOverflow] = 1;
                }
            }
        }
        g.sync();
        const int nsplit = *(volatile int *)split_ctr;
        const bool overflow = *(volatile int *)(B.ctl + kOverflow) != 0;
        if (gtid == 0) {
            B.ctl[kLevels] = level + 1;
            B.level_begin[level + 2] = next_base + 2 * nsplit;
            B.ctl[kNextBase] = next_base + 2 * nsplit;
            B.ctl[kNa] = overflow ? 0 : 2 * nsplit;
        }
        next_base += 2 * nsplit;
        na = overflow ? 0 : 2 * nsplit;
    }
}

template <int D>
__global__ void __launch_bounds__(kBuildThreads, D > 8 ? 2 : 1)
build_coop_kernel(const BuildArgs B) {
    cg::grid_group g = cg::this_grid();
    __shared__ typename BlockScanU64::TempStorage scan_tmp;
    __shared__ unsigned long long s_prefix;
    const int lane = threadIdx.x & 31;
    const int64_t n = B.n;
    const int gtid = blockIdx.x * kBuildThreads + threadIdx.x;
    const int gwarps = gridDim.x * kBuildThreads / 32;
    const int gwarp = gtid >> 5;
    const int nmax = (int)B.nmax;

    int level = 0;
    for (; level < kMaxLevels; level++) {
        const int cur = level & 1;
        const int na = B.ctl[kNa];
        if (na == 0) break;
        const int nchunks = B.ctl[kNchunks];
        if (nchunks == na) break;  // every active node fits one chunk
        const int next_base = B.ctl[kNextBase];
        const int *act = B.act[cur];
        int *act_next = B.act[cur ^ 1];
        const int *choff = B.choff + cur * nmax;
        int *choff_next = B.choff + (cur ^ 1) * nmax;
        int *done_a = B.done + cur * 2 * nmax, *done_b = done_a + nmax;
        int *done_next = B.done + (cur ^ 1) * 2 * nmax;
        const double *x = B.x[cur];
        const double *w = B.w[cur];
        const int *idx = B.idx[cur];
        auto chunk_end = [&](int s) { return s + 1 < na ? choff[s + 1] : nchunks; };

        // ---- phase A: per-chunk min / max / sum / weight; the warp finishing a
        // node's last chunk combines its partials (fixed order) and picks the split
        for (int c = gwarp; c < nchunks; c += gwarps) {
            const int s = chunk_slot_of(choff, na, c);
            const int node = act[s];
            const int4 ni = B.node_i[node];
            const int cb = ni.x + (c - choff[s]) * kChunk;
            const int ce = min(cb + kChunk, ni.x + ni.y);
            double lo[D], hi[D], sm[D], ws = 0.0;
#pragma unroll
            for (int d = 0; d < D; d++) {
                lo[d] = CUDART_INF;
                hi[d] = -CUDART_INF;
                sm[d] = 0.0;
            }
            #pragma unroll 4
            for (int i = cb + lane; i < ce; i += 32) {
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const double v = x[(int64_t)d * n + i];
                    lo[d] = fmin(lo[d], v);
                    hi[d] = fmax(hi[d], v);
                    sm[d] += v;
                }
                ws += w[i];
            }
#pragma unroll
            for (int d = 0; d < D; d++) {
                lo[d] = warp_min(lo[d]);
                hi[d] = warp_max(hi[d]);
                sm[d] = warp_sum(sm[d]);
            }
            ws = warp_sum(ws);
            const int c0 = choff[s], c1 = chunk_end(s);
            int last = 0;
            if (lane == 0) {
                double *p = B.part + (int64_t)c * (3 * D + 1);
#pragma unroll
                for (int d = 0; d < D; d++) {
                    p[d] = lo[d];
                    p[D + d] = hi[d];
                    p[2 * D + d] = sm[d];
                }
                p[3 * D] = ws;
                __threadfence();
                last = atomicAdd(done_a + s, 1) == c1 - c0 - 1;
            }
            if (!__shfl_sync(kFull, last, 0)) continue;
            __threadfence();
#pragma unroll
            for (int d = 0; d < D; d++) {
                lo[d] = CUDART_INF;
                hi[d] = -CUDART_INF;
                sm[d] = 0.0;
            }
            ws = 0.0;
            for (int cc = c0 + lane; cc < c1; cc += 32) {
                const double *p = B.part + (int64_t)cc * (3 * D + 1);
#pragma unroll
                for (int d = 0; d < D; d++) {
                    lo[d] = fmin(lo[d], __ldcg(p + d));
                    hi[d] = fmax(hi[d], __ldcg(p + D + d));
                    sm[d] += __ldcg(p + 2 * D + d);
                }
                ws += __ldcg(p + 3 * D);
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
                    B.node_box[(int64_t)node * 2 * D + d] = lo[d];
                    B.node_box[(int64_t)node * 2 * D + D + d] = hi[d];
                    B.node_c[(int64_t)node * D + d] = sm[d] / cnt;
                    const double wd = hi[d] - lo[d];
                    if (d > 0 && wd > best) {
                        best = wd;
                        sd = d;
                    }
                }
                B.node_wr[node] = make_double2(ws, 0.0);
                const bool leafy = ni.y <= B.leaf || best == 0.0;
                B.split_dim[s] = leafy ? -1 : sd;
                B.split_mid[s] = 0.5 * (lo[sd] + hi[sd]);
            }
        }
        g.sync();

        // ---- phase B: per-chunk inf-norm radius partial and left count; the
        // warp finishing a node's last chunk combines them, writes the per-chunk
        // left offsets and decides the split.  The slot's scan value packs
        // (is_split, chunks of its two children).
        for (int c = gwarp; c < nchunks; c += gwarps) {
            const int s = chunk_slot_of(choff, na, c);
            const int node = act[s];
            const int4 ni = B.node_i[node];
            const int cb = ni.x + (c - choff[s]) * kChunk;
            const int ce = min(cb + kChunk, ni.x + ni.y);
            const int sd = B.split_dim[s];
            const double mid = B.split_mid[s];
            double ctr[D];
#pragma unroll
            for (int d = 0; d < D; d++) ctr[d] = B.node_c[(int64_t)node * D + d];
            double rad = 0.0;
            int cnt = 0;
            #pragma unroll 4
            for (int i = cb + lane; i < ce; i += 32) {
#pragma unroll
                for (int d = 0; d < D; d++) rad = fmax(rad, fabs(x[(int64_t)d * n + i] - ctr[d]));
                if (sd >= 0) cnt += x[(int64_t)sd * n + i] < mid ? 1 : 0;
            }
            rad = warp_max(rad);
            cnt = warp_sum(cnt);
            const int c0 = choff[s], c1 = chunk_end(s);
            int last = 0;
            if (lane == 0) {
                B.part2[c] = rad;
                B.lcnt[c] = cnt;
                __threadfence();
                last = atomicAdd(done_b + s, 1) == c1 - c0 - 1;
            }
            if (!__shfl_sync(kFull, last, 0)) continue;
            __threadfence();
            rad = 0.0;
            int run = 0;
            for (int base = c0; base < c1; base += 32) {
                const int cc = base + lane;
                const int v = cc < c1 ? __ldcg(B.lcnt + cc) : 0;
                if (cc < c1) rad = fmax(rad, __ldcg(B.part2 + cc));
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                if (cc < c1) B.loff[cc] = run + incl - v;
                run += __shfl_sync(kFull, incl, 31);
            }
            rad = warp_max(rad);
            if (lane == 0) {
                double2 wr = B.node_wr[node];
                wr.y = rad;
                B.node_wr[node] = wr;
                const bool split = sd >= 0 && run > 0 && run < ni.y;
                if (!split) B.split_dim[s] = -1;
                B.nleft[s] = run;
                const unsigned long long ch =
                    split ? (unsigned long long)((run + kChunk - 1) / kChunk +
                                                 (ni.y - run + kChunk - 1) / kChunk)
                          : 0ull;
                B.sval[s] = (split ? 1ull : 0ull) | (ch << 32);
            }
        }
        g.sync();

        // ---- phase C: (1) scan over the slots with a decoupled look-back (CTA b
        // owns slots [b*per, (b+1)*per)) and child allocation; (2) the stable
        // scatter of every chunk (leaves -> final arrays, splits -> next buffers)
        {
            const int nb = gridDim.x;
            const int per = (na + nb - 1) / nb;
            const int npart = (na + per - 1) / per;  // CTAs that own slots
            const int s0 = min(na, (int)blockIdx.x * per), s1 = min(na, s0 + per);
            const int stamp = (level + 1) << 2;
            unsigned long long local = 0, agg = 0;
            if ((int)blockIdx.x < npart) {
                for (int s = s0 + threadIdx.x; s < s1; s += kBuildThreads) local += B.sval[s];
                BlockScanU64(scan_tmp).ExclusiveSum(local, local, agg);
            }
            if ((int)blockIdx.x < npart && threadIdx.x < 32) {
                // warp-wide look-back over 32 predecessors at a time
                if (lane == 0) {
                    B.lb_agg[blockIdx.x] = agg;
                    __threadfence();
                    atomicExch(B.lb_flag + blockIdx.x, stamp | 1);
                }
                unsigned long long prefix = 0;
                for (int p_end = (int)blockIdx.x; p_end > 0; p_end -= 32) {
                    const int p = p_end - 1 - lane;
                    int f = stamp | 2;
                    if (p >= 0) {
                        do {
                            f = *(volatile int *)(B.lb_flag + p);
                        } while ((f & ~3) != stamp);
                    }
                    __threadfence();
                    const unsigned inc = __ballot_sync(kFull, p < 0 || (f & 3) == 2);
                    const int k = inc ? __ffs(inc) - 1 : 32;
                    unsigned long long v = 0;
                    if (p >= 0 && lane < k) v = __ldcg(B.lb_agg + p);
                    else if (p >= 0 && lane == k) v = __ldcg(B.lb_incl + p);
                    prefix += warp_sum(v);
                    if (k < 32) break;
                }
                if (lane == 0) {
                    B.lb_incl[blockIdx.x] = prefix + agg;
                    __threadfence();
                    atomicExch(B.lb_flag + blockIdx.x, stamp | 2);
                    s_prefix = prefix;
                    if ((int)blockIdx.x == npart - 1) {
                        // the last owner holds the grand total: next level's control
                        const unsigned long long total = prefix + agg;
                        const int nsplit = (int)(total & 0xffffffffull);
                        const int nchunks_next = (int)(total >> 32);
                        if (next_base + 2 * nsplit > nmax) B.ctl[kOverflow] = 1;
                        B.ctl[kNa] = B.ctl[kOverflow] ? 0 : 2 * nsplit;
                        B.ctl[kNchunks] = nchunks_next;
                        B.ctl[kNextBase] = next_base + 2 * nsplit;
                        B.ctl[kLevels] = level + 1;
                        // level l+1 spans [next_base, next_base + 2*nsplit): its
                        // end is the start of level l+2
                        B.level_begin[level + 2] = next_base + 2 * nsplit;
                    }
                }
            }
            __syncthreads();
            unsigned long long carry = s_prefix;
            for (int base = s0; base < s1; base += kBuildThreads) {
                const int s = base + threadIdx.x;
                const unsigned long long v = s < s1 ? B.sval[s] : 0ull;
                unsigned long long ex, t;
                __syncthreads();
                BlockScanU64(scan_tmp).ExclusiveSum(v, ex, t);
                ex += carry;
                carry += t;
                if (s < s1 && (v & 1ull)) {
                    const int r = (int)(ex & 0xffffffffull);
                    const int coff = (int)(ex >> 32);
                    const int node = act[s];
                    int4 ni = B.node_i[node];
                    const int L = next_base + 2 * r, R = L + 1;
                    const int nl = B.nleft[s];
                    if (R < nmax) {
                        B.node_i[L] = make_int4(ni.x, nl, -1, -1);
                        B.node_i[R] = make_int4(ni.x + nl, ni.y - nl, -1, -1);
                        ni.z = L;
                        ni.w = R;
                        B.node_i[node] = ni;
                        act_next[2 * r] = L;
                        act_next[2 * r + 1] = R;
                        choff_next[2 * r] = coff;
                        choff_next[2 * r + 1] = coff + (nl + kChunk - 1) / kChunk;
                        done_next[2 * r] = done_next[2 * r + 1] = 0;
                        done_next[nmax + 2 * r] = done_next[nmax + 2 * r + 1] = 0;
                    }
                }
            }
        }
        for (int c = gwarp; c < nchunks; c += gwarps) {
            const int s = chunk_slot_of(choff, na, c);
            const int4 ni = B.node_i[act[s]];
            const int cb = ni.x + (c - choff[s]) * kChunk;
            const int ce = min(cb + kChunk, ni.x + ni.y);
            const int sd = B.split_dim[s];
            if (sd < 0) {
                #pragma unroll 4
            for (int i = cb + lane; i < ce; i += 32) {
#pragma unroll
                    for (int d = 0; d < D; d++) B.xf[(int64_t)d * n + i] = x[(int64_t)d * n + i];
                    B.wf[i] = w[i];
                    B.idxf[i] = idx[i];
                }
                continue;
            }
            // stable warp partition, 32 points per round, in order
            const double mid = B.split_mid[s];
            const int left_base = ni.x + B.loff[c];
            const int right_base = ni.x + B.nleft[s] + (cb - ni.x - B.loff[c]);
            double *xn = B.x[cur ^ 1];
            double *wn = B.w[cur ^ 1];
            int *idxn = B.idx[cur ^ 1];
            const unsigned lt = (1u << lane) - 1u;
            int nl = 0, nr = 0;
            // the next round's point is loaded while this round is scattered
            double yc[D], wc = 0.0;
            int ic = 0;
            if (cb + lane < ce) {
#pragma unroll
                for (int d = 0; d < D; d++) yc[d] = x[(int64_t)d * n + cb + lane];
                wc = w[cb + lane];
                ic = idx[cb + lane];
            }
            for (int base = cb; base < ce; base += 32) {
                const int i = base + lane;
                const bool in = i < ce;
                double yv[D];
#pragma unroll
                for (int d = 0; d < D; d++) yv[d] = yc[d];
                const double wv = wc;
                const int iv = ic;
                if (i + 32 < ce) {
#pragma unroll
                    for (int d = 0; d < D; d++) yc[d] = x[(int64_t)d * n + i + 32];
                    wc = w[i + 32];
                    ic = idx[i + 32];
                }
                double xs = yv[0];
#pragma unroll
                for (int d = 0; d < D; d++)
                    if (d == sd) xs = yv[d];
                const bool goes_left = in && xs < mid;
                const unsigned lm = __ballot_sync(kFull, goes_left);
                const unsigned rm = __ballot_sync(kFull, in && !goes_left);
                if (in) {
                    const int dst = goes_left ? left_base + nl + __popc(lm & lt)
                                              : right_base + nr + __popc(rm & lt);
#pragma unroll
                    for (int d = 0; d < D; d++) xn[(int64_t)d * n + dst] = yv[d];
                    wn[dst] = wv;
                    idxn[dst] = iv;
                }
                nl += __popc(lm);
                nr += __popc(rm);
            }
        }
        g.sync();
    }
    build_small_levels<D>(B, g, level);
}
