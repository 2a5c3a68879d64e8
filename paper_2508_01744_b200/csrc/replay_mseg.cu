// replay_mseg.cu — K2/MSEG<D,G>: G lanes per tuner (32/G tuners per warp) for K_act ≥ 2,
// with the active arms' state STREAMED every step from a tightly packed per-tuner buffer
// (L2-resident for the k_h = 4 quarter of C4, HBM-streamed in the first ~1,000 windows).
//
// Cost model: a warp instruction of per-tuner scalar work (response,
// reward median, Sherman–Morrison, stats) serves 32/G tuners, and scoring costs K·45/32
// warp instructions per tuner-step whatever G is; so small G minimises instructions, while
// G > 1 keeps enough warps resident (C4's multi-arm class is only ~16K tuners).  G = 4.
//
// Layout of the arm stream (workspace `mstream`): tuner at class-list position i owns
// rows r < 128/G; row r holds arms j = r·G + l (lane l of the segment), 38 words each:
//     word(i, r, e, l) = ((i·R + r)·W + e)·G + l,   R = 128/G, W = d(d+1)/2 + d + 3
// (packed A⁻¹, θ, r̄, ē, key|n).  A warp load touches one 32-B sector per tuner.
//
// The lexicographic argmax, near-tie data, pruning counts and the canonical 128-slot
// reduction (shared-memory scatter, aligned 128/G-slot block per lane, then a width-G
// butterfly — exactly ENV.md §4.8's pairwise tree) are segment-cooperative; the sorted
// EDP window lives in shared memory and is maintained by the segment's lane 0.
#include "step_common.cuh"

namespace agft {

namespace {

constexpr int kMsegTunersPerBlock = 16;       // blockDim = 16·G (G ≥ 2)
constexpr uint32_t kDeadKey = 0xFFu;

__device__ __forceinline__ uint64_t mpack(uint32_t key, uint32_t n) { return ((uint64_t)n << 32) | key; }
__device__ __forceinline__ uint32_t mkey(uint64_t m) { return (uint32_t)m; }
__device__ __forceinline__ uint32_t mn(uint64_t m) { return (uint32_t)(m >> 32); }

template <int G, typename T>
__device__ __forceinline__ T seg_max(T v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v = max(v, __shfl_xor_sync(kFull, v, off, G));
    return v;
}
template <int G>
__device__ __forceinline__ double seg_fmax(double v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, off, G));
    return v;
}
template <int G>
__device__ __forceinline__ double seg_fmin(double v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, off, G));
    return v;
}
template <int G>
__device__ __forceinline__ int seg_isum(int v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
    return v;
}

// canonical 128-slot pairwise sum of one tuner's (key, value) set (ENV.md §4.8):
// `buf` is the tuner's 128-double shared array, already holding value at slot key and
// +0.0 elsewhere; lane l reduces the aligned block [l·128/G, (l+1)·128/G) as a pairwise
// tree, then the width-G butterfly combines the blocks in tree order.
template <int G>
__device__ __forceinline__ double seg_tree_reduce(const double *buf, int l)
{
    constexpr int SL = 128 / G;
    double v[SL];
#pragma unroll
    for (int j = 0; j < SL; ++j) v[j] = buf[l * SL + j];
#pragma unroll
    for (int len = SL; len > 1; len >>= 1)
#pragma unroll
        for (int j = 0; j < len / 2; ++j) v[j] = xadd(v[2 * j], v[2 * j + 1]);
    double s = v[0];
#pragma unroll
    for (int off = 1; off < G; off <<= 1) s = xadd(s, __shfl_xor_sync(kFull, s, off, G));
    return s;
}

}  // namespace

template <int D, int G>
__global__ void __launch_bounds__(kMsegTunersPerBlock * G) mseg_kernel(const __grid_constant__ ReplayArgs a)
{
    constexpr int P = D * (D + 1) / 2;
    constexpr int W = P + D + 3;                 // words per arm slot
    constexpr int R = kMaxArms / G;              // rows per tuner
    constexpr int NSEG = kMsegTunersPerBlock;    // tuners per block
    __shared__ double s_win[kWindow * NSEG];     // sorted window column per tuner
    __shared__ double s_tree[kMaxArms * NSEG];   // canonical-tree scatter buffer per tuner
    __shared__ double s_dec[kMaxArms], s_pre[kMaxArms], s_pw[kMaxArms];
    const EnvConsts *ec = a.w.env;
    for (int q = threadIdx.x; q < kMaxArms; q += blockDim.x) {
        s_dec[q] = ec->dec[q];
        s_pre[q] = ec->pre[q];
        s_pw[q] = ec->pw[q];
    }
    for (int q = threadIdx.x; q < kMaxArms * NSEG; q += blockDim.x) s_tree[q] = 0.0;
    __syncthreads();
    const double invW = ec->invW, q_over = ec->q_over;

    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const int warp = threadIdx.x >> 5;
    const uint32_t wbase = blockIdx.x * NSEG + warp * (32 / G);
    if (wbase >= cnt) return;                                    // warp-uniform exit
    const int sgb = threadIdx.x / G;                              // segment within the block
    const int l = threadIdx.x % G;
    const uint32_t idx = blockIdx.x * NSEG + sgb;
    const bool valid = idx < cnt;
    const uint32_t pos = valid ? idx : cnt - 1;                   // dummy segments shadow a real tuner
    const uint32_t tb = a.list ? a.list[pos] : pos;
    agft_tuner_stats st = a.w.acc[tb];
    bool live = valid && !(st.flags & 1u);
    const agft_tuner_params prm = a.w.params[tb];
    // arm stream of this tuner (dummy segments get a private scratch: none — they never write)
    double *buf = a.w.mstream + (size_t)pos * R * W * G + l;
#define SLOT(r, e) buf[((r) * W + (e)) * G]
    double *tree = s_tree + sgb * kMaxArms;
    double *wcol = s_win + sgb;
    const SmemWindow win{wcol, NSEG};

    // ---- gather the active arms: active-order index j = r·G + l
    int K0 = 0;
    {
        const uint4 m4 = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
        for (int w = 0; w < 4; ++w) {
            uint32_t mm = mw[w];
            while (mm) {
                const int k = 32 * w + __ffs(mm) - 1;
                mm &= mm - 1u;
                if (valid && (K0 % G) == l) {
                    const int r = K0 / G;
#pragma unroll
                    for (int e = 0; e < P; ++e) SLOT(r, e) = a.w.ainv[((size_t)tb * P + e) * kMaxArms + k];
#pragma unroll
                    for (int q = 0; q < D; ++q) SLOT(r, P + q) = a.w.theta[((size_t)tb * D + q) * kMaxArms + k];
                    SLOT(r, P + D) = a.w.rbar[(size_t)tb * kMaxArms + k];
                    SLOT(r, P + D + 1) = a.w.ebar[(size_t)tb * kMaxArms + k];
                    SLOT(r, P + D + 2) = __longlong_as_double((long long)mpack(k, a.w.n[(size_t)tb * kMaxArms + k]));
                }
                ++K0;
            }
        }
    }
    const int rows = (K0 - l + G - 1) / G;                       // rows held by this lane
    int nact = K0;
    if (l == 0)
        for (int j = 0; j < kWindow; ++j) win.at(j) = a.w.wsorted[(size_t)tb * kWindow + j];
    uint32_t wcount = a.w.wmeta[(size_t)tb * 2], whead = a.w.wmeta[(size_t)tb * 2 + 1];
    const uint32_t M = a.median_window;
    double *ring = a.w.wring + (size_t)tb * kWindow;
    double *bg = a.w.b + (size_t)tb * D * kMaxArms;
    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;
    __syncwarp();

    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const uint32_t t = a.t0 + s;
        double x[D];
        RecView v;
        load_rec<D>(rp + s, x, v);
        const double alpha = prm.alpha0 / sqrt(1.0 + (double)t / a.tau);
        double w[P];
        {
            int e = 0;
#pragma unroll
            for (int r0 = 0; r0 < D; ++r0)
#pragma unroll
                for (int c = r0; c < D; ++c, ++e) w[e] = (r0 == c) ? x[r0] * x[r0] : 2.0 * x[r0] * x[c];
        }
        // ---- a4: this lane's arms (ascending keys along r)
        double s1 = -kInf, m1 = 0.0, s2 = -kInf, s2nf = -kInf, mmax = 0.0;
        int k1 = 0x7fffffff, r1 = 0;
        bool f1 = false;
        for (int r = 0; r < rows; ++r) {
            const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r, P + D + 2));
            const uint32_t key = mkey(meta);
            if (key == kDeadKey) continue;
            double q = 0.0, p = 0.0;
#pragma unroll
            for (int e = 0; e < P; ++e) q = fma(w[e], SLOT(r, e), q);
#pragma unroll
            for (int c = 0; c < D; ++c) p = fma(SLOT(r, P + c), x[c], p);
            const double bonus = alpha * sqrt(fmax(q, 0.0));
            const double sc = p + bonus, mg = fabs(p) + bonus;
            const bool fresh = mn(meta) == 0u;
            mmax = fmax(mmax, mg);
            if (sc > s1) {
                s2 = s1;
                if (!f1) s2nf = fmax(s2nf, s1);
                s1 = sc; m1 = mg; k1 = (int)key; r1 = r; f1 = fresh;
            } else {
                s2 = fmax(s2, sc);
                if (!fresh) s2nf = fmax(s2nf, sc);
            }
        }
        // ---- a5/a6: segment argmax (s desc, key asc)
        double bs = s1;
        int bk = k1;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            const double os = __shfl_xor_sync(kFull, bs, off, G);
            const int ok = __shfl_xor_sync(kFull, bk, off, G);
            if (os > bs || (os == bs && ok < bk)) { bs = os; bk = ok; }
        }
        const int kstar = bk;
        const bool owner = (k1 == kstar) && (s1 == bs);
        // rivals: the runner-up over the whole tuner (conservative near-tie data, ENV.md §4.5)
        const double lane_s2 = owner ? s2 : s1, lane_s2nf = owner ? s2nf : (f1 ? s2nf : fmax(s1, s2nf));
        const double g_s2 = seg_fmax<G>(lane_s2), g_s2nf = seg_fmax<G>(lane_s2nf);
        const double g_mmax = seg_fmax<G>(mmax);
        const unsigned own_bits = __ballot_sync(kFull, owner);
        const int own_lane = __ffs(G == 32 ? own_bits : (own_bits >> ((threadIdx.x & 31) / G * G)) & ((1u << G) - 1u)) - 1;
        const double mstar = __shfl_sync(kFull, m1, own_lane, G);
        const bool fstar = __shfl_sync(kFull, (int)f1, own_lane, G) != 0;
        const double rival = fstar ? g_s2nf : g_s2;
        const bool near = rival > -kInf && (bs - rival < a.tie_rel * fmax(mstar, g_mmax));

        // ---- a7: response (every lane; cheap, keeps the owner and lane 0 converged)
        const Response o = env_response(s_dec[kstar], s_pre[kstar], s_pw[kstar], v.I, v.P, v.g, v.invIm, v.invAm,
                                        v.wIm, v.nT, v.nE, invW, q_over, a.u_max, a.u_floor, a.p_idle, a.W);
        // ---- a8: reward + window on the segment's lane 0, broadcast
        double r = 0.0;
        int ok = 1;
        if (l == 0 && live) {
            bool fin;
            double oldest = ring_oldest(ring, wcount, whead, M);
            r = reward_and_push(win, ring, wcount, whead, M, o.edp, a.clip_lo, a.clip_hi, fin, oldest);
            ok = fin ? 1 : 0;
        }
        r = __shfl_sync(kFull, r, 0, G);
        ok = __shfl_sync(kFull, ok, 0, G);
        if (!ok) {
            if (live) st.flags |= 1u;
            live = false;
        }
        wcount = __shfl_sync(kFull, wcount, 0, G);
        whead = __shfl_sync(kFull, whead, 0, G);

        // ---- a9: Sherman–Morrison on the owner lane's slot
        if (owner && live) {
            double A[P], th[D], b[D];
#pragma unroll
            for (int e = 0; e < P; ++e) A[e] = SLOT(r1, e);
#pragma unroll
            for (int q = 0; q < D; ++q) {
                th[q] = SLOT(r1, P + q);
                b[q] = bg[(size_t)q * kMaxArms + kstar];
            }
            sm_update<D>(A, th, b, x, r);
#pragma unroll
            for (int e = 0; e < P; ++e) SLOT(r1, e) = A[e];
#pragma unroll
            for (int q = 0; q < D; ++q) {
                SLOT(r1, P + q) = th[q];
                bg[(size_t)q * kMaxArms + kstar] = b[q];
            }
            const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r1, P + D + 2));
            uint32_t n = mn(meta);
            double rb = SLOT(r1, P + D), eb = SLOT(r1, P + D + 1);
            welford(n, rb, eb, r, o.edp);
            SLOT(r1, P + D) = rb;
            SLOT(r1, P + D + 1) = eb;
            SLOT(r1, P + D + 2) = __longlong_as_double((long long)mpack((uint32_t)kstar, n));
        }
        __syncwarp();
        const int nact0 = nact;

        // ---- a10: pruning (ENV.md §4.8) on the post-update state
        if (a.prune_enable && __any_sync(kFull, live && nact > 1)) {
            const bool ext_on = t < a.ext_L;
            int next = 0, nq = 0;
            double best = kInf;
            for (int r0 = 0; r0 < rows; ++r0) {
                const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                const uint32_t key = mkey(meta);
                if (key == kDeadKey) continue;
                const uint32_t n = mn(meta);
                if (ext_on && n >= a.ext_n && SLOT(r0, P + D) < prm.extreme_reward_threshold) ++next;
                if (n >= a.hist_n) {
                    const double eb = SLOT(r0, P + D + 1);
                    ++nq;
                    best = fmin(best, eb);
                    tree[key] = eb;
                }
            }
            next = seg_isum<G>(next);
            nq = seg_isum<G>(nq);
            best = seg_fmin<G>(best);
            const bool hist_on = live && nact > 1 && t >= a.hist_t && nq >= 2;
            double thr = kInf;
            __syncwarp();
            if (__any_sync(kFull, hist_on)) {
                const double mu = xdiv(seg_tree_reduce<G>(tree, l), (double)(nq > 0 ? nq : 1));
                __syncwarp();
                for (int r0 = 0; r0 < rows; ++r0) {
                    const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                    const uint32_t key = mkey(meta);
                    if (key == kDeadKey || mn(meta) < a.hist_n) continue;
                    const double dv = xsub(SLOT(r0, P + D + 1), mu);
                    tree[key] = xmul(dv, dv);
                }
                __syncwarp();
                const double sd = xsqrt(xdiv(seg_tree_reduce<G>(tree, l), (double)(nq > 0 ? nq : 1)));
                if (hist_on) thr = xadd(best, xmul(prm.historical_k, sd));
            }
            __syncwarp();
            // clear the scatter slots this lane wrote (+0.0 elsewhere is the invariant)
            for (int r0 = 0; r0 < rows; ++r0) {
                const uint32_t key = mkey((uint64_t)__double_as_longlong(SLOT(r0, P + D + 2)));
                if (key != kDeadKey) tree[key] = 0.0;
            }
            // any removal?
            int nh = 0;
            if (thr < kInf)
                for (int r0 = 0; r0 < rows; ++r0) {
                    const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                    if (mkey(meta) != kDeadKey && mn(meta) >= a.hist_n && SLOT(r0, P + D + 1) > thr) ++nh;
                }
            nh = seg_isum<G>(nh);
            const bool any = live && nact > 1 && (next + nh) > 0;
            if (__any_sync(kFull, any)) {
                int kc = -1;
                for (int r0 = 0; r0 < rows; ++r0) {
                    const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                    const uint32_t key = mkey(meta);
                    if (key == kDeadKey) continue;
                    const uint32_t n = mn(meta);
                    const bool ext = ext_on && n >= a.ext_n && SLOT(r0, P + D) < prm.extreme_reward_threshold;
                    const bool hist = n >= a.hist_n && SLOT(r0, P + D + 1) > thr;
                    const double F = (double)(a.f_min_mhz + key * a.f_step_mhz);
                    if ((ext || hist) && F < a.cascade_limit) kc = max(kc, (int)key);
                }
                kc = seg_max<G>(kc);
                int remaining = 0;
                double br = -kInf;
                int bkey = 0x7fffffff;
                for (int r0 = 0; r0 < rows; ++r0) {
                    const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                    const uint32_t key = mkey(meta);
                    if (key == kDeadKey) continue;
                    const uint32_t n = mn(meta);
                    const double rb = SLOT(r0, P + D);
                    const bool ext = ext_on && n >= a.ext_n && rb < prm.extreme_reward_threshold;
                    const bool hist = n >= a.hist_n && SLOT(r0, P + D + 1) > thr;
                    const bool rm = ext || hist || (int)key < kc;
                    if (!rm) ++remaining;
                    else if (rb > br) { br = rb; bkey = (int)key; }     // AMB-11 candidate (lane-local)
                }
                remaining = seg_isum<G>(remaining);
#pragma unroll
                for (int off = G / 2; off > 0; off >>= 1) {
                    const double ob = __shfl_xor_sync(kFull, br, off, G);
                    const int okk = __shfl_xor_sync(kFull, bkey, off, G);
                    if (ob > br || (ob == br && okk < bkey)) { br = ob; bkey = okk; }
                }
                const int restore = remaining == 0 ? bkey : -1;
                int removed = 0;
                if (any)
                    for (int r0 = 0; r0 < rows; ++r0) {
                        const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
                        const uint32_t key = mkey(meta);
                        if (key == kDeadKey) continue;
                        const uint32_t n = mn(meta);
                        const bool ext = ext_on && n >= a.ext_n && SLOT(r0, P + D) < prm.extreme_reward_threshold;
                        const bool hist = n >= a.hist_n && SLOT(r0, P + D + 1) > thr;
                        const bool cas = !ext && !hist && (int)key < kc;
                        if ((ext || hist || cas) && (int)key != restore) {
                            if (ext) st.n_pruned_extreme++;
                            else if (hist) st.n_pruned_hist++;
                            else st.n_pruned_cascade++;
                            SLOT(r0, P + D + 2) = __longlong_as_double((long long)mpack(kDeadKey, n));
                            ++removed;
                        }
                    }
                nact -= seg_isum<G>(removed);
            }
        }

        // ---- a11 (every lane keeps an identical copy of the scalar stats; counters are
        // lane-local and summed over the segment at write-back)
        if (live) {
            stats_add(st, o, r, v.baseE, v.baseEDP, kstar, (uint32_t)nact0);
            st.near_tie_steps += (near && l == 0) ? 1u : 0u;
        }
        if (live && rec_on && l == 0) {
            if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
            if (a.gap) {
                const double den = fmax(mstar, g_mmax);
                a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] =
                    (g_s2 == -kInf) ? kInf : (den > 0.0 ? (bs - g_s2) / den : 0.0);
            }
        }
        if (a.chosen && live && l == 0) a.chosen[tb] = (uint32_t)kstar;
    }

    // ---- write back: arm j = r·G + l ↔ the j-th key of the launch-start mask
    uint32_t live_w[4] = {0u, 0u, 0u, 0u};
    if (valid) {
        const uint4 m4 = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
        int j = 0;
        for (int wd = 0; wd < 4; ++wd) {
            uint32_t mm = mw[wd];
            while (mm) {
                const int k = 32 * wd + __ffs(mm) - 1;
                mm &= mm - 1u;
                if ((j % G) == l) {
                    const int r0 = j / G;
                    const uint64_t meta = (uint64_t)__double_as_longlong(SLOT(r0, P + D + 2));
#pragma unroll
                    for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + k] = SLOT(r0, e);
#pragma unroll
                    for (int q = 0; q < D; ++q) a.w.theta[((size_t)tb * D + q) * kMaxArms + k] = SLOT(r0, P + q);
                    a.w.rbar[(size_t)tb * kMaxArms + k] = SLOT(r0, P + D);
                    a.w.ebar[(size_t)tb * kMaxArms + k] = SLOT(r0, P + D + 1);
                    a.w.n[(size_t)tb * kMaxArms + k] = mn(meta);
                    if (mkey(meta) != kDeadKey) live_w[k >> 5] |= 1u << (k & 31);
                }
                ++j;
            }
        }
    }
    // OR the live masks and sum the pruning counters over the segment
#pragma unroll
    for (int wd = 0; wd < 4; ++wd)
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) live_w[wd] |= __shfl_xor_sync(kFull, live_w[wd], off, G);
    const int ce = seg_isum<G>((int)st.n_pruned_extreme), ch = seg_isum<G>((int)st.n_pruned_hist),
              cc = seg_isum<G>((int)st.n_pruned_cascade);
    if (valid && l == 0) {
        const agft_tuner_stats st0 = a.w.acc[tb];
        st.n_pruned_extreme = st0.n_pruned_extreme + (ce - G * st0.n_pruned_extreme);
        st.n_pruned_hist = st0.n_pruned_hist + (ch - G * st0.n_pruned_hist);
        st.n_pruned_cascade = st0.n_pruned_cascade + (cc - G * st0.n_pruned_cascade);
        *reinterpret_cast<uint4 *>(a.w.active + (size_t)tb * 4) = make_uint4(live_w[0], live_w[1], live_w[2], live_w[3]);
        for (int j = 0; j < kWindow; ++j) a.w.wsorted[(size_t)tb * kWindow + j] = win.at(j);
        a.w.wmeta[(size_t)tb * 2] = wcount;
        a.w.wmeta[(size_t)tb * 2 + 1] = whead;
        st.n_active = (uint32_t)nact;
        a.w.acc[tb] = st;
    }
#undef SLOT
}

template <int D, int G>
static cudaError_t launch_mseg_dg(const ReplayArgs &a, cudaStream_t s)
{
    constexpr int per_block = kMsegTunersPerBlock;
    const uint32_t blocks = (a.n_tuners + per_block - 1) / per_block;
    mseg_kernel<D, G><<<blocks, kMsegTunersPerBlock * G, 0, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_mseg_d(const ReplayArgs &a, int G, cudaStream_t s)
{
    switch (G) {
    case 2: return launch_mseg_dg<D, 2>(a, s);
    case 8: return launch_mseg_dg<D, 8>(a, s);
    default: return launch_mseg_dg<D, 4>(a, s);
    }
}

cudaError_t launch_mseg(const ReplayArgs &a, uint32_t D, int G, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_mseg_d<1>(a, G, s);
    case 2: return launch_mseg_d<2>(a, G, s);
    case 3: return launch_mseg_d<3>(a, G, s);
    case 4: return launch_mseg_d<4>(a, G, s);
    case 5: return launch_mseg_d<5>(a, G, s);
    case 6: return launch_mseg_d<6>(a, G, s);
    default: return launch_mseg_d<7>(a, G, s);
    }
}

}  // namespace agft
