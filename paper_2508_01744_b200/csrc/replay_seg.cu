// replay_seg.cu — K2/SEG<G>: G lanes per tuner (32/G tuners per warp), for tuners with
// 2 ≤ K_act ≤ G active arms.  The active arms are compacted into the segment's lanes in
// ascending arm order (lane l ↔ l-th active arm) and their A⁻¹/θ live in registers for the
// whole launch.  Scores, the lexicographic argmax, the near-tie test and pruning are
// segment-cooperative (width-G shuffles, segment-masked ballots); the per-tuner scalar work
// (ENV-R, reward, Welford, stats) is executed redundantly by the segment's lanes, so one warp
// instruction serves 32/G tuners.  The sorted EDP window is spread 64/G entries per lane.
// The canonical 128-slot reduction of ENV.md §4.8 is reproduced exactly by scattering the
// segment's values to their arm slots in shared memory and reducing contiguous slot blocks
// per lane, then across lanes (the same pairwise tree, empty slots contributing +0.0).
//
// Control flow is warp-uniform: every collective runs on all 32 lanes; per-segment effects
// are predicated (a segment without a tuner or with a frozen tuner computes but never writes).
#include "step_common.cuh"

namespace agft {

namespace {

constexpr int kSegWarps = 2;

template <int G>
__device__ __forceinline__ uint32_t seg_bits(bool p, int sg)
{
    const uint32_t b = __ballot_sync(kFull, p);
    return G == 32 ? b : (b >> (sg * G)) & ((1u << G) - 1u);
}

template <int G>
__device__ __forceinline__ int seg_popc(bool p, int sg) { return __popc(seg_bits<G>(p, sg)); }

template <int G, typename T>
__device__ __forceinline__ T seg_sum_int(T v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
    return v;
}

// sorted window element idx (entries S[l*E + e] in lane l of the segment)
template <int G, int E>
__device__ __forceinline__ double win_at(const double (&S)[E], uint32_t idx)
{
    double v = S[0];
#pragma unroll
    for (int e = 1; e < E; ++e)
        if ((idx % E) == (uint32_t)e) v = S[e];
    return __shfl_sync(kFull, v, idx / E, G);
}

template <int G, int E>
__device__ __forceinline__ int win_count_less(const double (&S)[E], double v)
{
    int c = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) c += (S[e] < v) ? 1 : 0;
    return seg_sum_int<G>(c);
}

template <int G, int E>
__device__ __forceinline__ void win_remove(double (&S)[E], int po, int l)
{
    double nxt = __shfl_down_sync(kFull, S[0], 1, G);
    if (l == G - 1) nxt = kInf;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = l * E + e;
        const double up = (e + 1 < E) ? S[e + 1 < E ? e + 1 : e] : nxt;
        S[e] = (i < po) ? S[e] : up;
    }
}

template <int G, int E>
__device__ __forceinline__ void win_insert(double (&S)[E], double v, int pi, int l)
{
    const double prv = __shfl_up_sync(kFull, S[E - 1], 1, G);
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
        const int i = l * E + e;
        const double dn = (e > 0) ? S[e > 0 ? e - 1 : 0] : prv;
        S[e] = (i < pi) ? S[e] : ((i == pi) ? v : dn);
    }
}

// canonical 128-slot pairwise sum (ENV.md §4.8) of the segment's (key, value) pairs
template <int G>
__device__ __forceinline__ double seg_tree128(double *buf, int l, bool has, int key, double val)
{
    constexpr int SL = 128 / G;
#pragma unroll
    for (int j = 0; j < SL; ++j) buf[l * SL + j] = 0.0;
    __syncwarp();
    if (has) buf[key] = val;
    __syncwarp();
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
    __syncwarp();
    return s;
}

}  // namespace

template <int D, int G>
__global__ void __launch_bounds__(kSegWarps * 32) seg_kernel(const __grid_constant__ ReplayArgs a)
{
    constexpr int P = D * (D + 1) / 2;
    constexpr int E = kWindow / G;           // window entries per lane
    constexpr int NSEG = 32 / G;
    __shared__ double s_dec[kMaxArms], s_pre[kMaxArms], s_pw[kMaxArms];
    __shared__ double s_tree[kSegWarps * NSEG * kMaxArms];
    const EnvConsts *ec = a.w.env;
    for (int i = threadIdx.x; i < kMaxArms; i += blockDim.x) {
        s_dec[i] = ec->dec[i];
        s_pre[i] = ec->pre[i];
        s_pw[i] = ec->pw[i];
    }
    __syncthreads();
    const double invW = ec->invW, q_over = ec->q_over;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sg = lane / G, l = lane % G;
    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const uint32_t wbase = (blockIdx.x * kSegWarps + warp) * NSEG;
    if (wbase >= cnt) return;                                    // warp-uniform
    const uint32_t idx = wbase + sg;
    const bool valid = idx < cnt;
    const uint32_t tb = a.list ? a.list[valid ? idx : cnt - 1] : (valid ? idx : cnt - 1);
    double *tree = s_tree + (warp * NSEG + sg) * kMaxArms;

    agft_tuner_stats st = a.w.acc[tb];
    bool live = valid && !(st.flags & 1u);
    const agft_tuner_params prm = a.w.params[tb];

    // ---- compact the active arms into the segment's lanes (lane l ↔ l-th active arm)
    int key = 0;
    bool act = false;
    {
        const uint4 m4 = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
        int rem = l;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int c = __popc(mw[w]);
            if (!act && rem < c) {
                uint32_t mm = mw[w];
                for (int j = 0; j < rem; ++j) mm &= mm - 1u;
                key = 32 * w + __ffs(mm) - 1;
                act = true;
            } else if (!act) {
                rem -= c;
            }
        }
    }
    const bool slot = act;                                       // holds an arm (for write-back)
    double A[P], th[D];
    uint32_t n = 0;
    double rbar = 0.0, ebar = 0.0;
#pragma unroll
    for (int e = 0; e < P; ++e) A[e] = slot ? a.w.ainv[((size_t)tb * P + e) * kMaxArms + key] : 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) th[r] = slot ? a.w.theta[((size_t)tb * D + r) * kMaxArms + key] : 0.0;
    if (slot) {
        n = a.w.n[(size_t)tb * kMaxArms + key];
        rbar = a.w.rbar[(size_t)tb * kMaxArms + key];
        ebar = a.w.ebar[(size_t)tb * kMaxArms + key];
    }
    double S[E];
#pragma unroll
    for (int e = 0; e < E; ++e) S[e] = a.w.wsorted[(size_t)tb * kWindow + l * E + e];
    uint32_t wcount = a.w.wmeta[(size_t)tb * 2], whead = a.w.wmeta[(size_t)tb * 2 + 1];
    const uint32_t M = a.median_window;
    double *ring = a.w.wring + (size_t)tb * kWindow;
    double *bg = a.w.b + (size_t)tb * D * kMaxArms;
    int nact = seg_popc<G>(act, sg);
    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;

    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const uint32_t t = a.t0 + s;
        double x[D];
        RecView v;
        load_rec<D>(rp + s, x, v);
        const double alpha = prm.alpha0 / sqrt(1.0 + (double)t / a.tau);

        // ---- a4: Eq. 1 for this lane's arm
        double sc = -kInf, mg = 0.0;
        if (act) {
            double q = 0.0, p = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double zi = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) zi = fma(A[i <= c ? pidx<D>(i, c) : pidx<D>(c, i)], x[c], zi);
                q = fma(x[i], zi, q);
                p = fma(th[i], x[i], p);
            }
            const double bonus = alpha * sqrt(fmax(q, 0.0));
            sc = p + bonus;
            mg = fabs(p) + bonus;
        }
        // ---- a5/a6: lexicographic (s desc, k asc) argmax within the segment
        double bs = sc;
        int bk = act ? (key << 5) | lane : 0x7fffffff;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            const double os = __shfl_xor_sync(kFull, bs, off, G);
            const int ok = __shfl_xor_sync(kFull, bk, off, G);
            if (os > bs || (os == bs && ok < bk)) { bs = os; bk = ok; }
        }
        const int own = (bk & 31) % G;                           // owner lane within the segment
        const int kstar = (bk >> 5) & 127;
        const double mstar = __shfl_sync(kFull, mg, own, G);
        const bool fresh_star = __shfl_sync(kFull, (int)(n == 0u), own, G) != 0;
        const bool tie = act && l != own && (bs - sc < a.tie_rel * fmax(mstar, mg)) && !(fresh_star && n == 0u);
        const bool near = seg_bits<G>(tie, sg) != 0u;
        const int nact0 = nact;                                  // |F_available| before pruning
        double gapv = kInf;                                      // relative top-2 gap (recorded tuners)
        if (a.gap && __any_sync(kFull, rec_on && live)) {
            double s2 = (act && l != own) ? sc : -kInf, m2 = mg;
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const double os = __shfl_xor_sync(kFull, s2, off, G);
                const double om = __shfl_xor_sync(kFull, m2, off, G);
                if (os > s2) { s2 = os; m2 = om; }
            }
            const double den = fmax(mstar, m2);
            gapv = (s2 == -kInf) ? kInf : (den > 0.0 ? (bs - s2) / den : 0.0);
        }

        // ---- a7: response
        const Response o = env_response(s_dec[kstar], s_pre[kstar], s_pw[kstar], v.I, v.P, v.g, v.invIm, v.invAm,
                                        v.wIm, v.nT, v.nE, invW, q_over, a.u_max, a.u_floor, a.p_idle, a.W);
        // ---- a8: reward + window
        double r = 0.0;
        if (wcount > 0) {
            double ref;
            if (wcount & 1u) {
                ref = win_at<G, E>(S, wcount >> 1);
            } else {
                const double m0 = win_at<G, E>(S, (wcount >> 1) - 1), m1 = win_at<G, E>(S, wcount >> 1);
                ref = xmul(xadd(m0, m1), 0.5);
            }
            r = reward_of(o.edp, ref, a.clip_lo, a.clip_hi);
        }
        if (!isfinite(o.edp) || !isfinite(r)) {
            if (live) st.flags |= 1u;
            live = false;
        }
        if (wcount < M) {
            const int pi = win_count_less<G, E>(S, o.edp);
            win_insert<G, E>(S, o.edp, pi, l);
            if (live && l == 0) ring[wcount] = o.edp;
            ++wcount;
        } else {
            const double old = ring[whead];
            const int po = win_count_less<G, E>(S, old);
            win_remove<G, E>(S, po, l);
            const int pi = win_count_less<G, E>(S, o.edp);
            win_insert<G, E>(S, o.edp, pi, l);
            if (live && l == 0) ring[whead] = o.edp;
            whead = (whead + 1 == M) ? 0u : whead + 1;
        }

        // ---- a9: Sherman–Morrison on the owner lane
        if (live && l == own) {
            double b[D];
#pragma unroll
            for (int i = 0; i < D; ++i) b[i] = bg[(size_t)i * kMaxArms + kstar];
            sm_update<D>(A, th, b, x, r);
#pragma unroll
            for (int i = 0; i < D; ++i) bg[(size_t)i * kMaxArms + kstar] = b[i];
            welford(n, rbar, ebar, r, o.edp);
        }

        // ---- a10: pruning (ENV.md §4.8)
        if (a.prune_enable) {
            const bool ext = act && t < a.ext_L && n >= a.ext_n && rbar < prm.extreme_reward_threshold;
            const bool inq = act && n >= a.hist_n;
            const int next = seg_popc<G>(ext, sg), nq = seg_popc<G>(inq, sg);
            const bool need = live && t >= a.hist_t && nq >= 2;
            bool hist = false;
            if (__any_sync(kFull, need)) {
                double best = inq ? ebar : kInf;
#pragma unroll
                for (int off = G / 2; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(kFull, best, off, G));
                const double dq = (double)(nq > 0 ? nq : 1);
                const double mu = xdiv(seg_tree128<G>(tree, l, inq, key, ebar), dq);
                const double dv = xsub(ebar, mu);
                const double sd = xsqrt(xdiv(seg_tree128<G>(tree, l, inq, key, xmul(dv, dv)), dq));
                const double thr = xadd(best, xmul(prm.historical_k, sd));
                hist = need && inq && ebar > thr;
            }
            const int nh = seg_popc<G>(hist, sg);
            const bool any_rm = live && (next + nh) > 0;
            if (__any_sync(kFull, any_rm)) {
                const double F = (double)(a.f_min_mhz + (uint32_t)key * a.f_step_mhz);
                int kc = ((ext || hist) && F < a.cascade_limit) ? key : -1;
#pragma unroll
                for (int off = G / 2; off > 0; off >>= 1) kc = max(kc, __shfl_xor_sync(kFull, kc, off, G));
                const bool cas = act && !ext && !hist && key < kc;
                const int remaining = seg_popc<G>(act && !ext && !hist && !cas, sg);
                const bool cand = ext || hist || cas;
                double br = cand ? rbar : -kInf;
                int bkr = cand ? key : 0x7fffffff;
#pragma unroll
                for (int off = G / 2; off > 0; off >>= 1) {
                    const double ob = __shfl_xor_sync(kFull, br, off, G);
                    const int ok = __shfl_xor_sync(kFull, bkr, off, G);
                    if (ob > br || (ob == br && ok < bkr)) { br = ob; bkr = ok; }
                }
                const int restore = remaining == 0 ? bkr : -1;  // AMB-11
                const bool rm = any_rm && cand && key != restore;
                const int ce = seg_popc<G>(rm && ext, sg);
                const int ch = seg_popc<G>(rm && !ext && hist, sg);
                const int cc = seg_popc<G>(rm && !ext && !hist, sg);
                if (any_rm) {
                    st.n_pruned_extreme += ce;
                    st.n_pruned_hist += ch;
                    st.n_pruned_cascade += cc;
                    nact -= ce + ch + cc;
                }
                if (rm) act = false;
            }
        }

        // ---- a11
        if (live) {
            stats_add(st, o, r, v.baseE, v.baseEDP, kstar, (uint32_t)nact0);
            st.near_tie_steps += near ? 1u : 0u;
        }
        if (live && l == 0 && rec_on) {
            if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
            if (a.gap) a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = gapv;
        }
        if (a.chosen && live && l == 0) a.chosen[tb] = (uint32_t)kstar;
    }

    // ---- write back (segments of real tuners only)
    if (valid) {
        if (slot) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + key] = A[e];
#pragma unroll
            for (int r = 0; r < D; ++r) a.w.theta[((size_t)tb * D + r) * kMaxArms + key] = th[r];
            a.w.n[(size_t)tb * kMaxArms + key] = n;
            a.w.rbar[(size_t)tb * kMaxArms + key] = rbar;
            a.w.ebar[(size_t)tb * kMaxArms + key] = ebar;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) a.w.wsorted[(size_t)tb * kWindow + l * E + e] = S[e];
    }
    uint32_t words[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        uint32_t bits = (act && (key >> 5) == w) ? (1u << (key & 31)) : 0u;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) bits |= __shfl_xor_sync(kFull, bits, off, G);
        words[w] = bits;
    }
    if (valid && l == 0) {
        *reinterpret_cast<uint4 *>(a.w.active + (size_t)tb * 4) = make_uint4(words[0], words[1], words[2], words[3]);
        a.w.wmeta[(size_t)tb * 2] = wcount;
        a.w.wmeta[(size_t)tb * 2 + 1] = whead;
        st.n_active = (uint32_t)nact;
        a.w.acc[tb] = st;
    }
}

template <int D, int G>
static cudaError_t launch_seg_dg(const ReplayArgs &a, cudaStream_t s)
{
    constexpr int per_block = kSegWarps * (32 / G);
    const uint32_t blocks = (a.n_tuners + per_block - 1) / per_block;
    seg_kernel<D, G><<<blocks, kSegWarps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_seg_d(const ReplayArgs &a, int G, cudaStream_t s)
{
    switch (G) {
    case 8: return launch_seg_dg<D, 8>(a, s);
    case 16: return launch_seg_dg<D, 16>(a, s);
    default: return launch_seg_dg<D, 32>(a, s);
    }
}

cudaError_t launch_seg(const ReplayArgs &a, uint32_t D, int G, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_seg_d<1>(a, G, s);
    case 2: return launch_seg_d<2>(a, G, s);
    case 3: return launch_seg_d<3>(a, G, s);
    case 4: return launch_seg_d<4>(a, G, s);
    case 5: return launch_seg_d<5>(a, G, s);
    case 6: return launch_seg_d<6>(a, G, s);
    default: return launch_seg_d<7>(a, G, s);
    }
}

}  // namespace agft
