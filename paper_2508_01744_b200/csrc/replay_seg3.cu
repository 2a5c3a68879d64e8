// replay_seg3.cu — K2/SEG3<G>: the SEG mapping of replay_seg2.cu (G lanes per tuner, 32/G tuners per
// warp, two compacted arms per lane, 2 ≤ K_act ≤ 2G) with the per-step serial chain restructured.
//
// A tuner step is one dependency chain (argmax → ENV-R response → reward → update → pruning → next
// argmax, PAPER §4.2–4.3); with ~8 warps per SM the kernel runs at the speed of that chain, so this
// version shortens it without changing a single result bit of the exact parts (ENV.md §0):
//
//  1. Eq. 1 scores are software-pipelined: step t+1's scores of both slots are computed as soon as
//     step t's update has committed (only the chosen arm changed, PAPER Eqs. 3–5), so they overlap
//     step t's pruning pass instead of heading step t+1's chain.
//  2. Sherman–Morrison is split at its data dependency: z = A⁻¹x, δ = 1 + xᵀA⁻¹x and the new A⁻¹
//     entries do not depend on the reward, so they are computed right after the argmax, next to the
//     response; only θ += z(r − θᵀx)/δ and b += r x wait for r.  z and the A⁻¹ update are spread
//     over the segment's lanes (lane i computes z_i from the owner's column; each lane rewrites
//     ⌈P/G⌉ packed entries) instead of running on the owner lane alone.  δ reuses the chosen arm's
//     quadratic form from the scores and θᵀx its linear part (the same quantities, PAPER Eq. 1/5).
//  3. Historical pruning is screened: one butterfly gives min, max, Σē and Σē² over Q; from
//     them an approximate threshold with a rigorous rounding bound decides "no arm
//     can exceed best + k·σ" in the common case.  Only when an arm might be removed — a real
//     removal, or a mean within the bound of the threshold — does the warp run the exact canonical
//     128-slot trees of ENV.md §4.8 (identical to SEG2), so every pruning decision is bit-identical.
#include "seg_common.cuh"

namespace agft {

namespace {

#ifndef AGFT_SEG3_WARPS
#define AGFT_SEG3_WARPS 2
#endif
constexpr int kSeg3Warps = AGFT_SEG3_WARPS;
#ifndef AGFT_SEG3_MIN_BLOCKS
#define AGFT_SEG3_MIN_BLOCKS 4
#endif
constexpr int kSeg3MinBlocks = AGFT_SEG3_MIN_BLOCKS;
constexpr int kAS = 33;                 // A⁻¹ / b smem stride per packed entry (odd: the owner-column
                                        // reads of the distributed update fall in different banks)

template <int G>
__host__ __device__ constexpr bool env3_in_smem() { return G >= 8; }

template <int G>
constexpr size_t seg3_smem_bytes(int P, int D)
{
    return ((env3_in_smem<G>() ? 3 * kMaxArms : 0) + (size_t)kSeg3Warps * 2 * P * kAS +
            (size_t)kSeg3Warps * 2 * D * kAS + (size_t)kSeg3Warps * (32 / G) * tree_stride<G>()) * 8 +
           (size_t)kSeg3Warps * (32 / G) * sizeof(agft_tuner_stats);
}

// Eq. 1 score of one slot at x, with the packed quadratic form (and its magnitude, ENV.md §4.5)
template <int D, int P>
__device__ __forceinline__ void score_slot(bool act, const double (&w)[P], const double *Acol, const double (&th)[D],
                                           const double (&x)[D], double alpha, double &sc, double &mg)
{
    sc = -kInf;
    mg = 0.0;
    if (act) {
        const double q = quad_form<P>(w, Acol, kAS);
        double pp = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) pp = fma(th[i], x[i], pp);
        const double bonus = alpha * sqrt(fmax(q, 0.0));   // AMB-19
        sc = pp + bonus;
        mg = fabs(pp) + bonus;
    }
}

}  // namespace

template <int D, int G>
__global__ void __launch_bounds__(kSeg3Warps * 32, kSeg3MinBlocks) seg3_kernel(const __grid_constant__ ReplayArgs a)
{
    constexpr int P = D * (D + 1) / 2;
    constexpr int E = kWindow / G;
    constexpr int NSEG = 32 / G;
    constexpr int NE = (P + G - 1) / G;                              // packed entries per lane (update)
    extern __shared__ double sm[];
    constexpr bool kEnvS = env3_in_smem<G>();
    double *s_dec = sm, *s_pre = sm + kMaxArms, *s_pw = sm + 2 * kMaxArms;
    double *s_A = sm + (kEnvS ? 3 * kMaxArms : 0);                     // [warp][slot][P][kAS]
    double *s_B = s_A + kSeg3Warps * 2 * P * kAS;                      // [warp][slot][D][kAS]
    double *s_tree = s_B + kSeg3Warps * 2 * D * kAS;                   // [warp][seg][tree_stride]
    agft_tuner_stats *s_st = reinterpret_cast<agft_tuner_stats *>(s_tree + kSeg3Warps * NSEG * tree_stride<G>());
    const EnvConsts *ec = a.w.env;
    if (kEnvS) {
        for (int q = threadIdx.x; q < kMaxArms; q += blockDim.x) {
            s_dec[q] = ec->dec[q];
            s_pre[q] = ec->pre[q];
            s_pw[q] = ec->pw[q];
        }
    }
    for (int q = threadIdx.x; q < kSeg3Warps * NSEG * tree_stride<G>(); q += blockDim.x) s_tree[q] = 0.0;
    __syncthreads();
    const double invW = ec->invW, q_over = ec->q_over;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sg = lane / G, l = lane % G;
    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const uint32_t wbase = (blockIdx.x * kSeg3Warps + warp) * NSEG;
    if (wbase >= cnt) return;                                         // warp-uniform
    const uint32_t idx = wbase + sg;
    const bool valid = idx < cnt;
    const uint32_t tb = a.list ? a.list[valid ? idx : cnt - 1] : (valid ? idx : cnt - 1);
    double *tree = s_tree + (warp * NSEG + sg) * tree_stride<G>();
    double *A0 = s_A + (warp * 2 + 0) * P * kAS + lane;               // slot 0 column of this lane
    double *A1 = s_A + (warp * 2 + 1) * P * kAS + lane;
    double *B0 = s_B + (warp * 2 + 0) * D * kAS + lane;
    double *B1 = s_B + (warp * 2 + 1) * D * kAS + lane;
    agft_tuner_stats &st = s_st[warp * NSEG + sg];
    if (l == 0) st = a.w.acc[tb];
    __syncwarp();
    bool live = valid && !(st.flags & 1u);
    __shared__ PhState s_ph[kSeg3Warps * (32 / G)];
    PhState &ph = s_ph[warp * NSEG + sg];
    uint32_t phase = 0u;
    if (a.ph_enable) {
        if (l == 0) ph = a.w.ph[tb];
        __syncwarp();
        phase = ph.phase;
    }
    const agft_tuner_params prm = a.w.params[tb];

    // per-lane index tables of the distributed Sherman–Morrison update:
    //   zoff[c] = packed index of (l, c) (row l of the owner's A⁻¹, lanes l < D compute z_l),
    //   entries e = l + G·j of the packed triangle (row er[j], column ec_[j]) rewritten by this lane
    int zoff[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        const int r0 = l < c ? l : c, c0 = l < c ? c : l;
        zoff[c] = (l < D) ? (r0 * D - r0 * (r0 - 1) / 2 + (c0 - r0)) * kAS : 0;
    }
    // (row, column) of packed entry e, for the lanes' share of the A⁻¹ rewrite: s_rc[e] = row | col << 8
    __shared__ uint16_t s_rc[P];
    if (threadIdx.x < P) {
        int r0 = 0, rem = threadIdx.x;
        while (r0 < D - 1 && rem >= D - r0) { rem -= D - r0; ++r0; }
        s_rc[threadIdx.x] = (uint16_t)(r0 | ((r0 + rem) << 8));
    }
    __syncthreads();

    // ---- compact the active arms: lane l ← active-order arms l and G + l
    int key0 = 0, key1 = 0;
    bool act0 = false, act1 = false;
    {
        const uint4 m4 = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
        int j = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t mm = mw[w];
            while (mm) {
                const int k = 32 * w + __ffs(mm) - 1;
                mm &= mm - 1u;
                if (j == l) { key0 = k; act0 = true; }
                if (j == G + l) { key1 = k; act1 = true; }
                ++j;
            }
        }
    }
    const bool has0 = act0, has1 = act1;
    double th0[D], th1[D];
    uint32_t n0 = 0, n1 = 0;
    double rb0 = 0.0, rb1 = 0.0, eb0 = 0.0, eb1 = 0.0;
    double *bg = a.w.b + (size_t)tb * D * kMaxArms;
#pragma unroll
    for (int e = 0; e < P; ++e) {
        A0[e * kAS] = has0 ? a.w.ainv[((size_t)tb * P + e) * kMaxArms + key0] : 0.0;
        A1[e * kAS] = has1 ? a.w.ainv[((size_t)tb * P + e) * kMaxArms + key1] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
        th0[r] = has0 ? a.w.theta[((size_t)tb * D + r) * kMaxArms + key0] : 0.0;
        th1[r] = has1 ? a.w.theta[((size_t)tb * D + r) * kMaxArms + key1] : 0.0;
        B0[r * kAS] = has0 ? bg[(size_t)r * kMaxArms + key0] : 0.0;
        B1[r * kAS] = has1 ? bg[(size_t)r * kMaxArms + key1] : 0.0;
    }
    if (has0) {
        n0 = a.w.n[(size_t)tb * kMaxArms + key0];
        rb0 = a.w.rbar[(size_t)tb * kMaxArms + key0];
        eb0 = a.w.ebar[(size_t)tb * kMaxArms + key0];
    }
    if (has1) {
        n1 = a.w.n[(size_t)tb * kMaxArms + key1];
        rb1 = a.w.rbar[(size_t)tb * kMaxArms + key1];
        eb1 = a.w.ebar[(size_t)tb * kMaxArms + key1];
    }
    double S[E];
#pragma unroll
    for (int e = 0; e < E; ++e) S[e] = a.w.wsorted[(size_t)tb * kWindow + l * E + e];
    uint32_t wcount = a.w.wmeta[(size_t)tb * 2], whead = a.w.wmeta[(size_t)tb * 2 + 1];
    const uint32_t M = a.median_window;
    double *ring = a.w.wring + (size_t)tb * kWindow;
    double oldest = wcount == M ? ring[whead] : 0.0;
    int nact = spopc<G>(act0, sg) + spopc<G>(act1, sg);
    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;
    const double inv_tau = 1.0 / a.tau;
    const uint32_t *rawp = a.cl_enable ? a.raw + ((size_t)prm.trace_id * a.rec_stride + a.rec_off) * AGFT_ROW_WORDS
                                       : nullptr;
    uint32_t clq = 0u, clqb = 0u;
    if (rawp) {
        clq = a.w.clq[(size_t)tb * 2];
        clqb = a.w.clq[(size_t)tb * 2 + 1];
    }
    __syncwarp();

    // ---- the window's inputs: context x and the record fields the step consumes (ENV.md §3.2);
    // under ENV-C the tuner's and the baseline's server see their backlogs (§6)
    double x[D];
    double g, wIm, baseE, baseEDP, xl;
    uint32_t arr_cl = 0u;
    auto load_window = [&](uint32_t s) {
        const StepRec *rc = rp + s;
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = __ldg(&rc->x[i]);
        g = __ldg(&rc->g);
        wIm = __ldg(&rc->wIm);
        baseE = __ldg(&rc->baseE);
        baseEDP = __ldg(&rc->baseEDP);
        if (rawp) {
            const ClosedRec cr = closed_record(rawp + (size_t)s * AGFT_ROW_WORDS, clq, clqb, __ldg(&rc->I),
                                               __ldg(&rc->P), __ldg(&rc->invIm), __ldg(&rc->nT), __ldg(&rc->nE),
                                               ec, a);
            x[0] = cr.x0;
            g = cr.g;
            wIm = cr.wIm;
            baseE = cr.baseE;
            baseEDP = cr.baseEDP;
            arr_cl = cr.arr;
        }
        xl = 0.0;                                                     // x_l for the lane's b / z row
#pragma unroll
        for (int i = 0; i < D; ++i) xl = (l == i) ? x[i] : xl;
    };
    // Eq. 1 scores of both slots at the current x (state after the last committed update)
    double sc0, sc1, mg0, mg1;
    auto score_both = [&](uint32_t t) {
        const double alpha = phase ? 0.0 : alpha_t(prm.alpha0, t, inv_tau);   // Exploitation: Eq. 2
        double w[P];
        pair_weights<D>(x, w);
        score_slot<D, P>(act0, w, A0, th0, x, alpha, sc0, mg0);
        score_slot<D, P>(act1, w, A1, th1, x, alpha, sc1, mg1);
    };
    if (a.n_steps > 0) {
        load_window(0);
        score_both(a.t0);
    }

    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const uint32_t t = a.t0 + s;
        const StepRec *rc = rp + s;
        if (s + 1 < a.n_steps && l == 0) {
            prefetch_l1(rc + 1);
            if (rawp) prefetch_l1(rawp + (size_t)(s + 1) * AGFT_ROW_WORDS);
        }
        // off the chain: the reward's reference (median before this push) and Welford's 1/n
        double ref = 0.0;
        if (wcount > 0) {
            if (wcount & 1u) {
                ref = wat<G, E>(S, wcount >> 1);
            } else {
                const double m0 = wat<G, E>(S, (wcount >> 1) - 1), m1 = wat<G, E>(S, wcount >> 1);
                ref = xmul(xadd(m0, m1), 0.5);
            }
        }

        // ---- a5/a6: argmax of the (pipelined) scores over the active slots
        const bool pick1 = sc1 > sc0;
        double bs = pick1 ? sc1 : sc0;
        int bk = act0 || act1 ? (((pick1 ? key1 : key0) << 6) | (pick1 ? 32 : 0) | lane) : 0x7fffffff;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            const double os = __shfl_xor_sync(kFull, bs, off, G);
            const int ok = __shfl_xor_sync(kFull, bk, off, G);
            if (os > bs || (os == bs && ok < bk)) { bs = os; bk = ok; }
        }
        const int kstar = (bk >> 6) & 127;
        const int own = (bk & 31) % G;
        const int oslot = (bk >> 5) & 1;
        const bool is_own = (l == own);
        const double mstar = __shfl_sync(kFull, oslot ? mg1 : mg0, own, G);
        const uint32_t nstar = __shfl_sync(kFull, oslot ? n1 : n0, own, G);
        const bool fstar = nstar == 0u;
        const bool own0 = is_own && oslot == 0, own1 = is_own && oslot == 1;
        const double inv_n = xdiv(1.0, (double)(nstar + 1u));            // Welford's 1/n, off the chain
        const bool tie = (act0 && !own0 && (bs - sc0 < a.tie_rel * fmax(mstar, mg0)) && !(fstar && n0 == 0u)) ||
                         (act1 && !own1 && (bs - sc1 < a.tie_rel * fmax(mstar, mg1)) && !(fstar && n1 == 0u));
        const bool near = sbits<G>(tie, sg) != 0u;
        const int nact0 = nact;
        double gapv = kInf;
        if (a.gap && __any_sync(kFull, rec_on && live)) {
            double s2 = fmax(act0 && !own0 ? sc0 : -kInf, act1 && !own1 ? sc1 : -kInf);
            double m2 = (act0 && !own0 && sc0 == s2) ? mg0 : mg1;
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const double os = __shfl_xor_sync(kFull, s2, off, G);
                const double om = __shfl_xor_sync(kFull, m2, off, G);
                if (os > s2) { s2 = os; m2 = om; }
            }
            const double den = fmax(mstar, m2);
            gapv = (s2 == -kInf) ? kInf : (den > 0.0 ? (bs - s2) / den : 0.0);
        }

        // ---- a9, reward-independent half (distributed over the segment, off the response → reward
        // chain): z = A⁻¹x from the owner's column (lane i < D computes z_i), δ = 1 + xᵀz; the owner
        // forms θᵀx of its chosen slot
        const double *colA = s_A + (warp * 2 + oslot) * P * kAS + sg * G + own;
        double zl = 0.0;
        if (l < D) {
#pragma unroll
            for (int c = 0; c < D; ++c) zl = fma(colA[zoff[c]], x[c], zl);
        }
        double xz = xl * zl;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) xz += __shfl_xor_sync(kFull, xz, off, G);
        const double invd = 1.0 / (1.0 + xz);                           // Sherman–Morrison denominator
        double pstar = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) pstar = fma(oslot ? th1[i] : th0[i], x[i], pstar);

        // ---- a7: response
        const Response o = env_response(kEnvS ? s_dec[kstar] : __ldg(&ec->dec[kstar]),
                                        kEnvS ? s_pre[kstar] : __ldg(&ec->pre[kstar]),
                                        kEnvS ? s_pw[kstar] : __ldg(&ec->pw[kstar]), __ldg(&rc->I), __ldg(&rc->P),
                                        g, __ldg(&rc->invIm), __ldg(&rc->invAm), wIm,
                                        __ldg(&rc->nT), __ldg(&rc->nE), invW, q_over, a.u_max, a.u_floor,
                                        a.p_idle, a.W);
        if (rawp) clq = closed_carry(arr_cl + clq, o.u, a.cl_q_max);
        const double cur_baseE = baseE, cur_baseEDP = baseEDP;
        // ---- a8: reward
        double r = 0.0;
        if (wcount > 0) r = reward_of(o.edp, ref, a.clip_lo, a.clip_hi);
        if (!isfinite(o.edp) || !isfinite(r)) {
            if (live && l == 0) st.flags |= 1u;
            live = false;
        }
        if (a.ph_enable) {                                            // ENV.md §4.10 observe_reward
            if (live && l == 0) {
                ph.exploit_steps += phase;
                ph_observe(ph, r, t, a.ph_window, a.ph_delta, a.ph_lambda);
            }
            __syncwarp();
            phase = ph.phase;
        }
        // ---- a9, reward-dependent half + commit: A⁻¹ entries, b_i += r x_i (lane i), θ and Welford (owner)
        const double coef = (r - pstar) * invd;                         // RLS form of θ = A⁻¹ b (AMB-21)
        double anew[NE];                                                // this lane's packed entries
#pragma unroll
        for (int j = 0; j < NE; ++j) {
            const int e = l + G * j;
            const int rc_ = s_rc[e < P ? e : 0];
            const double zr = __shfl_sync(kFull, zl, rc_ & 0xff, G);
            const double zc = __shfl_sync(kFull, zl, rc_ >> 8, G);
            anew[j] = (e < P) ? fma(-zr * invd, zc, colA[(e < P ? e : 0) * kAS]) : 0.0;
        }
        __syncwarp();                                                   // owner-column reads done before the writes
        if (live) {
            double *wA = s_A + (warp * 2 + oslot) * P * kAS + sg * G + own;
#pragma unroll
            for (int j = 0; j < NE; ++j)
                if (l + G * j < P) wA[(l + G * j) * kAS] = anew[j];
            if (l < D) {
                double &bi = s_B[(warp * 2 + oslot) * D * kAS + l * kAS + sg * G + own];
                bi = xadd(bi, xmul(r, xl));                           // b exact, as Eq. 4 writes it
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const double zi = __shfl_sync(kFull, zl, i, G);
            if (live && own0) th0[i] = fma(zi, coef, th0[i]);
            if (live && own1) th1[i] = fma(zi, coef, th1[i]);
        }
        if (live && own0) welford_inv(n0, rb0, eb0, r, o.edp, inv_n);
        if (live && own1) welford_inv(n1, rb1, eb1, r, o.edp, inv_n);
        __syncwarp();

        // ---- the EDP window (median reference of the next step)
        if (wcount < M) {
            winsert<G, E>(S, o.edp, wless<G, E>(S, o.edp), l);
            if (live && l == 0) ring[wcount] = o.edp;
            ++wcount;
            if (wcount == M) oldest = M == 1 ? o.edp : ring[whead];
        } else {
            const double old = oldest;
            int c = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) c += ((S[e] < old) ? 1 : 0) + ((S[e] < o.edp) ? 0x10000 : 0);
            c = sisum<G>(c);
            const int po = c & 0xffff, pv = (c >> 16) - ((old < o.edp) ? 1 : 0);
            wremove<G, E>(S, po, l);
            winsert<G, E>(S, o.edp, pv, l);
            if (live && l == 0) ring[whead] = o.edp;
            whead = (whead + 1 == M) ? 0u : whead + 1;
            oldest = M == 1 ? o.edp : ring[whead];
        }

        // ---- software pipeline: step t+1's window inputs and Eq. 1 scores (state after this update)
        if (s + 1 < a.n_steps) {
            load_window(s + 1);
            score_both(t + 1);
        }

        // ---- a10: pruning (ENV.md §4.8) on the post-update state
        if (a.prune_enable) {
            const bool eon = t < a.ext_L;
            const bool ext0 = act0 && eon && n0 >= a.ext_n && rb0 < prm.extreme_reward_threshold;
            const bool ext1 = act1 && eon && n1 >= a.ext_n && rb1 < prm.extreme_reward_threshold;
            const bool q0 = act0 && n0 >= a.hist_n, q1 = act1 && n1 >= a.hist_n;
            const int next = spopc<G>(ext0, sg) + spopc<G>(ext1, sg);
            const int nq = spopc<G>(q0, sg) + spopc<G>(q1, sg);
            const bool need = live && t >= a.hist_t && nq >= 2;
            // screen: min, max, Σē, Σē² over Q in one butterfly; "no arm of Q can
            // exceed best + k·σ" is decided from them when it holds with a margin larger than the
            // rounding bound of either evaluation; otherwise (or when an arm is Extreme) → exact pass
            bool exact_me = live && next > 0;
            if (__any_sync(kFull, need)) {
                double mn = fmin(q0 ? eb0 : kInf, q1 ? eb1 : kInf);
                double mx = fmax(q0 ? eb0 : -kInf, q1 ? eb1 : -kInf);
                double s1 = (q0 ? eb0 : 0.0) + (q1 ? eb1 : 0.0);
                double s2 = (q0 ? eb0 * eb0 : 0.0) + (q1 ? eb1 * eb1 : 0.0);
#pragma unroll
                for (int off = G / 2; off > 0; off >>= 1) {
                    mn = fmin(mn, __shfl_xor_sync(kFull, mn, off, G));
                    mx = fmax(mx, __shfl_xor_sync(kFull, mx, off, G));
                    s1 += __shfl_xor_sync(kFull, s1, off, G);
                    s2 += __shfl_xor_sync(kFull, s2, off, G);
                }
                if (need && mx > mn) {                                // all equal: thr ≥ best = max, none removed
                    const double inq = 1.0 / (double)nq;
                    const double mu = s1 * inq, m2 = s2 * inq;
                    const double V = m2 - mu * mu;
                    bool safe = false;
                    if (V > 0.0) {
                        constexpr double u = 1.1102230246251565e-16;  // 2^-53
                        const double sd = sqrt(V);
                        const double thr = mn + prm.historical_k * sd;
                        const double dV = 256.0 * u * m2;              // |V_approx − V_exact| bound (×4 margin)
                        const double delta = prm.historical_k * (dV / sd + 8.0 * u * sd) + 8.0 * u * fabs(thr);
                        safe = mx < thr - 2.0 * delta;
                    }
                    exact_me = exact_me || !safe;
                }
            }
            if (__any_sync(kFull, exact_me)) {
                bool hist0 = false, hist1 = false;
                if (__any_sync(kFull, need)) {
                    double best = fmin(q0 ? eb0 : kInf, q1 ? eb1 : kInf);
#pragma unroll
                    for (int off = G / 2; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(kFull, best, off, G));
                    const double dq = (double)(nq > 0 ? nq : 1);
                    const double mu = xdiv(stree<G>(tree, l, q0, key0, eb0, q1, key1, eb1), dq);
                    const double d0 = xsub(eb0, mu), d1 = xsub(eb1, mu);
                    const double sd = xsqrt(xdiv(stree<G>(tree, l, q0, key0, xmul(d0, d0), q1, key1, xmul(d1, d1)), dq));
                    const double thr = xadd(best, xmul(prm.historical_k, sd));
                    hist0 = need && q0 && eb0 > thr;
                    hist1 = need && q1 && eb1 > thr;
                }
                const int nh = spopc<G>(hist0, sg) + spopc<G>(hist1, sg);
                const bool any_rm = live && (next + nh) > 0;
                if (__any_sync(kFull, any_rm)) {
                    int kc = -1;
                    if ((ext0 || hist0) && (double)(a.f_min_mhz + (uint32_t)key0 * a.f_step_mhz) < a.cascade_limit) kc = key0;
                    if ((ext1 || hist1) && (double)(a.f_min_mhz + (uint32_t)key1 * a.f_step_mhz) < a.cascade_limit) kc = max(kc, key1);
#pragma unroll
                    for (int off = G / 2; off > 0; off >>= 1) kc = max(kc, __shfl_xor_sync(kFull, kc, off, G));
                    const bool cas0 = act0 && !ext0 && !hist0 && key0 < kc;
                    const bool cas1 = act1 && !ext1 && !hist1 && key1 < kc;
                    const bool c0 = ext0 || hist0 || cas0, c1 = ext1 || hist1 || cas1;
                    const int remaining = spopc<G>(act0 && !c0, sg) + spopc<G>(act1 && !c1, sg);
                    double br = -kInf;
                    int bkr = 0x7fffffff;
                    if (c0) { br = rb0; bkr = key0; }
                    if (c1 && rb1 > br) { br = rb1; bkr = key1; }
#pragma unroll
                    for (int off = G / 2; off > 0; off >>= 1) {
                        const double ob = __shfl_xor_sync(kFull, br, off, G);
                        const int ok = __shfl_xor_sync(kFull, bkr, off, G);
                        if (ob > br || (ob == br && ok < bkr)) { br = ob; bkr = ok; }
                    }
                    const int restore = remaining == 0 ? bkr : -1;   // AMB-11
                    const bool rm0 = any_rm && c0 && key0 != restore, rm1 = any_rm && c1 && key1 != restore;
                    const int ce = spopc<G>(rm0 && ext0, sg) + spopc<G>(rm1 && ext1, sg);
                    const int ch = spopc<G>(rm0 && !ext0 && hist0, sg) + spopc<G>(rm1 && !ext1 && hist1, sg);
                    const int cc = spopc<G>(rm0 && !ext0 && !hist0, sg) + spopc<G>(rm1 && !ext1 && !hist1, sg);
                    if (any_rm) {
                        if (l == 0) {
                            st.n_pruned_extreme += ce;
                            st.n_pruned_hist += ch;
                            st.n_pruned_cascade += cc;
                        }
                        nact -= ce + ch + cc;
                    }
                    if (a.rf_enable) {
                        if (rm0 && ext0) atomicOr(a.w.extm + (size_t)tb * 4 + (key0 >> 5), 1u << (key0 & 31));
                        if (rm1 && ext1) atomicOr(a.w.extm + (size_t)tb * 4 + (key1 >> 5), 1u << (key1 & 31));
                    }
                    if (rm0) {
                        act0 = false;
                        sc0 = -kInf;                                  // pipelined score of a removed arm
                        tree[tslot<G>(key0)] = 0.0;
                    }
                    if (rm1) {
                        act1 = false;
                        sc1 = -kInf;
                        tree[tslot<G>(key1)] = 0.0;
                    }
                }
            }
        }

        // ---- a11
        if (live && l == 0) {
            stats_add(st, o, r, cur_baseE, cur_baseEDP, kstar, (uint32_t)nact0);
            st.near_tie_steps += near ? 1u : 0u;
            if (rec_on) {
                if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
                if (a.gap) a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = gapv;
            }
            if (a.chosen) a.chosen[tb] = (uint32_t)kstar;
        }
    }

    // ---- write back (segments of real tuners only)
    __syncwarp();
    if (valid) {
        if (has0) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + key0] = A0[e * kAS];
#pragma unroll
            for (int r = 0; r < D; ++r) {
                a.w.theta[((size_t)tb * D + r) * kMaxArms + key0] = th0[r];
                bg[(size_t)r * kMaxArms + key0] = B0[r * kAS];
            }
            a.w.n[(size_t)tb * kMaxArms + key0] = n0;
            a.w.rbar[(size_t)tb * kMaxArms + key0] = rb0;
            a.w.ebar[(size_t)tb * kMaxArms + key0] = eb0;
        }
        if (has1) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + key1] = A1[e * kAS];
#pragma unroll
            for (int r = 0; r < D; ++r) {
                a.w.theta[((size_t)tb * D + r) * kMaxArms + key1] = th1[r];
                bg[(size_t)r * kMaxArms + key1] = B1[r * kAS];
            }
            a.w.n[(size_t)tb * kMaxArms + key1] = n1;
            a.w.rbar[(size_t)tb * kMaxArms + key1] = rb1;
            a.w.ebar[(size_t)tb * kMaxArms + key1] = eb1;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) a.w.wsorted[(size_t)tb * kWindow + l * E + e] = S[e];
    }
    uint32_t words[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        uint32_t bits = ((act0 && (key0 >> 5) == w) ? (1u << (key0 & 31)) : 0u) |
                        ((act1 && (key1 >> 5) == w) ? (1u << (key1 & 31)) : 0u);
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) bits |= __shfl_xor_sync(kFull, bits, off, G);
        words[w] = bits;
    }
    if (valid && l == 0) {
        *reinterpret_cast<uint4 *>(a.w.active + (size_t)tb * 4) = make_uint4(words[0], words[1], words[2], words[3]);
        if (rawp) {
            a.w.clq[(size_t)tb * 2] = clq;
            a.w.clq[(size_t)tb * 2 + 1] = clqb;
        }
        a.w.wmeta[(size_t)tb * 2] = wcount;
        a.w.wmeta[(size_t)tb * 2 + 1] = whead;
        st.n_active = (uint32_t)nact;
        if (a.ph_enable) {
            a.w.ph[tb] = ph;
            ph_to_stats(ph, st);
        }
        a.w.acc[tb] = st;
    }
}

template <int D, int G>
static cudaError_t launch_seg3_dg(const ReplayArgs &a, cudaStream_t s)
{
    constexpr int P = D * (D + 1) / 2;
    constexpr int per_block = kSeg3Warps * (32 / G);
    const size_t smem = seg3_smem_bytes<G>(P, D);
    auto kern = seg3_kernel<D, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t blocks = (a.n_tuners + per_block - 1) / per_block;
    kern<<<blocks, kSeg3Warps * 32, smem, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_seg3_d(const ReplayArgs &a, int G, cudaStream_t s)
{
    switch (G) {
    case 4: return launch_seg3_dg<D, 4>(a, s);
    case 32: return launch_seg3_dg<D, 32>(a, s);
    case 8: return launch_seg3_dg<D, 8>(a, s);
    default: return launch_seg3_dg<D, 16>(a, s);
    }
}

cudaError_t launch_seg3(const ReplayArgs &a, uint32_t D, int G, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_seg3_d<1>(a, G, s);
    case 2: return launch_seg3_d<2>(a, G, s);
    case 3: return launch_seg3_d<3>(a, G, s);
    case 4: return launch_seg3_d<4>(a, G, s);
    case 5: return launch_seg3_d<5>(a, G, s);
    case 6: return launch_seg3_d<6>(a, G, s);
    default: return launch_seg3_d<7>(a, G, s);
    }
}

}  // namespace agft
