// replay_seg2.cu — K2/SEG<G>: G lanes per tuner (32/G tuners per warp), TWO compacted arms
// per lane, for tuners with 2 ≤ K_act ≤ 2G active arms (G = 4, 8, 16 → K ≤ 8, 16, 32).
//
// Why two arms per lane: the per-tuner scalar work of a step (ENV-R response, reward
// median, Sherman–Morrison, Welford, stats) is one warp instruction stream shared by the
// 32/G tuners of a warp, so halving G halves its cost per tuner-step; scoring costs the same
// lane-instructions either way.  Packed A⁻¹ of both slots lives in shared
// memory ([warp][slot][entry][lane], conflict-free), θ/n/r̄/ē/key in registers, per-segment
// stats in shared memory (lane 0 of the segment owns them), so registers stay low enough for
// ~10–12 warps per SM.
//
// Arm order: lane l holds active-order arms j = l (slot 0) and j = G + l (slot 1), so keys
// ascend along (slot, lane) and the lexicographic argmax compares (score desc, key asc).
// The canonical 128-slot reduction of ENV.md §4.8: values are scattered to their arm slots
// in a per-segment shared array, each lane reduces an aligned 128/G-slot block pairwise, and a
// width-G butterfly combines the blocks — the same pairwise tree, empty slots adding +0.0.
// Control flow is warp-uniform around every collective; per-segment effects are predicated.
#include "seg_common.cuh"
#include "rec_tile.cuh"

namespace agft {

namespace {

#ifndef AGFT_SEG2_WARPS
#define AGFT_SEG2_WARPS 2               // warps per block (A/B knob)
#endif
constexpr int kSeg2Warps = AGFT_SEG2_WARPS;
#ifndef AGFT_SEG2_MIN_BLOCKS
#define AGFT_SEG2_MIN_BLOCKS 4          // no effective register cap: spills cost more than occupancy gains (A/B)
#endif
constexpr int kSeg2MinBlocks = AGFT_SEG2_MIN_BLOCKS;

// b of both slots is staged in shared memory next to A⁻¹: its read-modify-write in the
// Sherman–Morrison step is on the serial chain, and a global-memory round trip there stalled the
// warp (ncu source attribution).  For G = 4 (eight tree buffers per warp) it fits
// at 4 blocks per SM only if the per-arm ENV-R constants are read through L1 instead of staged.
template <int G>
__host__ __device__ constexpr bool b_in_smem() { return true; }
template <int G>
__host__ __device__ constexpr bool env_in_smem() { return G >= 8; }

#ifndef AGFT_SCREEN_MIN_G
#define AGFT_SCREEN_MIN_G 8             // the screen for G ≥ this (A/B knob)
#endif
template <int G>
__host__ __device__ constexpr bool kScreen() { return G >= AGFT_SCREEN_MIN_G; }

template <int G>
constexpr size_t seg2_smem_bytes(int P, int D)
{
    return ((env_in_smem<G>() ? 3 * kMaxArms : 0) + (size_t)kSeg2Warps * 2 * P * 32 +
            (size_t)kSeg2Warps * (32 / G) * tree_stride<G>()) * 8 +
           (size_t)kSeg2Warps * (32 / G) * sizeof(agft_tuner_stats) +
           (b_in_smem<G>() ? (size_t)kSeg2Warps * 2 * D * 32 * 8 : 0);
}

}  // namespace

template <int D, int G>
__global__ void __launch_bounds__(kSeg2Warps * 32, kSeg2MinBlocks) seg2_kernel(const __grid_constant__ ReplayArgs a)
{
    const TlGuard tl_guard(a);
    constexpr int P = D * (D + 1) / 2;
    constexpr int E = kWindow / G;
    constexpr int NSEG = 32 / G;
    extern __shared__ double sm[];
    constexpr bool kEnvS = env_in_smem<G>();
    double *s_dec = sm, *s_pre = sm + kMaxArms, *s_pw = sm + 2 * kMaxArms;
    double *s_A = sm + (kEnvS ? 3 * kMaxArms : 0);                     // [warp][slot][P][32]
    double *s_tree = s_A + kSeg2Warps * 2 * P * 32;                    // [warp][seg][tree_stride]
    agft_tuner_stats *s_st = reinterpret_cast<agft_tuner_stats *>(s_tree + kSeg2Warps * NSEG * tree_stride<G>());
    double *s_B = reinterpret_cast<double *>(s_st + kSeg2Warps * NSEG);  // [warp][slot][D][32] (G ≥ 8)
    const EnvConsts *ec = a.w.env;
    if (kEnvS) {
        for (int q = threadIdx.x; q < kMaxArms; q += blockDim.x) {
            s_dec[q] = ec->dec[q];
            s_pre[q] = ec->pre[q];
            s_pw[q] = ec->pw[q];
        }
    }
    for (int q = threadIdx.x; q < kSeg2Warps * NSEG * tree_stride<G>(); q += blockDim.x) s_tree[q] = 0.0;
    __syncthreads();
    const double invW = ec->invW, q_over = ec->q_over;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sg = lane / G, l = lane % G;
    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const uint32_t wbase = (blockIdx.x * kSeg2Warps + warp) * NSEG;
    if (wbase >= cnt) return;                                         // warp-uniform
    const uint32_t idx = wbase + sg;
    const bool valid = idx < cnt;
    const uint32_t tb = a.list ? a.list[valid ? idx : cnt - 1] : (valid ? idx : cnt - 1);
    double *tree = s_tree + (warp * NSEG + sg) * tree_stride<G>();
    double *A0 = s_A + (warp * 2 + 0) * P * 32 + lane;                 // slot 0 column
    double *A1 = s_A + (warp * 2 + 1) * P * 32 + lane;                 // slot 1 column
    agft_tuner_stats &st = s_st[warp * NSEG + sg];
    if (l == 0) st = a.w.acc[tb];
    __syncwarp();
    bool live = valid && !(st.flags & 1u);
    __shared__ PhState s_ph[kSeg2Warps * (32 / G)];   // ENV.md §4.10 detector (lane 0 of the segment)
    PhState &ph = s_ph[warp * NSEG + sg];
    uint32_t phase = 0u;
    if (a.ph_enable) {
        if (l == 0) ph = a.w.ph[tb];
        __syncwarp();
        phase = ph.phase;
    }
    const agft_tuner_params prm = a.w.params[tb];

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
    const bool has0 = act0, has1 = act1;                              // slots holding an arm
    double th0[D], th1[D];
    uint32_t n0 = 0, n1 = 0;
    double rb0 = 0.0, rb1 = 0.0, eb0 = 0.0, eb1 = 0.0;
#pragma unroll
    for (int e = 0; e < P; ++e) {
        A0[e * 32] = has0 ? a.w.ainv[((size_t)tb * P + e) * kMaxArms + key0] : 0.0;
        A1[e * 32] = has1 ? a.w.ainv[((size_t)tb * P + e) * kMaxArms + key1] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
        th0[r] = has0 ? a.w.theta[((size_t)tb * D + r) * kMaxArms + key0] : 0.0;
        th1[r] = has1 ? a.w.theta[((size_t)tb * D + r) * kMaxArms + key1] : 0.0;
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
    double oldest = wcount == M ? ring[whead] : 0.0;                  // the value the next push evicts
    double *bg = a.w.b + (size_t)tb * D * kMaxArms;
    constexpr bool kBS = b_in_smem<G>();
    double *B0 = s_B + (warp * 2 + 0) * D * 32 + lane, *B1 = s_B + (warp * 2 + 1) * D * 32 + lane;
    if (kBS) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
            B0[r * 32] = has0 ? bg[(size_t)r * kMaxArms + key0] : 0.0;
            B1[r * 32] = has1 ? bg[(size_t)r * kMaxArms + key1] : 0.0;
        }
    }
    int nact = spopc<G>(act0, sg) + spopc<G>(act1, sg);
    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;
#if AGFT_TMA
    // a1: the warp's records by bulk copy when all its segments replay one trace (rec_tile.cuh)
    __shared__ __align__(128) StepRec s_rtile[kSeg2Warps][2 * kRecTile];
    __shared__ __align__(8) uint64_t s_rbar[kSeg2Warps][2];
    RecTile rt{s_rtile[warp], s_rbar[warp], rp, a.n_steps,
               __all_sync(kFull, prm.trace_id == __shfl_sync(kFull, prm.trace_id, 0))};
    rt.start(lane);
#endif
    const double inv_tau = 1.0 / a.tau;
    const uint32_t *rawp = a.cl_enable ? a.raw + ((size_t)prm.trace_id * a.rec_stride + a.rec_off) * AGFT_ROW_WORDS
                                       : nullptr;
    uint32_t clq = 0u, clqb = 0u;                                     // ENV-C backlogs (ENV.md §6)
    if (rawp) {
        clq = a.w.clq[(size_t)tb * 2];
        clqb = a.w.clq[(size_t)tb * 2 + 1];
    }
    __syncwarp();
    ScreenCache scr;                                                  // the incremental screen (G ≥ 8)
    scr.ok = false;
    scr.P = scr.B = scr.mx = scr.D = 0.0;
    scr.M = -kInf;

    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const uint32_t t = a.t0 + s;
        live = live && !(st.flags & kFlagSpd);                        // an SPD violation last step froze it
#if AGFT_TMA
        const StepRec *rc = rt.on ? rt.at(s, lane) : rp + s;
#define RF(f) (rt.on ? rc->f : __ldg(&rc->f))
#else
        const StepRec *rc = rp + s;
#define RF(f) __ldg(&rc->f)
#endif
        if (s + 1 < a.n_steps && l == 0) {
            if (!AGFT_TMA) prefetch_l1(rc + 1);
            if (rawp) prefetch_l1(rawp + (size_t)(s + 1) * AGFT_ROW_WORDS);
        }
        double x[D];
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = RF(x[i]);
        double g = RF(g), wIm = RF(wIm), baseE = RF(baseE), baseEDP = RF(baseEDP);
        uint32_t arr_cl = 0u;
        if (rawp) {                                                   // ENV-C: the servers see their backlog
            const ClosedRec cr = closed_record(rawp + (size_t)s * AGFT_ROW_WORDS, clq, clqb, RF(I),
                                               RF(P), RF(invIm), RF(nT), RF(nE),
                                               ec, a);
            x[0] = cr.x0;
            g = cr.g;
            wIm = cr.wIm;
            baseE = cr.baseE;
            baseEDP = cr.baseEDP;
            arr_cl = cr.arr;
        }
        const double alpha = phase ? 0.0 : alpha_t(prm.alpha0, t, inv_tau);   // Exploitation: Eq. 2
        // the reward's reference (median of the window before this step's push) depends only on
        // the window: computed here, off the response → reward chain
        // (branch-free — both lookups, then a select — so that no shuffle sits in a divergent region)
        double ref;
        {
            const double m0 = wat<G, E>(S, (wcount >> 1) - 1u), m1 = wat<G, E>(S, wcount >> 1);
            ref = wcount == 0u ? 0.0 : ((wcount & 1u) ? m1 : xmul(xadd(m0, m1), 0.5));
        }

        // ---- a4: both slots
        double x2[D];
#pragma unroll
        for (int i = 0; i < D; ++i) x2[i] = 2.0 * x[i];
        double sc0 = -kInf, mg0 = 0.0, sc1 = -kInf, mg1 = 0.0;
        if (act0) {
            const double q = quad_form_rows<D>(x, x2, A0, 32);
            double p = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) p = fma(th0[i], x[i], p);
            const double bonus = alpha * xsqrt_nb(q > 0.0 ? q : 0.0);
            sc0 = p + bonus;
            mg0 = fabs(p) + bonus;
        }
        if (act1) {
            const double q = quad_form_rows<D>(x, x2, A1, 32);
            double p = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) p = fma(th1[i], x[i], p);
            const double bonus = alpha * xsqrt_nb(q > 0.0 ? q : 0.0);
            sc1 = p + bonus;
            mg1 = fabs(p) + bonus;
        }
        // ---- a5/a6: lane best (slot 0 keys < slot 1 keys), then segment argmax
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
        const bool fstar = __shfl_sync(kFull, (int)((oslot ? n1 : n0) == 0u), own, G) != 0;
        const bool own0 = is_own && oslot == 0, own1 = is_own && oslot == 1;
        const double inv_n = xrcp_nb((double)((oslot ? n1 : n0) + 1u));   // Welford's 1/n, off the chain
        const bool tie = (act0 && !own0 && (bs - sc0 < a.tie_rel * (mstar > mg0 ? mstar : mg0)) && !(fstar && n0 == 0u)) ||
                         (act1 && !own1 && (bs - sc1 < a.tie_rel * (mstar > mg1 ? mstar : mg1)) && !(fstar && n1 == 0u));
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

        // ---- a7: response
        const Response o = env_response(kEnvS ? s_dec[kstar] : __ldg(&ec->dec[kstar]),
                                        kEnvS ? s_pre[kstar] : __ldg(&ec->pre[kstar]),
                                        kEnvS ? s_pw[kstar] : __ldg(&ec->pw[kstar]), RF(I), RF(P),
                                        g, RF(invIm), RF(invAm), wIm,
                                        RF(nT), RF(nE), invW, q_over, a.u_max, a.u_floor,
                                        a.p_idle, a.W);
        if (rawp) clq = closed_carry(arr_cl + clq, o.u, a.cl_q_max);
        // ---- a8: reward + segment window
        // (round 2: a8, a9 and the window update are branch-free — selects and predicated stores — so the
        // three independent chains after the reward (Sherman–Morrison, the window, Welford) form one basic
        // block the compiler can interleave; the arithmetic and its order are unchanged)
        const double r = wcount > 0u ? reward_of(o.edp, ref, a.clip_lo, a.clip_hi) : 0.0;
        {
            const bool bad = !isfinite(o.edp) || !isfinite(r);
            if (bad && live && l == 0) st.flags |= 1u;
            live = live && !bad;
        }
        if (a.ph_enable) {                                            // ENV.md §4.10 observe_reward
            __syncwarp();                                             // the last step's phase reads are done
            if (live && l == 0) {
                ph.exploit_steps += phase;
                ph_observe(ph, r, t, a.ph_window, a.ph_delta, a.ph_lambda);
            }
            __syncwarp();
            phase = ph.phase;
        }
        {
            // both ranks from ONE butterfly on the current window: #(S' < v) after removing `old` is
            // #(S < v) − [old < v], exactly (multiset identity); a window still filling removes nothing
            // (oldest = 0 there, below every EDP) and inserts at #(S < v)
            const bool full = wcount >= M;
            const double old = oldest;
            int c = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) c += ((S[e] < old) ? 1 : 0) + ((S[e] < o.edp) ? 0x10000 : 0);
            c = sisum<G>(c);
            const int po = full ? (c & 0xffff) : kWindow, pv = (c >> 16) - ((full && old < o.edp) ? 1 : 0);
            wremove<G, E>(S, po, l);
            winsert<G, E>(S, o.edp, pv, l);
            if (live && l == 0) ring[full ? whead : wcount] = o.edp;
            whead = full ? ((whead + 1 == M) ? 0u : whead + 1) : whead;
            wcount = full ? wcount : wcount + 1u;
            if (wcount == M) oldest = M == 1 ? o.edp : ring[whead];   // next step's eviction, off the chain
        }

        // ---- a9: Sherman–Morrison on the owner lane's slot (every lane runs it on its own column; the
        // owner's stores and results are kept)
        const bool upd = live && is_own;
        double scr_d = 0.0, scr_e = -kInf;                            // k*'s move within Q (screen_note)
        bool spd;
        {
            const uint32_t n_old = oslot ? n1 : n0;
            const double e_old = oslot ? eb1 : eb0, rb_old = oslot ? rb1 : rb0;
            double thv[D];
#pragma unroll
            for (int i = 0; i < D; ++i) thv[i] = oslot ? th1[i] : th0[i];
            if (kBS) spd = sm_update_smem_pred<D>(upd, oslot ? A1 : A0, 32, thv, oslot ? B1 : B0, 32, x, r);
            else spd = sm_update_smem_pred<D>(upd, oslot ? A1 : A0, 32, thv, bg + kstar, kMaxArms, x, r);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                th1[i] = oslot ? thv[i] : th1[i];
                th0[i] = oslot ? th0[i] : thv[i];
            }
            // Welford (ENV.md §4.7) with 1/(n+1) computed off the chain
            const double rb_new = xadd(rb_old, xmul(xsub(r, rb_old), inv_n));
            const double e_new = xadd(e_old, xmul(xsub(o.edp, e_old), inv_n));
            if (upd) {
                if (oslot) { n1 = n_old + 1u; rb1 = rb_new; eb1 = e_new; }
                else { n0 = n_old + 1u; rb0 = rb_new; eb0 = e_new; }
            }
            if (kScreen<G>() && upd) {
                if (n_old >= a.hist_n) {                              // a member of Q moved
                    scr_d = fabs(e_new - e_old);
                    scr_e = e_new;
                } else if (n_old + 1u >= a.hist_n) {                  // k* joined Q: membership changed
                    scr_d = kInf;
                }
            }
        }
        if (kScreen<G>() && a.prune_enable) {
            const double d = __shfl_sync(kFull, scr_d, own, G), e = __shfl_sync(kFull, scr_e, own, G);
            screen_note(scr, d, e);
        }
        if (!spd) atomicOr(&st.flags, kFlagFrozen | kFlagSpd);      // SPD guard: frozen from the next step

        // ---- a10: pruning (ENV.md §4.8)
        if (a.prune_enable) {
            const bool eon = t < a.ext_L;
            const bool ext0 = act0 && eon && n0 >= a.ext_n && rb0 < prm.extreme_reward_threshold;
            const bool ext1 = act1 && eon && n1 >= a.ext_n && rb1 < prm.extreme_reward_threshold;
            const bool q0 = act0 && n0 >= a.hist_n, q1 = act1 && n1 >= a.hist_n;
            const int next = spopc<G>(ext0, sg) + spopc<G>(ext1, sg);
            const int nq = spopc<G>(q0, sg) + spopc<G>(q1, sg);
            const bool need = live && t >= a.hist_t && nq >= 2;
            bool hist0 = false, hist1 = false;
            // the screen (seg_common.cuh) skips the exact trees when no arm of Q can be removed; on for
            // G ≥ 8 (A/B on the C4 day: −10% / −8% / −6% kernel time for G = 8 / 16 / 32, +9% for G = 4,
            // whose small Q sets are mostly pruned anyway — DESIGN.md §4)
            // (round 2: the full screen runs only when the cached bound of the last one no longer
            // decides — seg_common.cuh::ScreenCache)
            bool exact = need;
            if (kScreen<G>()) {
                const bool inc = need && screen_inc_safe(scr);
                exact = false;
                if (__any_sync(kFull, need && !inc)) {                // warp-wide call (butterflies)
                    ScreenCache fresh;
                    const bool safe = hist_screen_full<G>(q0, eb0, q1, eb1, nq, prm.historical_k, fresh);
                    if (need && !inc) scr = fresh;
                    exact = need && !inc && !safe;
                }
            }
            if (__any_sync(kFull, exact)) {
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
                const int restore = remaining == 0 ? bkr : -1;       // AMB-11
                const bool rm0 = any_rm && c0 && key0 != restore, rm1 = any_rm && c1 && key1 != restore;
                const int ce = spopc<G>(rm0 && ext0, sg) + spopc<G>(rm1 && ext1, sg);
                const int ch = spopc<G>(rm0 && !ext0 && hist0, sg) + spopc<G>(rm1 && !ext1 && hist1, sg);
                const int cc = spopc<G>(rm0 && !ext0 && !hist0, sg) + spopc<G>(rm1 && !ext1 && !hist1, sg);
                if (any_rm) {
                    scr.ok = false;                                   // Q lost members: the bound is void
                    if (l == 0) {
                        st.n_pruned_extreme += ce;
                        st.n_pruned_hist += ch;
                        st.n_pruned_cascade += cc;
                    }
                    nact -= ce + ch + cc;
                }
                if (a.rf_enable) {                    // ENV.md §4.11: Extreme removals stay out for good
                    if (rm0 && ext0) atomicOr(a.w.extm + (size_t)tb * 4 + (key0 >> 5), 1u << (key0 & 31));
                    if (rm1 && ext1) atomicOr(a.w.extm + (size_t)tb * 4 + (key1 >> 5), 1u << (key1 & 31));
                }
                if (rm0) {
                    act0 = false;
                    tree[tslot<G>(key0)] = 0.0;       // keep the tree buffer's non-Q slots at +0.0
                }
                if (rm1) {
                    act1 = false;
                    tree[tslot<G>(key1)] = 0.0;
                }
            }
        }

        // ---- a11
        if (live && l == 0) {
            stats_add(st, o, r, baseE, baseEDP, kstar, (uint32_t)nact0);
            st.near_tie_steps += near ? 1u : 0u;
            if (rec_on) {
                if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
                if (a.gap) a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = gapv;
            }
            if (a.chosen) a.chosen[tb] = (uint32_t)kstar;
        }
    }

#undef RF
    // ---- write back (segments of real tuners only)
    __syncwarp();
    if (valid) {
        if (has0) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + key0] = A0[e * 32];
#pragma unroll
            for (int r = 0; r < D; ++r) a.w.theta[((size_t)tb * D + r) * kMaxArms + key0] = th0[r];
            a.w.n[(size_t)tb * kMaxArms + key0] = n0;
            a.w.rbar[(size_t)tb * kMaxArms + key0] = rb0;
            a.w.ebar[(size_t)tb * kMaxArms + key0] = eb0;
            if (kBS) {
#pragma unroll
                for (int r = 0; r < D; ++r) bg[(size_t)r * kMaxArms + key0] = B0[r * 32];
            }
        }
        if (has1) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + key1] = A1[e * 32];
#pragma unroll
            for (int r = 0; r < D; ++r) a.w.theta[((size_t)tb * D + r) * kMaxArms + key1] = th1[r];
            a.w.n[(size_t)tb * kMaxArms + key1] = n1;
            a.w.rbar[(size_t)tb * kMaxArms + key1] = rb1;
            a.w.ebar[(size_t)tb * kMaxArms + key1] = eb1;
            if (kBS) {
#pragma unroll
                for (int r = 0; r < D; ++r) bg[(size_t)r * kMaxArms + key1] = B1[r * 32];
            }
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
        prof_add(a, a.w.acc + tb, st);
        a.w.acc[tb] = st;
    }
}

template <int D, int G>
static cudaError_t launch_seg2_dg(const ReplayArgs &a, cudaStream_t s)
{
    constexpr int P = D * (D + 1) / 2;
    constexpr int per_block = kSeg2Warps * (32 / G);
    const size_t smem = seg2_smem_bytes<G>(P, D);
    auto kern = seg2_kernel<D, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t blocks = (a.n_tuners + per_block - 1) / per_block;
    kern<<<blocks, kSeg2Warps * 32, smem, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D, int G>
static int occupancy_seg2_dg()
{
    constexpr int P = D * (D + 1) / 2;
    const size_t smem = seg2_smem_bytes<G>(P, D);
    auto kern = seg2_kernel<D, G>;
    int blocks = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kSeg2Warps * 32, smem) != cudaSuccess)
        return -1;
    return blocks * kSeg2Warps * (32 / G);
}

template <int D>
static int occupancy_seg2_d(int G)
{
    switch (G) {
    case 4: return occupancy_seg2_dg<D, 4>();
    case 32: return occupancy_seg2_dg<D, 32>();
    case 8: return occupancy_seg2_dg<D, 8>();
    default: return occupancy_seg2_dg<D, 16>();
    }
}

int occupancy_seg2(uint32_t D, int G)
{
    switch (D) {
    case 1: return occupancy_seg2_d<1>(G);
    case 2: return occupancy_seg2_d<2>(G);
    case 3: return occupancy_seg2_d<3>(G);
    case 4: return occupancy_seg2_d<4>(G);
    case 5: return occupancy_seg2_d<5>(G);
    case 6: return occupancy_seg2_d<6>(G);
    default: return occupancy_seg2_d<7>(G);
    }
}

template <int D>
static cudaError_t launch_seg2_d(const ReplayArgs &a, int G, cudaStream_t s)
{
    switch (G) {
    case 4: return launch_seg2_dg<D, 4>(a, s);
    case 32: return launch_seg2_dg<D, 32>(a, s);
    case 8: return launch_seg2_dg<D, 8>(a, s);
    default: return launch_seg2_dg<D, 16>(a, s);
    }
}

// K_act ≤ 2G
cudaError_t launch_seg2(const ReplayArgs &a, uint32_t D, int G, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_seg2_d<1>(a, G, s);
    case 2: return launch_seg2_d<2>(a, G, s);
    case 3: return launch_seg2_d<3>(a, G, s);
    case 4: return launch_seg2_d<4>(a, G, s);
    case 5: return launch_seg2_d<5>(a, G, s);
    case 6: return launch_seg2_d<6>(a, G, s);
    default: return launch_seg2_d<7>(a, G, s);
    }
}

}  // namespace agft
