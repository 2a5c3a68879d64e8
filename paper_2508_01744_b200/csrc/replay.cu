// replay.cu — K2: the fused tuner step loop (rows a1–a11), one warp per tuner.
//
// Per step (PAPER §4.2–4.3, ENV.md §4):  record → α_t → Eq. 1 score of every
// active arm → lexicographic (s desc, k asc) warp argmax → ENV-R response →
// EDP-median reward → Sherman–Morrison update of the chosen arm (Eqs. 3–5) →
// extreme / historical / cascade pruning → stats.
//
// Mapping: arm k lives in lane k%32, slot k/32 (S = ceil(K/32) ≤ 4 slots per lane).
// Packed A⁻¹ and θ of every slot stay resident in shared memory across all steps
// of the launch ([slot][entry][lane], conflict-free 8-byte accesses); n, r̄, ē and
// the scores live in registers.  The 64-entry EDP window is spread 2 per lane
// (sorted copy + chronological ring) and maintained with ballots and shuffles.
// The canonical 128-slot reduction of ENV.md §4.8 maps onto this layout exactly:
// levels 1–5 are the xor-butterfly across lanes (adjacent arms are adjacent lanes),
// levels 6–7 combine the four slot partials in-lane.
//
// MODE 0 is the replay (records from K1).  MODE 1 / 2 are the live two-phase step of
// agft_select / agft_observe (one window, WIDE mapping): select builds x_t from the tuner's
// MetricsSnapshot row, scores and picks k* and stops (no state change); observe takes the
// MEASURED (E, TPOT, TTFT) at k* in place of ENV-R and runs a8–a11 exactly as the replay does.
#include "env_t.cuh"
#include "step_common.cuh"
#include "des.cuh"

namespace agft {

namespace {

template <int S, typename T>
__device__ __forceinline__ T pick(const T (&v)[S], int j)
{
    T r = v[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (j == i) r = v[i];
    return r;
}

template <int S, typename T>
__device__ __forceinline__ void put(T (&v)[S], int j, T x)
{
#pragma unroll
    for (int i = 0; i < S; ++i)
        if (j == i) v[i] = x;
}

// canonical pairwise sum over 128 arm slots (ENV.md §4.8): value of arm 32*j + lane in v[j]
template <int S>
__device__ __forceinline__ double tree128(const double (&v)[S])
{
    double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < S; ++j) {
        double s = v[j];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) s = xadd(s, __shfl_xor_sync(kFull, s, off));
        part[j] = s;
    }
    return xadd(xadd(part[0], part[1]), xadd(part[2], part[3]));
}

__device__ __forceinline__ int popc_ballot(bool p) { return __popc(__ballot_sync(kFull, p)); }

// ---- the 64-entry EDP window: sorted S[0..63] with S[2l], S[2l+1] in lane l (+inf padded)
__device__ __forceinline__ double window_at(double lo, double hi, uint32_t idx)
{
    const double v = (idx & 1u) ? hi : lo;
    return __shfl_sync(kFull, v, idx >> 1);
}

__device__ __forceinline__ void window_remove(double &lo, double &hi, double old, int lane)
{
    const int po = popc_ballot(lo < old) + popc_ballot(hi < old);
    double nxt = __shfl_down_sync(kFull, lo, 1);
    if (lane == 31) nxt = kInf;
    const double nlo = (2 * lane < po) ? lo : hi;
    const double nhi = (2 * lane + 1 < po) ? hi : nxt;
    lo = nlo;
    hi = nhi;
}

__device__ __forceinline__ void window_insert(double &lo, double &hi, double v, int lane)
{
    const int pi = popc_ballot(lo < v) + popc_ballot(hi < v);
    const double prv = __shfl_up_sync(kFull, hi, 1);
    const double nlo = (2 * lane < pi) ? lo : ((2 * lane == pi) ? v : prv);
    const double nhi = (2 * lane + 1 < pi) ? hi : ((2 * lane + 1 == pi) ? v : lo);
    lo = nlo;
    hi = nhi;
}

constexpr int kWarpsPerBlock = 2;

}  // namespace

template <int D, int S, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
replay_kernel(const __grid_constant__ ReplayArgs a)
{
    const TlGuard tl_guard(a);
    constexpr int P = D * (D + 1) / 2;
    extern __shared__ double smem[];
    double *s_dec = smem, *s_pre = smem + kMaxArms, *s_pw = smem + 2 * kMaxArms;
    const EnvConsts *ec = a.w.env;
    constexpr bool kRep = MODE == 0 || MODE == 4;    // the replay (4: on the ENV-S server, ENV.md §7)
    if (kRep) {                                       // the live modes take no dynamic shared memory
        for (int i = threadIdx.x; i < kMaxArms; i += blockDim.x) {
            s_dec[i] = ec->dec[i];
            s_pre[i] = ec->pre[i];
            s_pw[i] = ec->pw[i];
        }
    }
    __syncthreads();
    const double invW = ec->invW, q_over = ec->q_over;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t widx = blockIdx.x * kWarpsPerBlock + warp;
    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    if (widx >= cnt) return;
    const uint64_t tb = a.list ? a.list[widx] : widx;
    agft_tuner_stats st = a.w.acc[tb];
    if (st.flags & 1u) {                              // frozen by an earlier anomaly
        if (MODE == 1 && lane == 0 && a.chosen) a.chosen[tb] = AGFT_NEVER;
        if (MODE == 1 && a.scores)
            for (uint32_t k = lane; k < a.K; k += 32) a.scores[tb * a.K + k] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    __shared__ PhState s_ph[kWarpsPerBlock];          // ENV.md §4.10 detector (lane 0 owns it)
    __shared__ uint32_t s_spd[kWarpsPerBlock];        // set by the owner lane on an SPD violation
    if (lane == 0) s_spd[warp] = 0u;
    __syncwarp();
    uint32_t phase = 0u;
    uint32_t extb = 0u;                               // bit j: arm 32j+lane was Extreme-pruned (ENV.md §4.11)
    if (a.rf_enable) {
#pragma unroll
        for (int j = 0; j < S; ++j)
            if ((a.w.extm[tb * 4 + j] >> lane) & 1u) extb |= 1u << j;
    }
    if (a.ph_enable) {
        if (lane == 0) s_ph[warp] = a.w.ph[tb];
        __syncwarp();
        phase = s_ph[warp].phase;
    }

    // Arm state: the replay stages A⁻¹ and θ in shared memory for the whole launch
    // ([slot][entry][lane]); a live window (MODE 1 / 2) reads and updates them in place in HBM
    // (arm index fastest: 32 consecutive arms = one coalesced 256-B row), with no dynamic shared
    // memory, so more tuners are in flight per SM.  Entry e of slot j: A[j * aJ + e * aS].
    constexpr bool kInPlace = !kRep;
    constexpr int aS = kInPlace ? kMaxArms : 32, aJ = kInPlace ? 32 : P * 32, tJ = kInPlace ? 32 : D * 32;
    double *sA = kInPlace ? a.w.ainv + (size_t)tb * P * kMaxArms : smem + 3 * kMaxArms + (size_t)warp * S * (P + D) * 32;
    double *sT = kInPlace ? a.w.theta + (size_t)tb * D * kMaxArms : sA + S * P * 32;
    const agft_tuner_params prm = a.w.params[tb];
    const uint32_t K = a.K;

    // ---- load resident state
    uint32_t n[S];
    double rbar[S], ebar[S];
    uint32_t act = 0;                                 // bit j: arm 32j+lane active
    // A single live window touches only what it needs (HBM-bound at large N): select reads the
    // active arms' A⁻¹, θ and n; observe reads the chosen arm's A⁻¹, θ (all arms' when refinement
    // may re-score them) plus n, r̄, ē for the pruning statistics, and writes back the chosen arm.
    const uint32_t kpend = MODE == 2 ? a.w.live[tb].kstar : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < S; ++j) {
        const uint32_t k = 32u * j + lane;
        const bool on = k < K && ((a.w.active[tb * 4 + j] >> lane) & 1u);
        if (on) act |= 1u << j;
        if (kRep) {
#pragma unroll
            for (int e = 0; e < P; ++e) sA[(j * P + e) * 32 + lane] = a.w.ainv[(tb * P + e) * kMaxArms + k];
#pragma unroll
            for (int i = 0; i < D; ++i) sT[(j * D + i) * 32 + lane] = a.w.theta[(tb * D + i) * kMaxArms + k];
        }
        n[j] = (MODE != 1 || on) ? a.w.n[tb * kMaxArms + k] : 0u;
        rbar[j] = MODE != 1 ? a.w.rbar[tb * kMaxArms + k] : 0.0;
        ebar[j] = MODE != 1 ? a.w.ebar[tb * kMaxArms + k] : 0.0;
    }
    double wlo = 0.0, whi = 0.0, rlo = 0.0, rhi = 0.0;
    uint32_t wcount = 0u, whead = 0u;
    if (MODE != 1 && MODE != 3) {                     // select / refine never touch the EDP window
        wlo = a.w.wsorted[tb * kWindow + 2 * lane];
        whi = a.w.wsorted[tb * kWindow + 2 * lane + 1];
        rlo = a.w.wring[tb * kWindow + 2 * lane];
        rhi = a.w.wring[tb * kWindow + 2 * lane + 1];
        wcount = a.w.wmeta[tb * 2];
        whead = a.w.wmeta[tb * 2 + 1];
    }
    const uint32_t M = a.median_window;

    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const uint32_t *rawp = (kRep && a.cl_enable) ? a.raw + ((size_t)prm.trace_id * a.rec_stride + a.rec_off) * AGFT_ROW_WORDS
                                                      : nullptr;
    uint32_t clq = 0u, clqb = 0u;                     // ENV-C backlogs (ENV.md §6)
    if (MODE == 0 && rawp) {
        clq = a.w.clq[tb * 2];
        clqb = a.w.clq[tb * 2 + 1];
    }
    double *bglob = a.w.b + tb * D * kMaxArms;
    // ENV-S (ENV.md §7): the tuner's server, its Philox key (the trace's, §1) and queue
    DesWarp des;
    DesReq *desq = nullptr;
    const Philox des_ph{(uint32_t)a.seed ^ (a.trace_base + prm.trace_id), (uint32_t)(a.seed >> 32)};
    if constexpr (MODE == 4) {
        des.load(a.w.des + tb, a.w.desr + tb * kDesR, lane);
        desq = a.w.desq + tb * kDesQ;
    }

    // ENV.md §4.11 mixed maturity-based refinement as of step t at context x (after pruning)
    auto refine = [&](uint32_t t, const double (&x)[D]) {
        int anchor = -1;
        if (t < a.rf_mature) {                    // Statistical: lowest ē among n ≥ min, not Extreme
            double be = kInf;
            int bk2 = 0x7fffffff;
#pragma unroll
            for (int j = 0; j < S; ++j) {
                const int k = 32 * j + lane;
                if (k < (int)K && !((extb >> j) & 1u) && n[j] >= a.rf_min_samples && ebar[j] < be) {
                    be = ebar[j];
                    bk2 = k;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(kFull, be, off);
                const int ok = __shfl_xor_sync(kFull, bk2, off);
                if (ob < be || (ob == be && ok < bk2)) { be = ob; bk2 = ok; }
            }
            anchor = bk2 == 0x7fffffff ? -1 : bk2;
        } else {                                  // Predictive: UCB argmax at x_t (Eq. 1's α_t)
            const double au = alpha_t(prm.alpha0, t, 1.0 / a.tau);
            double wv[P];
            {
                int e = 0;
#pragma unroll
                for (int r0 = 0; r0 < D; ++r0)
#pragma unroll
                    for (int c = r0; c < D; ++c, ++e) wv[e] = (r0 == c) ? x[r0] * x[r0] : 2.0 * x[r0] * x[c];
            }
            double bu = -kInf;
            int bk2 = 0x7fffffff;
#pragma unroll
            for (int j = 0; j < S; ++j) {
                if ((act >> j) & 1u) {
                    const double *Aj = sA + j * aJ + lane;
                    const double *Tj = sT + j * tJ + lane;
                    const double q = quad_form<P>(wv, Aj, aS);
                    double p = 0.0;
#pragma unroll
                    for (int i = 0; i < D; ++i) p = fma(Tj[i * aS], x[i], p);
                    const double u = p + au * xsqrt_nb(q > 0.0 ? q : 0.0);
                    if (u > bu) { bu = u; bk2 = 32 * j + lane; }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(kFull, bu, off);
                const int ok = __shfl_xor_sync(kFull, bk2, off);
                if (ob > bu || (ob == bu && ok < bk2)) { bu = ob; bk2 = ok; }
            }
            anchor = bk2 == 0x7fffffff ? -1 : bk2;
        }
        if (anchor >= 0) {
#pragma unroll
            for (int j = 0; j < S; ++j) {
                const int k = 32 * j + lane;
                const uint32_t dist = (uint32_t)(k > anchor ? k - anchor : anchor - k) * a.f_step_mhz;
                const bool in = k < (int)K && dist <= a.rf_half_mhz && dist % a.rf_step_mhz == 0u &&
                                !((extb >> j) & 1u);
                act = in ? (act | (1u << j)) : (act & ~(1u << j));
            }
            st.n_refine += 1u;
            st.last_anchor = (uint32_t)anchor;
        }
    };

    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const uint32_t t = a.t0 + s;
        if (s_spd[warp]) {                                // the last step's update broke A⁻¹'s SPD property
            st.flags |= kFlagFrozen | kFlagSpd;
            break;
        }
        double x[D];
        double g = 0.0, invIm = 0.0, invAm = 0.0, wIm = 0.0, nT = 0.0, nE = 0.0, baseE = 0.0, baseEDP = 0.0;
        uint32_t recI = 0u, recP = 0u, arr_cl = 0u;
        if constexpr (MODE == 4) {                    // ENV-S: the snapshot of the last window (§7)
            double xr[7];
            context_of(des.snap[0], des.snap[1], des.snap[2], des.snap[3], des.snap[4], des.snap[5], des.snap[6],
                       des.snap[7], a.W, a.kv_total, a.norm_lo, a.norm_hi, xr);
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = xr[i];
        } else if constexpr (MODE == 0 || MODE == 3) {
            const StepRec &rec = rp[s];
            if (s + 1 < a.n_steps && lane == 0) {
                prefetch_l1(&rp[s + 1]);
                if (rawp) prefetch_l1(rawp + (size_t)(s + 1) * AGFT_ROW_WORDS);
            }
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = rec.x[i];
            g = rec.g; invIm = rec.invIm; invAm = rec.invAm; wIm = rec.wIm;
            nT = rec.nT; nE = rec.nE; baseE = rec.baseE; baseEDP = rec.baseEDP;
            recI = rec.I; recP = rec.P;
            if (rawp) {                               // ENV-C: both servers see their backlog (§6)
                const ClosedRec cr = closed_record(rawp + (size_t)s * AGFT_ROW_WORDS, clq, clqb, recI, recP, invIm,
                                                   nT, nE, ec, a);
                x[0] = cr.x0;
                g = cr.g;
                wIm = cr.wIm;
                baseE = cr.baseE;
                baseEDP = cr.baseEDP;
                arr_cl = cr.arr;
            }
        } else if constexpr (MODE == 1) {             // live: §4.1 context of the tuner's own snapshot
            const uint4 *rw = reinterpret_cast<const uint4 *>(a.live_rows + tb * AGFT_ROW_WORDS);
            const uint4 r0 = rw[0], r1 = rw[1];
            double xr[7];
            context_of(r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, a.W, a.kv_total, a.norm_lo, a.norm_hi, xr);
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = xr[i];
        } else {                                      // live observe: the x_t of the selection
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = a.w.live[tb].x[i];
        }
        if constexpr (MODE == 3) {                    // the deferred refinement pass: nothing else
            refine(t, x);
            continue;
        }

        int nact = 0;
#pragma unroll
        for (int j = 0; j < S; ++j) nact += popc_ballot((act >> j) & 1u);

        // ---- a3: α_t = α0/√(1+t/τ)
        const uint32_t phase_sel = phase;
        const double alpha = phase ? 0.0 : alpha_t(prm.alpha0, t, 1.0 / a.tau);   // Exploitation: Eq. 2

        int kstar, own, jst;
        double sstar = 0.0, mstar = 0.0, s2 = -kInf, m2 = 0.0;
        bool near;
        if constexpr (MODE == 2) {
            kstar = (int)a.w.live[tb].kstar;
            near = a.w.live[tb].near != 0u;
            own = kstar & 31;
            jst = kstar >> 5;
        } else {
        // ---- a4: Eq. 1 scores.  q = Σ_{i≤j} w_ij A⁻¹_ij with w_ij = x_i x_j (×2 off-diagonal)
        double w[P];
        {
            int e = 0;
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int c = r; c < D; ++c, ++e) w[e] = (r == c) ? x[r] * x[r] : 2.0 * x[r] * x[c];
        }
        double sc[S], mg[S];
        double bs = -kInf;
        int bk = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            sc[j] = -kInf;
            mg[j] = 0.0;
            if (__ballot_sync(kFull, (act >> j) & 1u) == 0) continue;
            if ((act >> j) & 1u) {
                const double *Aj = sA + j * aJ + lane;
                const double *Tj = sT + j * tJ + lane;
                const double q = quad_form<P>(w, Aj, aS);
                double p = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) p = fma(Tj[i * aS], x[i], p);
                const double bonus = alpha * xsqrt_nb(q > 0.0 ? q : 0.0);   // AMB-19
                sc[j] = p + bonus;
                mg[j] = fabs(p) + bonus;
                if (sc[j] > bs) { bs = sc[j]; bk = 32 * j + lane; }  // ascending k: ties keep lowest
            }
        }
        // ---- a5/a6: lexicographic (s desc, k asc) warp argmax over F_available
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double os = __shfl_xor_sync(kFull, bs, off);
            const int ok = __shfl_xor_sync(kFull, bk, off);
            if (os > bs || (os == bs && ok < bk)) { bs = os; bk = ok; }
        }
        kstar = bk;
        own = kstar & 31;
        jst = kstar >> 5;
        sstar = bs;
        mstar = __shfl_sync(kFull, pick<S>(mg, jst), own);
        const bool fresh_star = __shfl_sync(kFull, pick<S>(n, jst) == 0u, own);

        // ---- near-tie flag (ENV.md §4.5)
        bool tie = false;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            if (!((act >> j) & 1u) || (32 * j + lane) == kstar) continue;
            const double sc_ = mstar > mg[j] ? mstar : mg[j];   // (scores are finite here)
            if (sstar - sc[j] < a.tie_rel * sc_ && !(fresh_star && n[j] == 0u)) tie = true;
            if (sc[j] > s2) { s2 = sc[j]; m2 = mg[j]; }
        }
        near = __ballot_sync(kFull, tie) != 0u;
        if constexpr (MODE == 1) {                    // select ends here: nothing changes until observe
            if (a.scores) {                           // agft_scores: every arm's Eq. 1 score (NaN if pruned)
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const uint32_t k = 32u * j + lane;
                    if (k < K) a.scores[tb * K + k] = ((act >> j) & 1u) ? sc[j] : __longlong_as_double(0x7ff8000000000000ll);
                }
            }
            if (lane == 0) {
                LivePend pd;
#pragma unroll
                for (int i = 0; i < 7; ++i) pd.x[i] = i < D ? x[i < D ? i : 0] : 0.0;
                pd.kstar = (uint32_t)kstar;
                pd.near = near ? 1u : 0u;
                a.w.live[tb] = pd;
                if (a.chosen) a.chosen[tb] = (uint32_t)kstar;
            }
            return;
        }
        }

        // the chosen arm's b (global memory) for the update below, loaded now so that its L2 round trip
        // overlaps the response, the reward and the window instead of stalling the update (round 2)
        double bpre[D];
        if (lane == own) {
#pragma unroll
            for (int i = 0; i < D; ++i) bpre[i] = bglob[(size_t)i * kMaxArms + kstar];
        }

        // ---- a7: ENV-R response at f = f_min + k*·step (ENV.md §3.3), exact arithmetic
        double E, tpot, ttft, edp;
        if constexpr (MODE == 2) {                    // live: the measured response, EDP = E·TPOT
            const double *m = a.live_resp + tb * 3;
            E = m[0];
            tpot = m[1];
            ttft = m[2];
            edp = xmul(E, tpot);
            if (!isfinite(E) || !isfinite(tpot) || !isfinite(ttft)) {
                st.flags |= 1u;
                break;
            }
        } else if constexpr (MODE == 4) {             // ENV-S: the window on the tuner's own server
            const DesOut o = des.window(t, rawp + (size_t)s * AGFT_ROW_WORDS, a.tc, des_ph, desq, s_dec[kstar],
                                        s_pre[kstar], s_pw[kstar], a, lane);
            E = o.E;
            tpot = o.tpot;
            ttft = o.ttft;
            edp = o.edp;
        } else {
        const double dec = s_dec[kstar], pre = s_pre[kstar], pw = s_pw[kstar];
        const double t_dec = xmul((double)recI, dec);
        const double t_pre = xmul((double)recP, pre);
        const double busy = xmul(xadd(t_dec, t_pre), g);
        const double u = xmul(busy, invW);
        const double q = u <= a.u_max ? xrcp_nb(xsub(1.0, u)) : xmul(u, q_over);
        if (rawp) clq = closed_carry(arr_cl + clq, u, a.cl_q_max);   // ENV-C: left queued (§6)
        tpot = xmul(xmul(xmul(xadd(dec, xmul(t_pre, invIm)), g), q), nT);
        double ue = u > 1.0 ? 1.0 : u;
        ue = ue < a.u_floor ? a.u_floor : ue;
        E = xmul(xmul(xadd(a.p_idle, xmul(pw, ue)), a.W), nE);
        ttft = xmul(xadd(xmul(t_pre, invAm), xmul(t_dec, wIm)), q);
        edp = xmul(E, tpot);
        }

        // ---- a8: reward = clip(1 − EDP/median(window)), then push EDP (AMB-3)
        double r = 0.0;
        if (wcount > 0) {
            double ref;
            if (wcount & 1u) {
                ref = window_at(wlo, whi, wcount >> 1);
            } else {
                const double m0 = window_at(wlo, whi, (wcount >> 1) - 1), m1 = window_at(wlo, whi, wcount >> 1);
                ref = xmul(xadd(m0, m1), 0.5);
            }
            r = xsub(1.0, xdiv_nb(edp, ref));
            r = r < a.clip_lo ? a.clip_lo : (r > a.clip_hi ? a.clip_hi : r);
        }
        if (!isfinite(edp) || !isfinite(r)) {         // anomaly: flag and freeze the tuner
            st.flags |= 1u;
            break;
        }
        if (a.ph_enable) {                            // ENV.md §4.10 observe_reward
            __syncwarp();                             // every lane's read of the last step's phase is done
            if (lane == 0) {
                s_ph[warp].exploit_steps += phase;
                ph_observe(s_ph[warp], r, t, a.ph_window, a.ph_delta, a.ph_lambda);
            }
            __syncwarp();
            phase = s_ph[warp].phase;
        }
        uint32_t ri;
        if (wcount < M) {
            ri = wcount;
            ++wcount;
        } else {
            const double old = window_at(rlo, rhi, whead);
            window_remove(wlo, whi, old, lane);
            ri = whead;
            whead = (whead + 1 == M) ? 0u : whead + 1;
        }
        window_insert(wlo, whi, edp, lane);
        if (lane == (int)(ri >> 1)) {
            if (ri & 1u) rhi = edp; else rlo = edp;
        }

        // ---- a9: rank-1 update of the chosen arm (Eqs. 3–5) by its owner lane
        bool spd = true;
        if (lane == own) {
            double *Aj = sA + jst * aJ + lane;
            double *Tj = sT + jst * tJ + lane;
            double Ap[P];
#pragma unroll
            for (int e = 0; e < P; ++e) Ap[e] = Aj[e * aS];
            double z[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double acc = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const int lo = i < c ? i : c, hi = i < c ? c : i;
                    acc = fma(Ap[lo * D - lo * (lo - 1) / 2 + (hi - lo)], x[c], acc);
                }
                z[i] = acc;
            }
            double xz = 0.0, px = 0.0;
            double th[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                xz = fma(x[i], z[i], xz);
                th[i] = Tj[i * aS];
                px = fma(th[i], x[i], px);
            }
            const double invd = xrcp_nb(1.0 + xz);              // Sherman–Morrison denominator
            {
                int e = 0;
#pragma unroll
                for (int r0 = 0; r0 < D; ++r0)
#pragma unroll
                    for (int c = r0; c < D; ++c, ++e) {
                        const double v = fma(-z[r0] * invd, z[c], Ap[e]);
                        Aj[e * aS] = v;
                        if (c == r0) spd = spd && v > 0.0;
                    }
                spd = spd && spd_quad_ok(xz);
            }
            const double coef = (r - px) * invd;                // RLS form of θ = A⁻¹ b (AMB-21)
#pragma unroll
            for (int i = 0; i < D; ++i) {
                Tj[i * aS] = fma(z[i], coef, th[i]);
                bglob[(size_t)i * kMaxArms + kstar] = xadd(bpre[i], xmul(r, x[i]));   // b exact, as Eq. 4 writes it
            }
            const uint32_t nn = pick<S>(n, jst) + 1u;
            const double inv = xrcp_nb((double)nn);
            put<S>(n, jst, nn);
            put<S>(rbar, jst, xadd(pick<S>(rbar, jst), xmul(xsub(r, pick<S>(rbar, jst)), inv)));
            put<S>(ebar, jst, xadd(pick<S>(ebar, jst), xmul(xsub(edp, pick<S>(ebar, jst)), inv)));
        }
        if (!spd) s_spd[warp] = 1u;                       // SPD guard: frozen from the next step

        // ---- a10: §4.3 pruning on the post-update state
        if (a.prune_enable) {
            bool ext[S], inq[S], hist[S];
            int next = 0, nq = 0;
#pragma unroll
            for (int j = 0; j < S; ++j) {
                const bool on = (act >> j) & 1u;
                ext[j] = on && t < a.ext_L && n[j] >= a.ext_n && rbar[j] < prm.extreme_reward_threshold;
                inq[j] = on && n[j] >= a.hist_n;
                hist[j] = false;
                next += popc_ballot(ext[j]);
                nq += popc_ballot(inq[j]);
            }
            if (t >= a.hist_t && nq >= 2) {
                double best = kInf;
                double v[S], v2[S];
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    if (inq[j] && ebar[j] < best) best = ebar[j];
                    v[j] = inq[j] ? ebar[j] : 0.0;
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(kFull, best, off));
                const double mu = xdiv(tree128<S>(v), (double)nq);
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const double dv = xsub(ebar[j], mu);
                    v2[j] = inq[j] ? xmul(dv, dv) : 0.0;
                }
                const double sd = xsqrt(xdiv(tree128<S>(v2), (double)nq));
                const double thr = xadd(best, xmul(prm.historical_k, sd));
                int nh = 0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    hist[j] = inq[j] && ebar[j] > thr;
                    nh += popc_ballot(hist[j]);
                }
                next += nh;
            }
            if (next > 0) {
                // cascade: all active arms below the highest removed arm under the limit
                int kc = -1;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const uint32_t k = 32u * j + lane;
                    const double F = (double)(a.f_min_mhz + k * a.f_step_mhz);
                    if ((ext[j] || hist[j]) && F < a.cascade_limit) kc = (int)k;
                }
                kc = __reduce_max_sync(kFull, kc);
                bool cas[S];
                int remaining = 0;
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const bool on = (act >> j) & 1u;
                    const int k = 32 * j + lane;
                    cas[j] = on && !ext[j] && !hist[j] && k < kc;
                    remaining += popc_ballot(on && !ext[j] && !hist[j] && !cas[j]);
                }
                int restore = -1;
                if (remaining == 0) {                   // AMB-11: keep the removed arm with max r̄
                    double br = -kInf;
                    int bkr = 0x7fffffff;
#pragma unroll
                    for (int j = 0; j < S; ++j)
                        if ((ext[j] || hist[j] || cas[j]) && rbar[j] > br) { br = rbar[j]; bkr = 32 * j + lane; }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const double ob = __shfl_xor_sync(kFull, br, off);
                        const int ok = __shfl_xor_sync(kFull, bkr, off);
                        if (ob > br || (ob == br && ok < bkr)) { br = ob; bkr = ok; }
                    }
                    restore = bkr;
                }
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    const int k = 32 * j + lane;
                    const bool rm = (ext[j] || hist[j] || cas[j]) && k != restore;
                    const int ce = popc_ballot(rm && ext[j]);
                    const int ch = popc_ballot(rm && !ext[j] && hist[j]);
                    const int cc = popc_ballot(rm && !ext[j] && !hist[j]);
                    st.n_pruned_extreme += ce;
                    st.n_pruned_hist += ch;
                    st.n_pruned_cascade += cc;
                    if (rm) act &= ~(1u << j);
                    if (rm && ext[j]) extb |= 1u << j;
                }
            }
        }

        // ---- ENV.md §4.11 mixed maturity-based refinement (after pruning); on the class schedule
        // a separate pass (MODE 3) applies it at the sub-chunk end instead (rf_defer)
        if (a.rf_enable && !a.rf_defer && ((t + 1u) % a.rf_period == 0u || (a.ph_enable && phase != phase_sel)))
            refine(t, x);

        // ---- a11: stats (ENV.md §4.9 order) and trajectory record
        st.sum_energy = xadd(st.sum_energy, E);
        st.sum_tpot = xadd(st.sum_tpot, tpot);
        st.sum_ttft = xadd(st.sum_ttft, ttft);
        st.sum_edp = xadd(st.sum_edp, edp);
        st.sum_reward = xadd(st.sum_reward, r);
        st.base_energy = xadd(st.base_energy, baseE);
        st.base_edp = xadd(st.base_edp, baseEDP);
        st.traj_hash = (st.traj_hash ^ (uint64_t)kstar) * kFnvPrime;
        st.sum_active += (uint64_t)nact;
        st.steps += 1;
        st.last_arm = (uint32_t)kstar;
        st.near_tie_steps += near ? 1u : 0u;
        if (a.traj && prm.record_slot != AGFT_NO_RECORD && lane == 0)
            a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
        if (a.gap && prm.record_slot != AGFT_NO_RECORD) {
            // relative top-2 gap: (s* − s2)/max(m*, m2), +inf when only one arm is active
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double os = __shfl_xor_sync(kFull, s2, off);
                const double om = __shfl_xor_sync(kFull, m2, off);
                if (os > s2) { s2 = os; m2 = om; }
            }
            if (lane == 0) {
                const double den = fmax(mstar, m2);
                a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] =
                    (s2 == -kInf) ? kInf : (den > 0.0 ? (sstar - s2) / den : 0.0);
            }
        }
        if (a.chosen && lane == 0) a.chosen[tb] = (uint32_t)kstar;
    }

    // ---- write back the resident state
#pragma unroll
    for (int j = 0; j < S; ++j) {
        const uint32_t k = 32u * j + lane;
        if (kRep) {
#pragma unroll
            for (int e = 0; e < P; ++e) a.w.ainv[(tb * P + e) * kMaxArms + k] = sA[(j * P + e) * 32 + lane];
#pragma unroll
            for (int i = 0; i < D; ++i) a.w.theta[(tb * D + i) * kMaxArms + k] = sT[(j * D + i) * 32 + lane];
        }
        if (kRep || k == kpend) {                // a live window changed only the chosen arm's counters
            a.w.n[tb * kMaxArms + k] = n[j];
            a.w.rbar[tb * kMaxArms + k] = rbar[j];
            a.w.ebar[tb * kMaxArms + k] = ebar[j];
        }
        const uint32_t bits = __ballot_sync(kFull, (act >> j) & 1u);
        if (lane == 0) a.w.active[tb * 4 + j] = bits;
    }
    if constexpr (MODE == 4) des.save(a.w.des + tb, a.w.desr + tb * kDesR, lane);
    if (MODE == 0 && rawp && lane == 0) {
        a.w.clq[tb * 2] = clq;
        a.w.clq[tb * 2 + 1] = clqb;
    }
    if (MODE != 3) {
        a.w.wsorted[tb * kWindow + 2 * lane] = wlo;
        a.w.wsorted[tb * kWindow + 2 * lane + 1] = whi;
        a.w.wring[tb * kWindow + 2 * lane] = rlo;
        a.w.wring[tb * kWindow + 2 * lane + 1] = rhi;
    }
    int nact_end = 0;
#pragma unroll
    for (int j = 0; j < S; ++j) nact_end += popc_ballot((act >> j) & 1u);
    if (lane == 0) {
        if (MODE != 3) {
            a.w.wmeta[tb * 2] = wcount;
            a.w.wmeta[tb * 2 + 1] = whead;
        }
        st.n_active = (uint32_t)nact_end;
        if (a.ph_enable) {
            a.w.ph[tb] = s_ph[warp];
            ph_to_stats(s_ph[warp], st);
        }
        prof_add(a, a.w.acc + tb, st);
        a.w.acc[tb] = st;
    }
    if (a.rf_enable) {
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const uint32_t bits = __ballot_sync(kFull, (extb >> j) & 1u);
            if (lane == 0) a.w.extm[tb * 4 + j] = bits;
        }
    }
}

template <int D, int S, int MODE>
static cudaError_t launch_ds(const ReplayArgs &a, cudaStream_t s)
{
    constexpr int P = D * (D + 1) / 2;
    const size_t smem = (MODE == 0 || MODE == 4) ? (3 * kMaxArms + (size_t)kWarpsPerBlock * S * (P + D) * 32) * sizeof(double) : 0;
    auto kern = replay_kernel<D, S, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t blocks = (a.n_tuners + kWarpsPerBlock - 1) / kWarpsPerBlock;
    kern<<<blocks, kWarpsPerBlock * 32, smem, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D, int S>
static int occupancy_ds()
{
    constexpr int P = D * (D + 1) / 2;
    const size_t smem = (3 * kMaxArms + (size_t)kWarpsPerBlock * S * (P + D) * 32) * sizeof(double);
    auto kern = replay_kernel<D, S, 0>;
    int blocks = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kWarpsPerBlock * 32, smem) != cudaSuccess)
        return -1;
    return blocks * kWarpsPerBlock;                   // one tuner per warp
}

template <int D>
static int occupancy_d(uint32_t K)
{
    switch ((K + 31) / 32) {
    case 1: return occupancy_ds<D, 1>();
    case 2: return occupancy_ds<D, 2>();
    case 3: return occupancy_ds<D, 3>();
    default: return occupancy_ds<D, 4>();
    }
}

int occupancy_wide(uint32_t D, uint32_t K)
{
    switch (D) {
    case 1: return occupancy_d<1>(K);
    case 2: return occupancy_d<2>(K);
    case 3: return occupancy_d<3>(K);
    case 4: return occupancy_d<4>(K);
    case 5: return occupancy_d<5>(K);
    case 6: return occupancy_d<6>(K);
    default: return occupancy_d<7>(K);
    }
}

template <int D, int MODE>
static cudaError_t launch_d(const ReplayArgs &a, cudaStream_t s)
{
    const uint32_t slots = (a.K + 31) / 32;
    switch (slots) {
    case 1: return launch_ds<D, 1, MODE>(a, s);
    case 2: return launch_ds<D, 2, MODE>(a, s);
    case 3: return launch_ds<D, 3, MODE>(a, s);
    default: return launch_ds<D, 4, MODE>(a, s);
    }
}

template <int MODE>
static cudaError_t launch_mode(const ReplayArgs &a, uint32_t D, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_d<1, MODE>(a, s);
    case 2: return launch_d<2, MODE>(a, s);
    case 3: return launch_d<3, MODE>(a, s);
    case 4: return launch_d<4, MODE>(a, s);
    case 5: return launch_d<5, MODE>(a, s);
    case 6: return launch_d<6, MODE>(a, s);
    default: return launch_d<7, MODE>(a, s);
    }
}

cudaError_t launch_replay(const ReplayArgs &a, uint32_t D, cudaStream_t s)
{
    return a.cl_enable == 2u ? launch_mode<4>(a, D, s) : launch_mode<0>(a, D, s);   // ENV-S (ENV.md §7)
}

cudaError_t launch_live(const ReplayArgs &a, uint32_t D, int mode, cudaStream_t s)
{
    return mode == 1 ? launch_mode<1>(a, D, s) : launch_mode<2>(a, D, s);
}

cudaError_t launch_refine(const ReplayArgs &a, uint32_t D, cudaStream_t s) { return launch_mode<3>(a, D, s); }

}  // namespace agft
