// replay_lane.cu — K2/LANE<D, KL, MB>: one LANE per tuner for tuners with 2 ≤ K_act ≤ KL
// active arms, with the Eq. 1 arm scores computed in batches of MB windows.
//
// Why: after the first ~1,000 windows of C4 the multi-arm tuners keep 2–32
// arms, and a step of one tuner is a long serial chain (argmax → ENV-R response → median
// reward → Sherman–Morrison → Welford → pruning) whose latency, not its arithmetic, sets the
// rate.  The SEG kernels spend G lanes on that chain for every tuner; LANE runs 32 tuners'
// chains in one warp instruction stream.  The arm state of a tuner (K × 336 B) no longer
// fits on chip at one tuner per lane, so it lives in an L2-resident per-tuner stream and is
// read once per MB windows:
//
//   phase A (every MB windows): for every active arm, load A⁻¹ and θ once and score the
//     arm at all MB upcoming contexts (the trace is open-loop, so x_t is known ahead);
//     the scores go to a per-lane shared-memory table tab[j][slot], together with an
//     upper bound M_j of every arm's score magnitude m_k = |θ·x| + α√q (ENV.md §4.3).
//   phase B (every window): argmax = scan of tab[j] over the active slots.  Only the arm
//     chosen at a window changes (Eqs. 3–5), so right after its Sherman–Morrison update it
//     is re-scored for the remaining windows of the batch — every table entry is then the
//     score of the CURRENT state, exactly what a per-window rescoring would compute (the
//     same function of the same operands).  The chosen arm stays in registers ("hot")
//     until another arm is chosen.
//
// The near-tie rule (ENV.md §4.5) is decided from the table: if s* − s₂ ≥ tie_rel·M_j no
// arm can be within tolerance; otherwise (and for recorded tuners, whose score gap is
// written out) the exact rule is evaluated with fresh magnitudes.  Historical pruning
// (ENV.md §4.8) is screened per window with a one-pass mean/variance and a rigorous
// margin; when the screen cannot exclude a removal, the canonical 128-slot tree is
// evaluated exactly over the member arms (a stack that merges adjacent subtrees in the
// full tree's order; empty slots add +0.0, which is exact).  Extreme pruning only looks at
// the chosen arm once t ≥ L_E is excluded (n and r̄ change for no other arm).
#include "step_common.cuh"

namespace agft {

namespace {

constexpr int kLStride = 42;   // stream words per arm slot: packed A⁻¹ (≤ 28), θ (≤ 7), b (≤ 7); 336 B
constexpr int kLSlots = 32;    // stream slots per tuner

template <int KL, int MB>
__host__ __device__ constexpr size_t lane_smem_bytes()
{
    // dec/pre/pw [3][128] + per lane: tab[MB][KL], mmax[MB], window[64], rbar[KL], ebar[KL] (f64),
    // n[KL] (u32), key[KL] (u8)
    return (size_t)3 * kMaxArms * 8 + (size_t)(MB * KL + MB + kWindow + 2 * KL) * 32 * 8 + (size_t)KL * 32 * 4 +
           (size_t)KL * 32;
}

template <int D>
__device__ __forceinline__ void load_x(const StepRec *__restrict__ rc, double (&x)[D])
{
    const double2 *q = reinterpret_cast<const double2 *>(rc->x);
#pragma unroll
    for (int i = 0; i < D; i += 2) {
        const double2 v = __ldg(q + i / 2);
        x[i] = v.x;
        if (i + 1 < D) x[i + 1 < D ? i + 1 : i] = v.y;
    }
}

// Eq. 1 score s = θ·x + α√max(xᵀA⁻¹x, 0) and magnitude m = |θ·x| + α√max(q, 0) (ENV.md §4.3).
// The one function phase A, the re-scoring and the exact near-tie path share, so that a
// table entry and a fresh evaluation of the same state are bit-identical.
// q = Σ_i x_i (A_ii x_i + 2 Σ_{c>i} A_ic x_c) over the packed upper triangle.
template <int D>
__device__ __forceinline__ void score_mag(const double (&A)[D * (D + 1) / 2], const double (&th)[D],
                                          const double (&x)[D], double alpha, double &s, double &m)
{
    double t[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double inner = 0.0;
#pragma unroll
        for (int c = i + 1; c < D; ++c) inner = fma(A[pidx<D>(i, c)], x[c], inner);
        t[i] = fma(2.0, inner, A[pidx<D>(i, i)] * x[i]);
    }
    double q0 = 0.0, q1 = 0.0, p0 = 0.0, p1 = 0.0;
#pragma unroll
    for (int i = 0; i < D; i += 2) {
        q0 = fma(x[i], t[i], q0);
        p0 = fma(th[i], x[i], p0);
        if (i + 1 < D) {
            q1 = fma(x[i + 1 < D ? i + 1 : i], t[i + 1 < D ? i + 1 : i], q1);
            p1 = fma(th[i + 1 < D ? i + 1 : i], x[i + 1 < D ? i + 1 : i], p1);
        }
    }
    const double q = q0 + q1, p = p0 + p1;
    const double bonus = alpha * sqrt(fmax(q, 0.0));
    s = p + bonus;
    m = fabs(p) + bonus;
}

template <int D>
__device__ __forceinline__ void load_arm(const double *__restrict__ slot, double (&A)[D * (D + 1) / 2],
                                         double (&th)[D])
{
    constexpr int P = D * (D + 1) / 2;
    double w[P + D + 1];
    const double2 *q = reinterpret_cast<const double2 *>(slot);
#pragma unroll
    for (int e = 0; e < P + D; e += 2) {
        const double2 v = __ldcg(q + e / 2);
        w[e] = v.x;
        w[e + 1] = v.y;
    }
#pragma unroll
    for (int e = 0; e < P; ++e) A[e] = w[e];
#pragma unroll
    for (int r = 0; r < D; ++r) th[r] = w[P + r];
}

template <int D>
__device__ __forceinline__ void load_hot(const double *slot, double (&A)[D * (D + 1) / 2], double (&th)[D],
                                         double (&b)[D])
{
    constexpr int P = D * (D + 1) / 2;
    double w[P + 2 * D + 1];
    const double2 *q = reinterpret_cast<const double2 *>(slot);
#pragma unroll
    for (int e = 0; e < P + 2 * D; e += 2) {
        const double2 v = __ldcg(q + e / 2);
        w[e] = v.x;
        w[e + 1] = v.y;
    }
#pragma unroll
    for (int e = 0; e < P; ++e) A[e] = w[e];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        th[r] = w[P + r];
        b[r] = w[P + D + r];
    }
}

template <int D>
__device__ __forceinline__ void store_hot(double *slot, const double (&A)[D * (D + 1) / 2], const double (&th)[D],
                                          const double (&b)[D])
{
    constexpr int P = D * (D + 1) / 2;
    double w[P + 2 * D + 1];
#pragma unroll
    for (int e = 0; e < P; ++e) w[e] = A[e];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        w[P + r] = th[r];
        w[P + D + r] = b[r];
    }
    w[P + 2 * D] = 0.0;
    double2 *q = reinterpret_cast<double2 *>(slot);
#pragma unroll
    for (int e = 0; e < P + 2 * D; e += 2) __stcg(q + e / 2, make_double2(w[e], w[e + 1]));
}

// ENV.md §4.8 tree128 over the member slots, exact: slots are in ascending arm order, and a
// stack merges adjacent subtrees in the order of the full 128-slot pairwise tree (the
// level at which consecutive members k < k' join is msb(k ^ k')); empty slots would add
// +0.0, which is exact, so they are simply absent.  SQ: sum (ē − μ)² instead of ē.
template <int KL, bool SQ>
__device__ double tree_canon(uint32_t members, const uint8_t *ky, const double *ebr, double mu)
{
    double vs[9];
    int lv[9];
    int top = 0, prev = 0;
    for (int sl = 0; sl < KL; ++sl) {
        if (!((members >> sl) & 1u)) continue;
        const int k = ky[sl * 32];
        const double e = ebr[sl * 32];
        const double v = SQ ? xmul(xsub(e, mu), xsub(e, mu)) : e;
        if (top > 0) {
            const int g = 31 - __clz(prev ^ k);
            while (top >= 2 && lv[top - 1] < g) {
                vs[top - 2] = xadd(vs[top - 2], vs[top - 1]);
                --top;
            }
            lv[top] = g;
        } else {
            lv[0] = 99;
        }
        vs[top++] = v;
        prev = k;
    }
    while (top >= 2) {
        vs[top - 2] = xadd(vs[top - 2], vs[top - 1]);
        --top;
    }
    return top ? vs[0] : 0.0;
}

}  // namespace

template <int D, int KL, int MB>
__global__ void __launch_bounds__(32, 1) lane_kernel(const __grid_constant__ ReplayArgs a)
{
    constexpr int P = D * (D + 1) / 2;
    static_assert(KL <= kLSlots, "LANE: at most 32 slots per tuner");
    extern __shared__ double sm[];
    double *s_dec = sm, *s_pre = sm + kMaxArms, *s_pw = sm + 2 * kMaxArms;
    const int lane = threadIdx.x;
    double *const tab = sm + 3 * kMaxArms + lane;            // tab[(j * KL + slot) * 32]
    double *const mmx = tab + MB * KL * 32;                  // mmx[j * 32]
    double *const wsm = mmx + MB * 32;                       // sorted EDP window [64][32]
    double *const rbr = wsm + kWindow * 32;                  // r̄ [KL][32]
    double *const ebr = rbr + KL * 32;                       // ē [KL][32]
    uint32_t *const nn =
        reinterpret_cast<uint32_t *>(sm + 3 * kMaxArms + (MB * KL + MB + kWindow + 2 * KL) * 32) + lane;   // n [KL][32]
    uint8_t *const ky = reinterpret_cast<uint8_t *>(nn - lane + KL * 32) + lane;                             // key [KL][32]

    const EnvConsts *ec = a.w.env;
    for (int q = lane; q < kMaxArms; q += 32) {
        s_dec[q] = ec->dec[q];
        s_pre[q] = ec->pre[q];
        s_pw[q] = ec->pw[q];
    }
    __syncthreads();                                         // the only block-wide sync: lanes are independent below
    const double invW = ec->invW, q_over = ec->q_over;

    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const uint32_t i = blockIdx.x * 32 + lane;
    if (i >= cnt) return;
    const uint32_t tb = a.list ? a.list[i] : i;
    agft_tuner_stats st = a.w.acc[tb];
    if (st.flags & 1u) return;
    const agft_tuner_params prm = a.w.params[tb];

    // ---- compact the active arms into slots (ascending arm index = ascending frequency)
    int kact0 = 0;
    {
        const uint4 m4 = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t mm = mw[w];
            while (mm) {
                const int k = 32 * w + __ffs(mm) - 1;
                mm &= mm - 1u;
                if (kact0 < KL) ky[kact0 * 32] = (uint8_t)k;
                ++kact0;
            }
        }
    }
    if (kact0 > KL) {                                        // scheduling bug: never silently wrong
        st.flags |= 4u;
        a.w.acc[tb] = st;
        return;
    }
    uint32_t act = kact0 >= 32 ? kFull : ((1u << kact0) - 1u);
    double *const strm = a.w.mstream + (size_t)tb * kLSlots * kLStride;
    for (int sl = 0; sl < kact0; ++sl) {
        const int k = ky[sl * 32];
        double *dst = strm + sl * kLStride;
#pragma unroll
        for (int e = 0; e < P; ++e) dst[e] = a.w.ainv[((size_t)tb * P + e) * kMaxArms + k];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            dst[P + r] = a.w.theta[((size_t)tb * D + r) * kMaxArms + k];
            dst[P + D + r] = a.w.b[((size_t)tb * D + r) * kMaxArms + k];
        }
        nn[sl * 32] = a.w.n[(size_t)tb * kMaxArms + k];
        rbr[sl * 32] = a.w.rbar[(size_t)tb * kMaxArms + k];
        ebr[sl * 32] = a.w.ebar[(size_t)tb * kMaxArms + k];
    }
    for (int j = 0; j < kWindow; ++j) wsm[j * 32] = a.w.wsorted[(size_t)tb * kWindow + j];
    uint32_t wcount = a.w.wmeta[(size_t)tb * 2], whead = a.w.wmeta[(size_t)tb * 2 + 1];
    const uint32_t M = a.median_window;
    double *ring = a.w.wring + (size_t)tb * kWindow;
    const SmemWindow win{wsm, 32};
    double oldest = ring_oldest(ring, wcount, whead, M);

    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;
    const bool exact_tie = rec_on && a.gap != nullptr;       // the gap output needs exact magnitudes
    const double inv_tau = 1.0 / a.tau;
    const double kh = prm.historical_k;

    double hA[P], hth[D], hb[D];                             // the hot (last chosen) arm
    int hot = -1;
    double al[MB];
    int kstar = ky[0];

    for (uint32_t s0 = 0; s0 < a.n_steps; s0 += MB) {
        const int len = (a.n_steps - s0) < (uint32_t)MB ? (int)(a.n_steps - s0) : MB;
        // ================= phase A: every active arm scored at the next `len` contexts
        if (hot >= 0) store_hot<D>(strm + hot * kLStride, hA, hth, hb);
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            al[j] = alpha_t(prm.alpha0, a.t0 + s0 + j, inv_tau);
            mmx[j * 32] = 0.0;
        }
        for (int sl = 0; sl < KL; ++sl) {
            if (!((act >> sl) & 1u)) continue;
            double A[P], th[D];
            load_arm<D>(strm + sl * kLStride, A, th);
#pragma unroll
            for (int j = 0; j < MB; ++j) {
                if (j < len) {
                    double x[D];
                    load_x<D>(rp + s0 + j, x);
                    double sc, mg;
                    score_mag<D>(A, th, x, al[j], sc, mg);
                    tab[(j * KL + sl) * 32] = sc;
                    mmx[j * 32] = fmax(mmx[j * 32], mg);
                }
            }
        }

        // ================= phase B: the serial step chain
        for (int j = 0; j < len; ++j) {
            const uint32_t s = s0 + j, t = a.t0 + s;
            const StepRec *rc = rp + s;

            // ---- a5/a6: lexicographic argmax (score desc, arm asc) over the active slots
            double b1 = -kInf, b2 = -kInf;
            int k1 = __ffs(act) - 1, k2 = -1;
            const double *trow = tab + j * KL * 32;
#pragma unroll
            for (int sl = 0; sl < KL; ++sl) {
                if ((act >> sl) & 1u) {
                    const double v = trow[sl * 32];
                    if (v > b1) {
                        b2 = b1;
                        k2 = k1;
                        b1 = v;
                        k1 = sl;
                    } else if (v > b2) {
                        b2 = v;
                        k2 = sl;
                    }
                }
            }
            if (b2 == -kInf) k2 = -1;
            // ---- near-tie rule (ENV.md §4.5): screened with the magnitude bound
            bool near = false;
            double gapv = kInf;
            const double mmj = mmx[j * 32];
            if (!(b1 - b2 >= a.tie_rel * mmj) || exact_tie) {
                double x[D];
                load_x<D>(rc, x);
                const double alj = alpha_t(prm.alpha0, t, inv_tau);
                // fresh (score, magnitude) of slot sl at this window: the hot arm from registers
                auto fresh = [&](int sl, double &sc, double &mg) {
                    double A[P], th[D];
                    if (sl == hot) {
#pragma unroll
                        for (int e = 0; e < P; ++e) A[e] = hA[e];
#pragma unroll
                        for (int r = 0; r < D; ++r) th[r] = hth[r];
                    } else {
                        load_arm<D>(strm + sl * kLStride, A, th);
                    }
                    score_mag<D>(A, th, x, alj, sc, mg);
                };
                double sc, ms, m2 = 0.0;
                fresh(k1, sc, ms);
                if (exact_tie && k2 >= 0) fresh(k2, sc, m2);
                const uint32_t n1 = nn[k1 * 32];
                for (int sl = 0; sl < KL; ++sl) {
                    if (!((act >> sl) & 1u) || sl == k1) continue;
                    if (!(b1 - trow[sl * 32] < a.tie_rel * mmj)) continue;        // outside any tolerance
                    double mg;
                    fresh(sl, sc, mg);
                    if (b1 - sc < a.tie_rel * fmax(ms, mg) && !(n1 == 0u && nn[sl * 32] == 0u)) near = true;
                }
                if (exact_tie) {
                    const double den = fmax(ms, m2);
                    gapv = (k2 < 0) ? kInf : (den > 0.0 ? (b1 - b2) / den : 0.0);
                }
            }
            const int ks = k1;
            kstar = ky[ks * 32];

            // ---- the chosen arm into registers
            if (ks != hot) {
                if (hot >= 0) store_hot<D>(strm + hot * kLStride, hA, hth, hb);
                load_hot<D>(strm + ks * kLStride, hA, hth, hb);
                hot = ks;
            }

            // ---- a7: response; a8: reward against the window median, push
            const Response o = env_response(s_dec[kstar], s_pre[kstar], s_pw[kstar], __ldg(&rc->I), __ldg(&rc->P),
                                            __ldg(&rc->g), __ldg(&rc->invIm), __ldg(&rc->invAm), __ldg(&rc->wIm),
                                            __ldg(&rc->nT), __ldg(&rc->nE), invW, q_over, a.u_max, a.u_floor,
                                            a.p_idle, a.W);
            bool ok;
            const double r = reward_and_push(win, ring, wcount, whead, M, o.edp, a.clip_lo, a.clip_hi, ok, oldest);
            if (!ok) {
                st.flags |= 1u;
                goto done;
            }

            // ---- a9: Sherman–Morrison on the hot arm (Eqs. 3–5), Welford (ENV.md §4.7)
            {
                double x[D];
                load_x<D>(rc, x);
                sm_update<D>(hA, hth, hb, x, r);
                uint32_t nk = nn[ks * 32];
                double rb = rbr[ks * 32], eb = ebr[ks * 32];
                welford(nk, rb, eb, r, o.edp);
                nn[ks * 32] = nk;
                rbr[ks * 32] = rb;
                ebr[ks * 32] = eb;
            }
            // ---- the updated arm re-scored at the remaining contexts of the batch
#pragma unroll
            for (int jj = 1; jj < MB; ++jj) {
                if (jj > j && jj < len) {
                    double x[D];
                    load_x<D>(rp + s0 + jj, x);
                    double sc, mg;
                    score_mag<D>(hA, hth, x, al[jj], sc, mg);
                    tab[(jj * KL + ks) * 32] = sc;
                    mmx[jj * 32] = fmax(mmx[jj * 32], mg);
                }
            }

            const uint32_t nact0 = (uint32_t)__popc(act);
            // ---- a10: pruning (ENV.md §4.8) on the post-update state
            if (a.prune_enable) {
                uint32_t ext = 0u, hist = 0u;
                if (t < a.ext_L) {
                    for (int sl = 0; sl < KL; ++sl)
                        if (((act >> sl) & 1u) && nn[sl * 32] >= a.ext_n && rbr[sl * 32] < prm.extreme_reward_threshold)
                            ext |= 1u << sl;
                }
                if (t >= a.hist_t) {
                    uint32_t q = 0u;
                    int nq = 0;
                    double sum = 0.0, sum2 = 0.0, best = kInf, worst = -kInf;
#pragma unroll
                    for (int sl = 0; sl < KL; ++sl) {
                        if (((act >> sl) & 1u) && nn[sl * 32] >= a.hist_n) {
                            const double e = ebr[sl * 32];
                            q |= 1u << sl;
                            ++nq;
                            sum += e;
                            sum2 = fma(e, e, sum2);
                            best = fmin(best, e);
                            worst = fmax(worst, e);
                        }
                    }
                    if (nq >= 2) {
                        // screen: |sd_approx − sd_exact| ≤ √|var_a − var_x| ≤ 1e-7·max ē (var errors ≤ 1e-14·E[ē²]),
                        // so worst ≤ thr_a − margin proves worst < thr_exact (no historical removal)
                        const double dq = (double)nq;
                        const double mu_a = sum / dq;
                        const double sd_a = sqrt(fmax(sum2 / dq - mu_a * mu_a, 0.0));
                        const double thr_a = best + kh * sd_a;
                        const double margin = (kh * 1e-6 + 1e-12) * worst;
                        if (worst > thr_a - margin || a.force_exact) {
                            const double mu = xdiv(tree_canon<KL, false>(q, ky, ebr, 0.0), dq);
                            const double sd = xsqrt(xdiv(tree_canon<KL, true>(q, ky, ebr, mu), dq));
                            const double thr = xadd(best, xmul(kh, sd));
                            for (int sl = 0; sl < KL; ++sl)
                                if (((q >> sl) & 1u) && ebr[sl * 32] > thr) hist |= 1u << sl;
                        }
                    }
                }
                const uint32_t R = ext | hist;
                if (R) {
                    int kc = -1;                                      // highest removed slot below the cascade frequency
                    for (int sl = 0; sl < KL; ++sl)
                        if (((R >> sl) & 1u) &&
                            (double)(a.f_min_mhz + (uint32_t)ky[sl * 32] * a.f_step_mhz) < a.cascade_limit)
                            kc = sl;
                    const uint32_t cas = kc > 0 ? (act & ~R & ((1u << kc) - 1u)) : 0u;
                    const uint32_t rm = (R | cas) & act;
                    uint32_t remaining = act & ~rm;
                    uint32_t keep = 0u;
                    if (remaining == 0u) {                            // AMB-11: keep the best r̄ (ties: lowest arm)
                        int bk = -1;
                        double br = -kInf;
                        for (int sl = 0; sl < KL; ++sl)
                            if (((rm >> sl) & 1u) && (bk < 0 || rbr[sl * 32] > br)) {
                                bk = sl;
                                br = rbr[sl * 32];
                            }
                        keep = 1u << bk;
                    }
                    const uint32_t gone = rm & ~keep;
                    st.n_pruned_extreme += __popc(gone & ext);
                    st.n_pruned_hist += __popc(gone & ~ext & hist);
                    st.n_pruned_cascade += __popc(gone & ~ext & ~hist);
                    act = remaining | keep;
                }
            }

            // ---- a11
            stats_add(st, o, r, __ldg(&rc->baseE), __ldg(&rc->baseEDP), kstar, nact0);
            st.near_tie_steps += near ? 1u : 0u;
            if (rec_on) {
                if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)kstar;
                if (a.gap) a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = gapv;
            }
        }
    }
done:
    if (a.chosen) a.chosen[tb] = (uint32_t)kstar;
    if (hot >= 0) store_hot<D>(strm + hot * kLStride, hA, hth, hb);
    for (int sl = 0; sl < kact0; ++sl) {
        const int k = ky[sl * 32];
        const double *src = strm + sl * kLStride;
#pragma unroll
        for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + k] = src[e];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            a.w.theta[((size_t)tb * D + r) * kMaxArms + k] = src[P + r];
            a.w.b[((size_t)tb * D + r) * kMaxArms + k] = src[P + D + r];
        }
        a.w.n[(size_t)tb * kMaxArms + k] = nn[sl * 32];
        a.w.rbar[(size_t)tb * kMaxArms + k] = rbr[sl * 32];
        a.w.ebar[(size_t)tb * kMaxArms + k] = ebr[sl * 32];
    }
    uint32_t words[4] = {0u, 0u, 0u, 0u};
    for (int sl = 0; sl < kact0; ++sl)
        if ((act >> sl) & 1u) {
            const int k = ky[sl * 32];
            words[k >> 5] |= 1u << (k & 31);
        }
    *reinterpret_cast<uint4 *>(a.w.active + (size_t)tb * 4) = make_uint4(words[0], words[1], words[2], words[3]);
    for (int j = 0; j < kWindow; ++j) a.w.wsorted[(size_t)tb * kWindow + j] = wsm[j * 32];
    a.w.wmeta[(size_t)tb * 2] = wcount;
    a.w.wmeta[(size_t)tb * 2 + 1] = whead;
    st.n_active = (uint32_t)__popc(act);
    a.w.acc[tb] = st;
}

template <int D, int KL, int MB>
static cudaError_t launch_lane_dk(const ReplayArgs &a, cudaStream_t s)
{
    constexpr size_t smem = lane_smem_bytes<KL, MB>();
    auto kern = lane_kernel<D, KL, MB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t blocks = (a.n_tuners + 31) / 32;
    kern<<<blocks, 32, smem, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_lane_d(const ReplayArgs &a, int KL, cudaStream_t s)
{
    switch (KL) {
    case 8: return launch_lane_dk<D, 8, 8>(a, s);
    case 16: return launch_lane_dk<D, 16, 8>(a, s);
    default: return launch_lane_dk<D, 32, 4>(a, s);
    }
}

// 1 ≤ K_act ≤ KL (KL ∈ {8, 16, 32}).  Instantiated for d = 7 (the paper's context) and d = 4
// (C1); lane_supported() tells the scheduler which d it may route here.
bool lane_supported(uint32_t D) { return D == 4 || D == 7; }

cudaError_t launch_lane(const ReplayArgs &a, uint32_t D, int KL, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 4: return launch_lane_d<4>(a, KL, s);
    case 7: return launch_lane_d<7>(a, KL, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace agft
