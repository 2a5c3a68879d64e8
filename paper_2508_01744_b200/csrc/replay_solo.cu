// replay_solo.cu — K2/SOLO: one LANE per tuner, for tuners whose action space has
// collapsed to a single frequency (K_act = 1; 73% of C4's tuner-steps).
//
// With one active arm the argmax of Eq. 1 is that arm and pruning can change nothing
// (the non-empty guard restores it, AMB-11), so a step is: ENV-R response → EDP-median
// reward → Sherman–Morrison update (Eqs. 3–5) → Welford → stats, all per thread with no
// cross-lane communication.  Arm state (A⁻¹, θ, b: 49 doubles at d = 7) lives in
// registers for the whole launch; the sorted 64-entry EDP window lives in shared memory
// ([entry][thread], conflict-free) and is maintained by one binary search plus an
// insertion-sort walk from the evicted slot; the chronological ring stays in global
// memory (one 8-byte read + write per step).
#include "step_common.cuh"

namespace agft {

namespace {
#ifndef AGFT_SOLO_THREADS
#define AGFT_SOLO_THREADS 64            // threads per block (A/B knob)
#endif
constexpr int kSoloThreads = AGFT_SOLO_THREADS;
#ifndef AGFT_SOLO_MIN_BLOCKS
#define AGFT_SOLO_MIN_BLOCKS 4          // as SEG2: an occupancy cap (≤ 168 regs) spilled and measured slower
#endif
constexpr int kSoloMinBlocks = AGFT_SOLO_MIN_BLOCKS;
}

template <int D>
__global__ void __launch_bounds__(kSoloThreads, kSoloMinBlocks) solo_kernel(const __grid_constant__ ReplayArgs a)
{
    const TlGuard tl_guard(a);
    constexpr int P = D * (D + 1) / 2;
    __shared__ double S_[kWindow * kSoloThreads];
    const uint32_t cnt = a.count ? *a.count : a.n_tuners;
    const uint32_t i = blockIdx.x * kSoloThreads + threadIdx.x;
    if (i >= cnt) return;                                        // no collectives below
    const uint32_t tb = a.list ? a.list[i] : i;
    double *S = S_ + threadIdx.x;                                // S[j * kSoloThreads]
#define SW(j) S[(j) * kSoloThreads]

    agft_tuner_stats st = a.w.acc[tb];
    if (st.flags & 1u) return;
    __shared__ PhState s_ph[kSoloThreads];                       // ENV.md §4.10 detector of this lane
    PhState &ph = s_ph[threadIdx.x];
    if (a.ph_enable) ph = a.w.ph[tb];
    const agft_tuner_params prm = a.w.params[tb];
    int k = 0;
    {
        const uint4 m = *reinterpret_cast<const uint4 *>(a.w.active + (size_t)tb * 4);
        k = m.x ? __ffs(m.x) - 1 : m.y ? 31 + __ffs(m.y) : m.z ? 63 + __ffs(m.z) : 95 + __ffs(m.w);
    }
    double A[P], th[D], b[D];
#pragma unroll
    for (int e = 0; e < P; ++e) A[e] = a.w.ainv[((size_t)tb * P + e) * kMaxArms + k];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        th[r] = a.w.theta[((size_t)tb * D + r) * kMaxArms + k];
        b[r] = a.w.b[((size_t)tb * D + r) * kMaxArms + k];
    }
    uint32_t n = a.w.n[(size_t)tb * kMaxArms + k];
    double rbar = a.w.rbar[(size_t)tb * kMaxArms + k], ebar = a.w.ebar[(size_t)tb * kMaxArms + k];
    const EnvConsts *ec = a.w.env;
    const double dec = ec->dec[k], pre = ec->pre[k], pw = ec->pw[k], invW = ec->invW, q_over = ec->q_over;
    for (int j = 0; j < kWindow; ++j) SW(j) = a.w.wsorted[(size_t)tb * kWindow + j];
    uint32_t wcount = a.w.wmeta[(size_t)tb * 2], whead = a.w.wmeta[(size_t)tb * 2 + 1];
    const uint32_t M = a.median_window;
    double *ring = a.w.wring + (size_t)tb * kWindow;
    const StepRec *rp = a.records + (size_t)prm.trace_id * a.rec_stride + a.rec_off;
    const bool rec_on = prm.record_slot != AGFT_NO_RECORD;
    const uint32_t *rawp = a.cl_enable ? a.raw + ((size_t)prm.trace_id * a.rec_stride + a.rec_off) * AGFT_ROW_WORDS
                                       : nullptr;
    uint32_t clq = 0u, clqb = 0u;                                // ENV-C backlogs (ENV.md §6)
    if (rawp) {
        clq = a.w.clq[(size_t)tb * 2];
        clqb = a.w.clq[(size_t)tb * 2 + 1];
    }

    const SmemWindow win{S, kSoloThreads};
    double oldest = ring_oldest(ring, wcount, whead, M);
    for (uint32_t s = 0; s < a.n_steps; ++s) {
        const StepRec *rc = rp + s;                       // shared by the lanes of a trace: L1 broadcast
        if (s + 1 < a.n_steps) {
            prefetch_l1(rc + 1);
            if (rawp) prefetch_l1(rawp + (size_t)(s + 1) * AGFT_ROW_WORDS);
        }
        // off the chain: the reward's reference (median of the window before this push) and
        // Welford's 1/n depend only on the tuner's state at the start of the step
        const double ref = wcount > 0 ? win.median(wcount) : 0.0;
        const double inv_n = xrcp_nb((double)(n + 1u));
        // a7: response at the only active frequency
        const uint32_t rI = __ldg(&rc->I), rP = __ldg(&rc->P);
        const double rinvIm = __ldg(&rc->invIm), rnT = __ldg(&rc->nT), rnE = __ldg(&rc->nE);
        double g = __ldg(&rc->g), wIm = __ldg(&rc->wIm), baseE = __ldg(&rc->baseE), baseEDP = __ldg(&rc->baseEDP);
        double x0 = __ldg(&rc->x[0]);
        uint32_t arr = 0u;
        if (rawp) {                                              // ENV-C: the servers see their backlog
            const ClosedRec cr = closed_record(rawp + (size_t)s * AGFT_ROW_WORDS, clq, clqb, rI, rP, rinvIm, rnT,
                                               rnE, ec, a);
            x0 = cr.x0;
            g = cr.g;
            wIm = cr.wIm;
            baseE = cr.baseE;
            baseEDP = cr.baseEDP;
            arr = cr.arr;
        }
        const Response o = env_response(dec, pre, pw, rI, rP, g, rinvIm, __ldg(&rc->invAm), wIm, rnT, rnE, invW,
                                        q_over, a.u_max, a.u_floor, a.p_idle, a.W);
        if (rawp) clq = closed_carry(arr + clq, o.u, a.cl_q_max);
        // a8: reward against the median of the window, then push the EDP
        const double r = wcount > 0 ? reward_of(o.edp, ref, a.clip_lo, a.clip_hi) : 0.0;
        if (!isfinite(o.edp) || !isfinite(r)) {
            st.flags |= 1u;
            break;
        }
        push_edp(win, ring, wcount, whead, M, o.edp, oldest);
        if (a.ph_enable) {                                       // ENV.md §4.10 (one arm: α is moot)
            ph.exploit_steps += ph.phase;
            ph_observe(ph, r, a.t0 + s, a.ph_window, a.ph_delta, a.ph_lambda);
        }
        // a9: Eqs. 3–5 on the (only) chosen arm, Welford means
        double x[D];
#pragma unroll
        for (int q = 0; q < D; ++q) x[q] = __ldg(&rc->x[q]);
        x[0] = x0;
        if (!sm_update<D>(A, th, b, x, r)) {                    // SPD guard: freeze (flags bit 1)
            st.flags |= kFlagFrozen | kFlagSpd;
            break;
        }
        welford_inv(n, rbar, ebar, r, o.edp, inv_n);
        // a11
        stats_add(st, o, r, baseE, baseEDP, k, 1u);
        if (rec_on) {
            if (a.traj) a.traj[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = (uint8_t)k;
            if (a.gap) a.gap[(size_t)prm.record_slot * a.rec_stride + a.rec_off + s] = kInf;
        }
    }
    if (a.chosen) a.chosen[tb] = (uint32_t)k;

#pragma unroll
    for (int e = 0; e < P; ++e) a.w.ainv[((size_t)tb * P + e) * kMaxArms + k] = A[e];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        a.w.theta[((size_t)tb * D + r) * kMaxArms + k] = th[r];
        a.w.b[((size_t)tb * D + r) * kMaxArms + k] = b[r];
    }
    a.w.n[(size_t)tb * kMaxArms + k] = n;
    a.w.rbar[(size_t)tb * kMaxArms + k] = rbar;
    a.w.ebar[(size_t)tb * kMaxArms + k] = ebar;
    for (int j = 0; j < kWindow; ++j) a.w.wsorted[(size_t)tb * kWindow + j] = SW(j);
    a.w.wmeta[(size_t)tb * 2] = wcount;
    a.w.wmeta[(size_t)tb * 2 + 1] = whead;
    if (rawp) {
        a.w.clq[(size_t)tb * 2] = clq;
        a.w.clq[(size_t)tb * 2 + 1] = clqb;
    }
    st.n_active = 1;
    if (a.ph_enable) {
        a.w.ph[tb] = ph;
        ph_to_stats(ph, st);
    }
    prof_add(a, a.w.acc + tb, st);
    a.w.acc[tb] = st;
#undef SW
}

template <int D>
static cudaError_t launch_solo_d(const ReplayArgs &a, cudaStream_t s)
{
    const uint32_t blocks = (a.n_tuners + kSoloThreads - 1) / kSoloThreads;
    solo_kernel<D><<<blocks, kSoloThreads, 0, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

template <int D>
static int occupancy_solo_d()
{
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, solo_kernel<D>, kSoloThreads, 0) != cudaSuccess) return -1;
    return blocks * kSoloThreads;                     // one tuner per lane
}

int occupancy_solo(uint32_t D)
{
    switch (D) {
    case 1: return occupancy_solo_d<1>();
    case 2: return occupancy_solo_d<2>();
    case 3: return occupancy_solo_d<3>();
    case 4: return occupancy_solo_d<4>();
    case 5: return occupancy_solo_d<5>();
    case 6: return occupancy_solo_d<6>();
    default: return occupancy_solo_d<7>();
    }
}

cudaError_t launch_solo(const ReplayArgs &a, uint32_t D, cudaStream_t s)
{
    if (a.n_tuners == 0 || a.n_steps == 0) return cudaSuccess;
    switch (D) {
    case 1: return launch_solo_d<1>(a, s);
    case 2: return launch_solo_d<2>(a, s);
    case 3: return launch_solo_d<3>(a, s);
    case 4: return launch_solo_d<4>(a, s);
    case 5: return launch_solo_d<5>(a, s);
    case 6: return launch_solo_d<6>(a, s);
    default: return launch_solo_d<7>(a, s);
    }
}

}  // namespace agft
