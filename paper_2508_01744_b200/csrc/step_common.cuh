// step_common.cuh — per-step pieces shared by the replay kernels (WIDE / SEG / SOLO):
// the ENV-R response, the reward clip, Welford and stats accumulation, all in the exact
// IEEE arithmetic ENV.md §0 prescribes.
#pragma once
#include "agft_internal.cuh"

namespace agft {

constexpr double kInf = __builtin_huge_val();

// ENV.md §3.3: response at the chosen frequency (per-arm constants dec/pre/pw).
struct Response {
    double E, tpot, ttft, edp, u;   // u: the window's utilisation busy/W (ENV-C backlog, ENV.md §6)
};

__device__ __forceinline__ Response env_response(double dec, double pre, double pw, uint32_t I, uint32_t P,
                                                 double g, double invIm, double invAm, double wIm, double nT,
                                                 double nE, double invW, double q_over, double u_max,
                                                 double u_floor, double p_idle, double W)
{
    Response o;
    const double t_dec = xmul((double)I, dec);
    const double t_pre = xmul((double)P, pre);
    const double busy = xmul(xadd(t_dec, t_pre), g);
    const double u = xmul(busy, invW);
    const double q = u <= u_max ? xrcp_nb(xsub(1.0, u)) : xmul(u, q_over);
    o.tpot = xmul(xmul(xmul(xadd(dec, xmul(t_pre, invIm)), g), q), nT);
    double ue = u > 1.0 ? 1.0 : u;                  // (fmin/fmax compile to ~7 instructions each: NaN rules)
    ue = ue < u_floor ? u_floor : ue;
    o.E = xmul(xmul(xadd(p_idle, xmul(pw, ue)), W), nE);
    o.ttft = xmul(xadd(xmul(t_pre, invAm), xmul(t_dec, wIm)), q);
    o.edp = xmul(o.E, o.tpot);
    o.u = u;
    return o;
}

// ---- ENV-C closed loop (ENV.md §6): the window as the tuner's server (carried backlog q) and
// the f_max baseline server (backlog qb) see it.  Returns x1 (normalised), g and wIm of the
// tuner's server and the baseline's (E, EDP); advances qb.  Exact arithmetic (ENV.md §0).
struct ClosedRec {
    double x0, g, wIm, baseE, baseEDP;
    uint32_t arr;
};

__device__ __forceinline__ uint32_t closed_carry(uint32_t D, double u, uint32_t q_max)
{
    const uint32_t served = u > 1.0 ? (uint32_t)floor(xdiv((double)D, u)) : D;
    return min(q_max, D - served);
}

__device__ __forceinline__ double rho_penalty(uint32_t running, uint32_t waiting, uint32_t cap)
{
    const double rho = xdiv((double)(running + waiting), (double)cap);
    return rho > 1.0 ? xmul(rho, xsqrt(rho)) : 1.0;
}

__device__ __forceinline__ ClosedRec closed_record(const uint32_t *__restrict__ rw, uint32_t q, uint32_t &qb,
                                                   uint32_t I, uint32_t P, double invIm, double nT, double nE,
                                                   const EnvConsts *ec, const ReplayArgs &a)
{
    ClosedRec c;
    const uint4 r0 = __ldg(reinterpret_cast<const uint4 *>(rw));
    const uint4 r1 = __ldg(reinterpret_cast<const uint4 *>(rw) + 1);
    const uint32_t wr = r0.x, run = r0.y;
    c.arr = r1.z + r1.w;
    const uint32_t wq = wr + q, wb = wr + qb;
    {
        const double lo = a.norm_lo[0], hi = a.norm_hi[0];
        double xv = 0.0;
        if (hi > lo) {
            xv = xdiv(xsub(wq > 0 ? 1.0 : 0.0, lo), xsub(hi, lo));
            xv = xv < 0.0 ? 0.0 : (xv > 1.0 ? 1.0 : xv);
        }
        c.x0 = xv;
    }
    c.g = rho_penalty(run, wq, a.cap);
    c.wIm = xmul((double)wq, invIm);
    const double gb = rho_penalty(run, wb, a.cap);
    const double bdec = ec->base_dec, bpre = ec->base_pre, bpw = ec->base_pw;
    const double bt_dec = xmul((double)I, bdec);
    const double bt_pre = xmul((double)P, bpre);
    const double bu = xmul(xmul(xadd(bt_dec, bt_pre), gb), ec->invW);
    const double bq = bu <= a.u_max ? xdiv(1.0, xsub(1.0, bu)) : xmul(bu, ec->q_over);
    const double btpot = xmul(xmul(xmul(xadd(bdec, xmul(bt_pre, invIm)), gb), bq), nT);
    double bue = bu > 1.0 ? 1.0 : bu;
    bue = bue < a.u_floor ? a.u_floor : bue;
    c.baseE = xmul(xmul(xadd(a.p_idle, xmul(bpw, bue)), a.W), nE);
    c.baseEDP = xmul(c.baseE, btpot);
    qb = closed_carry(c.arr + qb, bu, a.cl_q_max);
    return c;
}

// L1 prefetch of the next window's 128-B step record: its fields head the next step's serial
// chain (context → scores), so the L2 round trip is taken off it (no register cost)
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// a8: r = clip(1 − EDP/ref) (AMB-3)
__device__ __forceinline__ double reward_of(double edp, double ref, double lo, double hi)
{
    double r = xsub(1.0, xdiv_nb(edp, ref));
    return r < lo ? lo : (r > hi ? hi : r);
}

// Welford means with one reciprocal (ENV.md §4.7)
__device__ __forceinline__ void welford(uint32_t &n, double &rbar, double &ebar, double r, double edp)
{
    n += 1u;
    const double inv = xdiv(1.0, (double)n);
    rbar = xadd(rbar, xmul(xsub(r, rbar), inv));
    ebar = xadd(ebar, xmul(xsub(edp, ebar), inv));
}

// the same with 1/(n+1) computed earlier, off the reward chain (identical values)
__device__ __forceinline__ void welford_inv(uint32_t &n, double &rbar, double &ebar, double r, double edp, double inv)
{
    n += 1u;
    rbar = xadd(rbar, xmul(xsub(r, rbar), inv));
    ebar = xadd(ebar, xmul(xsub(edp, ebar), inv));
}

// ENV.md §4.10 observe_reward: the Page-Hinkley detector on the reward of step t (after a8)
__device__ __forceinline__ void ph_observe(PhState &p, double r, uint32_t t, uint32_t W, double delta, double lambda)
{
    p.n += 1u;
    const double inv = xdiv(1.0, (double)p.n);
    p.mean = xadd(p.mean, xmul(xsub(r, p.mean), inv));
    p.cum = xadd(p.cum, xsub(xsub(r, p.mean), delta));
    if (p.cum < p.min) p.min = p.cum;
    p.quiet += 1u;
    if (xsub(p.cum, p.min) > lambda) {               // drift alarm: reset, re-enter Exploration
        p.alarms += 1u;
        p.quiet = 0u;
        p.n = 0u;
        p.mean = 0.0;
        p.cum = 0.0;
        p.min = 0.0;
        p.phase = 0u;
    } else if (p.phase == 0u && p.quiet >= W) {       // W quiet observations: Exploitation (Eq. 2)
        p.phase = 1u;
        if (p.first_exploit_t == AGFT_NEVER) p.first_exploit_t = t;
    }
}

__device__ __forceinline__ void ph_to_stats(const PhState &p, agft_tuner_stats &st)
{
    st.exploit_steps = p.exploit_steps;
    st.ph_alarms = p.alarms;
    st.first_exploit_t = p.first_exploit_t;
    st.phase = p.phase;
}

// a11: stats in ENV.md §4.9 order
__device__ __forceinline__ void stats_add(agft_tuner_stats &st, const Response &o, double r, double baseE,
                                          double baseEDP, int kstar, uint32_t nact)
{
    st.sum_energy = xadd(st.sum_energy, o.E);
    st.sum_tpot = xadd(st.sum_tpot, o.tpot);
    st.sum_ttft = xadd(st.sum_ttft, o.ttft);
    st.sum_edp = xadd(st.sum_edp, o.edp);
    st.sum_reward = xadd(st.sum_reward, r);
    st.base_energy = xadd(st.base_energy, baseE);
    st.base_edp = xadd(st.base_edp, baseEDP);
    st.traj_hash = (st.traj_hash ^ (uint64_t)kstar) * kFnvPrime;
    st.sum_active += nact;
    st.steps += 1u;
    st.last_arm = (uint32_t)kstar;
}

// Eq. 1's quadratic form xᵀA⁻¹x = Σ_e w_e·A⁻¹_e over the packed upper triangle (w_e = x_i x_j,
// doubled off the diagonal), in four independent FMA chains (ILP; scores are
// tolerance-compared, ENV.md §4.3)
template <int P>
__device__ __forceinline__ double quad_form(const double (&w)[P], const double *A, int stride)
{
    double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
#pragma unroll
    for (int e = 0; e < P; e += 4) {
        q0 = fma(w[e], A[e * stride], q0);
        if (e + 1 < P) q1 = fma(w[e + 1 < P ? e + 1 : e], A[(e + 1 < P ? e + 1 : e) * stride], q1);
        if (e + 2 < P) q2 = fma(w[e + 2 < P ? e + 2 : e], A[(e + 2 < P ? e + 2 : e) * stride], q2);
        if (e + 3 < P) q3 = fma(w[e + 3 < P ? e + 3 : e], A[(e + 3 < P ? e + 3 : e) * stride], q3);
    }
    return (q0 + q1) + (q2 + q3);
}

// The same form row by row without the pair weights: xᵀA⁻¹x = Σ_i x_i (A_ii x_i + Σ_{j>i} A_ij (2x_j)),
// x2 = 2x (exact).  7 + 28 FP64 instructions per arm and 2·D registers of weights instead of
// D(D+1)/2 + the 49 instructions that build them once per step (SEG2: two arms per lane)
template <int D>
__device__ __forceinline__ double quad_form_rows(const double (&x)[D], const double (&x2)[D], const double *A,
                                                 int stride)
{
    double q0 = 0.0, q1 = 0.0;
    int e = 0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double in = A[e * stride] * x[i];
        ++e;
#pragma unroll
        for (int j = i + 1; j < D; ++j, ++e) in = fma(A[e * stride], x2[j], in);
        if (i & 1) q1 = fma(x[i], in, q1);
        else q0 = fma(x[i], in, q0);
    }
    return q0 + q1;
}

template <int D>
__device__ __forceinline__ void pair_weights(const double (&x)[D], double (&w)[D * (D + 1) / 2])
{
    int e = 0;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c, ++e) w[e] = (r == c) ? x[r] * x[r] : 2.0 * x[r] * x[c];
}

// a3: α_t = α0/√(1 + t/τ) (AMB-1), via one reciprocal square root
__device__ __forceinline__ double alpha_t(double alpha0, uint32_t t, double inv_tau)
{
    return alpha0 * rsqrt(fma((double)t, inv_tau, 1.0));
}

// packed upper-triangle index of (r, c), r ≤ c, for a D×D symmetric matrix
template <int D>
__device__ __forceinline__ constexpr int pidx(int r, int c)
{
    return r * D - r * (r - 1) / 2 + (c - r);
}

// SPD guard of a rank-1 update (SURVEY §5 failure detection; A⁻¹ stays symmetric
// positive definite with eigenvalues in (0, 1] since λ_min(A) ≥ 1): xᵀA⁻¹x must not be negative
// beyond rounding and every updated diagonal entry must stay positive.  A violation (a corrupted
// or numerically broken arm) freezes the tuner with flags bit 1 (kFlagSpd).
constexpr uint32_t kFlagFrozen = 1u, kFlagSpd = 2u;
__device__ __forceinline__ bool spd_quad_ok(double xz) { return xz > -1e-12; }

// Sherman–Morrison update of one arm held in registers (Eqs. 3–5, AMB-21):
// z = A⁻¹x, δ = 1 + xᵀz, A⁻¹ ← A⁻¹ − z zᵀ/δ, θ ← θ + z (r − θ·x)/δ, b ← b + r x (exact).
// Returns the SPD guard.
template <int D>
__device__ __forceinline__ bool sm_update(double (&A)[D * (D + 1) / 2], double (&th)[D], double (&b)[D],
                                          const double (&x)[D], double r)
{
    double z[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) acc = fma(A[i <= c ? pidx<D>(i, c) : pidx<D>(c, i)], x[c], acc);
        z[i] = acc;
    }
    double xz = 0.0, px = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        xz = fma(x[i], z[i], xz);
        px = fma(th[i], x[i], px);
    }
    const double invd = xrcp_nb(1.0 + xz);
    bool ok = spd_quad_ok(xz);
#pragma unroll
    for (int r0 = 0; r0 < D; ++r0) {
        const double zr = -z[r0] * invd;
#pragma unroll
        for (int c = r0; c < D; ++c) A[pidx<D>(r0, c)] = fma(zr, z[c], A[pidx<D>(r0, c)]);
        ok = ok && A[pidx<D>(r0, r0)] > 0.0;
    }
    const double coef = (r - px) * invd;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        th[i] = fma(z[i], coef, th[i]);
        b[i] = xadd(b[i], xmul(r, x[i]));
    }
    return ok;
}

// ---- the sorted EDP window of ONE tuner in a strided shared-memory column (lane-private)
// S[j * stride], j < 64, +inf padded; ring (chronological) in global memory.
struct SmemWindow {
    double *S;
    int stride;
    __device__ __forceinline__ double &at(int j) const { return S[j * stride]; }

    __device__ __forceinline__ double median(uint32_t n) const
    {
        return (n & 1u) ? at(n >> 1) : xmul(xadd(at((n >> 1) - 1), at(n >> 1)), 0.5);
    }
    // #(S[0..n) < v): branch-free binary search (n ≤ 64)
    __device__ __forceinline__ int count_less(int n, double v) const
    {
        int lo = 0;
#pragma unroll
        for (int step = 64; step > 0; step >>= 1)
            if (lo + step <= n && at(lo + step - 1) < v) lo += step;
        return lo;
    }
    // insert into a window holding n < M values: position by binary search, then a
    // fixed-length shift whose loads are independent (pipelined, no data-dependent exit)
    __device__ __forceinline__ void insert(uint32_t n, double v) const
    {
        const int p = count_less((int)n, v);
        for (int j = (int)n; j > p; --j) at(j) = at(j - 1);
        at(p) = v;
    }
    // #(S[0..64) < v) in two dependent shared-memory round trips instead of seven: the 8 block
    // maxima S[8i+7] say how many whole blocks are below v, then the 8 entries of the next block.
    // Entries past the count are +inf, so this equals count_less(n, v) for any n ≤ 64 and finite v.
    __device__ __forceinline__ int count_less64(double v) const
    {
        int c = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) c += at(8 * i + 7) < v ? 1 : 0;
        if (c == 8) return 64;
        int r = 8 * c;
#pragma unroll
        for (int k = 0; k < 7; ++k) r += at(8 * c + k) < v ? 1 : 0;
        return r;
    }
    // replace `old` (present) by v in a full window of M values: both positions (independent),
    // then shift the elements between them by one slot
    __device__ __forceinline__ void replace(uint32_t M, double old, double v) const
    {
        const int po = count_less64(old);                   // S[po] == old
        const int lv = count_less64(v);                     // #(S < v), old included
        // the shifts move up to 63 entries and their lengths differ between the lanes of a warp:
        // 8 entries per iteration (all 8 loads issued before the 8 stores) instead of one, so the
        // divergent loop runs ≤ 8 times and its loads overlap
        if (v < old) {                                      // v lands at lv ≤ po: shift [lv, po) up
            for (int j0 = po; j0 > lv; j0 -= 8) {
                double t[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) t[k] = at(max(j0 - 1 - k, 0));
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (j0 - k > lv) at(j0 - k) = t[k];
            }
            at(lv) = v;
        } else if (v > old) {                               // v lands at lv − 1 ≥ po: shift (po, lv) down
            const int pn = lv - 1;
            for (int j0 = po; j0 < pn; j0 += 8) {
                double t[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) t[k] = at(min(j0 + 1 + k, kWindow - 1));
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (j0 + k < pn) at(j0 + k) = t[k];
            }
            at(pn) = v;
        }                                                   // v == old: the multiset is unchanged
    }
};

__device__ __forceinline__ void push_edp(const SmemWindow &win, double *ring, uint32_t &wcount, uint32_t &whead,
                                         uint32_t M, double edp, double &oldest);

// a8 for a lane-private window: reward against the median of the window, then push edp.
// `oldest` carries the ring value that the next push evicts (ring[whead] of a full window),
// loaded one step ahead so its global-memory latency overlaps the step.
__device__ __forceinline__ double reward_and_push(const SmemWindow &win, double *ring, uint32_t &wcount,
                                                  uint32_t &whead, uint32_t M, double edp, double clip_lo,
                                                  double clip_hi, bool &finite_ok, double &oldest)
{
    double r = 0.0;
    if (wcount > 0) r = reward_of(edp, win.median(wcount), clip_lo, clip_hi);
    finite_ok = isfinite(edp) && isfinite(r);
    if (!finite_ok) return r;
    push_edp(win, ring, wcount, whead, M, edp, oldest);
    return r;
}

// push edp into a lane-private window (the second half of reward_and_push)
__device__ __forceinline__ void push_edp(const SmemWindow &win, double *ring, uint32_t &wcount, uint32_t &whead,
                                         uint32_t M, double edp, double &oldest)
{
    if (wcount < M) {
        win.insert(wcount, edp);
        ring[wcount] = edp;
        ++wcount;
    } else {
        win.replace(M, oldest, edp);
        ring[whead] = edp;
        whead = (whead + 1 == M) ? 0u : whead + 1;
    }
    if (wcount == M) oldest = ring[whead];
}

__device__ __forceinline__ double ring_oldest(const double *ring, uint32_t wcount, uint32_t whead, uint32_t M)
{
    return wcount == M ? ring[whead] : 0.0;
}

// The update with the packed A⁻¹ held in shared memory (entry e at Ac[e * stride], each read once),
// every store predicated on `on` and no branch: the warp runs it in one basic block with the
// independent work of the step (window, Welford), so the compiler can interleave them.  Lanes with
// on = false read their own (valid) column and discard the result.  Returns the SPD guard.
template <int D>
__device__ __forceinline__ bool sm_update_smem_pred(bool on, double *Ac, int stride, double (&th)[D], double *bcol,
                                                    int bstride, const double (&x)[D], double r)
{
    constexpr int P = D * (D + 1) / 2;
    double Ap[P];
#pragma unroll
    for (int e = 0; e < P; ++e) Ap[e] = Ac[e * stride];
    double z[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) acc = fma(Ap[i <= c ? pidx<D>(i, c) : pidx<D>(c, i)], x[c], acc);
        z[i] = acc;
    }
    double xz = 0.0, px = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        xz = fma(x[i], z[i], xz);
        px = fma(th[i], x[i], px);
    }
    const double invd = xrcp_nb(1.0 + xz);
    bool ok = spd_quad_ok(xz);
#pragma unroll
    for (int r0 = 0; r0 < D; ++r0) {
        const double zr = -z[r0] * invd;
#pragma unroll
        for (int c = r0; c < D; ++c) {
            const double v = fma(zr, z[c], Ap[pidx<D>(r0, c)]);
            if (on) Ac[pidx<D>(r0, c) * stride] = v;
            if (c == r0) ok = ok && v > 0.0;
        }
    }
    const double coef = (r - px) * invd;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double t = fma(z[i], coef, th[i]);
        th[i] = on ? t : th[i];
        double &bi = bcol[(size_t)i * bstride];
        const double nb = xadd(bi, xmul(r, x[i]));
        if (on) bi = nb;
    }
    return ok || !on;
}

}  // namespace agft
