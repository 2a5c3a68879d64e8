// trace.cu — K1: ENV-T trace rows + per-window step records (rows a0, a2 and the
// row-only part of a7), plus the workspace init and export kernels.
//
// One thread per (trace, step): six Philox4x32-10 draws (ENV.md §1-2), integer
// row synthesis, then the record of ENV.md §3.2 including the f_max baseline
// response.  HBM-write bound: 128 B (+48 B raw) per (trace, step).
#include "env_t.cuh"

namespace agft {

__global__ void __launch_bounds__(256) trace_kernel(const __grid_constant__ TraceArgs a)
{
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (uint64_t)a.n_traces * a.n_steps) return;
    const uint32_t lr = (uint32_t)(gid / a.n_steps);          // local trace
    const uint32_t s = (uint32_t)(gid - (uint64_t)lr * a.n_steps);
    const uint32_t t = a.t0 + s;                              // global step
    const uint32_t r = a.trace_base + lr;                     // global trace id (Philox key)
    const agft_trace_cfg &c = a.tc;
    const Philox ph{(uint32_t)a.seed ^ r, (uint32_t)(a.seed >> 32)};

    uint32_t pattern = c.pattern_mode < 3 ? c.pattern_mode : (c.pattern_mode == 3 ? r % 3u : 1u + r % 2u);
    const uint32_t p = prototype_of(c, ph, t);                // segment prototype (Table 1 mix)
    // rate multiplier (diurnal knots, burst)
    double m = 1.0;
    if (pattern >= 1) {
        const uint32_t sday = t % (24u * c.steps_per_hour);
        const uint32_t h = sday / c.steps_per_hour;
        const double fr = xdiv((double)(sday - h * c.steps_per_hour), (double)c.steps_per_hour);
        m = xadd(c.knot[h], xmul(xsub(c.knot[(h + 1) % 24], c.knot[h]), fr));
        if (pattern == 2 && ph(t / c.burst_steps, 2u, 0u, 0u).x < c.burst_p32) m = xmul(m, c.burst_mult);
    }
    const double lam = xmul(xmul(c.lambda0, c.conc_mult[p]), m);

    const uint4 U0 = ph(t, 3u, 0u, 0u), U1 = ph(t, 3u, 1u, 0u), U2 = ph(t, 3u, 2u, 0u), U3 = ph(t, 3u, 3u, 0u);
    const uint32_t U[12] = {U0.x, U0.y, U0.z, U0.w, U1.x, U1.y, U1.z, U1.w, U2.x, U2.y, U2.z, U2.w};
    double z = unit32(U[0]);
#pragma unroll
    for (int i = 1; i < 12; ++i) z = xadd(z, unit32(U[i]));
    z = xsub(z, 6.0);
    const double W = a.env.window_s;
    const double mu = xmul(lam, W);
    const double va = xadd(xadd(mu, xmul(xsqrt(mu), z)), 0.5);
    const uint32_t arr = va < 0.0 ? 0u : (uint32_t)floor(va);
    const uint32_t ctx = c.ctx_lo[p] + (uint32_t)(((uint64_t)U3.x * (uint64_t)(c.ctx_hi[p] - c.ctx_lo[p] + 1)) >> 32);
    const uint32_t gen = c.gen_lo[p] + (uint32_t)(((uint64_t)U3.y * (uint64_t)(c.gen_hi[p] - c.gen_lo[p] + 1)) >> 32);
    const uint32_t h0 = (uint32_t)floor(xadd(xmul((double)arr, c.hit_rate[p]), 0.5));
    const uint32_t hits = min(arr, h0);
    const uint32_t misses = arr - hits;
    const uint32_t ctot = (uint32_t)floor(xadd(xmul(lam, xadd(c.e2e0, xmul((double)gen, c.tau_ref))), 0.5));
    const uint32_t running = min(ctot, c.cap);
    const uint32_t waiting = ctot - running;
    const uint32_t iters = running > 0 ? (uint32_t)floor(xdiv(W, xadd(c.t_iter0, xmul(c.t_iter1, (double)running)))) : 0u;
    const uint32_t decode = running * iters;
    const uint32_t prefill = arr * ctx - hits * (ctx / 2);
    const uint32_t kv_used = min(c.kv_total, running * (ctx + gen / 2));
    const uint4 N = ph(t, 4u, 0u, 0u);

    if (a.raw) {
        uint4 *o = reinterpret_cast<uint4 *>(a.raw + gid * AGFT_ROW_WORDS);
        o[0] = make_uint4(waiting, running, prefill, decode);
        o[1] = make_uint4(iters, kv_used, hits, misses);
        o[2] = N;
    }

    // ---- ENV.md §3.2 record: context (§4.1) + row-only response terms
    StepRec rec;
    context_of(waiting, running, prefill, decode, iters, kv_used, hits, misses, W, c.kv_total, a.norm_lo,
               a.norm_hi, rec.x);
    rec.I = iters;
    rec.P = prefill;
    const double rho = xdiv((double)(running + waiting), (double)a.cap);
    rec.g = rho > 1.0 ? xmul(rho, xsqrt(rho)) : 1.0;
    rec.invIm = xdiv(1.0, (double)(iters > 0 ? iters : 1u));
    rec.invAm = xdiv(1.0, (double)(arr > 0 ? arr : 1u));
    rec.wIm = xmul((double)waiting, rec.invIm);
    rec.nT = xadd(1.0, xmul(a.env.sigma_t, xsub(xmul(2.0, unit53(N.x, N.y)), 1.0)));
    rec.nE = xadd(1.0, xmul(a.env.sigma_e, xsub(xmul(2.0, unit53(N.z, N.w)), 1.0)));
    const EnvConsts &ec = *a.envc;
    double bE, bT;
    response(rec, ec.base_dec, ec.base_pre, ec.base_pw, W, ec.invW, ec.q_over, a.env.u_max,
             a.env.u_floor, a.env.p_idle, bE, bT);
    rec.baseE = bE;
    rec.baseEDP = xmul(bE, bT);

    uint4 *o = reinterpret_cast<uint4 *>(a.records + gid);
    const uint4 *src = reinterpret_cast<const uint4 *>(&rec);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = src[i];
}

cudaError_t launch_trace(const TraceArgs &a, cudaStream_t s)
{
    const uint64_t n = (uint64_t)a.n_traces * a.n_steps;
    if (n == 0) return cudaSuccess;
    const uint32_t blocks = (uint32_t)((n + 255) / 256);
    trace_kernel<<<blocks, 256, 0, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- workspace init
struct InitArgs {
    Ws w;
    uint32_t N, K, D, des;
    uint32_t f_min_mhz, f_step_mhz, f_max_hw_mhz;
    agft_env env;
};

__global__ void init_env_kernel(const __grid_constant__ InitArgs a)
{
    // ENV.md §3 / §3.1: per-arm and baseline constants, exactly as written.
    EnvConsts &e = *a.w.env;
    const int k = threadIdx.x;
    const double fmax = xdiv((double)a.f_max_hw_mhz, 1000.0);
    auto consts = [&](uint32_t F, double &dec, double &pre, double &pw) {
        const double f = xdiv((double)F, 1000.0);
        dec = xdiv(a.env.c_decode, xadd(a.env.beta, xmul(xsub(1.0, a.env.beta), xdiv(f, fmax))));
        pre = xdiv(a.env.c_prefill, f);
        pw = xadd(xmul(a.env.k_lin, f), xmul(a.env.k_cube, xmul(xmul(f, f), f)));
    };
    if (k < kMaxArms) {
        double dec = 0.0, pre = 0.0, pw = 0.0;
        if ((uint32_t)k < a.K) consts(a.f_min_mhz + (uint32_t)k * a.f_step_mhz, dec, pre, pw);
        e.dec[k] = dec;
        e.pre[k] = pre;
        e.pw[k] = pw;
    }
    if (k == 0) {
        consts(a.f_max_hw_mhz, e.base_dec, e.base_pre, e.base_pw);
        e.invW = xdiv(1.0, a.env.window_s);
        e.q_over = xdiv(1.0, xmul(a.env.u_max, xsub(1.0, a.env.u_max)));
        e.fmax = fmax;
    }
}

__global__ void init_tuner_kernel(const __grid_constant__ InitArgs a)
{
    const uint32_t P = a.D * (a.D + 1) / 2;
    const uint64_t total = (uint64_t)a.N * kMaxArms;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t tb = i / kMaxArms;
        const uint32_t k = (uint32_t)(i % kMaxArms);
        // AMB-2: A = I (so A⁻¹ = I), b = 0, θ = 0, n = 0, r̄ = ē = 0
        uint32_t e = 0;
        for (uint32_t r = 0; r < a.D; ++r)
            for (uint32_t c = r; c < a.D; ++c, ++e)
                a.w.ainv[(tb * P + e) * kMaxArms + k] = (r == c) ? 1.0 : 0.0;
        for (uint32_t r = 0; r < a.D; ++r) {
            a.w.theta[(tb * a.D + r) * kMaxArms + k] = 0.0;
            a.w.b[(tb * a.D + r) * kMaxArms + k] = 0.0;
        }
        a.w.n[tb * kMaxArms + k] = 0;
        a.w.rbar[tb * kMaxArms + k] = 0.0;
        a.w.ebar[tb * kMaxArms + k] = 0.0;
        if (k < kWindow) {
            a.w.wsorted[tb * kWindow + k] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
            a.w.wring[tb * kWindow + k] = 0.0;
        }
        if (k < 4) {
            const uint32_t lo = 32u * k;
            uint32_t bits = 0;
            if (a.K > lo) bits = (a.K - lo >= 32u) ? kFull : ((1u << (a.K - lo)) - 1u);
            a.w.active[tb * 4 + k] = bits;
            a.w.extm[tb * 4 + k] = 0u;
        }
        if (k < 2) {
            a.w.wmeta[tb * 2 + k] = 0;
            a.w.clq[tb * 2 + k] = 0;                    // ENV-C: no backlog at t = 0 (ENV.md §6)
        }
        if (a.des && k < (uint32_t)kDesR) {            // ENV-S (ENV.md §7): idle server, empty slots
            DesSlot sl = {};
            a.w.desr[tb * kDesR + k] = sl;
            if (k == 0) {
                DesScal sc = {};
                a.w.des[tb] = sc;
            }
        }
        if (k == 0) {
            agft_tuner_stats st = {};
            st.traj_hash = kFnvOffset;
            st.n_active = a.K;
            st.first_exploit_t = AGFT_NEVER;
            st.last_anchor = AGFT_NEVER;
            a.w.acc[tb] = st;
            PhState ph = {};
            ph.first_exploit_t = AGFT_NEVER;
            a.w.ph[tb] = ph;
        }
    }
}

cudaError_t launch_init(const Ws &w, const agft_config &cfg, cudaStream_t s)
{
    InitArgs a;
    a.w = w;
    a.N = cfg.n_tuners;
    a.K = cfg.grid.n_arms;
    a.D = cfg.d;
    a.des = cfg.closed.enable == 2u ? 1u : 0u;
    a.f_min_mhz = cfg.grid.f_min_mhz;
    a.f_step_mhz = cfg.grid.f_step_mhz;
    a.f_max_hw_mhz = cfg.grid.f_max_hw_mhz;
    a.env = cfg.env;
    init_env_kernel<<<1, kMaxArms, 0, s>>>(a); note_launches(1);
    const uint64_t total = (uint64_t)a.N * kMaxArms;
    uint32_t blocks = (uint32_t)((total + 255) / 256);
    if (blocks > 148u * 32u) blocks = 148u * 32u;
    init_tuner_kernel<<<blocks, 256, 0, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- export one tuner's arms
__global__ void export_kernel(Ws w, uint32_t tuner, uint32_t K, uint32_t D, double *ainv, double *b,
                              double *theta, uint32_t *n, double *rbar, double *ebar, uint32_t *mask)
{
    const uint32_t k = threadIdx.x;
    const uint32_t P = D * (D + 1) / 2;
    const uint64_t tb = tuner;
    if (k < K) {
        if (ainv)
            for (uint32_t e = 0; e < P; ++e) ainv[k * P + e] = w.ainv[(tb * P + e) * kMaxArms + k];
        for (uint32_t i = 0; i < D; ++i) {
            if (b) b[k * D + i] = w.b[(tb * D + i) * kMaxArms + k];
            if (theta) theta[k * D + i] = w.theta[(tb * D + i) * kMaxArms + k];
        }
        if (n) n[k] = w.n[tb * kMaxArms + k];
        if (rbar) rbar[k] = w.rbar[tb * kMaxArms + k];
        if (ebar) ebar[k] = w.ebar[tb * kMaxArms + k];
    }
    if (mask && k < 4) mask[k] = w.active[tb * 4 + k];
}

cudaError_t launch_export(const Ws &w, uint32_t tuner, uint32_t K, uint32_t D, double *ainv, double *b,
                          double *theta, uint32_t *n, double *rbar, double *ebar, uint32_t *mask,
                          cudaStream_t s)
{
    export_kernel<<<1, kMaxArms, 0, s>>>(w, tuner, K, D, ainv, b, theta, n, rbar, ebar, mask); note_launches(1);
    return cudaGetLastError();
}

}  // namespace agft
