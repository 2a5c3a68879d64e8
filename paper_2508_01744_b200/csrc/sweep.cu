// sweep.cu — K4: the offline frequency sweep of ENV.md §5 (
// P:257-262 "we iterated through all core frequencies … and calculated the corresponding
// EDP", Table 6 P:550-567 Offline vs Online) and K5: per-tuner regret against it.
//
// K4 mapping: one CTA per trace (256 threads), windows in tiles of 32 whose step records (4 KB)
// are staged in shared memory and broadcast to every arm.  Per-arm sums are folded in ascending t
// (ENV.md §5's left-to-right order, so chunked sweeps equal one sweep), the EDP also into the
// running sum of the window's prototype (runs split at segment boundaries).  k° per window
// (smallest arm index on ties) comes from warp min-reductions on the EDP bit patterns; its EDP
// and energy are folded in window order.  FP64-ALU bound: ~22 FP64 operations per (window, arm),
// the record read once per (trace, window) for 107 arms.
#include "env_t.cuh"

namespace agft {

namespace {

constexpr int kTile = 32;
constexpr int kThreads2 = 256;
constexpr int kWarps2 = kThreads2 / 32;
constexpr int kMaxArmsSw = 128;
constexpr int kLd = kTile + 1;                // arm-major tables [k][w], odd stride: conflict-free both ways
constexpr size_t kSweepSmem = 3 * (size_t)kMaxArmsSw * kLd * 8 + 2 * kTile * 8 +
                              3 * (size_t)kMaxArmsSw * 8;
#ifndef AGFT_SWEEP_ILP
#define AGFT_SWEEP_ILP 7                      // 8 warps × 7 = 56 arms per pass: two passes cover K = 107
#endif
constexpr int kIlp = AGFT_SWEEP_ILP;          // independent ENV-R evaluations in flight per thread
constexpr uint32_t kNoArm = 0xFFu;
constexpr double kInf = __builtin_huge_val();

struct SweepArgs {
    const StepRec *records;   // [n_traces][n_steps]
    double *S;                // [n_traces][K][3]   ΣE, ΣTPOT, ΣEDP
    double *SP;               // [n_traces][5][K]   Σ EDP per prototype
    uint32_t *NP;             // [n_traces][5]
    double *O;                // [n_traces][2]      Σ EDP°, Σ E°
    uint8_t *best;            // [n_traces][n_steps] k°, or null
    const EnvConsts *env;
    agft_trace_cfg tc;
    uint64_t seed;
    uint32_t trace_base, n_traces, t0, n_steps, K;
    double W, p_idle, u_floor, u_max;
};

// K4 v2 (v1 ran one 128-thread CTA per trace — 256 CTAs, ~7 warps per SM, 5.5% of
// the FP64 pipe).  The per-(trace, arm) sums must be folded left to right in t (ENV.md §5), but
// the ENV-R evaluations feeding them are independent, so the two are split inside the CTA:
//   A. all 256 threads evaluate the tile's 32 windows × 128 arm slots (16 evaluations each,
//      kIlp in flight) into shared memory E / TPOT / EDP tables [window][arm];
//   B. warps 0–3 (thread k = arm k) fold the tile into their sums in window order, while warps
//      4–7 find each window's k° (8 windows per warp) and one of them folds the oracle sums —
// so the FP64 evaluations run at 16 warps per SM (two CTAs of 110 KB) and the serial folds,
// ~1/20 of the arithmetic, overlap each other.  Results are bit-identical to v1.
// v3 (v2 issued ~89 warp instructions per (window, arm) evaluation, 29 of them FP64):
// phase A maps lane = window and warp = arm subset, so a lane converts its record's fields once per
// tile and every evaluation is the ENV-R arithmetic plus three conflict-free stores; the tables are
// arm-major with an odd stride (stores by window, folds by arm, k° scans all conflict-free); no
// evaluation of the padding slots k ≥ K (their EDP rows hold +inf for the k° scan).
__global__ void __launch_bounds__(kThreads2, 2) sweep_kernel(const __grid_constant__ SweepArgs a)
{
    extern __shared__ __align__(16) double sw[];
    double *s_E = sw, *s_T = s_E + kMaxArmsSw * kLd, *s_D = s_T + kMaxArmsSw * kLd;   // [k][kLd]
    double *s_oe = s_D + kMaxArmsSw * kLd, *s_oE = s_oe + kTile;
    double *s_dec = s_oE + kTile, *s_pre = s_dec + kMaxArmsSw, *s_pw = s_pre + kMaxArmsSw;
    const uint32_t r = blockIdx.x;                                               // local trace
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const EnvConsts &ec = *a.env;
    const double invW = ec.invW, q_over = ec.q_over;
    const Philox ph{(uint32_t)a.seed ^ (a.trace_base + r), (uint32_t)(a.seed >> 32)};
    const int K = (int)a.K;
    for (int q = tid; q < kMaxArmsSw; q += kThreads2) {
        s_dec[q] = q < K ? ec.dec[q] : 0.0;
        s_pre[q] = q < K ? ec.pre[q] : 0.0;
        s_pw[q] = q < K ? ec.pw[q] : 0.0;
    }
    for (int q = K * kLd + tid; q < kMaxArmsSw * kLd; q += kThreads2) s_D[q] = kInf;   // padding rows
    // phase B accumulators: warps 0–3, thread tid = arm
    const bool acc = warp < 4, arm = acc && tid < K;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, sp[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (arm) {
        const double *S = a.S + ((size_t)r * a.K + tid) * 3;
        s0 = S[0];
        s1 = S[1];
        s2 = S[2];
#pragma unroll
        for (int p = 0; p < 5; ++p) sp[p] = a.SP[((size_t)r * 5 + p) * a.K + tid];
    }
    double o0 = 0.0, o1 = 0.0;                                                   // warp 4, lane 0
    uint32_t np[5] = {0u, 0u, 0u, 0u, 0u};                                       // thread 0
    if (tid == 128) {
        o0 = a.O[2 * r];
        o1 = a.O[2 * r + 1];
    }
    if (tid == 0) {
#pragma unroll
        for (int p = 0; p < 5; ++p) np[p] = a.NP[r * 5 + p];
    }
    const StepRec *rp = a.records + (size_t)r * a.n_steps;
    // phase A lane = window: its record's six ENV-R fields straight from global memory (L1 after the
    // CTA's first warp), the next tile's loaded one tile ahead (no staging copy, no barrier for it)
    struct Fld {
        double g, invIm, nT, nE;
        uint2 ip;
    };
    auto load_fld = [&](uint32_t b) {
        Fld f;
        const StepRec *rc = rp + min(b + (uint32_t)lane, a.n_steps - 1);
        f.g = __ldg(&rc->g);
        f.invIm = __ldg(&rc->invIm);
        f.nT = __ldg(&rc->nT);
        f.nE = __ldg(&rc->nE);
        f.ip = __ldg(reinterpret_cast<const uint2 *>(&rc->I));
        return f;
    };
    Fld nxt = load_fld(0);
    __syncthreads();                                                             // arm constants, padding rows

    for (uint32_t base = 0; base < a.n_steps; base += kTile) {
        const int nw = (int)min((uint32_t)kTile, a.n_steps - base);
        const Fld cur = nxt;
        if (base + kTile < a.n_steps) nxt = load_fld(base + kTile);
        // ---- A: ENV-R (ENV.md §3.3) for window w = lane at arms warp, warp + 8, … (kIlp in flight)
        {
            const int w = lane;
            const double I = (double)cur.ip.x, P = (double)cur.ip.y, g = cur.g, invIm = cur.invIm, nT = cur.nT,
                         nE = cur.nE;
            for (int k0 = warp; k0 < K; k0 += kWarps2 * kIlp) {
                double E[kIlp], tp[kIlp];
#pragma unroll
                for (int j = 0; j < kIlp; ++j) {
                    const int k = min(k0 + kWarps2 * j, K - 1);
                    response_f(I, P, g, invIm, nT, nE, s_dec[k], s_pre[k], s_pw[k], a.W, invW, q_over, a.u_max,
                               a.u_floor, a.p_idle, E[j], tp[j]);
                }
#pragma unroll
                for (int j = 0; j < kIlp; ++j) {
                    const int k = k0 + kWarps2 * j;
                    if (k < K && w < nw) {
                        s_E[k * kLd + w] = E[j];
                        s_T[k * kLd + w] = tp[j];
                        s_D[k * kLd + w] = xmul(E[j], tp[j]);
                    }
                }
            }
        }
        __syncthreads();
        if (acc) {
            // ---- B1: per-arm folds in window order; prototype runs split at segment boundaries
            int w = 0;
            while (w < nw) {                                                     // uniform over warps 0–3
                const uint32_t t = a.t0 + base + (uint32_t)w;
                const uint32_t p = prototype_of(a.tc, ph, t);
                const int wend = w + (int)min((uint32_t)(nw - w), a.tc.seg_steps - t % a.tc.seg_steps);
                if (tid == 0) np[p] += (uint32_t)(wend - w);
                double cur = p == 0 ? sp[0] : p == 1 ? sp[1] : p == 2 ? sp[2] : p == 3 ? sp[3] : sp[4];
                if (arm) {
                    for (; w < wend; ++w) {
                        const double ed = s_D[tid * kLd + w];
                        s0 = xadd(s0, s_E[tid * kLd + w]);
                        s1 = xadd(s1, s_T[tid * kLd + w]);
                        s2 = xadd(s2, ed);
                        cur = xadd(cur, ed);
                    }
                }
                w = wend;
                if (p == 0) sp[0] = cur;
                else if (p == 1) sp[1] = cur;
                else if (p == 2) sp[2] = cur;
                else if (p == 3) sp[3] = cur;
                else sp[4] = cur;
            }
        } else {
            // ---- B2: per-window oracle arm k° (smallest index on ties), 8 windows per warp.  EDP > 0
            // (ENV.md §3.3) and empty slots hold +inf, so doubles order like their bit patterns: min
            // of the high words, then of the low words among the ties, then the smallest arm index.
            for (int j = 0; j < kTile / 4; ++j) {
                const int w = (warp - 4) * (kTile / 4) + j;
                if (w >= nw) break;                                              // warp-uniform
                double bv = s_D[lane * kLd + w];
                int bk = lane;
#pragma unroll
                for (int q = 1; q < kMaxArmsSw / 32; ++q) {
                    const double v = s_D[(lane + 32 * q) * kLd + w];
                    if (v < bv) {
                        bv = v;
                        bk = lane + 32 * q;
                    }
                }
                const uint64_t bits = (uint64_t)__double_as_longlong(bv);
                const uint32_t hi = (uint32_t)(bits >> 32), lo = (uint32_t)bits;
                const uint32_t mhi = __reduce_min_sync(kFull, hi);
                const uint32_t mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xFFFFFFFFu);
                const uint32_t kmin = __reduce_min_sync(kFull, (hi == mhi && lo == mlo) ? (uint32_t)bk : 0xFFFFFFFFu);
                if (lane == j) {
                    s_oe[w] = __longlong_as_double((long long)(((uint64_t)mhi << 32) | mlo));
                    s_oE[w] = s_E[kmin * kLd + w];                               // E at k°, as evaluated
                    if (a.best) a.best[(size_t)r * a.n_steps + base + w] = (uint8_t)kmin;
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");                       // warps 4–7: all k° written
            if (tid == 128) {                                                    // ENV.md §5: in window order
                for (int w = 0; w < nw; ++w) {
                    o0 = xadd(o0, s_oe[w]);
                    o1 = xadd(o1, s_oE[w]);
                }
            }
        }
        __syncthreads();
    }
    if (arm) {
        double *S = a.S + ((size_t)r * a.K + tid) * 3;
        S[0] = s0;
        S[1] = s1;
        S[2] = s2;
#pragma unroll
        for (int p = 0; p < 5; ++p) a.SP[((size_t)r * 5 + p) * a.K + tid] = sp[p];
    }
    if (tid == 128) {
        a.O[2 * r] = o0;
        a.O[2 * r + 1] = o1;
    }
    if (tid == 0) {
#pragma unroll
        for (int p = 0; p < 5; ++p) a.NP[r * 5 + p] = np[p];
    }
}

// K5a: Table-6 "Offline" arms — k_off(r, p) for p < 5 (kNoArm if the prototype never
// occurred) and k_off(r) in slot 5; smallest index on ties
__global__ void offline_kernel(const double *S, const double *SP, const uint32_t *NP, uint32_t n_traces, uint32_t K,
                               uint8_t *koff)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_traces * 6u) return;
    const uint32_t r = i / 6u, p = i % 6u;
    if (p < 5 && NP[r * 5 + p] == 0u) {
        koff[i] = (uint8_t)kNoArm;
        return;
    }
    uint32_t kb = 0;
    double bv = 0.0;
    for (uint32_t k = 0; k < K; ++k) {
        const double v = p < 5 ? SP[((size_t)r * 5 + p) * K + k] : S[((size_t)r * K + k) * 3 + 2];
        if (k == 0 || v < bv) {
            bv = v;
            kb = k;
        }
    }
    koff[i] = (uint8_t)kb;
}

// K5b: per-tuner regret against the per-window oracle and the best fixed arm (ENV.md §5)
__global__ void regret_kernel(Ws w, uint32_t N, uint32_t K, const double *S, const double *O, const uint8_t *koff,
                              double *regret)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t r = w.params[i].trace_id;
    const double e = w.acc[i].sum_edp;
    regret[2 * (size_t)i] = xsub(e, O[2 * r]);
    regret[2 * (size_t)i + 1] = xsub(e, S[((size_t)r * K + koff[r * 6 + 5]) * 3 + 2]);
}

}  // namespace

cudaError_t launch_sweep(const Ws &w, const agft_config &c, const void *records, uint32_t t0, uint32_t n_steps,
                         double *S, double *SP, uint32_t *NP, double *O, uint8_t *best, cudaStream_t s)
{
    if (n_steps == 0) return cudaSuccess;
    SweepArgs a;
    a.records = static_cast<const StepRec *>(records);
    a.S = S;
    a.SP = SP;
    a.NP = NP;
    a.O = O;
    a.best = best;
    a.env = w.env;
    a.tc = c.trace;
    a.seed = c.env_seed;
    a.trace_base = c.trace_base;
    a.n_traces = c.n_traces;
    a.t0 = t0;
    a.n_steps = n_steps;
    a.K = c.grid.n_arms;
    a.W = c.env.window_s;
    a.p_idle = c.env.p_idle;
    a.u_floor = c.env.u_floor;
    a.u_max = c.env.u_max;
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    if (e != cudaSuccess) return e;
    sweep_kernel<<<c.n_traces, kThreads2, kSweepSmem, s>>>(a); note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_regret(const Ws &w, const agft_config &c, const double *S, const double *SP, const uint32_t *NP,
                          const double *O, uint8_t *koff, double *regret, cudaStream_t s)
{
    const uint32_t nk = c.n_traces * 6u;
    offline_kernel<<<(nk + 127) / 128, 128, 0, s>>>(S, SP, NP, c.n_traces, c.grid.n_arms, koff); note_launches(1);
    if (regret) {
        regret_kernel<<<(c.n_tuners + 255) / 256, 256, 0, s>>>(w, c.n_tuners, c.grid.n_arms, S, O, koff, regret);
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace agft
