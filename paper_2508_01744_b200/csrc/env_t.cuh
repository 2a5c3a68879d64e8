// env_t.cuh — device pieces of ENV.md §1–§3 shared by the trace kernel (K1) and the
// offline sweep (K4): Philox4x32-10, the segment prototype, the §3.3 response.
// (CUDA path only; the oracle has its own, independent implementation.)
#pragma once
#include "agft_internal.cuh"

namespace agft {

struct Philox {
    uint32_t k0, k1;
    __device__ __forceinline__ uint4 operator()(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) const
    {
        uint32_t a = k0, b = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
            const uint32_t n0 = hi1 ^ c1 ^ a, n2 = hi0 ^ c3 ^ b;
            c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
            a += 0x9E3779B9u;
            b += 0xBB67AE85u;
        }
        return make_uint4(c0, c1, c2, c3);
    }
};

__device__ __forceinline__ double unit32(uint32_t v) { return xmul((double)v, 0x1p-32); }
__device__ __forceinline__ double unit53(uint32_t a, uint32_t b)
{
    const uint64_t m = ((uint64_t)a << 21) ^ ((uint64_t)b >> 11);
    return xmul((double)m, 0x1p-53);
}

// ENV.md §3.3 response at one frequency (given its §3.1 constants), from the record's fields
// (I and P already converted to double: exact, they are < 2^32).
__device__ __forceinline__ void response_f(double I, double P, double g, double invIm, double nT, double nE,
                                           double dec, double pre, double pw, double W, double invW,
                                           double q_over, double u_max, double u_floor, double p_idle, double &E,
                                           double &tpot)
{
    const double t_dec = xmul(I, dec);
    const double t_pre = xmul(P, pre);
    const double busy = xmul(xadd(t_dec, t_pre), g);
    const double u = xmul(busy, invW);
    const double q = u <= u_max ? xrcp_nb(xsub(1.0, u)) : xmul(u, q_over);
    tpot = xmul(xmul(xmul(xadd(dec, xmul(t_pre, invIm)), g), q), nT);
    double ue = u > 1.0 ? 1.0 : u;                  // (fmin/fmax compile to ~7 instructions each: NaN rules)
    ue = ue < u_floor ? u_floor : ue;
    E = xmul(xmul(xadd(p_idle, xmul(pw, ue)), W), nE);
}

__device__ __forceinline__ void response(const StepRec &r, double dec, double pre, double pw,
                                         double W, double invW, double q_over, double u_max,
                                         double u_floor, double p_idle, double &E, double &tpot)
{
    response_f((double)r.I, (double)r.P, r.g, r.invIm, r.nT, r.nE, dec, pre, pw, W, invW, q_over, u_max, u_floor,
               p_idle, E, tpot);
}

// §4.1 context x1..x7 from one window's MetricsSnapshot counters (ENV.md §3.2), then
// the per-dimension normalisation clamp((raw − lo)/(hi − lo), 0, 1), 0 when hi = lo (AMB-14/15).
__device__ __forceinline__ void context_of(uint32_t waiting, uint32_t running, uint32_t prefill, uint32_t decode,
                                           uint32_t iters, uint32_t kv_used, uint32_t hits, uint32_t misses,
                                           double W, uint32_t kv_total, const double *norm_lo,
                                           const double *norm_hi, double (&x)[7])
{
    double raw[7];
    raw[0] = waiting > 0 ? 1.0 : 0.0;
    raw[1] = xdiv((double)prefill, W);
    raw[2] = xdiv((double)decode, W);
    raw[3] = xdiv((double)((uint64_t)prefill + (uint64_t)decode), (double)(iters > 0 ? iters : 1u));
    raw[4] = (double)running;
    raw[5] = xdiv((double)kv_used, (double)kv_total);
    raw[6] = (hits + misses) > 0 ? xdiv((double)hits, (double)(hits + misses)) : 0.0;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
        const double lo = norm_lo[i], hi = norm_hi[i];
        double xv = 0.0;
        if (hi > lo) {
            xv = xdiv(xsub(raw[i], lo), xsub(hi, lo));
            xv = xv < 0.0 ? 0.0 : (xv > 1.0 ? 1.0 : xv);
        }
        x[i] = xv;
    }
}

// ENV.md §2.2: the Table-1 prototype of the 10-minute segment holding window t
__device__ __forceinline__ uint32_t prototype_of(const agft_trace_cfg &c, const Philox &ph, uint32_t t)
{
    const uint32_t v = ph(t / c.seg_steps, 1u, 0u, 0u).x >> 24;
    uint32_t p = 0, cum = 0;
    for (; p < 5; ++p) {
        cum += c.weight[p];
        if (v < cum) break;
    }
    return p >= 5 ? 4u : p;
}

}  // namespace agft
