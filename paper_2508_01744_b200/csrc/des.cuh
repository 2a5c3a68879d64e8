// des.cuh — ENV.md §7 ENV-S on the device: one tuner's discrete-event continuous-batching server
// (SPEC inference_sim), driven by the warp that owns the tuner in the WIDE
// replay kernel (MODE 4).  The 128 running slots live in registers, four per lane (slot k = 32·j +
// lane, so ascending k is j-major, then lane — the oracle's slot order); the FIFO queue of ≤ 512
// requests and the scalars live in the workspace.  Every control decision is warp-uniform (the
// queue head and the counters are the same in every lane); the order-dependent sums (first-token
// latencies) are added in ascending slot order, one shuffle per contributing slot.
#pragma once
#include "env_t.cuh"

namespace agft {

constexpr int kDesS = 4;                                 // running slots per lane
constexpr double kDesOver = 0.004;                       // s per iteration (SPEC batch_overhead)

struct DesOut {
    double E, tpot, ttft, edp;
};

struct DesWarp {
    double arr[kDesS];
    uint32_t ctx[kDesS], gen[kDesS], done[kDesS], flags[kDesS];
    uint32_t store;                                       // word `lane` of the template set (lanes < 16)
    double clock;
    uint32_t qhead, qlen, nrun, kv, dropped;
    uint32_t snap[8];

    __device__ __forceinline__ void load(const DesScal *sc, const DesSlot *sl, int lane)
    {
        clock = sc->clock;
        qhead = sc->qhead;
        qlen = sc->qlen;
        nrun = sc->nrun;
        kv = sc->kv;
        dropped = sc->dropped;
        store = lane < 16 ? sc->store[lane] : 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) snap[i] = sc->snap[i];
#pragma unroll
        for (int j = 0; j < kDesS; ++j) {
            const DesSlot s = sl[32 * j + lane];
            arr[j] = s.arr;
            ctx[j] = s.ctx;
            gen[j] = s.gen;
            done[j] = s.done;
            flags[j] = s.flags;
        }
    }
    __device__ __forceinline__ void save(DesScal *sc, DesSlot *sl, int lane) const
    {
        if (lane == 0) {
            sc->clock = clock;
            sc->qhead = qhead;
            sc->qlen = qlen;
            sc->nrun = nrun;
            sc->kv = kv;
            sc->dropped = dropped;
#pragma unroll
            for (int i = 0; i < 8; ++i) sc->snap[i] = snap[i];
        }
        if (lane < 16) sc->store[lane] = store;
#pragma unroll
        for (int j = 0; j < kDesS; ++j) {
            DesSlot s;
            s.arr = arr[j];
            s.ctx = ctx[j];
            s.gen = gen[j];
            s.done = done[j];
            s.flags = flags[j];
            sl[32 * j + lane] = s;
        }
    }

    // window t (ENV.md §7): the row's arrivals into the queue, then iterations until (t+1)·W at the
    // chosen frequency's §3.1 constants; returns the window's (E, TPOT, TTFT, EDP), updates snap
    __device__ __forceinline__ DesOut window(uint32_t t, const uint32_t *row, const agft_trace_cfg &tc, const Philox &ph,
                             DesReq *q, double dec, double pre, double pw, const ReplayArgs &a, int lane)
    {
        // ---- arrivals: a = hits + misses of the row, evenly spaced; lanes draw 32 at a time
        const uint32_t na = __ldg(row + 6) + __ldg(row + 7);
        const uint32_t p = prototype_of(tc, ph, t);
        const uint32_t pool = p == 4 ? 5u : 500u;
        const double tW = xmul((double)t, a.W);
        for (uint32_t base = 0; base < na; base += 32) {
            const uint32_t i = base + (uint32_t)lane;
            const bool real = i < na;
            const uint4 u = ph(t, 5u, i, 0u);
            const uint32_t c = tc.ctx_lo[p] + (uint32_t)(((uint64_t)u.x * (tc.ctx_hi[p] - tc.ctx_lo[p] + 1u)) >> 32);
            const uint32_t g = tc.gen_lo[p] + (uint32_t)(((uint64_t)u.y * (tc.gen_hi[p] - tc.gen_lo[p] + 1u)) >> 32);
            const uint32_t tm = (uint32_t)(((uint64_t)u.z * pool) >> 32);
            const double ar = xadd(tW, xmul(xdiv(xadd((double)i, 0.5), (double)na), a.W));
            const bool fits = real && (uint64_t)c + g <= a.kv_total;
            const uint32_t fm = __ballot_sync(kFull, fits);
            const uint32_t pos = qlen + (uint32_t)__popc(fm & ((1u << lane) - 1u));
            const bool keep = fits && pos < (uint32_t)kDesQ;
            if (keep) {
                DesReq r;
                r.arr = ar;
                r.ctx = c;
                r.gen = g;
                r.tmpl = tm;
                r.pad = 0u;
                q[(qhead + pos) % kDesQ] = r;
            }
            const uint32_t nk = (uint32_t)__popc(__ballot_sync(kFull, keep));
            dropped += (uint32_t)__popc(__ballot_sync(kFull, real)) - nk;
            qlen += nk;
        }
        __syncwarp();                                         // the queue writes before the head reads

        // ---- the engine (ENV.md §7), warp-uniform control; the queue head is kept in registers
        const double t_end = xmul((double)(t + 1u), a.W);
        DesReq h;
        if (qlen > 0u) h = q[qhead];
        uint32_t P = 0, Dc = 0, I = 0, hits = 0, misses = 0, n_tok = 0, n_first = 0;
        double busy = 0.0, sdec = 0.0, sfirst = 0.0;
        uint32_t g_n = 0xFFFFFFFFu;                          // running count the penalty g was computed for
        double g = 1.0;
        while (clock < t_end) {
            uint32_t npre = 0, fresh[kDesS];
#pragma unroll
            for (int j = 0; j < kDesS; ++j) fresh[j] = 0u;
            while (qlen > 0u) {                               // admission: FIFO, head of line
                if (!(h.arr <= clock) || nrun >= (uint32_t)kDesR || (uint64_t)kv + h.ctx + h.gen > a.kv_total) break;
                const uint32_t wd = h.tmpl >> 5, bit = 1u << (h.tmpl & 31u);
                const uint32_t hit = (__shfl_sync(kFull, store, (int)wd) & bit) ? 1u : 0u;
                if (lane == (int)wd) store |= bit;
                hits += hit;
                misses += 1u - hit;
                npre += h.ctx - (hit ? h.ctx / 2u : 0u);
                kv += h.ctx + h.gen;
                {                                             // the lowest free slot (j-major, then lane)
                    static_assert(kDesS == 4, "four slots per lane");
                    const uint32_t fm0 = __ballot_sync(kFull, !(flags[0] & 1u)), fm1 = __ballot_sync(kFull, !(flags[1] & 1u)),
                                   fm2 = __ballot_sync(kFull, !(flags[2] & 1u)), fm3 = __ballot_sync(kFull, !(flags[3] & 1u));
                    const int js = fm0 ? 0 : fm1 ? 1 : fm2 ? 2 : 3;
                    const uint32_t fm = fm0 ? fm0 : fm1 ? fm1 : fm2 ? fm2 : fm3;
                    const int owner = __ffs(fm) - 1;
#pragma unroll
                    for (int j = 0; j < kDesS; ++j) {          // (no early exit: the slots stay in registers)
                        if (j == js && lane == owner) {
                            arr[j] = h.arr;
                            ctx[j] = h.ctx;
                            gen[j] = h.gen;
                            done[j] = 0u;
                            flags[j] = 1u;
                        }
                        if (j == js) fresh[j] |= 1u << owner;
                    }
                }
                nrun += 1u;
                qhead = (qhead + 1u) % (uint32_t)kDesQ;
                qlen -= 1u;
                if (qlen > 0u) h = q[qhead];
            }
            uint32_t ndec = 0;
#pragma unroll
            for (int j = 0; j < kDesS; ++j) ndec += (uint32_t)__popc(__ballot_sync(kFull, (flags[j] & 3u) == 3u));
            if (npre == 0u && ndec == 0u) {                   // idle until the next arrival
                double nxt = t_end;
                if (qlen > 0u && h.arr < t_end) nxt = h.arr;
                clock = nxt;
                continue;
            }
            if (nrun != g_n) {                                // the penalty changes only with nrun
                const double rho = xdiv((double)nrun, (double)a.cap);
                g = rho > 1.0 ? xmul(rho, xsqrt(rho)) : 1.0;
                g_n = nrun;
            }
            const double tp = xmul((double)npre, pre), td = ndec > 0u ? dec : 0.0;
            const double dt = xadd(kDesOver, xmul(tp > td ? tp : td, g));
            clock = xadd(clock, dt);
            uint32_t kv_free = 0;
#pragma unroll
            for (int j = 0; j < kDesS; ++j) {                 // one token per prefilled request, slot order
                const bool act = (flags[j] & 3u) == 3u;
                if (act) done[j] += 1u;
                uint32_t fm = __ballot_sync(kFull, act && done[j] == 1u);
                while (fm) {
                    const int src = __ffs(fm) - 1;
                    fm &= fm - 1u;
                    sfirst = xadd(sfirst, xsub(clock, __shfl_sync(kFull, arr[j], src)));
                    n_first += 1u;
                }
                const bool ret = act && done[j] == gen[j];
                kv_free += __reduce_add_sync(kFull, ret ? ctx[j] + gen[j] : 0u);
                nrun -= (uint32_t)__popc(__ballot_sync(kFull, ret));
                if (ret) flags[j] = 0u;
            }
            kv -= kv_free;
#pragma unroll
            for (int j = 0; j < kDesS; ++j)
                if ((fresh[j] >> lane) & 1u) flags[j] |= 2u;
            P += npre;
            Dc += ndec;
            I += 1u;
            n_tok += ndec;
            busy = xadd(busy, dt);
            sdec = xadd(sdec, xmul(dt, (double)ndec));
        }
        DesOut o;
        const double u = xdiv(busy, a.W);
        double ue = busy > 0.0 ? (u > 1.0 ? 1.0 : u) : 0.0;
        if (busy > 0.0 && ue < a.u_floor) ue = a.u_floor;
        o.E = xmul(xadd(a.p_idle, xmul(pw, ue)), a.W);
        o.tpot = n_tok > 0u ? xdiv(sdec, (double)n_tok) : dec;
        o.ttft = n_first > 0u ? xdiv(sfirst, (double)n_first) : 0.0;
        o.edp = xmul(o.E, o.tpot);
        snap[0] = qlen;
        snap[1] = nrun;
        snap[2] = P;
        snap[3] = Dc;
        snap[4] = I;
        snap[5] = kv;
        snap[6] = hits;
        snap[7] = misses;
        return o;
    }
};

}  // namespace agft
