// seg_common.cuh — warp-segment helpers of the SEG kernels (G lanes per tuner, 32/G tuners per
// warp): segment ballots and sums, the segment-distributed sorted EDP window (E = 64/G entries per
// lane), and the canonical 128-slot reduction tree of ENV.md §4.8 over a per-segment buffer.
#pragma once
#include "step_common.cuh"

namespace agft {

template <int G>
__device__ __forceinline__ uint32_t sbits(bool p, int sg)
{
    const uint32_t b = __ballot_sync(kFull, p);
    return G == 32 ? b : (b >> (sg * G)) & ((1u << G) - 1u);
}
template <int G>
__device__ __forceinline__ int spopc(bool p, int sg) { return __popc(sbits<G>(p, sg)); }
template <int G>
__device__ __forceinline__ int sisum(int v)
{
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
    return v;
}

// sorted window element idx (S[l*E + e] in lane l of the segment)
// (a binary mux tree on the bits of idx % E: a select chain here was compiled into a dynamically
// indexed local-memory copy of the window — STL ×E/2 + LDL on the reward's serial chain)
template <int G, int E>
__device__ __forceinline__ double wat(const double (&S)[E], uint32_t idx)
{
    const uint32_t j = idx % E;
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = S[e];
#pragma unroll
    for (int b = 1; b < E; b <<= 1) {
        const bool up = (j & (uint32_t)b) != 0u;
#pragma unroll
        for (int e = 0; e + b < E; e += 2 * b) v[e] = up ? v[e + b] : v[e];
    }
    return __shfl_sync(kFull, v[0], idx / E, G);
}
template <int G, int E>
__device__ __forceinline__ int wless(const double (&S)[E], double v)
{
    int c = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) c += (S[e] < v) ? 1 : 0;
    return sisum<G>(c);
}
template <int G, int E>
__device__ __forceinline__ void wremove(double (&S)[E], int po, int l)
{
    double nxt = __shfl_down_sync(kFull, S[0], 1, G);
    if (l == G - 1) nxt = kInf;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double up = (e + 1 < E) ? S[e + 1 < E ? e + 1 : e] : nxt;
        S[e] = (l * E + e < po) ? S[e] : up;
    }
}
template <int G, int E>
__device__ __forceinline__ void winsert(double (&S)[E], double v, int pi, int l)
{
    const double prv = __shfl_up_sync(kFull, S[E - 1], 1, G);
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
        const int i = l * E + e;
        const double dn = (e > 0) ? S[e > 0 ? e - 1 : 0] : prv;
        S[e] = (i < pi) ? S[e] : ((i == pi) ? v : dn);
    }
}

// per-segment tree buffer: slot k at k + k/SL (one pad per 128/G-slot block, odd stride) so
// that the lanes' block reads fall in different banks
template <int G>
__host__ __device__ constexpr int tree_stride() { return 128 + G + 1; }
template <int G>
__device__ __forceinline__ int tslot(int k) { return k + k / (128 / G); }

// canonical tree: scatter (has0,key0,v0), (has1,key1,v1) of every lane to `buf`, reduce aligned
// blocks pairwise, butterfly.  Slots outside the scattered set must hold +0.0: the caller scatters
// the same set Q (active arms with n ≥ hist_n) in both trees of a step, Q only grows between steps
// except by pruning, and a pruned arm's slot is zeroed when it is removed (no restore pass here)
template <int G>
__device__ __forceinline__ double stree(double *buf, int l, bool h0, int k0, double v0, bool h1, int k1, double v1)
{
    constexpr int SL = 128 / G;
    if (h0) buf[tslot<G>(k0)] = v0;
    if (h1) buf[tslot<G>(k1)] = v1;
    __syncwarp();
    double v[SL];
#pragma unroll
    for (int j = 0; j < SL; ++j) v[j] = buf[l * (SL + 1) + j];
#pragma unroll
    for (int len = SL; len > 1; len >>= 1)
#pragma unroll
        for (int j = 0; j < len / 2; ++j) v[j] = xadd(v[2 * j], v[2 * j + 1]);
    double s = v[0];
#pragma unroll
    for (int off = 1; off < G; off <<= 1) s = xadd(s, __shfl_xor_sync(kFull, s, off, G));
    __syncwarp();                                     // reads done before the next scatter / zeroing
    return s;
}

// Historical-pruning screen (ENV.md §4.8).  Historical pruning removes arm k ∈ Q iff
// ē_k > thr = best + k_h·σ, with μ and σ from the canonical 128-slot trees.  From min, max, Σē and
// Σē² over Q (one butterfly, any order) this returns true only when max ē_Q < thr_lo ≤ thr, so that
// the exact evaluation would remove nothing and may be skipped:
//   V = Σē²/n − μ² is within 27u·m2 of the true population variance V* (u = 2⁻⁵³, m2 = Σē²/n; sums
//   of ≤ 64 positive terms, one product, one subtraction), taken as dV = 64u·m2; the exact path's σ
//   is ≥ √V*·(1 − 8u) (its μ error only adds n·ε² to Σ(ē − μ)², and the tree / division / square
//   root round by ≤ 8u), so thr_lo = (best + k_h·√(V − dV)(1 − 8u))(1 − 16u) ≤ thr.
// All equal means (max = min = best) remove nothing either: thr ≥ best.  Called warp-wide.
// The screen's state carried between steps (per segment, replicated in its G lanes).  A full screen that
// finds Q safe also leaves a lower bound of the exact threshold that stays valid while Q's membership is
// unchanged and its means move: with D ≥ Σ|Δē| over the changes since (ℓ1 ≥ ℓ2), the true minimum
// drops by at most D and the true σ by at most D/√n (σ = ‖Pē‖/√n, P the centring projection), so
//   thr ≥ (1 − 16u)·(mn + k_h(1 − 8u)√V* − D·(1 + k_h/√n)),   √V* ≥ √(V − dV)  (k_h ≥ 0, ē > 0),
// and max ē ≤ max(mx, M), M the largest changed mean.  P = mn + k_h·sd_lo and B ≥ 1 + k_h/√n carry the
// full screen's part; the check rounds every term the safe way (screen_inc_safe).
struct ScreenCache {
    double P, B, mx, D, M;
    bool ok;
};

// full screen over the segment (warp-wide call: butterflies); fills c when the result is "safe"
template <int G>
__device__ __forceinline__ bool hist_screen_full(bool q0, double e0, bool q1, double e1, int nq, double kh,
                                                 ScreenCache &c)
{
    double mn = fmin(q0 ? e0 : kInf, q1 ? e1 : kInf);
    double mx = fmax(q0 ? e0 : -kInf, q1 ? e1 : -kInf);
    double s1 = (q0 ? e0 : 0.0) + (q1 ? e1 : 0.0);
    double s2 = (q0 ? e0 * e0 : 0.0) + (q1 ? e1 * e1 : 0.0);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(kFull, mn, off, G));
        mx = fmax(mx, __shfl_xor_sync(kFull, mx, off, G));
        s1 += __shfl_xor_sync(kFull, s1, off, G);
        s2 += __shfl_xor_sync(kFull, s2, off, G);
    }
    constexpr double u = 0x1p-53;
    c.ok = false;
    c.mx = mx;
    c.D = 0.0;
    c.M = -kInf;
    c.B = (1.0 + kh * rsqrt((double)(nq > 0 ? nq : 1))) * (1.0 + 8.0 * u);
    if (!(mx > mn)) {                                  // all equal: thr ≥ best, nothing is removed
        c.P = mn;
        c.ok = kh >= 0.0;
        return true;
    }
    const double inq = xrcp_nb((double)(nq > 0 ? nq : 1));
    const double m2 = s2 * inq, mu = s1 * inq;
    const double V = m2 - mu * mu;
    const double dV = 64.0 * u * m2;
    if (!(V - dV > 0.0)) return false;
    const double sd_lo = xsqrt_nb(V - dV) * (1.0 - 8.0 * u);
    c.P = mn + kh * sd_lo;
    const double thr_lo = c.P * (1.0 - 16.0 * u);
    const bool safe = mx < thr_lo;
    c.ok = safe && kh >= 0.0;
    return safe;
}

// the cached bound after the changes noted since the full screen:
//   R = ((P(1 − 8u) − D·B)(1 − 20u)) ≤ (1 − 16u)(P(1 − 6u) − D·B_true) ≤ thr   (P(1 − 6u) ≤ the exact
// mn + k_h(1 − 8u)√V*; every rounding safe-side; a negative R fails the test since every mean is > 0;
// host replay against the oracle's canonical trees: tests/test_screen_bound.py)
__device__ __forceinline__ bool screen_inc_safe(const ScreenCache &c)
{
    constexpr double u = 0x1p-53;
    const double R = (c.P * (1.0 - 8.0 * u) - c.D * c.B) * (1.0 - 20.0 * u);
    return c.ok && fmax(c.mx, c.M) < R;
}

// one mean of Q moved by dlt (to enew); dlt = +inf marks a change of Q's membership (the bound is void)
__device__ __forceinline__ void screen_note(ScreenCache &c, double dlt, double enew)
{
    constexpr double u = 0x1p-53;
    c.D = (c.D + dlt) * (1.0 + 8.0 * u);               // ≥ the true Σ|Δ| (each rounding covered)
    c.M = fmax(c.M, enew);
}

// Historical-pruning screen (ENV.md §4.8).  Historical pruning removes arm k ∈ Q iff
// ē_k > thr = best + k_h·σ, with μ and σ from the canonical 128-slot trees.  From min, max, Σē and
// Σē² over Q (one butterfly, any order) this returns true only when max ē_Q < thr_lo ≤ thr, so that
// the exact evaluation would remove nothing and may be skipped:
//   V = Σē²/n − μ² is within 27u·m2 of the true population variance V* (u = 2⁻⁵³, m2 = Σē²/n; sums
//   of ≤ 64 positive terms, one product, one subtraction), taken as dV = 64u·m2; the exact path's σ
//   is ≥ √V*·(1 − 8u) (its μ error only adds n·ε² to Σ(ē − μ)², and the tree / division / square
//   root round by ≤ 8u), so thr_lo = (best + k_h·√(V − dV)(1 − 8u))(1 − 16u) ≤ thr.
// All equal means (max = min = best) remove nothing either: thr ≥ best.  Called warp-wide.
template <int G>
__device__ __forceinline__ bool hist_screen_safe(bool q0, double e0, bool q1, double e1, int nq, double kh)
{
    ScreenCache c;
    return hist_screen_full<G>(q0, e0, q1, e1, nq, kh, c);
}

}  // namespace agft
