// rec_tile.cuh — a1: the step records of a warp's trace streamed into shared memory
// by 1-D bulk copies (cp.async.bulk, the TMA engine's non-tensor form) in double-buffered tiles of
// kRecTile windows, completion signalled on an mbarrier per buffer.
//
// Used by a warp whose tuners all replay the same trace (the class lists keep a trace's tuners
// adjacent, so this is the common case); a warp that spans two traces reads its records with __ldg
// as before.  Compile-time opt-in (AGFT_TMA=1): measured against the L1-prefetch path, DESIGN.md §4.
#pragma once
#include "step_common.cuh"

#ifndef AGFT_TMA
#define AGFT_TMA 0
#endif

namespace agft {

constexpr int kRecTile = 8;                     // windows per tile (1 KB)

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// arm the barrier for `bytes` of transactions and issue the bulk copy global → shared
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of dst first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Per-warp record stream: buf [2][kRecTile] StepRec and bar [2] in shared memory.
struct RecTile {
    StepRec *buf;
    uint64_t *bar;
    const StepRec *src;      // the trace's records for this launch (window s at src + s)
    uint32_t n;              // windows in this launch
    bool on;                 // warp-uniform: every lane replays the same trace

    // lane 0 of the warp: barriers + the first tile (call warp-wide, then __syncwarp)
    __device__ __forceinline__ void start(int lane)
    {
        if (!on) return;
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            mbar_fence_init();
            if (n > 0) bulk_load(buf, src, min((uint32_t)kRecTile, n) * (uint32_t)sizeof(StepRec), bar);
        }
        __syncwarp();
    }
    // record of window s (warp-uniform s): at a tile boundary, wait for the tile and issue the next
    __device__ __forceinline__ const StepRec *at(uint32_t s, int lane)
    {
        const uint32_t ti = s / kRecTile, slot = s % kRecTile, b = ti & 1u;
        if (slot == 0) {
            mbar_wait(bar + b, (ti >> 1) & 1u);
            __syncwarp();                                  // all lanes are done with the other buffer
            const uint32_t next = (ti + 1) * kRecTile;
            if (lane == 0 && next < n)
                bulk_load(buf + (b ^ 1u) * kRecTile, src + next, min((uint32_t)kRecTile, n - next) * (uint32_t)sizeof(StepRec),
                          bar + (b ^ 1u));
        }
        return buf + b * kRecTile + slot;
    }
};

}  // namespace agft
