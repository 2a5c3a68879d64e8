// schedule.cu — per-sub-chunk tuner classification and stable partition into class lists.
//
// Pruning only ever removes arms (AMB-12), so a tuner's class can only move toward
// SOLO.  Between sub-chunks the host library classifies every tuner by its active-arm
// count and builds order-preserving per-class lists (so tuners sharing a trace stay
// adjacent and read their step records as warp-wide broadcasts):
//   K_act > 64 → WIDE (warp per tuner, arms in smem)
//   2..64 → SEG8 / SEG16 / SEG32 / SEG64 (SEG2 with G = 4 / 8 / 16 / 32 lanes per tuner, two arms per lane)
//   1 → SOLO (lane per tuner)
#include "agft_internal.cuh"

namespace agft {

// WIDE (>64) / SEG64 / SEG32 / SEG16 / SEG8 / SOLO
__device__ __forceinline__ int class_of(const Ws &w, uint32_t tb)
{
    if (w.acc[tb].flags & 1u) return -1;                    // frozen: not scheduled
    const uint4 m = *reinterpret_cast<const uint4 *>(w.active + (size_t)tb * 4);
    const int k = __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
    if (k <= 1) return kClsSolo;
    if (k <= 8) return kClsSeg8;
    if (k <= 16) return kClsSeg16;
    if (k <= 32) return kClsSeg32;
    if (k <= 64) return kClsSeg64;
    return kClsWide;
}

// per-block counts of each class
__global__ void __launch_bounds__(kPartBlock) class_count_kernel(Ws w, uint32_t N)
{
    __shared__ uint32_t cnt[kNumCls];
    if (threadIdx.x < kNumCls) cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t tb = blockIdx.x * kPartBlock + threadIdx.x;
    const int c = tb < N ? class_of(w, tb) : -1;
#pragma unroll
    for (int k = 0; k < kNumCls; ++k) {
        const uint32_t b = __ballot_sync(kFull, c == k);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&cnt[k], __popc(b));
    }
    __syncthreads();
    if (threadIdx.x < kNumCls) w.blkcnt[threadIdx.x * gridDim.x + blockIdx.x] = cnt[threadIdx.x];
}

// exclusive scan of the block counts, per class (one block)
__global__ void class_scan_kernel(Ws w, uint32_t nblk)
{
    const int c = threadIdx.x;
    if (c >= kNumCls) return;
    uint32_t run = 0;
    for (uint32_t b = 0; b < nblk; ++b) {
        const uint32_t v = w.blkcnt[c * nblk + b];
        w.blkcnt[c * nblk + b] = run;
        run += v;
    }
    w.counts[c] = run;
}

// stable scatter into the class lists
__global__ void __launch_bounds__(kPartBlock) class_scatter_kernel(Ws w, uint32_t N)
{
    __shared__ uint32_t wcnt[kNumCls][kPartBlock / 32];
    const uint32_t tb = blockIdx.x * kPartBlock + threadIdx.x;
    const int c = tb < N ? class_of(w, tb) : -1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t myrank = 0;
#pragma unroll
    for (int k = 0; k < kNumCls; ++k) {
        const uint32_t b = __ballot_sync(kFull, c == k);
        if (lane == 0) wcnt[k][warp] = __popc(b);
        if (c == k) myrank = __popc(b & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (c >= 0) {
        uint32_t off = w.blkcnt[c * gridDim.x + blockIdx.x];
        for (int i = 0; i < warp; ++i) off += wcnt[c][i];
        w.lists[(size_t)c * N + off + myrank] = tb;
    }
}

cudaError_t launch_classify(const Ws &w, uint32_t N, cudaStream_t s)
{
    const uint32_t nblk = (N + kPartBlock - 1) / kPartBlock;
    class_count_kernel<<<nblk, kPartBlock, 0, s>>>(w, N); note_launches(1);
    class_scan_kernel<<<1, 32, 0, s>>>(w, nblk); note_launches(1);
    class_scatter_kernel<<<nblk, kPartBlock, 0, s>>>(w, N); note_launches(1);
    return cudaGetLastError();
}

}  // namespace agft
