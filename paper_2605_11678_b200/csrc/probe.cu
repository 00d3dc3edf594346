// probe.cu -- diagnostic: per-SM bulk-copy (TMA engine) streaming bandwidth as a
// function of CTAs, stage size and ring depth.  A producer thread streams
// `per_cta` bytes through an mbarrier ring of `stages` x `stage_bytes`; the
// consumer warp only waits and releases each stage (no compute).
#include "common.cuh"
#include "kernels.h"

namespace lsb {

__global__ void __launch_bounds__(64, 1) bulk_stream_kernel(const uint8_t* src, uint64_t per_cta,
                                                            int stage_bytes, int stages,
                                                            uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // per_cta's top bit set: every CTA streams the SAME bytes (L2-resident, hot lines)
  const bool shared = (per_cta >> 63) != 0;
  per_cta &= ~(1ull << 63);
  const uint8_t* base = shared ? src : src + blockIdx.x * per_cta;
  const int n = static_cast<int>(per_cta / stage_bytes);
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t round = 0;
      for (int i = 0; i < n; ++i) {
        if (round) mbar_wait(&empty[s], (round - 1) & 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        bulk_g2s(smem + s * stage_bytes, base + static_cast<uint64_t>(i) * stage_bytes, stage_bytes, &full[s]);
        if (++s == stages) {
          s = 0;
          ++round;
        }
      }
    }
  } else {
    int s = 0;
    uint32_t round = 0;
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) {
      mbar_wait(&full[s], round & 1);
      acc += reinterpret_cast<const uint32_t*>(smem + s * stage_bytes)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == stages) {
        s = 0;
        ++round;
      }
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

cudaError_t launch_bulk_stream(const void* src, uint64_t per_cta, int stage_bytes, int stages, int grid,
                               uint32_t* sink, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(stages) * stage_bytes + 2 * stages * 8;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(bulk_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024);
  if (e != cudaSuccess) return e;
  return launch_k(bulk_stream_kernel, dim3(grid), dim3(64), smem, st,
                  static_cast<const uint8_t*>(src), per_cta, stage_bytes, stages, sink);
}

}  // namespace lsb
