// gemv_ect.cu -- decode-time (batch 1) GEMV straight from ECT pages (compact
// residency / streaming form, ect.py): 12 KiB pages are decoded in registers
// and fed to mma.sync, never expanded in memory.
//
// Roofline: HBM.  Moved bytes per launch = n_pages * (12288 + 16) (pages +
// escape masks) + K*4 + N*4; the plain-equivalent figure divides N*K*2 by
// the same time.  The kernel is bound by the consumers' integer issue rate
// (~2.4 ALU/FMA ops per decoded word), so everything around the decode is
// cut to a few instructions per page:
//   * chunks of up to 4 pages (never straddling an m-tile) are one ring slot:
//     one bulk copy of the pages (contiguous in the blob) + one of their
//     escape masks, one mbarrier wait and one arrive per warp per chunk;
//   * the per-page escape mask (16 B: one bit per 64 words = 4 lanes of a warp)
//     says where code-15 words are, so the per-code escape test and the patch
//     run only for those lanes (~1 % of lane groups for BF16 weights);
//   * pages never depend on the previous kernel: the producer fills the ring
//     and (K <= 4096) the consumers decode the first chunk before
//     griddepcontrol.wait / x staging;
//   * same stream-K split, fix-up (one all-consumer barrier per m-tile, the
//     rest on warps 0-3) and fused epilogues as gemv.cu (shared
//     gemv_common.cuh), so plain and ECT launches give bit-identical results.
// LS_GEMV_CHUNK / LS_GEMV_SLOTS are tuning knobs (4 x 4 measured best,
// DESIGN.md §8c).
#include "common.cuh"
#include "gemv_common.cuh"
#include "kernels.h"

namespace lsb {

namespace {
constexpr int kWarps = 16;                 // 8 row blocks x 2 k-parts of every page
constexpr int kConsumers = kWarps * 32;
constexpr int kThreads = kConsumers + 32;  // + producer warp
#ifndef LS_GEMV_CHUNK
#define LS_GEMV_CHUNK 4
#endif
#ifndef LS_GEMV_SLOTS
#define LS_GEMV_SLOTS 4
#endif
constexpr int kChunk = LS_GEMV_CHUNK;      // pages per ring slot
constexpr int kMaskBytes = 16;             // escape mask per page (1 bit per 64 words)
constexpr int kSlotBytes = kChunk * (kEctPageBytes + kMaskBytes);
constexpr int kMaxSlots = LS_GEMV_SLOTS;
constexpr int kSmemBudget = 227 * 1024;

__host__ __device__ inline int ect_slots(int n_kb, int max_slots) {
  const int avail = (kSmemBudget - n_kb * kTileCols * 4 - 4 * kTileRows * 4 - 64 - 2 * kMaxSlots * 8 - 16) /
                    kSlotBytes;
  const int cap = max_slots > 0 && max_slots < kMaxSlots ? max_slots : kMaxSlots;
  return avail > cap ? cap : avail;
}

size_t ect_smem(int n_kb, int max_slots) {
  return static_cast<size_t>(ect_slots(n_kb, max_slots)) * kSlotBytes +
         static_cast<size_t>(n_kb) * kTileCols * 4 + 4 * kTileRows * 4 + 64 + 2 * kMaxSlots * 8 + 16;
}
}  // namespace

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1) gemv_ect_kernel(const GemvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = a.n_kb * kTileCols;
  const int NQ = ect_slots(a.n_kb, a.max_slots);
  uint8_t* slots = smem;
  uint32_t* xq = reinterpret_cast<uint32_t*>(smem + NQ * kSlotBytes);  // B words (gemv.cu layout)
  float* red = reinterpret_cast<float*>(xq + K);                        // 2 x [2][128]
  float* scratch = red + 4 * kTileRows;
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + 16);
  uint64_t* empty = full + kMaxSlots;
  int* flag = reinterpret_cast<int*>(empty + kMaxSlots);

  pdl_trigger();
  const int G = gridDim.x, c = blockIdx.x;
  const long T = static_cast<long>(a.n_mt) * a.n_kb;
  const long t0 = c * T / G, t1 = (c + 1) * T / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EctHeader* h = reinterpret_cast<const EctHeader*>(a.ct_blob);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
#if defined(LS_GEMV_EXP) && (LS_GEMV_EXP & 32)  // diagnostic: launch + setup only
  return;
#endif

  if (warp == kWarps) {  // ---- producer warp: one chunk (<= 4 pages + masks) per slot ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* masks =
          h->off_escmask ? a.ct_blob + h->off_escmask + static_cast<long>(a.ct_page0) * kMaskBytes : nullptr;
      int kb = static_cast<int>(t0 % a.n_kb), s = 0;
      uint32_t round = 0;
      for (long t = t0; t < t1;) {
        int np = a.n_kb - kb;
        if (np > kChunk) np = kChunk;
        if (np > t1 - t) np = static_cast<int>(t1 - t);
        if (round) mbar_wait(&empty[s], (round - 1) & 1);
        uint8_t* dst = slots + s * kSlotBytes;
        mbar_arrive_expect_tx(&full[s], np * (kEctPageBytes + (masks ? kMaskBytes : 0)));
        bulk_g2s_evict_first(dst, a.w + t * kEctPageBytes, np * kEctPageBytes, &full[s], pol);
        if (masks)
          bulk_g2s_evict_first(dst + kChunk * kEctPageBytes, masks + t * kMaskBytes, np * kMaskBytes, &full[s],
                               pol);
        t += np;
        kb += np;
        if (kb == a.n_kb) kb = 0;
        if (++s == NQ) {
          s = 0;
          ++round;
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const int tid = threadIdx.x;
  const uint32_t e0p = (h->e0 << 7) | (h->e0 << 23);
  const uint32_t* exc_off = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_excoff) + a.ct_page0;
  const uint32_t* exc = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_exc);
  const bool has_mask = h->off_escmask != 0;

  const int g = lane >> 2, t4 = lane & 3;
  const int rb = warp & 7, kh = warp >> 3;  // row block, k-part (k-steps 2 kh, 2 kh + 1)
  const int wreg = rb * 2 + kh;             // warp region: page words [512 wreg, +512)
  const int f0 = (wreg * 32 + lane) * 2;    // this lane's two fragments in a page
  // B words: column g = 0 -> hi, 1 -> lo; columns g >= 2 repeat them and only
  // reach C columns >= 2, which lanes t4 != 0 hold and the flush ignores
  const uint32_t* xb = xq + kh * 32 + (g & 1) * 16 + t4 * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};

  auto frags = [&](const uint8_t* pg, uint32_t page, bool esc, uint32_t (&af)[2][4]) {
    const uint4 sm = *reinterpret_cast<const uint4*>(pg + f0 * 8);
    const uint2 nib = *reinterpret_cast<const uint2*>(pg + kEctPageWords + f0 * 4);
    uint4 w0 = ect_decode8(make_uint2(sm.x, sm.y), nib.x, e0p);
    uint4 w1 = ect_decode8(make_uint2(sm.z, sm.w), nib.y, e0p);
    if (esc) {  // this lane's 16 words hold an escape (rare, divergent)
      ect_patch16(w0, w1, ect_escapes(nib.x), ect_escapes(nib.y), page, f0 * 8, exc_off, exc);
    }
    af[0][0] = w0.x; af[0][1] = w0.y; af[0][2] = w0.z; af[0][3] = w0.w;
    af[1][0] = w1.x; af[1][1] = w1.y; af[1][2] = w1.z; af[1][3] = w1.w;
  };
  // without a mask section every lane takes the escape test (the slot's mask
  // area then holds stale bytes, overridden by no_mask)
  const uint32_t no_mask = has_mask ? 0u : 0xffffffffu;
  const int esh = 8 * (wreg & 3) + (lane >> 2);  // mask bit of this lane's 64-word group
  auto lane_esc = [&](const uint8_t* st, int q) -> bool {
    const uint32_t m = *reinterpret_cast<const uint32_t*>(st + kChunk * kEctPageBytes + q * kMaskBytes + (wreg >> 2) * 4);
    return ((m | no_mask) >> esh) & 1u;
  };

  int kb = static_cast<int>(t0 % a.n_kb), mt = static_cast<int>(t0 / a.n_kb), s = 0;
  int rem = static_cast<int>(t1 - t0), par = 0;
  uint32_t t = static_cast<uint32_t>(t0), round = 0;
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  // K <= 4096 (QKV, O, gate|up): the first chunk's pages do not depend on the
  // previous kernel -- decode them into registers while it drains, then stage x
  uint32_t fr0[kChunk][2][4];
  bool have0 = false;
  if (K <= 8 * kConsumers && min(min(kChunk, a.n_kb - kb), rem) == kChunk) {
    mbar_wait_u32(full0, 0);
#pragma unroll
    for (int q = 0; q < kChunk; ++q) frags(slots + q * kEctPageBytes, t + q, lane_esc(slots, q), fr0[q]);
    have0 = true;
  }
#if defined(LS_GEMV_EXP) && (LS_GEMV_EXP & 16)  // diagnostic: no x prologue (wrong results)
  pdl_wait();
#else
  if (K <= 8 * kConsumers) gemv_stage_x<kConsumers, 4>(a, xq, scratch, K, tid, lane, warp);
  else gemv_stage_x<kConsumers>(a, xq, scratch, K, tid, lane, warp);
#endif
  named_bar(1, kConsumers);
  auto advance = [&](int np) {
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty0 + 8 * s);
    if (++s == NQ) {
      s = 0;
      ++round;
    }
    t += np;
    rem -= np;
    kb += np;
    if (kb == a.n_kb) {
      gemv_flush<EPI, kConsumers, 2>(a, acc, red, par, flag, mt, G, T, c, tid, g, t4, rb, kh);
      kb = 0;
      ++mt;
    }
  };
  if (have0) {  // the chunk decoded before x was staged
#pragma unroll
    for (int q = 0; q < kChunk; ++q) {
      const uint4 bw = *reinterpret_cast<const uint4*>(xb + (kb + q) * 64);
      mma_bf16_16816(acc, fr0[q][0], bw.x, bw.y);
      mma_bf16_16816(acc, fr0[q][1], bw.z, bw.w);
    }
    advance(kChunk);
  }
  while (rem > 0) {
    const int np = min(min(kChunk, a.n_kb - kb), rem);
    const uint8_t* st = slots + s * kSlotBytes;
    if (np == kChunk) {
      uint4 bw[kChunk];
#pragma unroll
      for (int q = 0; q < kChunk; ++q)
        bw[q] = *reinterpret_cast<const uint4*>(xb + (kb + q) * 64);
      uint32_t fr[kChunk][2][4];
      mbar_wait_u32(full0 + 8 * s, round & 1);
#pragma unroll
      for (int q = 0; q < kChunk; ++q)
        frags(st + q * kEctPageBytes, t + q, lane_esc(st, q), fr[q]);
#pragma unroll
      for (int q = 0; q < kChunk; ++q) {
        mma_bf16_16816(acc, fr[q][0], bw[q].x, bw[q].y);
        mma_bf16_16816(acc, fr[q][1], bw[q].z, bw[q].w);
      }
    } else {
      mbar_wait_u32(full0 + 8 * s, round & 1);
      for (int q = 0; q < np; ++q) {
        const uint4 bw = *reinterpret_cast<const uint4*>(xb + (kb + q) * 64);
        uint32_t fr[2][4];
        frags(st + q * kEctPageBytes, t + q, lane_esc(st, q), fr);
        mma_bf16_16816(acc, fr[0], bw.x, bw.y);
        mma_bf16_16816(acc, fr[1], bw.z, bw.w);
      }
    }
    advance(np);
  }
  if (kb != 0) gemv_flush<EPI, kConsumers, 2>(a, acc, red, par, flag, mt, G, T, c, tid, g, t4, rb, kh);
}

template <int EPI>
static cudaError_t launch_ect_t(const GemvArgs& a, int grid, cudaStream_t st) {
  static DeviceFlags attr_set;
  if (!attr_set.done()) {
    cudaError_t e =
        cudaFuncSetAttribute(gemv_ect_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return e;
    // one shared-memory carveout for every in-step kernel: a decode-attention CTA
    // can then share an SM with a GEMV CTA without a reconfiguration drain
    e = cudaFuncSetAttribute(gemv_ect_kernel<EPI>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr_set.mark();
  }
  return launch_k(gemv_ect_kernel<EPI>, dim3(grid), dim3(kThreads), ect_smem(a.n_kb, a.max_slots), st, a);
}

cudaError_t launch_gemv_ect(int epi, const GemvArgs& a, int grid, cudaStream_t st) {
  if (ect_slots(a.n_kb, a.max_slots) < 2 || ect_smem(a.n_kb, a.max_slots) > static_cast<size_t>(kSmemBudget))
    return cudaErrorInvalidValue;
  switch (epi) {
    case GEMV_F32: return launch_ect_t<GEMV_F32>(a, grid, st);
    case GEMV_RESID: return launch_ect_t<GEMV_RESID>(a, grid, st);
    case GEMV_SILU: return launch_ect_t<GEMV_SILU>(a, grid, st);
    case GEMV_QKV: return launch_ect_t<GEMV_QKV>(a, grid, st);
    case GEMV_ARGMAX: return launch_ect_t<GEMV_ARGMAX>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lsb
