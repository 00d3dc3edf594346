// gemv.cu -- decode-time (batch 1) matrix-vector product over tiled weights.
//
// Roofline: HBM.  Algorithmic bytes per launch = N*K*2 (weights, read once)
// + K*4 (x) + N*4 (y).  Design for B200:
//   * persistent grid (<= 148 CTAs, one per SM); the flattened (m-tile,
//     k-block) tile sequence is split into equal contiguous ranges (stream-K),
//     so every SM streams the same number of 16 KiB tiles regardless of shape;
//   * one producer warp issues 1-D bulk copies (TMA engine, L2 evict-first)
//     into an 8-stage shared-memory ring guarded by mbarriers -- 128 KiB in
//     flight per SM, no registers spent on loads;
//   * eight consumer warps dot the swizzled tile rows with x (fp32, resident
//     in shared memory, RMSNorm fused in the prologue) and keep per-row
//     partials in registers across a CTA's whole k-range;
//   * m-tiles split across CTAs are fixed up deterministically: partials land
//     in a workspace slot per contributor and the last arriving CTA sums them
//     in contributor order (bit-reproducible), then runs the fused epilogue
//     (residual add / SiLU*up / q,k-norm + RoPE + KV-cache append / argmax).
#include "common.cuh"
#include "gemv_common.cuh"
#include "kernels.h"

namespace lsb {

constexpr int kGemvMaxStages = 16;
// Shared-memory budget per CTA.  Measured: capping it at 113 KiB so two GEMV
// CTAs (of consecutive PDL-chained launches) can share an SM is a net loss
// (decode layer 127 -> 193 us): the shallower ring costs more than the overlap
// gains, so each GEMV owns its SM's shared memory.
#ifndef LS_GEMV_SMEM_KB
#define LS_GEMV_SMEM_KB 227
#endif
constexpr int kGemvSmemBudget = LS_GEMV_SMEM_KB * 1024;

// Ring depth from the shared-memory left after x (fp32, K floats): 12 x 16 KiB
// plain tiles or 16 x 12 KiB ECT pages (192 KiB in flight per SM) for K = 4096.
template <bool CT>
__host__ __device__ inline int gemv_stages(int n_kb) {
  constexpr int stage = CT ? kEctPageBytes : kTileBytes;
  constexpr int cap = CT ? 16 : 12;
  const int avail = (kGemvSmemBudget - n_kb * kTileCols * 4 - 2560) / stage;
  return avail > cap ? cap : avail;
}
// NW consumer warps = 8 row blocks x NW/8 k-parts of every tile (16: two k-steps
// per warp -- the launched configuration; 32 would exceed 1024 threads with the
// producer warp).
template <int NW>
struct GemvShape {
  static constexpr int kConsumers = NW * 32;
  static constexpr int kThreads = kConsumers + 32;
  static constexpr int kQ = NW / 8;  // k-parts per tile
};

#ifndef LS_GEMV_EXP
#define LS_GEMV_EXP 0
#endif
__device__ __forceinline__ void gemv_mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
#if LS_GEMV_EXP & 2  // diagnostic build: operands consumed, no tensor-core work
  asm volatile("" ::"r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
#else
  mma_bf16_16816(c, a, b0, b1);
#endif
}

// Consumers run the dot products on the tensor cores: mma.sync m16n8k16 with
// the weight tile as A (16 rows x 16 k per warp and k-step, fetched by one
// ldmatrix.x4 from the swizzled tile -- conflict-free -- or decoded straight
// from an ECT page, which stores words in A-fragment order) and x as B with
// two live columns, bf16(x) and bf16(x - bf16(x)) (x to ~16 mantissa bits).
// Per 8 weight words a thread spends ~0.25 instructions instead of 16 FMA +
// convert ops, which is what lets the ECT decode (~2.5 ops/word) fit under
// the HBM stream.  Warp w owns rows 16 (w % 8) .. +15 and k-steps 2 (w / 8),
// +1 of every tile (16 warps hide the decode latency); the two k-halves are
// summed in a fixed order at flush.  x lives in shared memory pre-arranged so
// a lane's four B words for two k-steps are one 16-byte load, and an ECT page
// keeps a lane's two fragments for its k-step pair adjacent (one 16-byte +
// one 8-byte load).  Plain and ECT tiles give bit-identical results.
template <int EPI, bool CT, int NW>
__global__ void __launch_bounds__(GemvShape<NW>::kThreads, 1) gemv_kernel(const GemvArgs a) {
  constexpr int kGemvConsumers = GemvShape<NW>::kConsumers;
  constexpr int kQ = GemvShape<NW>::kQ;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kStage = CT ? kEctPageBytes : kTileBytes;
  const int K = a.n_kb * kTileCols;
  uint8_t* stages = smem;
  const int NS = gemv_stages<CT>(a.n_kb);
  // x as bf16x2 B words: [kb][half h][column hi|lo][t4][b0(2h), b1(2h), b0(2h+1), b1(2h+1)]
  uint32_t* xq = reinterpret_cast<uint32_t*>(smem + NS * kStage);
  float* red = reinterpret_cast<float*>(xq + K);  // 2 x [kQ][128]: one slice per k-part
  float* scratch = red + 2 * kQ * kTileRows;      // 16 floats for block reductions
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + 16);
  uint64_t* empty = full + kGemvMaxStages;
  int* flag = reinterpret_cast<int*>(empty + kGemvMaxStages);

  pdl_trigger();
  const int G = gridDim.x, c = blockIdx.x;
  const long T = static_cast<long>(a.n_mt) * a.n_kb;
  const long t0 = c * T / G, t1 = (c + 1) * T / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvConsumers / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kGemvConsumers / 32) {  // ---- producer warp ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // stage / round counters advance incrementally: no 64-bit div or mod per tile
      const uint8_t* src = a.w + t0 * kStage;
      int s = 0;
      uint32_t round = 0;
      for (int n = static_cast<int>(t1 - t0); n > 0; --n) {
        if (round) mbar_wait(&empty[s], (round - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kStage);
        bulk_g2s_evict_first(stages + s * kStage, src, kStage, &full[s], pol);
        src += kStage;
        if (++s == NS) {
          s = 0;
          ++round;
        }
      }
    }
    return;
  }

  // ---- consumers: x -> shared (fp32), optional fused RMSNorm ----
  const int tid = threadIdx.x;
  const uint32_t* exc_off = nullptr;
  const uint32_t* exc = nullptr;
  uint32_t e0p = 0;
  if constexpr (CT) {  // weights are not produced by the previous kernel
    const EctHeader* h = reinterpret_cast<const EctHeader*>(a.ct_blob);
    e0p = (h->e0 << 7) | (h->e0 << 23);
    exc_off = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_excoff) + a.ct_page0;
    exc = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_exc);
  }
  gemv_stage_x<kGemvConsumers>(a, xq, scratch, K, tid, lane, warp);
  named_bar(1, kGemvConsumers);

  const int g = lane >> 2, t4 = lane & 3;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // mma C: rows g, g+8 x columns (hi, lo) in lanes t4 == 0
  int cur_mt = t0 < t1 ? static_cast<int>(t0 / a.n_kb) : -1;

  const int rb = warp & 7, kh = warp >> 3;  // row block, k-part
  int par = 0;  // red buffer of the next flush
  auto flush = [&](int mt) {
    gemv_flush<EPI, kGemvConsumers, kQ>(a, acc, red, par, flag, mt, G, T, c, tid, g, t4, rb, kh);
  };

  // B words: column g = 0 -> hi, g = 1 -> lo; columns g >= 2 repeat them and
  // only reach C columns >= 2 (lanes t4 != 0), which the flush ignores
  const uint32_t* xb = xq + (kQ == 2 ? kh : kh >> 1) * 32 + (g & 1) * 16 + t4 * 4 +
                       (kQ == 2 ? 0 : (kh & 1) * 2);
  // ldmatrix.x4 row address of this lane inside a plain tile (k-step added per use)
  const int lr = rb * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
  const int lc = lane >> 4;  // 0: k 0-7 of the step, 1: k 8-15
  // ECT: this lane's fragments (k-steps 2kh, 2kh+1 for kQ = 2; k-step kh for kQ = 4)
  const int f0 = kQ == 2 ? ((rb * 2 + kh) * 32 + lane) * 2 : ((rb * 2 + (kh >> 1)) * 32 + lane) * 2 + (kh & 1);
  int kb = t0 < t1 ? static_cast<int>(t0 - static_cast<long>(cur_mt) * a.n_kb) : 0;
  int s = 0;
  uint32_t round = 0;
  uint32_t tile = static_cast<uint32_t>(t0);
  // ECT, two k-steps per warp: pages are consumed in pairs (same m-tile), so a
  // warp has four independent decode chains in flight and the per-page
  // barrier / bookkeeping cost is shared
  auto ect_frags = [&](const uint8_t* st, uint32_t pg_idx, uint32_t (&af)[2][4]) {
    const uint4 sm = *reinterpret_cast<const uint4*>(st + f0 * 8);
    const uint2 nib = *reinterpret_cast<const uint2*>(st + kEctPageWords + f0 * 4);
#if LS_GEMV_EXP & 1  // diagnostic build: no decode (wrong results, timing only)
    af[0][0] = sm.x; af[0][1] = sm.y; af[0][2] = nib.x; af[0][3] = sm.x ^ nib.x;
    af[1][0] = sm.z; af[1][1] = sm.w; af[1][2] = nib.y; af[1][3] = sm.z ^ nib.y;
    return;
#endif
    uint4 w0 = ect_decode8(make_uint2(sm.x, sm.y), nib.x, e0p);
    uint4 w1 = ect_decode8(make_uint2(sm.z, sm.w), nib.y, e0p);
    if (ect_escapes(nib.x) | ect_escapes(nib.y)) {
      w0 = ect_patch8(w0, ect_escapes(nib.x), pg_idx, f0 * 8, exc_off, exc);
      w1 = ect_patch8(w1, ect_escapes(nib.y), pg_idx, f0 * 8 + 8, exc_off, exc);
    }
    af[0][0] = w0.x; af[0][1] = w0.y; af[0][2] = w0.z; af[0][3] = w0.w;
    af[1][0] = w1.x; af[1][1] = w1.y; af[1][2] = w1.z; af[1][3] = w1.w;
  };
  for (int n = static_cast<int>(t1 - t0), mt = cur_mt; n > 0; --n, ++tile) {
    if (kb == a.n_kb) {
      kb = 0;
      ++mt;
      flush(cur_mt);
      cur_mt = mt;
    }
    if constexpr (CT && kQ == 2) {
      if (n > 3 && kb + 3 < a.n_kb) {  // four pages of one m-tile
        int ss[4];
        uint32_t rr[4];
        ss[0] = s;
        rr[0] = round;
#pragma unroll
        for (int q = 1; q < 4; ++q) {
          ss[q] = ss[q - 1] + 1 == NS ? 0 : ss[q - 1] + 1;
          rr[q] = ss[q - 1] + 1 == NS ? rr[q - 1] + 1 : rr[q - 1];
        }
        uint4 bw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          bw[q] = *reinterpret_cast<const uint4*>(xb + (kb + q) * 64);
        uint32_t fr[4][2][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mbar_wait(&full[ss[q]], rr[q] & 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) ect_frags(stages + ss[q] * kStage, tile + q, fr[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          gemv_mma(acc, fr[q][0], bw[q].x, bw[q].y);
          gemv_mma(acc, fr[q][1], bw[q].z, bw[q].w);
        }
        __syncwarp();
        if (lane == 0)
#pragma unroll
          for (int q = 0; q < 4; ++q) mbar_arrive(&empty[ss[q]]);
        kb += 4;
        s = ss[3] + 1 == NS ? 0 : ss[3] + 1;
        round = ss[3] + 1 == NS ? rr[3] + 1 : rr[3];
        n -= 3;
        tile += 3;
        continue;
      }
      if (n > 1 && kb + 1 < a.n_kb) {
        const int s1 = s + 1 == NS ? 0 : s + 1;
        const uint32_t round1 = s + 1 == NS ? round + 1 : round;
        const uint4 bw0 = *reinterpret_cast<const uint4*>(xb + kb * 64);
        const uint4 bw1 = *reinterpret_cast<const uint4*>(xb + (kb + 1) * 64);
        uint32_t fa[2][4], fb[2][4];
        // both pages first, so the two pages' loads and decode chains interleave
        mbar_wait(&full[s], round & 1);
        mbar_wait(&full[s1], round1 & 1);
        ect_frags(stages + s * kStage, tile, fa);
        ect_frags(stages + s1 * kStage, tile + 1, fb);
        gemv_mma(acc, fa[0], bw0.x, bw0.y);
        gemv_mma(acc, fa[1], bw0.z, bw0.w);
        gemv_mma(acc, fb[0], bw1.x, bw1.y);
        gemv_mma(acc, fb[1], bw1.z, bw1.w);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[s]);
          mbar_arrive(&empty[s1]);
        }
        kb += 2;
        s = s1 + 1 == NS ? 0 : s1 + 1;
        round = s1 + 1 == NS ? round1 + 1 : round1;
        --n;
        ++tile;
        continue;
      }
    }
    mbar_wait(&full[s], round & 1);
    const uint8_t* st = stages + s * kStage;
    if constexpr (kQ == 4) {  // one k-step per warp and tile
      const uint2 bw = *reinterpret_cast<const uint2*>(xb + kb * 64);
      uint32_t af[4];
      if constexpr (CT) {
        const uint2 sm = *reinterpret_cast<const uint2*>(st + f0 * 8);
        const uint32_t nib = *reinterpret_cast<const uint32_t*>(st + kEctPageWords + f0 * 4);
        uint4 w0 = ect_decode8(sm, nib, e0p);
        const uint32_t esc = ect_escapes(nib);
        if (esc) w0 = ect_patch8(w0, esc, tile, f0 * 8, exc_off, exc);
        af[0] = w0.x; af[1] = w0.y; af[2] = w0.z; af[3] = w0.w;
      } else {
        ldsm_x4(af, st + lr * 128 + (((2 * kh + lc) ^ (lr & 7)) << 4));
      }
      gemv_mma(acc, af, bw.x, bw.y);
    } else {
    const uint4 bw = *reinterpret_cast<const uint4*>(xb + kb * 64);
    uint32_t af[2][4];
    if constexpr (CT) {
      ect_frags(st, tile, af);
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q)
        ldsm_x4(af[q], st + lr * 128 + (((2 * (2 * kh + q) + lc) ^ (lr & 7)) << 4));
    }
    gemv_mma(acc, af[0], bw.x, bw.y);
    gemv_mma(acc, af[1], bw.z, bw.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++kb;
    if (++s == NS) {
      s = 0;
      ++round;
    }
  }
  if (cur_mt >= 0) flush(cur_mt);
}

int gemv_grid(int n_mt, int n_kb, int num_sms) {
  long T = static_cast<long>(n_mt) * n_kb;
  return static_cast<int>(T < num_sms ? T : num_sms);
}

int gemv_max_contrib(int n_mt, int n_kb, int grid) {
  long T = static_cast<long>(n_mt) * n_kb;
  int best = 1;
  for (int mt = 0; mt < n_mt; ++mt) {
    long first = static_cast<long>(mt) * n_kb, last = first + n_kb - 1;
    int cf = static_cast<int>(((first + 1) * grid - 1) / T);
    int cl = static_cast<int>(((last + 1) * grid - 1) / T);
    if (cl - cf + 1 > best) best = cl - cf + 1;
  }
  return best;
}

template <bool CT>
static size_t gemv_smem(int n_kb) {
  return static_cast<size_t>(gemv_stages<CT>(n_kb)) * (CT ? kEctPageBytes : kTileBytes) +
         static_cast<size_t>(n_kb) * kTileCols * 4 + 2 * 2 * kTileRows * 4 + 16 * 4 +
         2 * kGemvMaxStages * 8 + 16;
}

template <int EPI, bool CT, int NW>
static cudaError_t launch_t(const GemvArgs& a, int grid, cudaStream_t st) {
  static DeviceFlags attr_set;
  if (!attr_set.done()) {
    cudaError_t e = cudaFuncSetAttribute(gemv_kernel<EPI, CT, NW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set.mark();
  }
  return launch_k(gemv_kernel<EPI, CT, NW>, dim3(grid), dim3(GemvShape<NW>::kThreads),
                  gemv_smem<CT>(a.n_kb), st, a);
}

template <bool CT, int NW>
static cudaError_t launch_ct(int epi, const GemvArgs& a, int grid, cudaStream_t st) {
  if (gemv_smem<CT>(a.n_kb) > kGemvSmemBudget) return cudaErrorInvalidValue;
  switch (epi) {
    case GEMV_F32: return launch_t<GEMV_F32, CT, NW>(a, grid, st);
    case GEMV_RESID: return launch_t<GEMV_RESID, CT, NW>(a, grid, st);
    case GEMV_SILU: return launch_t<GEMV_SILU, CT, NW>(a, grid, st);
    case GEMV_QKV: return launch_t<GEMV_QKV, CT, NW>(a, grid, st);
    case GEMV_ARGMAX: return launch_t<GEMV_ARGMAX, CT, NW>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemv(int epi, const GemvArgs& a, int grid, cudaStream_t st) {
#if LS_GEMV_ECT_LEGACY  // diagnostic build: ECT pages through the generic kernel
  return a.ct_blob ? launch_ct<true, 16>(epi, a, grid, st) : launch_ct<false, 16>(epi, a, grid, st);
#else
  return a.ct_blob ? launch_gemv_ect(epi, a, grid, st) : launch_ct<false, 16>(epi, a, grid, st);
#endif
}

}  // namespace lsb
