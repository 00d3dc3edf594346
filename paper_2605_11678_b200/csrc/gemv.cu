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

constexpr int kGemvMaxStages = 12;

// Ring depth from the shared-memory left after x (fp32, K floats): 12 stages
// (192 KiB in flight per SM) for K = 4096, 11 for K = 12288.
__host__ __device__ inline int gemv_stages(int n_kb) {
  const int avail = (227 * 1024 - n_kb * kTileCols * 4 - 1024) / kTileBytes;
  return avail > kGemvMaxStages ? kGemvMaxStages : avail;
}
constexpr int kGemvConsumers = 256;  // 8 warps
constexpr int kGemvThreads = kGemvConsumers + 32;

__device__ __forceinline__ int cta_of_tile(long t, int G, long T) {
  return static_cast<int>(((t + 1) * G - 1) / T);
}

template <int EPI>
__global__ void __launch_bounds__(kGemvThreads, 1) gemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int K = a.n_kb * kTileCols;
  uint8_t* stages = smem;
  const int NS = gemv_stages(a.n_kb);
  float* xs = reinterpret_cast<float*>(smem + NS * kTileBytes);
  float* red = xs + K;
  float* scratch = red + kTileRows;  // 8 floats for block reductions
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
      const uint8_t* src = a.w + t0 * kTileBytes;
      int s = 0;
      uint32_t round = 0;
      for (int n = static_cast<int>(t1 - t0); n > 0; --n) {
        if (round) mbar_wait(&empty[s], (round - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kTileBytes);
        bulk_g2s_evict_first(stages + s * kTileBytes, src, kTileBytes, &full[s], pol);
        src += kTileBytes;
        if (++s == NS) {
          s = 0;
          ++round;
        }
      }
    }
    return;
  }

  // ---- consumers: x -> shared (fp32), optional fused RMSNorm ----
  pdl_wait();  // x, workspace and outputs belong to the previous kernel until here
  const int tid = threadIdx.x;
  float ss = 0.f;
  for (int k = tid; k < K; k += kGemvConsumers) {
    float v = a.x[k];
    xs[k] = v;
    ss = fmaf(v, v, ss);
  }
  if (a.norm_w) {
    ss = warp_sum(ss);
    if (lane == 0) scratch[warp] = ss;
    named_bar(1, kGemvConsumers);
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kGemvConsumers / 32; ++w) tot += scratch[w];
    const float rstd = rsqrtf(tot / K + a.eps);
    for (int k = tid; k < K; k += kGemvConsumers) xs[k] = xs[k] * rstd * bf2f(a.norm_w[k]);
  }
  named_bar(1, kGemvConsumers);

  const int rr = lane >> 3, ch = lane & 7;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int cur_mt = t0 < t1 ? static_cast<int>(t0 / a.n_kb) : -1;

  auto flush = [&](int mt) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v = acc[j];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      if (ch == 0) red[warp * 16 + rr + 4 * j] = v;
      acc[j] = 0.f;
    }
    named_bar(1, kGemvConsumers);
    const long first = static_cast<long>(mt) * a.n_kb, last = first + a.n_kb - 1;
    const int c_first = cta_of_tile(first, G, T);
    const int n_contrib = cta_of_tile(last, G, T) - c_first + 1;
    if (n_contrib == 1) {
      if (tid < kTileRows) gemv_epilogue<EPI>(a, mt, red, tid);
      named_bar(1, kGemvConsumers);
      return;
    }
    const int slot = c - c_first;
    float* mine = a.ws + (static_cast<long>(mt) * a.max_contrib + slot) * kTileRows;
    if (tid < kTileRows) mine[tid] = red[tid];
    __threadfence();
    named_bar(1, kGemvConsumers);
    if (tid == 0) {
      const int old = atomicAdd(&a.counters[mt], 1);
      *flag = (old == n_contrib - 1);
    }
    named_bar(1, kGemvConsumers);
    if (*flag) {
      __threadfence();
      if (tid < kTileRows) {
        const float* base = a.ws + static_cast<long>(mt) * a.max_contrib * kTileRows;
        float s = 0.f;
        for (int j = 0; j < n_contrib; ++j) s += __ldcg(base + j * kTileRows + tid);
        red[tid] = s;
      }
      named_bar(1, kGemvConsumers);
      if (tid < kTileRows) gemv_epilogue<EPI>(a, mt, red, tid);
      if (tid == 0) a.counters[mt] = 0;
    }
    named_bar(1, kGemvConsumers);
  };

  int kb = t0 < t1 ? static_cast<int>(t0 - static_cast<long>(cur_mt) * a.n_kb) : 0;
  int s = 0;
  uint32_t round = 0;
  for (int n = static_cast<int>(t1 - t0), mt = cur_mt; n > 0; --n) {
    if (kb == a.n_kb) {
      kb = 0;
      ++mt;
      flush(cur_mt);
      cur_mt = mt;
    }
    mbar_wait(&full[s], round & 1);
    const uint8_t* st = stages + s * kTileBytes;
    const float* xk = xs + kb * kTileCols;
    const float4* xa = reinterpret_cast<const float4*>(xk + ((ch ^ rr) << 3));
    const float4* xb = reinterpret_cast<const float4*>(xk + ((ch ^ (rr + 4)) << 3));
    const float4 a0 = xa[0], a1 = xa[1], b0 = xb[0], b1 = xb[1];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = warp * 16 + rr + 4 * j;
      const uint4 wv = *reinterpret_cast<const uint4*>(st + row * 128 + ch * 16);
      acc[j] += (j & 1) ? dot8(wv, b0, b1) : dot8(wv, a0, a1);
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

static size_t gemv_smem(int n_kb) {
  return static_cast<size_t>(gemv_stages(n_kb)) * kTileBytes + static_cast<size_t>(n_kb) * kTileCols * 4 +
         kTileRows * 4 + 16 * 4 + 2 * kGemvMaxStages * 8 + 16;
}

template <int EPI>
static cudaError_t launch_t(const GemvArgs& a, int grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemv_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  return launch_k(gemv_kernel<EPI>, dim3(grid), dim3(kGemvThreads), gemv_smem(a.n_kb), st, a);
}

cudaError_t launch_gemv(int epi, const GemvArgs& a, int grid, cudaStream_t st) {
  if (gemv_smem(a.n_kb) > 227 * 1024) return cudaErrorInvalidValue;
  switch (epi) {
    case GEMV_F32: return launch_t<GEMV_F32>(a, grid, st);
    case GEMV_RESID: return launch_t<GEMV_RESID>(a, grid, st);
    case GEMV_SILU: return launch_t<GEMV_SILU>(a, grid, st);
    case GEMV_QKV: return launch_t<GEMV_QKV>(a, grid, st);
    case GEMV_ARGMAX: return launch_t<GEMV_ARGMAX>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lsb
