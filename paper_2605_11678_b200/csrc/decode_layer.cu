// decode_layer.cu -- one persistent kernel per LM decode layer (batch 1).
//
// A decode layer is ~386 MB of weights read once: QKV GEMV -> GQA attention ->
// O GEMV (+residual) -> gate|up GEMV (+SiLU*up) -> down GEMV (+residual).  As
// five launches each pays launch latency, a prologue and a drain tail, and
// HBM idles between them.  Here one 148-CTA persistent grid runs all five
// phases separated by grid barriers, while the producer warp of every CTA
// streams ITS tiles of all four weight matrices back to back through one
// bulk-copy (TMA engine) ring: weights never depend on activations, so the
// next phase's tiles are already in shared memory when a barrier releases.
// The GEMV consumers, the deterministic stream-K fix-up and the fused
// epilogues are those of gemv.cu; attention is the split-context scheme of
// attention.cu with one (kv head, split) work item per CTA.
//
// Co-residency: 1 CTA per SM (shared memory) and grid == #SMs.  PDL dependents
// are released only after the last grid barrier, so a following kernel can
// never occupy an SM this grid still needs.
#include "common.cuh"
#include "gemv_common.cuh"
#include "kernels.h"

namespace lsb {

namespace {

constexpr int kThreads = 288;    // 8 consumer warps + 1 producer warp
constexpr int kConsumers = 256;
constexpr int kMaxStages = 12;
constexpr int kAttnChunk = 64;   // positions per attention work item

__device__ __forceinline__ int cta_of_tile_dl(long t, int G, long T) {
  return static_cast<int>(((t + 1) * G - 1) / T);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over the consumer warps of every CTA (generation counter).
__device__ void grid_sync(unsigned* bar, unsigned& gen, int tid) {
  named_bar(1, kConsumers);
  if (tid == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(&bar[1], gen + 1);
    } else {
      while (ld_acquire(&bar[1]) == gen) __nanosleep(64);
    }
  }
  ++gen;
  named_bar(1, kConsumers);
}

struct Ring {
  uint8_t* stages;
  uint64_t* full;
  uint64_t* empty;
  int ns, s;
  uint32_t round;
};

}  // namespace

int decode_layer_stages(int max_kb) {
  const int fixed = max_kb * kTileCols * 4 + 2 * kAttnChunk * 128 * 2 + 8 * 1024 + 2048;
  const int avail = (227 * 1024 - fixed) / kTileBytes;
  return avail > kMaxStages ? kMaxStages : avail;
}

__global__ void __launch_bounds__(kThreads, 1) decode_layer_kernel(const DecodeLayerArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int NS = a.stages;
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  int max_k = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) max_k = max(max_k, a.n_kb[p] * kTileCols);
  uint8_t* stages = smem;
  float* xs = reinterpret_cast<float*>(smem + NS * kTileBytes);
  bf16* kvs = reinterpret_cast<bf16*>(xs + max_k);                  // [2][kAttnChunk][hd]
  float* comb = reinterpret_cast<float*>(kvs + 2 * kAttnChunk * a.hd);  // 8 KiB scratch
  float* red = comb + 2048;
  float* scratch = red + kTileRows;
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + 16);
  uint64_t* empty = full + kMaxStages;
  int* flag = reinterpret_cast<int*>(empty + kMaxStages);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumers / 32) {  // ---- producer: all four weight matrices, back to back ----
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t round = 0;
      for (int p = 0; p < 4; ++p) {
        const long T = static_cast<long>(a.n_mt[p]) * a.n_kb[p];
        const int Ge = static_cast<int>(T < G ? T : G);  // CTAs with work in this phase
        if (c >= Ge) continue;
        const long t0 = c * T / Ge, t1 = (c + 1) * T / Ge;
        const uint8_t* src = a.w[p] + t0 * kTileBytes;
        for (long n = t1 - t0; n > 0; --n) {
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
    }
    return;
  }

  pdl_wait();
  unsigned gen = ld_acquire(&a.barrier[1]);
  Ring ring{stages, full, empty, NS, 0, 0};
  const int rr = lane >> 3, ch = lane & 7;

  // ---- one GEMV phase: x (global, fp32) -> consumers -> fused epilogue ----
  auto gemv_phase = [&](int p, const float* x, const bf16* norm_w, int epi, float* out, int n_valid) {
    const long T = static_cast<long>(a.n_mt[p]) * a.n_kb[p];
    const int Ge = static_cast<int>(T < G ? T : G);  // contiguous non-empty ranges
    if (c >= Ge) return;
    const int K = a.n_kb[p] * kTileCols;
    float ss = 0.f;
    for (int k = tid; k < K; k += kConsumers) {
      const float v = __ldcg(x + k);  // written by other CTAs before the barrier
      xs[k] = v;
      ss = fmaf(v, v, ss);
    }
    if (norm_w) {
      ss = warp_sum(ss);
      if (lane == 0) scratch[warp] = ss;
      named_bar(1, kConsumers);
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumers / 32; ++w) tot += scratch[w];
      const float rstd = rsqrtf(tot / K + a.eps);
      for (int k = tid; k < K; k += kConsumers) xs[k] = xs[k] * rstd * bf2f(norm_w[k]);
    }
    named_bar(1, kConsumers);
    const long t0 = c * T / Ge, t1 = (c + 1) * T / Ge;
    GemvArgs ea{};
    ea.n_mt = a.n_mt[p];
    ea.n_kb = a.n_kb[p];
    ea.out = out;
    ea.n_valid = n_valid;
    ea.eps = a.eps;
    ea.hq = a.hq;
    ea.hkv = a.hkv;
    ea.hd = a.hd;
    ea.pos = a.pos;
    ea.qn_w = a.qn_w;
    ea.kn_w = a.kn_w;
    ea.rope = a.rope;
    ea.q_out = a.q;
    ea.k_cache = a.k_cache;
    ea.v_cache = a.v_cache;
    ea.cache_head_stride = a.cache_head_stride;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    int cur_mt = static_cast<int>(t0 / a.n_kb[p]);
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
      named_bar(1, kConsumers);
      const long first = static_cast<long>(mt) * a.n_kb[p], last = first + a.n_kb[p] - 1;
      const int c_first = cta_of_tile_dl(first, Ge, T);
      const int n_contrib = cta_of_tile_dl(last, Ge, T) - c_first + 1;
      if (n_contrib == 1) {
        if (tid < kTileRows) gemv_epilogue_any(epi, ea, mt, red, tid);
        named_bar(1, kConsumers);
        return;
      }
      float* mine = a.ws + (static_cast<long>(mt) * a.max_contrib + (c - c_first)) * kTileRows;
      if (tid < kTileRows) mine[tid] = red[tid];
      __threadfence();
      named_bar(1, kConsumers);
      if (tid == 0) *flag = atomicAdd(&a.counters[mt], 1) == n_contrib - 1;
      named_bar(1, kConsumers);
      if (*flag) {
        __threadfence();
        if (tid < kTileRows) {
          const float* base = a.ws + static_cast<long>(mt) * a.max_contrib * kTileRows;
          float s = 0.f;
          for (int j = 0; j < n_contrib; ++j) s += __ldcg(base + j * kTileRows + tid);
          red[tid] = s;
        }
        named_bar(1, kConsumers);
        if (tid < kTileRows) gemv_epilogue_any(epi, ea, mt, red, tid);
        if (tid == 0) a.counters[mt] = 0;
      }
      named_bar(1, kConsumers);
    };
    int kb = static_cast<int>(t0 - static_cast<long>(cur_mt) * a.n_kb[p]);
    for (long n = t1 - t0, mt = cur_mt; n > 0; --n) {
      if (kb == a.n_kb[p]) {
        kb = 0;
        ++mt;
        flush(cur_mt);
        cur_mt = static_cast<int>(mt);
      }
      mbar_wait(&ring.full[ring.s], ring.round & 1);
      const uint8_t* st = ring.stages + ring.s * kTileBytes;
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
      if (lane == 0) mbar_arrive(&ring.empty[ring.s]);
      ++kb;
      if (++ring.s == ring.ns) {
        ring.s = 0;
        ++ring.round;
      }
    }
    flush(cur_mt);
  };

  // 1. QKV GEMV (+ RMSNorm prologue, q/k norm + RoPE + KV-cache append)
  gemv_phase(0, a.h, a.attn_norm, GEMV_QKV, a.q, a.n_mt[0] * kTileRows);
  grid_sync(a.barrier, gen, tid);

  // 2. attention: work item (kv head, split) per CTA, partials merged by the last
  {
    const int items = a.hkv * a.n_split;
    const int HD = a.hd, G_ = a.hq / a.hkv, E = HD / 32;
    const float sl2 = a.scale * 1.4426950408889634f;
    const int W = HD + 2;
    for (int item = c; item < items; item += G) {
      const int kh = item / a.n_split, split = item % a.n_split;
      const int n_ctx = a.pos + 1;
      const int chunk = (n_ctx + a.n_split - 1) / a.n_split;
      const int p0 = split * chunk, p1 = min(n_ctx, p0 + chunk);
      const int np = max(p1 - p0, 0);
      const bf16* kb = a.k_cache + static_cast<long>(kh) * a.cache_head_stride + static_cast<long>(p0) * HD;
      const bf16* vb = a.v_cache + static_cast<long>(kh) * a.cache_head_stride + static_cast<long>(p0) * HD;
      bf16* ks = kvs;
      bf16* vs = kvs + kAttnChunk * HD;
      for (int i = tid; i < np * HD / 8; i += kConsumers) {  // KV written in phase 1 by other CTAs
        reinterpret_cast<uint4*>(ks)[i] = __ldcg(reinterpret_cast<const uint4*>(kb) + i);
        reinterpret_cast<uint4*>(vs)[i] = __ldcg(reinterpret_cast<const uint4*>(vb) + i);
      }
      named_bar(1, kConsumers);
      // warp w < G_ handles query head kh*G_ + w over all np positions (lane = dims)
      if (warp < G_) {
        const int hq_i = kh * G_ + warp;
        float qv[4];
        for (int e = 0; e < E; ++e) qv[e] = __ldcg(a.q + hq_i * HD + lane * E + e) * sl2;
        float m = -INFINITY, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < np; ++j) {
          float sc = 0.f;
          for (int e = 0; e < E; ++e) sc = fmaf(qv[e], bf2f(ks[j * HD + lane * E + e]), sc);
          sc = warp_sum(sc);
          const float mn = fmaxf(m, sc);
          const float corr = exp2f(m - mn), pe = exp2f(sc - mn);
          l = l * corr + pe;
          for (int e = 0; e < E; ++e) acc[e] = acc[e] * corr + pe * bf2f(vs[j * HD + lane * E + e]);
          m = mn;
        }
        float* rec = a.attn_ws + (static_cast<long>(hq_i) * a.n_split + split) * W;
        for (int e = 0; e < E; ++e) rec[2 + lane * E + e] = acc[e];
        if (lane == 0) {
          rec[0] = m;
          rec[1] = l;
        }
      }
      __threadfence();
      named_bar(1, kConsumers);
      if (tid == 0) *flag = atomicAdd(&a.attn_cnt[kh], 1) == a.n_split - 1;
      named_bar(1, kConsumers);
      if (*flag) {
        __threadfence();
        for (int idx = tid; idx < G_ * HD; idx += kConsumers) {
          const int g = idx / HD, dd = idx % HD, h = kh * G_ + g;
          const float* r = a.attn_ws + static_cast<long>(h) * a.n_split * W;
          float M = -INFINITY;
          for (int sp = 0; sp < a.n_split; ++sp) M = fmaxf(M, __ldcg(r + sp * W));
          float L = 0.f, O = 0.f;
          for (int sp = 0; sp < a.n_split; ++sp) {
            const float ms = __ldcg(r + sp * W);
            if (ms == -INFINITY) continue;
            const float f = exp2f(ms - M);
            L += __ldcg(r + sp * W + 1) * f;
            O += __ldcg(r + sp * W + 2 + dd) * f;
          }
          a.attn[h * HD + dd] = O / L;
        }
        if (tid == 0) a.attn_cnt[kh] = 0;
      }
      named_bar(1, kConsumers);
    }
  }
  grid_sync(a.barrier, gen, tid);

  // 3. O GEMV + residual
  gemv_phase(1, a.attn, nullptr, GEMV_RESID, a.h, a.n_mt[1] * kTileRows);
  grid_sync(a.barrier, gen, tid);
  // 4. gate|up GEMV (+ RMSNorm prologue, SiLU*up)
  gemv_phase(2, a.h, a.mlp_norm, GEMV_SILU, a.mlp, a.ffn);
  grid_sync(a.barrier, gen, tid);
  // 5. down GEMV + residual
  gemv_phase(3, a.mlp, nullptr, GEMV_RESID, a.h, a.n_mt[3] * kTileRows);
  grid_sync(a.barrier, gen, tid);
  pdl_trigger();  // only now may a dependent kernel take SMs
  (void)comb;
}

cudaError_t launch_decode_layer(const DecodeLayerArgs& a, int num_sms, cudaStream_t st) {
  int max_kb = 0;
  for (int p = 0; p < 4; ++p) max_kb = a.n_kb[p] > max_kb ? a.n_kb[p] : max_kb;
  const size_t smem = static_cast<size_t>(a.stages) * kTileBytes + max_kb * kTileCols * 4 +
                      2ull * kAttnChunk * a.hd * 2 + 8 * 1024 + kTileRows * 4 + 64 +
                      2 * kMaxStages * 8 + 16;
  if (smem > 227 * 1024 || a.stages < 2 || a.hd > 128 || (a.pos + a.n_split) / a.n_split > kAttnChunk)
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_k(decode_layer_kernel, dim3(num_sms), dim3(kThreads), smem, st, a);
}

}  // namespace lsb
