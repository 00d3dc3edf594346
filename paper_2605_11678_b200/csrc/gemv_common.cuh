// gemv_common.cuh -- pieces shared by the stand-alone decode GEMV (gemv.cu) and
// the persistent decode-layer kernel (decode_layer.cu): the swizzled-row dot
// product and the fused fix-up epilogues.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace lsb {

__device__ __forceinline__ float dot8(uint4 w, const float4& a, const float4& b) {
  float s = bf16_lo(w.x) * a.x;
  s = fmaf(bf16_hi(w.x), a.y, s);
  s = fmaf(bf16_lo(w.y), a.z, s);
  s = fmaf(bf16_hi(w.y), a.w, s);
  s = fmaf(bf16_lo(w.z), b.x, s);
  s = fmaf(bf16_hi(w.z), b.y, s);
  s = fmaf(bf16_lo(w.w), b.z, s);
  s = fmaf(bf16_hi(w.w), b.w, s);
  return s;
}

// x pairs held in registers by the GEMV prologue: K <= 2 * kXRegPairs * 512
constexpr int kXRegPairs = 12;

// pair i = (x[2i], x[2i+1]) -> (hi, lo) bf16 B words in the layout of gemv_kernel's xq
__device__ __forceinline__ void gemv_stage_pair(uint32_t* xq, int i, float v0, float v1) {
  const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
  const float2 hf = __bfloat1622float2(hi);
  const __nv_bfloat162 lo = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
  const int kb = i >> 5, pp = i & 31;  // pair within the k-block: 16 h + 8 (ks&1) + 4 (b1) + t4
  const int h = pp >> 4, slot = ((pp >> 3) & 1) * 2 + ((pp >> 2) & 1), t4i = pp & 3;
  const int base = kb * 64 + h * 32 + t4i * 4 + slot;
  xq[base] = *reinterpret_cast<const uint32_t*>(&hi);
  xq[base + 16] = *reinterpret_cast<const uint32_t*>(&lo);
}

// Prologue for K beyond the register path: two passes over x in global memory.
static __device__ __noinline__ void gemv_stage_x_loop(const float* x, const bf16* norm_w, float eps, uint32_t* xq,
                                               float* scratch, int K, int tid, int lane, int warp,
                                               int n_consumers) {
  float rstd = 1.f;
  if (norm_w) {
    float ss = 0.f;
    for (int i = tid; i < K / 2; i += n_consumers) {
      const float2 v = reinterpret_cast<const float2*>(x)[i];
      ss = fmaf(v.x, v.x, ss);
      ss = fmaf(v.y, v.y, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) scratch[warp] = ss;
    named_bar(1, n_consumers);
    float tot = 0.f;
    for (int w = 0; w < n_consumers / 32; ++w) tot += scratch[w];
    rstd = rsqrtf(tot / K + eps);
  }
  for (int i = tid; i < K / 2; i += n_consumers) {
    float2 v = reinterpret_cast<const float2*>(x)[i];
    if (norm_w) {
      const float2 nw = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(norm_w)[i]);
      v.x = v.x * rstd * nw.x;
      v.y = v.y * rstd * nw.y;
    }
    gemv_stage_pair(xq, i, v.x, v.y);
  }
}

__device__ __forceinline__ int cta_of_tile(long t, int G, long T) {
  return static_cast<int>(((t + 1) * G - 1) / T);
}

template <int EPI>
__device__ void gemv_epilogue(const GemvArgs& a, int mt, const float* red, int tid) {
  // tid in [0,128): one output row each
  const int row = mt * kTileRows + tid;
  float y = red[tid];
  if constexpr (EPI == GEMV_F32 || EPI == GEMV_RESID) {
    if (row < a.n_valid) {
      if (a.bias) y += a.bias[row];
      if constexpr (EPI == GEMV_F32) a.out[row] = y;
      else a.out[row] += y;
    }
  } else if constexpr (EPI == GEMV_SILU) {
    if (tid < 64) {
      const int f = mt * 64 + tid;
      if (f < a.n_valid) a.out[f] = silu(y) * red[tid + 64];
    }
  } else if constexpr (EPI == GEMV_QKV) {
    const int hd = a.hd, h2 = hd >> 1;
    const int q_rows = a.hq * hd, k_rows = a.hkv * hd;
    if (row >= q_rows + 2 * k_rows) return;
    const int d = row % hd;
    const int head_base = tid - d;  // rows of one head never straddle a tile (hd | 128)
    const bool is_v = row >= q_rows + k_rows;
    if (is_v) {
      const int kh = (row - q_rows - k_rows) / hd;
      a.v_cache[(long)kh * a.cache_head_stride + (long)a.pos * hd + d] = f2bf(y);
      return;
    }
    const bool is_q = row < q_rows;
    float rstd = 1.0f;
    const bf16* nw = is_q ? a.qn_w : a.kn_w;
    if (nw) {
      float ss = 0.f;
      for (int i = 0; i < hd; ++i) ss = fmaf(red[head_base + i], red[head_base + i], ss);
      rstd = rsqrtf(ss / hd + a.eps);
    }
    auto normed = [&](int dd) {
      float v = red[head_base + dd] * rstd;
      return nw ? v * bf2f(nw[dd]) : v;
    };
    const int f = d < h2 ? d : d - h2;
    const float2 cs = a.rope[(long)a.pos * h2 + f];
    float v = normed(d);
    float o = d < h2 ? v * cs.x - normed(d + h2) * cs.y : v * cs.x + normed(d - h2) * cs.y;
    if (is_q) {
      a.q_out[row] = o;
    } else {
      const int kh = (row - q_rows) / hd;
      a.k_cache[(long)kh * a.cache_head_stride + (long)a.pos * hd + d] = f2bf(o);
    }
  } else if constexpr (EPI == GEMV_ARGMAX) {
    unsigned long long key = 0ull;
    if (row < a.n_valid) {
      a.out[row] = y;
      key = argmax_key(y, static_cast<uint32_t>(row + a.key_row0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if ((tid & 31) == 0 && key) atomicMax(a.amax, key);
  }
}


__device__ inline void gemv_epilogue_any(int epi, const GemvArgs& a, int mt, const float* red,
                                         int tid) {
  switch (epi) {
    case GEMV_F32: gemv_epilogue<GEMV_F32>(a, mt, red, tid); break;
    case GEMV_RESID: gemv_epilogue<GEMV_RESID>(a, mt, red, tid); break;
    case GEMV_SILU: gemv_epilogue<GEMV_SILU>(a, mt, red, tid); break;
    case GEMV_QKV: gemv_epilogue<GEMV_QKV>(a, mt, red, tid); break;
    default: gemv_epilogue<GEMV_ARGMAX>(a, mt, red, tid); break;
  }
}

// Consumer prologue shared by the decode GEMVs: x (fp32, optional fused
// RMSNorm) -> the (hi, lo) bf16 B-word layout in shared memory.  Contains the
// kernel's pdl_wait.  Ends without a barrier (callers sync the NC consumers).
template <int NC, int RP = kXRegPairs>
__device__ __forceinline__ void gemv_stage_x(const GemvArgs& a, uint32_t* xq, float* scratch, int K, int tid,
                                             int lane, int warp) {
  constexpr int kXRegPairs = RP;  // register pairs per thread on the one-round-trip path
  // x pairs i = tid + j * consumers live in registers between the load, the
  // RMSNorm reduction and the scatter (one global round trip after pdl_wait);
  // the norm weights do not come from the previous kernel and load before it.
  const int KP = K / 2;
  if (KP <= kXRegPairs * NC) {
    float2 xv[kXRegPairs];
    uint32_t nv[kXRegPairs];  // bf16 pairs (norm weights do not come from the previous kernel)
#pragma unroll
    for (int j = 0; j < kXRegPairs; ++j) {
      const int i = tid + j * NC;
      nv[j] = 0x3f803f80u;  // (1, 1)
      if (a.norm_w && i < KP) nv[j] = reinterpret_cast<const uint32_t*>(a.norm_w)[i];
    }
    pdl_wait();  // x, workspace and outputs belong to the previous kernel until here
#pragma unroll
    for (int j = 0; j < kXRegPairs; ++j) {
      const int i = tid + j * NC;
      xv[j] = i < KP ? reinterpret_cast<const float2*>(a.x)[i] : make_float2(0.f, 0.f);
    }
    float rstd = 1.f;
    if (a.norm_w) {  // sum of squares: per-thread pairs in j order, warps in order
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < kXRegPairs; ++j) {
        ss = fmaf(xv[j].x, xv[j].x, ss);
        ss = fmaf(xv[j].y, xv[j].y, ss);
      }
      ss = warp_sum(ss);
      if (lane == 0) scratch[warp] = ss;
      named_bar(1, NC);
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < NC / 32; ++w) tot += scratch[w];
      rstd = rsqrtf(tot / K + a.eps);
    }
#pragma unroll
    for (int j = 0; j < kXRegPairs; ++j) {
      const int i = tid + j * NC;
      if (i < KP) gemv_stage_pair(xq, i, xv[j].x * rstd * bf16_lo(nv[j]), xv[j].y * rstd * bf16_hi(nv[j]));
    }
  } else {
    pdl_wait();
    gemv_stage_x_loop(a.x, a.norm_w, a.eps, xq, scratch, K, tid, lane, warp, NC);
  }
}

// End of an m-tile: the NC consumer warps' partials (acc: rows g, g + 8 of row
// block rb, k-part kh) -> red, k-parts summed in order, then either the fused
// epilogue or the deterministic stream-K fix-up (workspace slot per
// contributing CTA, last arriver sums in contributor order).  Zeroes acc.
// red holds two [kQ][128] buffers used alternately (par flips per call): after
// the one all-consumer barrier only warps 0-3 (one thread per row) finish the
// m-tile -- fix-up and epilogue under their own barrier -- while the other
// warps go on decoding; the next call's barrier orders buffer reuse.
__device__ __forceinline__ int gemv_cta_of_tile(long t, int G, long T) {
  if (T * G < (1l << 32))  // 32-bit division when it fits (all decode shapes)
    return static_cast<int>((static_cast<uint32_t>(t + 1) * static_cast<uint32_t>(G) - 1u) /
                            static_cast<uint32_t>(T));
  return cta_of_tile(t, G, T);
}

template <int EPI, int NC, int kQ>
__device__ __forceinline__ void gemv_flush(const GemvArgs& a, float (&acc)[4], float* red_base, int& par,
                                           int* flag, int mt, int G, long T, int c, int tid, int g, int t4,
                                           int rb, int kh) {
  float* red = red_base + par * kQ * kTileRows;
  par ^= 1;
  if (t4 == 0) {
    red[kh * kTileRows + rb * 16 + g] = acc[0] + acc[1];
    red[kh * kTileRows + rb * 16 + g + 8] = acc[2] + acc[3];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = 0.f;
  named_bar(1, NC);
  if (tid >= kTileRows) return;
  float v = red[tid];
#pragma unroll
  for (int q = 1; q < kQ; ++q) v += red[q * kTileRows + tid];
  const long first = static_cast<long>(mt) * a.n_kb, last = first + a.n_kb - 1;
  const int c_first = gemv_cta_of_tile(first, G, T);
  const int n_contrib = gemv_cta_of_tile(last, G, T) - c_first + 1;
  if (n_contrib == 1) {
    red[tid] = v;
    named_bar(2, kTileRows);
    gemv_epilogue<EPI>(a, mt, red, tid);
    return;
  }
  float* mine = a.ws + (static_cast<long>(mt) * a.max_contrib + (c - c_first)) * kTileRows;
  mine[tid] = v;
  named_bar(2, kTileRows);
  if (tid == 0) {
    __threadfence();  // cumulative: orders the 128 rows' stores (via the barrier) before the count
    const int old = atomicAdd(&a.counters[mt], 1);
    *flag = (old == n_contrib - 1);
  }
  named_bar(2, kTileRows);
  if (*flag) {
    __threadfence();
    const float* base = a.ws + static_cast<long>(mt) * a.max_contrib * kTileRows;
    float s = 0.f;
    for (int j = 0; j < n_contrib; ++j) s += __ldcg(base + j * kTileRows + tid);
    red[tid] = s;
    named_bar(2, kTileRows);
    gemv_epilogue<EPI>(a, mt, red, tid);
    if (tid == 0) a.counters[mt] = 0;
  }
}

}  // namespace lsb
