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
      key = argmax_key(y, static_cast<uint32_t>(row));
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

}  // namespace lsb
