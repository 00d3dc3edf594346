// elementwise.cu -- row norms, q/k-norm + RoPE + KV append for prefill,
// embeddings, the action-expert input/output heads and small glue kernels.
// All HBM-bound and tiny next to the weight streams; one CTA per row where a
// row reduction is needed, vectorised 16-byte accesses where rows allow.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace lsb {

__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// RMSNorm over rows of an fp32 [T x D] residual stream -> bf16 GEMM operand.
// Rows with D % 4 == 0 and D <= 4096 (every hidden size here): a thread holds
// its float4 groups (group v * 256 + tid) in registers -- x is read once, in
// one round trip, and the norm weights are fetched before pdl_wait.
constexpr int kNormMaxV = 4;  // float4 per thread (256 threads -> D <= 4096)

__global__ void rmsnorm_rows_kernel(const float* x, const bf16* w, bf16* out, int D, float eps) {
  pdl_trigger();
  __shared__ float sh[32];
  const float* xr = x + static_cast<long>(blockIdx.x) * D;
  bf16* o = out + static_cast<long>(blockIdx.x) * D;
  const int ng = D / 4;
  if (D % 4 == 0 && ng <= 256 * kNormMaxV) {
    uint2 wv[kNormMaxV];
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) wv[v] = reinterpret_cast<const uint2*>(w)[v * 256 + threadIdx.x];
    pdl_wait();
    float4 xv[kNormMaxV];
    float ss = 0.f;
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        xv[v] = reinterpret_cast<const float4*>(xr)[v * 256 + threadIdx.x];
        ss = fmaf(xv[v].x, xv[v].x, ss);
        ss = fmaf(xv[v].y, xv[v].y, ss);
        ss = fmaf(xv[v].z, xv[v].z, ss);
        ss = fmaf(xv[v].w, xv[v].w, ss);
      }
    const float rstd = rsqrtf(block_sum(ss, sh) / D + eps);
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        uint2 r;
        r.x = pack_bf16x2(xv[v].x * rstd * bf16_lo(wv[v].x), xv[v].y * rstd * bf16_hi(wv[v].x));
        r.y = pack_bf16x2(xv[v].z * rstd * bf16_lo(wv[v].y), xv[v].w * rstd * bf16_hi(wv[v].y));
        reinterpret_cast<uint2*>(o)[v * 256 + threadIdx.x] = r;
      }
    return;
  }
  pdl_wait();
  float ss = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  const float rstd = rsqrtf(block_sum(ss, sh) / D + eps);
  for (int i = threadIdx.x; i < D; i += blockDim.x) o[i] = f2bf(xr[i] * rstd * bf2f(w[i]));
}

cudaError_t launch_rmsnorm_rows(const float* x, const bf16* w, bf16* out, int T, int D, float eps,
                                cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_k(rmsnorm_rows_kernel, dim3(T), dim3(256), 0, st, x, w, out, D, eps);
}

__global__ void layernorm_rows_kernel(const float* x, const bf16* w, const bf16* b, bf16* out,
                                      int D, long ld_out, float eps) {
  pdl_trigger();
  __shared__ float sh[32];
  const float* xr = x + static_cast<long>(blockIdx.x) * D;
  const int ng = D / 4;
  if (D % 4 == 0 && ng <= 256 * kNormMaxV && ld_out % 4 == 0) {  // register path (see rmsnorm)
    uint2 wv[kNormMaxV], bv[kNormMaxV];
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        wv[v] = reinterpret_cast<const uint2*>(w)[v * 256 + threadIdx.x];
        bv[v] = reinterpret_cast<const uint2*>(b)[v * 256 + threadIdx.x];
      }
    pdl_wait();
    float4 xv[kNormMaxV];
    float s1 = 0.f;
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        xv[v] = reinterpret_cast<const float4*>(xr)[v * 256 + threadIdx.x];
        s1 += xv[v].x + xv[v].y + xv[v].z + xv[v].w;
      }
    const float mean = block_sum(s1, sh) / D;
    float v2 = 0.f;
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        const float d0 = xv[v].x - mean, d1 = xv[v].y - mean, d2 = xv[v].z - mean, d3 = xv[v].w - mean;
        v2 = fmaf(d0, d0, v2);
        v2 = fmaf(d1, d1, v2);
        v2 = fmaf(d2, d2, v2);
        v2 = fmaf(d3, d3, v2);
      }
    const float rstd = rsqrtf(block_sum(v2, sh) / D + eps);
    bf16* o = out + static_cast<long>(blockIdx.x) * ld_out;
#pragma unroll
    for (int v = 0; v < kNormMaxV; ++v)
      if (v * 256 + static_cast<int>(threadIdx.x) < ng) {
        uint2 r;
        r.x = pack_bf16x2((xv[v].x - mean) * rstd * bf16_lo(wv[v].x) + bf16_lo(bv[v].x),
                          (xv[v].y - mean) * rstd * bf16_hi(wv[v].x) + bf16_hi(bv[v].x));
        r.y = pack_bf16x2((xv[v].z - mean) * rstd * bf16_lo(wv[v].y) + bf16_lo(bv[v].y),
                          (xv[v].w - mean) * rstd * bf16_hi(wv[v].y) + bf16_hi(bv[v].y));
        reinterpret_cast<uint2*>(o)[v * 256 + threadIdx.x] = r;
      }
    return;
  }
  pdl_wait();
  float s = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) s += xr[i];
  const float mean = block_sum(s, sh) / D;
  float v2 = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float d = xr[i] - mean;
    v2 = fmaf(d, d, v2);
  }
  const float rstd = rsqrtf(block_sum(v2, sh) / D + eps);
  bf16* o = out + static_cast<long>(blockIdx.x) * ld_out;
  for (int i = threadIdx.x; i < D; i += blockDim.x)
    o[i] = f2bf((xr[i] - mean) * rstd * bf2f(w[i]) + bf2f(b[i]));
}

// Narrow rows (ViT: D = 1152): one warp per row, the row in registers (<= 12
// float4 per lane), shuffles only -- no block barriers, 8 rows per CTA.
constexpr int kLnWarpMaxV = 12;
__global__ void __launch_bounds__(256) layernorm_rows_warp_kernel(const float* x, const bf16* w, const bf16* b,
                                                                  bf16* out, int T, int D, long ld_out,
                                                                  float eps) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int ng = D / 4;
  uint2 wv[kLnWarpMaxV], bv[kLnWarpMaxV];
#pragma unroll
  for (int v = 0; v < kLnWarpMaxV; ++v)
    if (v * 32 + lane < ng) {
      wv[v] = reinterpret_cast<const uint2*>(w)[v * 32 + lane];
      bv[v] = reinterpret_cast<const uint2*>(b)[v * 32 + lane];
    }
  pdl_wait();
  if (row >= T) return;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long>(row) * D);
  float4 xv[kLnWarpMaxV];
  float s1 = 0.f;
#pragma unroll
  for (int v = 0; v < kLnWarpMaxV; ++v)
    if (v * 32 + lane < ng) {
      xv[v] = xr[v * 32 + lane];
      s1 += xv[v].x + xv[v].y + xv[v].z + xv[v].w;
    }
  const float mean = warp_sum(s1) / D;
  float v2 = 0.f;
#pragma unroll
  for (int v = 0; v < kLnWarpMaxV; ++v)
    if (v * 32 + lane < ng) {
      const float d0 = xv[v].x - mean, d1 = xv[v].y - mean, d2 = xv[v].z - mean, d3 = xv[v].w - mean;
      v2 = fmaf(d0, d0, v2);
      v2 = fmaf(d1, d1, v2);
      v2 = fmaf(d2, d2, v2);
      v2 = fmaf(d3, d3, v2);
    }
  const float rstd = rsqrtf(warp_sum(v2) / D + eps);
  uint2* o = reinterpret_cast<uint2*>(out + static_cast<long>(row) * ld_out);
#pragma unroll
  for (int v = 0; v < kLnWarpMaxV; ++v)
    if (v * 32 + lane < ng) {
      uint2 r;
      r.x = pack_bf16x2((xv[v].x - mean) * rstd * bf16_lo(wv[v].x) + bf16_lo(bv[v].x),
                        (xv[v].y - mean) * rstd * bf16_hi(wv[v].x) + bf16_hi(bv[v].x));
      r.y = pack_bf16x2((xv[v].z - mean) * rstd * bf16_lo(wv[v].y) + bf16_lo(bv[v].y),
                        (xv[v].w - mean) * rstd * bf16_hi(wv[v].y) + bf16_hi(bv[v].y));
      o[v * 32 + lane] = r;
    }
}

cudaError_t launch_layernorm_rows(const float* x, const bf16* w, const bf16* b, bf16* out, int T,
                                  int D, long ld_out, float eps, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (D % 4 == 0 && D / 4 <= 32 * kLnWarpMaxV && ld_out % 4 == 0)
    return launch_k(layernorm_rows_warp_kernel, dim3((T + 7) / 8), dim3(256), 0, st, x, w, b, out, T, D, ld_out,
                    eps);
  return launch_k(layernorm_rows_kernel, dim3(T), dim3(256), 0, st, x, w, b, out, D, ld_out, eps);
}

// Prefill q/k RMSNorm + RoPE; K,V appended to the cache at positions pos0+t.
// One CTA per token, one warp per head.
__global__ void qk_norm_rope_kernel(const bf16* qkv, int hq, int hkv, int hd, const bf16* qn_w,
                                    const bf16* kn_w, float eps, const float2* rope, int pos0,
                                    bf16* q_out, bf16* k_cache, bf16* v_cache,
                                    int cache_head_stride) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = hq + 2 * hkv;
  const int row_len = nh * hd;
  const int pos = pos0 + t;
  const int h2 = hd / 2;
  for (int head = warp; head < nh; head += blockDim.x >> 5) {
    const bf16* src = qkv + static_cast<long>(t) * row_len + head * hd;
    const bool is_q = head < hq, is_k = !is_q && head < hq + hkv;
    if (!is_q && !is_k) {
      const int vh = head - hq - hkv;
      bf16* dst = v_cache + static_cast<long>(vh) * cache_head_stride + static_cast<long>(pos) * hd;
      for (int d = lane; d < hd; d += 32) dst[d] = src[d];
      continue;
    }
    float ss = 0.f;
    for (int d = lane; d < hd; d += 32) {
      const float v = bf2f(src[d]);
      ss = fmaf(v, v, ss);
    }
    const bf16* nw = is_q ? qn_w : kn_w;
    const float rstd = nw ? rsqrtf(warp_sum(ss) / hd + eps) : 1.0f;
    auto normed = [&](int d) {
      const float v = bf2f(src[d]) * rstd;
      return nw ? v * bf2f(nw[d]) : v;
    };
    bf16* dst = is_q ? q_out + (static_cast<long>(t) * hq + head) * hd
                     : k_cache + static_cast<long>(head - hq) * cache_head_stride +
                           static_cast<long>(pos) * hd;
    for (int d = lane; d < hd; d += 32) {
      const int f = d < h2 ? d : d - h2;
      const float2 cs = rope[static_cast<long>(pos) * h2 + f];
      const float v = normed(d);
      const float o = d < h2 ? v * cs.x - normed(d + h2) * cs.y : v * cs.x + normed(d - h2) * cs.y;
      dst[d] = f2bf(o);
    }
  }
}

// Head dim 128: lane l holds dims 2l, 2l+1 and 64+2l, 64+2l+1 -- the RoPE pairs
// (d, d + 64) never leave the lane -- and a warp issues every load of its heads
// (x, norm weights, cos/sin; the tables before pdl_wait) before computing.
constexpr int kQkMaxHeadsPerWarp = 8;

__global__ void qk_norm_rope128_kernel(const bf16* qkv, int hq, int hkv, const bf16* qn_w,
                                       const bf16* kn_w, float eps, const float2* rope, int pos0,
                                       bf16* q_out, bf16* k_cache, bf16* v_cache, int cache_head_stride) {
  constexpr int hd = 128;
  pdl_trigger();
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nh = hq + 2 * hkv;
  const int pos = pos0 + t;
  const float4 cs = reinterpret_cast<const float4*>(rope + static_cast<long>(pos) * (hd / 2))[lane];
  uint32_t wq[2] = {0x3f803f80u, 0x3f803f80u}, wk[2] = {0x3f803f80u, 0x3f803f80u};  // bf16 1.0
  if (qn_w) { wq[0] = reinterpret_cast<const uint32_t*>(qn_w)[lane]; wq[1] = reinterpret_cast<const uint32_t*>(qn_w)[32 + lane]; }
  if (kn_w) { wk[0] = reinterpret_cast<const uint32_t*>(kn_w)[lane]; wk[1] = reinterpret_cast<const uint32_t*>(kn_w)[32 + lane]; }
  pdl_wait();
  const uint32_t* row = reinterpret_cast<const uint32_t*>(qkv + static_cast<long>(t) * nh * hd);
  uint32_t xa[kQkMaxHeadsPerWarp], xb[kQkMaxHeadsPerWarp];
#pragma unroll
  for (int i = 0; i < kQkMaxHeadsPerWarp; ++i) {
    const int head = warp + i * nw;
    if (head < nh) {
      xa[i] = row[head * (hd / 2) + lane];
      xb[i] = row[head * (hd / 2) + 32 + lane];
    }
  }
#pragma unroll
  for (int i = 0; i < kQkMaxHeadsPerWarp; ++i) {
    const int head = warp + i * nw;
    if (head >= nh) break;
    uint32_t* dst;
    if (head >= hq + hkv) {  // V: straight into the cache
      dst = reinterpret_cast<uint32_t*>(v_cache + static_cast<long>(head - hq - hkv) * cache_head_stride +
                                        static_cast<long>(pos) * hd);
      dst[lane] = xa[i];
      dst[32 + lane] = xb[i];
      continue;
    }
    const bool is_q = head < hq;
    const bf16* nwp = is_q ? qn_w : kn_w;
    const uint2 o = qk_norm_rope128_lane(xa[i], xb[i], nwp != nullptr, is_q ? wq[0] : wk[0],
                                         is_q ? wq[1] : wk[1], cs, eps);
    dst = is_q ? reinterpret_cast<uint32_t*>(q_out + (static_cast<long>(t) * hq + head) * hd)
               : reinterpret_cast<uint32_t*>(k_cache + static_cast<long>(head - hq) * cache_head_stride +
                                             static_cast<long>(pos) * hd);
    dst[lane] = o.x;
    dst[32 + lane] = o.y;
  }
}

cudaError_t launch_qk_norm_rope(const bf16* qkv, int T, int hq, int hkv, int hd, const bf16* qn_w,
                                const bf16* kn_w, float eps, const float2* rope, int pos0,
                                bf16* q_out, bf16* k_cache, bf16* v_cache, int cache_head_stride,
                                cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (hd == 128 && hq + 2 * hkv <= 8 * kQkMaxHeadsPerWarp)
    return launch_k(qk_norm_rope128_kernel, dim3(T), dim3(256), 0, st, qkv, hq, hkv, qn_w, kn_w, eps, rope,
                    pos0, q_out, k_cache, v_cache, cache_head_stride);
  return launch_k(qk_norm_rope_kernel, dim3(T), dim3(256), 0, st, qkv, hq, hkv, hd, qn_w, kn_w, eps, rope, pos0, q_out,
                                         k_cache, v_cache, cache_head_stride);
}

__global__ void embed_rows_kernel(const bf16* table, const int* ids, int D, float* out, long ld) {
  pdl_trigger();
  pdl_wait();
  const int id = ids[blockIdx.x];
  const bf16* src = table + static_cast<long>(id) * D;
  float* dst = out + static_cast<long>(blockIdx.x) * ld;
  for (int i = threadIdx.x; i < D; i += blockDim.x) dst[i] = bf2f(src[i]);
}

cudaError_t launch_embed_rows(const bf16* table, const int* ids, int n, int D, float* out,
                              long ld_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(embed_rows_kernel, dim3(n), dim3(256), 0, st, table, ids, D, out, ld_out);
}

// x[t, :] += add[t % period, :]   (learned ViT position embedding per image)
__global__ void add_rows_kernel(float* x, const bf16* add, int D, int period) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const bf16* a = add + static_cast<long>(t % period) * D;
  float* xr = x + static_cast<long>(t) * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) xr[i] += bf2f(a[i]);
}

cudaError_t launch_add_rows_bf16(float* x, const bf16* add, int T, int D, long period,
                                 cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_k(add_rows_kernel, dim3(T), dim3(256), 0, st, x, add, D, static_cast<int>(period));
}

__global__ void cast_kernel(const float* x, bf16* out, long n) {
  pdl_trigger();
  pdl_wait();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    out[i] = f2bf(x[i]);
}

cudaError_t launch_cast_f32_bf16(const float* x, bf16* out, long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(cast_kernel, dim3(296), dim3(256), 0, st, x, out, n);
}

// Greedy decode bookkeeping: key -> token id (+ history), re-arm the key.
__global__ void argmax_to_token_kernel(const unsigned long long* key, int* token_out, int* history,
                                       int step, unsigned long long* key_reset) {
  pdl_trigger();
  pdl_wait();
  const unsigned long long k = *key;
  const int idx = static_cast<int>(0xffffffffu - static_cast<uint32_t>(k & 0xffffffffull));
  *token_out = idx;
  if (history) history[step] = idx;
  if (key_reset) *key_reset = 0ull;
}

cudaError_t launch_argmax_to_token(const unsigned long long* key, int* token_out, int* history,
                                   int step, unsigned long long* key_reset, cudaStream_t st) {
  return launch_k(argmax_to_token_kernel, dim3(1), dim3(1), 0, st, key, token_out, history, step, key_reset);
}

__global__ void fill_u64_kernel(unsigned long long* p, unsigned long long v, int n) {
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

cudaError_t launch_fill_u64(unsigned long long* p, unsigned long long v, int n, cudaStream_t st) {
  return launch_k(fill_u64_kernel, dim3(1), dim3(128), 0, st, p, v, n);
}

// Sinusoidal flow-time features: out[i] = sin(t * f_i) | cos(t * f_i), f_i = 1e4^(-i/(dim/2)).
__global__ void time_embed_kernel(const float* t_table, int step, int dim, float* out) {
  pdl_trigger();
  pdl_wait();
  const float t = t_table[step];
  const int half = dim / 2;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float f = expf(-9.210340371976184f * i / half);  // ln(1e4)
    out[i] = sinf(t * f);
    out[half + i] = cosf(t * f);
  }
}

cudaError_t launch_time_embed(const float* t_table, int step, int dim, float* out, cudaStream_t st) {
  return launch_k(time_embed_kernel, dim3(1), dim3(128), 0, st, t_table, step, dim, out);
}

// Action-token input: h[i, :] = W_in . a_i + b_in + temb   (K = action dim, tiny).
__global__ void action_in_kernel(const float* actions, const bf16* w_in, const bf16* b_in,
                                 const float* temb, int a_dim, int D, float* out) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float s = bf2f(b_in[d]) + temb[d];
    for (int k = 0; k < a_dim; ++k) s = fmaf(bf2f(w_in[d * a_dim + k]), actions[i * a_dim + k], s);
    out[static_cast<long>(i) * D + d] = s;
  }
}

cudaError_t launch_action_in(const float* actions, const bf16* w_in, const bf16* b_in,
                             const float* temb, int n_tok, int a_dim, int D, float* out,
                             cudaStream_t st) {
  return launch_k(action_in_kernel, dim3(n_tok), dim3(256), 0, st, actions, w_in, b_in, temb, a_dim, D, out);
}

// Final RMSNorm + velocity head (D -> a_dim) + explicit Euler step a += dt * v.
__global__ void action_out_euler_kernel(const float* h, const bf16* norm_w, float eps,
                                        const bf16* w_out, const bf16* b_out, int D, int a_dim,
                                        float dt, float* actions, float* velocity) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sh[32];
  __shared__ float part[8][8];
  const int i = blockIdx.x;
  const float* hr = h + static_cast<long>(i) * D;
  float ss = 0.f;
  for (int d = threadIdx.x; d < D; d += blockDim.x) ss = fmaf(hr[d], hr[d], ss);
  const float rstd = rsqrtf(block_sum(ss, sh) / D + eps);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < a_dim; ++k) {
    float s = 0.f;
    for (int d = threadIdx.x; d < D; d += blockDim.x)
      s = fmaf(hr[d] * rstd * bf2f(norm_w[d]), bf2f(w_out[k * D + d]), s);
    s = warp_sum(s);
    if (lane == 0) part[k][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < a_dim) {
    const int k = threadIdx.x;
    float v = bf2f(b_out[k]);
    for (int w = 0; w < (blockDim.x >> 5); ++w) v += part[k][w];
    if (velocity) velocity[i * a_dim + k] = v;
    actions[i * a_dim + k] += dt * v;
  }
}

cudaError_t launch_action_out_euler(const float* h, const bf16* norm_w, float eps,
                                    const bf16* w_out, const bf16* b_out, int n_tok, int D,
                                    int a_dim, float dt, float* actions, float* velocity,
                                    cudaStream_t st) {
  if (a_dim > 8) return cudaErrorInvalidValue;
  return launch_k(action_out_euler_kernel, dim3(n_tok), dim3(256), 0, st, h, norm_w, eps, w_out, b_out, D, a_dim, dt,
                                                 actions, velocity);
}

// SiLU in place (time-MLP hidden).
__global__ void silu_kernel(float* x, int n) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = silu(x[i]);
}

cudaError_t launch_silu_inplace(float* x, int n, cudaStream_t st) {
  return launch_k(silu_kernel, dim3((n + 255) / 256), dim3(256), 0, st, x, n);
}

// x += y (tensor-parallel partial sums after the all-reduce), float4 vectorised.
__global__ void add_f32_kernel(float* __restrict__ x, const float* __restrict__ y, long n) {
  pdl_trigger();
  pdl_wait();
  const long n4 = n / 4;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(x)[i];
    const float4 b = reinterpret_cast<const float4*>(y)[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    reinterpret_cast<float4*>(x)[i] = a;
  }
  for (long i = 4 * n4 + blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    x[i] += y[i];
}

cudaError_t launch_add_f32(float* x, const float* y, long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long blocks = std::min<long>((n / 4 + 255) / 256 + 1, 1184);
  return launch_k(add_f32_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, x, y, n);
}

}  // namespace lsb
