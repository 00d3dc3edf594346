// attention.cu -- GQA attention kernels.
//
// decode_attention: one query token per head against the bf16 KV cache
//   (flash-decoding split over the context; per-split partials combined by
//   the last-arriving CTA in split order -> deterministic).  HBM-bound on the
//   KV bytes: hkv * n_ctx * hd * 2 (K,V) * 2 B per launch.
// flash_attention: many queries (LM prefill, ViT, action expert) with
//   bf16 mma.sync m16n8k16 tiles, online softmax in fp32, causal /
//   block-diagonal (per image) / two-segment KV (expert: VLM cache + own).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace lsb {

// ------------------------------- decode ---------------------------------------
//
// grid (hkv, n_split) launched as clusters of n_split CTAs (<= 16) along y, kDecThreads
// threads.  Each CTA owns <= kDecChunk consecutive positions of one KV head:
// its K and V rows are contiguous in the cache, so two 1-D bulk copies (TMA
// engine) land them in shared memory with one mbarrier wait.  Scores: one
// thread per (query head, position) dot product, K rows read with a per-lane
// rotation (conflict-free); softmax per head by one warp; P.V: one thread per
// (head, dim pair).  The split partials (max, sum, O) never leave the chip:
// after a cluster barrier CTA z merges a 1/n_split slice of the G x HD outputs
// reading every peer's partial over DSMEM, in split order (deterministic).

constexpr int kDecChunk = 128;
constexpr int kDecThreads = 256;  // 2 scores / 1 output pair per thread per head group
constexpr int kDecMaxSplits = 16;

// rows of the K / V / score buffers a CTA lays out: its share of the positions
// rounded up to 8 (the launch reserves kDecChunk)
__host__ __device__ inline int dec_cap(int n_ctx, int n_split) {
  return ((n_ctx + n_split - 1) / n_split + 7) & ~7;
}

template <int HD, int G>
__global__ void __launch_bounds__(kDecThreads) decode_attn_kernel(const DecodeAttnArgs a) {
  namespace cg = cooperative_groups;
  constexpr int HP = HD / 2;  // bf16 pairs per row
  extern __shared__ __align__(16) uint8_t dsm[];
  // cap: positions per split rounded up to 8 (shared memory sized to the launch,
  // so the CTA fits beside a GEMV CTA on the same SM)
  const int cap = dec_cap(a.n_ctx, a.n_split);
  bf16* ks = reinterpret_cast<bf16*>(dsm);
  bf16* vs = ks + cap * HD;
  float* qs = reinterpret_cast<float*>(vs + cap * HD);  // [G][HD], pre-scaled
  float* ps = qs + G * HD;                              // [G][cap] scores -> probs
  float* recv_o = ps + G * cap;                         // [S][slice] partial O pushed by every split
  float* recv_ml = recv_o + G * HD + kDecMaxSplits;  // [S][2G] partial (max, sum) per head
  __shared__ __align__(8) uint64_t bar;
  __shared__ float sm_ml[2 * G];                               // partial max (log2), sum
  pdl_trigger();
  const int kh = blockIdx.x, split = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // peers may write our shared memory only once we run: announce it now, wait
  // for everyone's announcement right before the first remote store
  if (a.n_split > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int chunk = (a.n_ctx + a.n_split - 1) / a.n_split;
  const int p0 = split * chunk, p1 = min(a.n_ctx, p0 + chunk);
  const int np = max(p1 - p0, 0);
  // positions < n_ctx - 1 were cached by earlier steps: their bulk copies go out
  // before griddepcontrol.wait; only the newest position (appended by the QKV
  // GEMV this kernel follows) waits for it
  const int n_old = max(min(p1, a.n_ctx - 1) - p0, 0);
  const long off = static_cast<long>(kh) * a.cache_head_stride + static_cast<long>(p0) * HD;
  if (threadIdx.x == 0 && np > 0) {
    mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(2 * np * HD * 2));
    if (n_old > 0) {
      const uint32_t bytes = static_cast<uint32_t>(n_old * HD * 2);
      bulk_g2s(ks, a.k_cache + off, bytes, &bar);
      bulk_g2s(vs, a.v_cache + off, bytes, &bar);
    }
  }
  pdl_wait();
  if (threadIdx.x == 0 && np > n_old) {
    const uint32_t bytes = static_cast<uint32_t>((np - n_old) * HD * 2);
    const long o2 = off + static_cast<long>(n_old) * HD;
    bulk_g2s(ks + n_old * HD, a.k_cache + o2, bytes, &bar);
    bulk_g2s(vs + n_old * HD, a.v_cache + o2, bytes, &bar);
  }
  const float sl2 = a.scale * 1.4426950408889634f;
  for (int i = threadIdx.x; i < G * HD; i += kDecThreads) qs[i] = a.q[kh * G * HD + i] * sl2;
  __syncthreads();
  if (np > 0) mbar_wait(&bar, 0);
  // ---- scores (log2 domain) ----
  for (int idx = threadIdx.x; idx < G * cap; idx += kDecThreads) {
    const int g = idx / cap, p = idx % cap;
    float sc = -INFINITY;
    if (p < np) {
      const uint32_t* kr = reinterpret_cast<const uint32_t*>(ks + p * HD);
      const float2* qg = reinterpret_cast<const float2*>(qs + g * HD);
      float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
      for (int j = 0; j < HP; ++j) {
        const int jj = (j + p) & (HP - 1);  // rotate: lanes hit distinct banks
        const uint32_t kv = kr[jj];
        const float2 qv = qg[jj];
        s0 = fmaf(bf16_lo(kv), qv.x, s0);
        s1 = fmaf(bf16_hi(kv), qv.y, s1);
      }
      sc = s0 + s1;
    }
    ps[idx] = sc;
  }
  __syncthreads();
  // ---- softmax per head: warp g (strided) ----
  for (int g = warp; g < G; g += kDecThreads / 32) {
    float mx = -INFINITY;
    for (int p = lane; p < cap; p += 32) mx = fmaxf(mx, ps[g * cap + p]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int p = lane; p < cap; p += 32) {
      const float v = ps[g * cap + p];
      const float e = v == -INFINITY ? 0.f : exp2f(v - mx);
      ps[g * cap + p] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    if (lane == 0) {
      sm_ml[g] = mx;
      sm_ml[G + g] = sum;
    }
  }
  __syncthreads();
  // ---- O = P V: one thread per (head, dim pair); partials pushed to their owners ----
  namespace cg = cooperative_groups;
  const int S = a.n_split;
  constexpr int GHD = G * HD;
  const int SL = (GHD + S - 1) / S;  // slice length owned by each split CTA (>=)
  auto owner = [&](int i) { return (i * S + S - 1) / GHD; };
  if (S > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (S > 1 && threadIdx.x < S) {  // (max, sum) of every head -> CTA threadIdx.x
    cg::cluster_group cluster = cg::this_cluster();
    float* dst = cluster.map_shared_rank(recv_ml, static_cast<int>(threadIdx.x)) + split * 2 * G;
#pragma unroll
    for (int g = 0; g < 2 * G; ++g) dst[g] = sm_ml[g];
  }
  for (int idx = threadIdx.x; idx < G * HP; idx += kDecThreads) {
    const int g = idx / HP, dp = idx % HP;
    const uint32_t* vc = reinterpret_cast<const uint32_t*>(vs) + dp;
    const float* pg = ps + g * cap;
    float o0 = 0.f, o1 = 0.f;
#pragma unroll 8
    for (int p = 0; p < np; ++p) {
      const uint32_t v = vc[p * HP];
      const float w = pg[p];
      o0 = fmaf(w, bf16_lo(v), o0);
      o1 = fmaf(w, bf16_hi(v), o1);
    }
    if (a.n_split == 1) {
      const float l = sm_ml[G + g], inv = l > 0.f ? 1.0f / l : 0.f;
      a.out[(kh * G + g) * HD + 2 * dp] = o0 * inv;
      a.out[(kh * G + g) * HD + 2 * dp + 1] = o1 * inv;
    } else {  // push to the CTA owning outputs i, i+1 (remote DSMEM stores)
      cg::cluster_group cluster = cg::this_cluster();
      const int i0 = g * HD + 2 * dp;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + u, r = owner(i);
        cluster.map_shared_rank(recv_o, r)[split * SL + (i - r * GHD / S)] = u ? o1 : o0;
      }
    }
  }
  if (S == 1) return;
  // ---- one cluster barrier, then every CTA merges its own slice from local smem ----
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const int lo = split * GHD / S, hi = (split + 1) * GHD / S;
  for (int i = lo + threadIdx.x; i < hi; i += kDecThreads) {
    const int g = i / HD;
    float M = -INFINITY;
    for (int z = 0; z < S; ++z) M = fmaxf(M, recv_ml[z * 2 * G + g]);
    float L = 0.f, O = 0.f;
    for (int z = 0; z < S; ++z) {
      const float mz = recv_ml[z * 2 * G + g];
      if (mz == -INFINITY) continue;
      const float f = exp2f(mz - M);
      L = fmaf(recv_ml[z * 2 * G + G + g], f, L);
      O = fmaf(recv_o[z * SL + (i - lo)], f, O);
    }
    a.out[kh * GHD + i] = L > 0.f ? O / L : 0.f;
  }
}

int decode_attn_max_ctx() { return kDecMaxSplits * kDecChunk; }

int decode_attn_splits(int n_ctx) {
  // >= 64 positions per split, <= kDecChunk: measured in context (the PDL chain
  // QKV GEMV -> attention -> O GEMV) at ctx 1045, 16 x 66 positions beat 9 x 117
  // by 1.4 ms per inference (isolated, 9 splits is faster: 7.9 vs 9.7 us)
  int s = (n_ctx + 63) / 64;
  const int smin = (n_ctx + kDecChunk - 1) / kDecChunk;
  if (s > kDecMaxSplits) s = kDecMaxSplits;
  if (s < smin) s = smin;
  return s < 1 ? 1 : s;
}

template <int HD, int G>
static cudaError_t decode_launch(const DecodeAttnArgs& a, cudaStream_t st) {
  const auto bytes = [](int cap) {
    return 2ull * cap * HD * 2 + 4ull * (G * (HD + cap) + G * HD + kDecMaxSplits + kDecMaxSplits * 2 * G);
  };
  // shared memory for the full kDecChunk rows whatever the split's share: smaller
  // CTAs pack more of a cluster onto one SM (sized to ~67 positions, 42 KiB:
  // +2.7 ms per inference; 112 rows, which fits beside a 3-slot QKV / O GEMV
  // CTA: +0.26 ms)
  const size_t smem = bytes(kDecChunk);
  static DeviceFlags attr;
  if (!attr.done()) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes(kDecChunk)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(decode_attn_kernel<HD, G>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(decode_attn_kernel<HD, G>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr.mark();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.hkv, a.n_split);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = take_launch_pdl() ? 1 : 0;
  la[1].id = cudaLaunchAttributeClusterDimension;
  la[1].val.clusterDim.x = 1;
  la[1].val.clusterDim.y = static_cast<unsigned>(a.n_split);
  la[1].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = a.n_split > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, decode_attn_kernel<HD, G>, a);
}

template <int HD>
static cudaError_t decode_hd(const DecodeAttnArgs& a, cudaStream_t st) {
  if (a.n_split < 1 || a.n_split > kDecMaxSplits || (a.n_ctx + a.n_split - 1) / a.n_split > kDecChunk)
    return cudaErrorInvalidValue;
  switch (a.hq / a.hkv) {
    case 1: return decode_launch<HD, 1>(a, st);
    case 2: return decode_launch<HD, 2>(a, st);
    case 4: return decode_launch<HD, 4>(a, st);
    case 8: return decode_launch<HD, 8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_decode_attention(const DecodeAttnArgs& a, cudaStream_t st) {
  switch (a.hd) {
    case 32: return decode_hd<32>(a, st);
    case 64: return decode_hd<64>(a, st);
    case 128: return decode_hd<128>(a, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------- flash ----------------------------------------

constexpr int kMaxKvSplits = 8;  // split-KV CTAs form one (portable-size) cluster

template <int HD>
struct FlashCfg {
  static constexpr int kDK = (HD + 15) / 16 * 16;  // QK^T contraction, padded to k16
  static constexpr int kLd = kDK + 8;              // smem row pitch (bank spread)
  static constexpr int kND = HD / 8;               // PV n-tiles of 8
  static constexpr int kBM = 64, kBN = 64;
};

// G > 1 (GQA packing): one CTA = G query heads of one KV head, 4 warps per head,
// so each K/V block is loaded once for all G heads.  NS: K/V block stages in
// flight (2 = double buffering; the split-KV expert launch, one CTA per SM with a
// few blocks each, keeps NS - 1 blocks ahead so L2/HBM latency is not exposed
// per block).
//
// KG = 2 (key groups): a second set of 4 G warps takes every other key block of
// the same queries (own running max / sum / O, merged in group order at the end),
// halving the per-warp chain -- the split-KV expert launch has one CTA per SM and
// only a few blocks per CTA, so its latency, not its math, is the cost.
template <int HD, int G = 1, int NS = 2, int KG = 1>
__global__ void __launch_bounds__(128 * G * KG) flash_kernel(const FlashArgs a) {
  static_assert(NS % KG == 0, "whole rounds of KG blocks per stage group");
  using Cfg = FlashCfg<HD>;
  constexpr int NT = 128 * G * KG;
  constexpr int NR = NS / KG;  // rounds of KG blocks in flight
  constexpr int DK = Cfg::kDK, LD = Cfg::kLd, ND = Cfg::kND, BM = Cfg::kBM, BN = Cfg::kBN;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  extern __shared__ __align__(16) uint8_t fsm[];
  bf16* qs = reinterpret_cast<bf16*>(fsm);
  bf16* ks_buf = qs + G * BM * LD;      // [NS][BN][LD]: K and V block stages
  bf16* vs_buf = ks_buf + NS * BN * LD;
  pdl_trigger();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kg = warp / (4 * G);                     // key group
  const int hw = (warp >> 2) % G, wr = warp & 3;      // head of this warp within the CTA, row block
  const int h = static_cast<int>(blockIdx.y) * G + hw, kvh = static_cast<int>(blockIdx.y) * G / (a.hq / a.hkv);
  const int q0 = blockIdx.x * BM;
  const int g = lane >> 2, t4 = lane & 3;
  const float sl2 = a.scale * 1.4426950408889634f;

  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int qi[2] = {q0 + wr * 16 + g, q0 + wr * 16 + g + 8};

  const int n_keys = a.len1 + a.len2;
  int k_begin = 0, k_end = n_keys;
  if (a.seg_len > 0) {
    const int img = q0 / a.seg_len;
    k_begin = img * a.seg_len;
    k_end = min(n_keys, k_begin + a.seg_len);
  }
  if (a.causal) k_end = min(k_end, q0 + BM + a.q_offset);
  const int splits = a.kv_splits > 1 ? a.kv_splits : 1;
  if (splits > 1) {  // this CTA's contiguous share of the key blocks
    const int nblk = (k_end - k_begin + BN - 1) / BN;
    const int per = (nblk + splits - 1) / splits;
    const int b0 = k_begin + static_cast<int>(blockIdx.z) * per * BN;
    k_end = min(k_end, b0 + per * BN);
    k_begin = b0;
  }

  // K/V block loader: cp.async 16-byte chunks (zero-filled past the end), one
  // commit group per block, so block j+1 streams in while block j is computed.
  // A thread always copies chunk column c of rows r0, r0 + 128 / (DK / 8), ...:
  // its per-segment base pointers are fixed, a row costs one multiply-add.
  constexpr int CPR = DK / 8;          // 16-byte chunks per (padded) row
  constexpr int RSTEP = NT / CPR;      // rows between a thread's chunks
  const int lc = threadIdx.x % CPR, lr0 = threadIdx.x / CPR;
  const bool col_ok = lc < CH;
  const long hoff1 = static_cast<long>(kvh) * a.k1_head_stride + lc * 8;
  const long hoff2 = static_cast<long>(kvh) * a.k2_head_stride + lc * 8;
  auto load_row = [&](bf16* kd, bf16* vd, int j, bool ok) {
    const bf16 *kp = a.k1, *vp = a.v1;
    if (ok) {
      const long off = j < a.len1 ? hoff1 + static_cast<long>(j) * a.k1_tok_stride
                                  : hoff2 + static_cast<long>(j - a.len1) * a.k2_tok_stride;
      kp = (j < a.len1 ? a.k1 : a.k2) + off;
      vp = (j < a.len1 ? a.v1 : a.v2) + off;
    }
    cp_async16(kd, kp, ok);
    cp_async16(vd, vp, ok);
  };
  auto load_kv_nocommit = [&](int buf, int j0) {
    bf16* kb = ks_buf + buf * BN * LD;
    bf16* vb = vs_buf + buf * BN * LD;
    if constexpr (NT % CPR == 0) {
#pragma unroll
      for (int r = lr0; r < BN; r += RSTEP)
        load_row(kb + r * LD + lc * 8, vb + r * LD + lc * 8, j0 + r, col_ok && j0 + r < k_end);
    } else {  // chunk count per row does not divide the CTA (head dim 72)
      for (int i = threadIdx.x; i < BN * CPR; i += NT) {
        const int r = i / CPR, c = i % CPR, j = j0 + r;
        const long hc = (c - lc) * 8;  // load_row's bases are for column lc
        bf16* kd = kb + r * LD + c * 8;
        bf16* vd = vb + r * LD + c * 8;
        const bool ok = c < CH && j < k_end;
        const bf16 *kp = a.k1, *vp = a.v1;
        if (ok) {
          const long off = (j < a.len1 ? hoff1 + static_cast<long>(j) * a.k1_tok_stride
                                       : hoff2 + static_cast<long>(j - a.len1) * a.k2_tok_stride) + hc;
          kp = (j < a.len1 ? a.k1 : a.k2) + off;
          vp = (j < a.len1 ? a.v1 : a.v2) + off;
        }
        cp_async16(kd, kp, ok);
        cp_async16(vd, vp, ok);
      }
    }
  };
  // ldmatrix source row / column of this lane for K^T fragments: matrices
  // 0..3 = dims +0, +8, +16, +24 of a k-step pair, rows = the 8 keys of n-tile
  const int kl_row = lane & 7, kl_col = (lane >> 3) * 8;
  const int q_lo = q0 + a.q_offset;  // smallest query position of the tile (causal)
  // the first K/V block is requested before griddepcontrol.wait when it lies in
  // a segment the previous kernel did not write (the expert over the VLM cache)
  // the first NS - 1 blocks are requested before griddepcontrol.wait when they lie
  // in a segment the previous kernel did not write (the expert over the VLM cache)
  const int nblk = k_begin < k_end ? (k_end - k_begin + BN - 1) / BN : 0;
  // round r = blocks r KG .. r KG + KG - 1 (block jb in stage jb % NS), one
  // cp.async group per round; NR - 1 rounds are requested ahead
  auto issue_round = [&](int r) {
#pragma unroll
    for (int i = 0; i < KG; ++i) {
      const int jb = r * KG + i;
      if (jb < nblk) load_kv_nocommit(jb % NS, k_begin + jb * BN);
    }
    cp_async_commit();
  };
  int issued = 0;  // rounds
  while (issued < NR - 1 && issued * KG < nblk && a.k1_ready &&
         k_begin + min(nblk, (issued + 1) * KG) * BN <= a.len1) {
    issue_round(issued);
    ++issued;
  }
  pdl_wait();
  // ---- Q tile -> smem (zero padded), after griddepcontrol.wait ----
  for (int i = threadIdx.x; i < G * BM * (DK / 8); i += NT) {
    const int hh = i / (BM * (DK / 8)), rc = i % (BM * (DK / 8));
    const int r = rc / (DK / 8), c = rc % (DK / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (q0 + r < a.Tq && c < CH)
      v = *reinterpret_cast<const uint4*>(a.q + static_cast<long>(q0 + r) * a.q_tok_stride +
                                          static_cast<long>(blockIdx.y * G + hh) * a.q_head_stride + c * 8);
    *reinterpret_cast<uint4*>(qs + (hh * BM + r) * LD + c * 8) = v;
  }
  __syncthreads();
  uint32_t qf[DK / 16][4];
  {
    const bf16* qr = qs + (hw * BM + wr * 16) * LD;
#pragma unroll
    for (int kk = 0; kk < DK / 16; ++kk) {
      qf[kk][0] = *reinterpret_cast<const uint32_t*>(qr + g * LD + kk * 16 + 2 * t4);
      qf[kk][1] = *reinterpret_cast<const uint32_t*>(qr + (g + 8) * LD + kk * 16 + 2 * t4);
      qf[kk][2] = *reinterpret_cast<const uint32_t*>(qr + g * LD + kk * 16 + 8 + 2 * t4);
      qf[kk][3] = *reinterpret_cast<const uint32_t*>(qr + (g + 8) * LD + kk * 16 + 8 + 2 * t4);
    }
  }
  float o[ND][4];
#pragma unroll
  for (int j = 0; j < ND; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  for (; issued < NR - 1; ++issued) issue_round(issued);  // (empty groups keep the count uniform)
  for (int r = 0; r * KG < nblk; ++r) {
    // round r + NR - 1 into the stages round r - 1 used (freed by the loop's final barrier)
    issue_round(r + NR - 1);
    cp_async_wait<NR - 1>();  // round r has landed
    __syncthreads();
    const int jb = r * KG + kg;
    if (jb >= nblk) {  // this group has no block in the last round
      __syncthreads();
      continue;
    }
    const int j0 = k_begin + jb * BN;
    const bf16* ks = ks_buf + (jb % NS) * BN * LD;
    const bf16* vs = vs_buf + (jb % NS) * BN * LD;
    // S = Q K^T  (16 x 64 per warp); K^T fragments by ldmatrix (two k-steps per x4)
    float s[BN / 8][4];
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
      const bf16* kr = ks + (nt * 8 + kl_row) * LD + kl_col;
#pragma unroll
      for (int kk = 0; kk + 1 < DK / 16; kk += 2) {
        uint32_t b[4];
        ldsm_x4(b, kr + kk * 16);
        mma_bf16_16816(s[nt], qf[kk], b[0], b[1]);
        mma_bf16_16816(s[nt], qf[kk + 1], b[2], b[3]);
      }
      if constexpr ((DK / 16) & 1) {  // odd k-step count (head dim 72 -> 80)
        constexpr int kk = DK / 16 - 1;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(ks + (nt * 8 + g) * LD + kk * 16 + 2 * t4);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(ks + (nt * 8 + g) * LD + kk * 16 + 8 + 2 * t4);
        mma_bf16_16816(s[nt], qf[kk], b0, b1);
      }
    }
    // masks only where a block can hold masked keys: the range end, causal diagonal
    const bool edge = j0 + BN > k_end || (a.causal && j0 + BN - 1 > q_lo);
    if (edge) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = j0 + nt * 8 + 2 * t4 + e;
            bool ok = j < k_end;
            if (a.causal) ok = ok && (j <= qi[r] + a.q_offset);
            if (!ok) s[nt][2 * r + e] = -INFINITY;
          }
    }
    // online softmax (rows g and g+8 of this warp), log2 domain: p = 2^(s sl2 - m)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * r], s[nt][2 * r + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mnew = fmaxf(mrow[r], mx * sl2);
      const float base = mnew == -INFINITY ? 0.f : mnew;
      const float corr = exp2f(mrow[r] - base);
      float rs = 0.f;
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float p = exp2f(fmaf(s[nt][2 * r + e], sl2, -base));
          s[nt][2 * r + e] = p;
          rs += p;
        }
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      lrow[r] = lrow[r] * corr + rs;
      mrow[r] = mnew;
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        o[j][2 * r] *= corr;
        o[j][2 * r + 1] *= corr;
      }
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dt = 0; dt < ND; ++dt) {
        uint32_t b0, b1;
        ldsm_x2_trans(b0, b1, vs + (kk * 16 + (lane & 15)) * LD + dt * 8);
        mma_bf16_16816(o[dt], pa, b0, b1);
      }
    }
    __syncthreads();  // everyone is done with the round's stages before the next prefetch overwrites them
  }
  if constexpr (KG > 1) {
    // ---- key groups -> group 0 (group order, deterministic); the K/V stages are free ----
    cp_async_wait<0>();
    float* xg = reinterpret_cast<float*>(ks_buf);  // [KG - 1][4 G warps][32 lanes][ND * 4 + 4]
    constexpr int W = ND * 4 + 4;
    const int slot = (warp % (4 * G)) * 32 + lane;
    if (kg > 0) {
      float* d = xg + ((kg - 1) * 4 * G * 32 + slot) * W;
#pragma unroll
      for (int j = 0; j < ND; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[j * 4 + e] = o[j][e];
      d[ND * 4 + 0] = mrow[0];
      d[ND * 4 + 1] = mrow[1];
      d[ND * 4 + 2] = lrow[0];
      d[ND * 4 + 3] = lrow[1];
    }
    __syncthreads();
    // (group-k warps stay resident: the merges below use block-wide barriers)
#pragma unroll
    for (int q = 1; q < KG; ++q) {
      if (kg > 0) break;
      const float* d = xg + ((q - 1) * 4 * G * 32 + slot) * W;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float m2 = d[ND * 4 + r], l2 = d[ND * 4 + 2 + r];
        const float mn = fmaxf(mrow[r], m2);
        const float base = mn == -INFINITY ? 0.f : mn;
        const float c1 = exp2f(mrow[r] - base), c2 = exp2f(m2 - base);
        lrow[r] = lrow[r] * c1 + l2 * c2;
        mrow[r] = mn;
#pragma unroll
        for (int j = 0; j < ND; ++j) {
          o[j][2 * r] = o[j][2 * r] * c1 + d[j * 4 + 2 * r] * c2;
          o[j][2 * r + 1] = o[j][2 * r + 1] * c1 + d[j * 4 + 2 * r + 1] * c2;
        }
      }
    }
  }
  if (splits > 1) {
    // ---- split-KV merge inside the thread-block cluster (the splits of one
    // (q tile, head)): partials stay in each CTA's shared memory; after a
    // cluster barrier CTA z merges rows [z*BM/S, (z+1)*BM/S) reading its peers'
    // partials over DSMEM (fixed split order -> deterministic), then a second
    // barrier keeps every CTA alive until its peers are done reading ----
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int W = HD + 2;
    constexpr int RT = G * BM;                   // merged rows (G heads x BM queries)
    float* rec = reinterpret_cast<float*>(fsm);  // [RT][W]: o unnormalised, m, l
    __syncthreads();                             // K/V buffers are free
#pragma unroll
    for (int r = 0; r < 2 && kg == 0; ++r) {
      const int row = hw * BM + wr * 16 + g + 8 * r;
#pragma unroll
      for (int dt = 0; dt < ND; ++dt) {
        rec[row * W + dt * 8 + 2 * t4] = o[dt][2 * r];
        rec[row * W + dt * 8 + 2 * t4 + 1] = o[dt][2 * r + 1];
      }
      if (t4 == 0) {
        rec[row * W + HD] = mrow[r];
        rec[row * W + HD + 1] = lrow[r];
      }
    }
    cluster.sync();
    const int z = static_cast<int>(cluster.block_rank());
    const int r_lo = z * RT / splits, r_hi = (z + 1) * RT / splits;
    __shared__ float wz[RT / 2 + 1][kMaxKvSplits + 1];  // merge weights, then 1/L
    for (int row = r_lo + threadIdx.x; row < r_hi; row += NT) {
      float mz[kMaxKvSplits], M = -INFINITY;
#pragma unroll
      for (int p = 0; p < kMaxKvSplits; ++p) {
        mz[p] = p < splits ? cluster.map_shared_rank(rec, p)[row * W + HD] : -INFINITY;
        M = fmaxf(M, mz[p]);
      }
      float L = 0.f;
#pragma unroll
      for (int p = 0; p < kMaxKvSplits; ++p) {
        const float w = (p < splits && mz[p] != -INFINITY) ? exp2f(mz[p] - M) : 0.f;
        wz[row - r_lo][p] = w;
        if (p < splits) L = fmaf(cluster.map_shared_rank(rec, p)[row * W + HD + 1], w, L);
      }
      wz[row - r_lo][kMaxKvSplits] = L > 0.f ? 1.0f / L : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (r_hi - r_lo) * (HD / 2); i += NT) {
      const int rr = i / (HD / 2), d = 2 * (i % (HD / 2)), row = r_lo + rr;
      float v0 = 0.f, v1 = 0.f;
#pragma unroll
      for (int p = 0; p < kMaxKvSplits; ++p) {
        if (p < splits) {
          const float2 pv = *reinterpret_cast<const float2*>(cluster.map_shared_rank(rec, p) + row * W + d);
          v0 = fmaf(pv.x, wz[rr][p], v0);
          v1 = fmaf(pv.y, wz[rr][p], v1);
        }
      }
      const int qrow = q0 + row % BM, hrow = static_cast<int>(blockIdx.y) * G + row / BM;
      if (qrow < a.Tq) {
        const float inv = wz[rr][kMaxKvSplits];
        bf16* op = a.out + static_cast<long>(qrow) * a.o_tok_stride + static_cast<long>(hrow) * a.o_head_stride;
        *reinterpret_cast<uint32_t*>(op + d) = pack_bf16x2(v0 * inv, v1 * inv);
      }
    }
    cluster.sync();
    return;
  }
  // normalise + store
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (qi[r] >= a.Tq || kg > 0) continue;
    const float inv = lrow[r] > 0.f ? 1.0f / lrow[r] : 0.f;
    bf16* op = a.out + static_cast<long>(qi[r]) * a.o_tok_stride + static_cast<long>(h) * a.o_head_stride;
#pragma unroll
    for (int dt = 0; dt < ND; ++dt)
      *reinterpret_cast<uint32_t*>(op + dt * 8 + 2 * t4) =
          pack_bf16x2(o[dt][2 * r] * inv, o[dt][2 * r + 1] * inv);
  }
}

template <int HD, int G = 1, int NS = 2, int KG = 1>
static cudaError_t flash_hd(const FlashArgs& a, cudaStream_t st) {
  using Cfg = FlashCfg<HD>;
  const size_t smem = static_cast<size_t>(G * Cfg::kBM + 2 * NS * Cfg::kBN) * Cfg::kLd * 2;
  static DeviceFlags attr;
  if (!attr.done()) {
    cudaError_t e = cudaFuncSetAttribute(flash_kernel<HD, G, NS, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr.mark();
  }
  const int splits = a.kv_splits > 1 ? a.kv_splits : 1;
  dim3 grid((a.Tq + Cfg::kBM - 1) / Cfg::kBM, a.hq / G, splits);
  if (splits > kMaxKvSplits || (splits > 1 && a.seg_len > 0) ||
      static_cast<size_t>(G * Cfg::kBM) * (HD + 2) * 4 > smem || a.hq % G || (a.hq / a.hkv) % G)
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(128 * G * KG);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = take_launch_pdl() ? 1 : 0;
  la[1].id = cudaLaunchAttributeClusterDimension;
  la[1].val.clusterDim.x = 1;
  la[1].val.clusterDim.y = 1;
  la[1].val.clusterDim.z = static_cast<unsigned>(splits);
  cfg.attrs = la;
  cfg.numAttrs = splits > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, flash_kernel<HD, G, NS, KG>, a);
}

int flash_kv_splits(int Tq, int hq, int n_keys, int num_sms) {
  const int units = (Tq + 63) / 64 * hq;
  const int nblk = (n_keys + 63) / 64;
  if (units * 2 > num_sms || nblk < 4) return 1;
  // one wave of ~1 CTA per SM (measured in context, expert 32 heads x 1109 keys:
  // 4 splits 25.1 us, 8 splits 28.9 us, 2 splits 32.6 us per layer)
  int s = num_sms / units;
  s = s < nblk / 2 ? s : nblk / 2;            // >= 2 key blocks per split
  s = s < kMaxKvSplits ? s : kMaxKvSplits;    // one portable cluster per (q tile, head)
  return s < 1 ? 1 : s;
}

long flash_ws_floats(int Tq, int hq, int hd, int kv_splits) {
  return static_cast<long>((Tq + 63) / 64) * hq * kv_splits * 64 * (hd + 2);
}

cudaError_t launch_flash_attention(const FlashArgs& a, cudaStream_t st) {
  if (a.Tq <= 0) return cudaSuccess;
  switch (a.hd) {
    case 32: return flash_hd<32>(a, st);
    case 64: return flash_hd<64>(a, st);
    case 72: return flash_hd<72>(a, st);
    case 128: {
      if (a.g_pack == 2) return flash_hd<128, 2>(a, st);
      if (a.kv_splits <= 1) {  // causal prefill (LS_DIAG_FLASH_NSP: 2 = two CTAs per SM)
        static const int nsp = [] {
          const char* v = std::getenv("LS_DIAG_FLASH_NSP");
          return v ? std::atoi(v) : 2;
        }();
        return nsp <= 2 ? flash_hd<128>(a, st) : nsp == 3 ? flash_hd<128, 1, 3>(a, st) : flash_hd<128, 1, 4>(a, st);
      }
      // split-KV (the expert): a few key blocks per CTA, one CTA per SM -- keep
      // more blocks in flight (LS_DIAG_FLASH_NS: 2..4, diagnostics)
      static const int ns = [] {
        const char* v = std::getenv("LS_DIAG_FLASH_NS");
        return v ? std::atoi(v) : 4;
      }();
      static const int kgs = [] {  // LS_DIAG_FLASH_KG: key groups (diagnostics)
        const char* v = std::getenv("LS_DIAG_FLASH_KG");
        return v ? std::atoi(v) : 2;
      }();
      if (kgs == 2 && ns >= 4) return flash_hd<128, 1, 4, 2>(a, st);
      return ns <= 2 ? flash_hd<128>(a, st) : ns == 3 ? flash_hd<128, 1, 3>(a, st) : flash_hd<128, 1, 4>(a, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace lsb
