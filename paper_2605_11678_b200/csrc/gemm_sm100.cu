// gemm_sm100.cu -- tcgen05 tensor-core GEMM for the dense (prefill / ViT /
// action-expert) contractions:  Y[T x N] = X[T x K] . W[N x K]^T.
//
// Roofline: tensor pipe (2*T*N*K FLOP per launch) for T >= ~256; weight-HBM
// bound for the 64-token expert.  B200 mapping:
//   * weights are the MMA "A" operand (M = 128 output features per CTA),
//     tokens are "B" (N = BN tokens), so the 64-token expert still issues
//     full-height M=128 MMAs;
//   * A tiles are pre-swizzled in HBM (see common.cuh), one 16 KiB 1-D bulk
//     copy per stage; B tiles come through a 2-D TMA tensor map with
//     SWIZZLE_128B -- both land in the UMMA K-major SW128 layout;
//   * warp 0: TMA producer, warp 1: TMEM allocator + single-thread MMA issuer
//     (tcgen05.mma.cta_group::1.kind::f16, accumulator in TMEM), warps 2-5:
//     epilogue (tcgen05.ld -> shared-memory transpose -> fused bias / GELU /
//     SiLU*up / residual -> 16-byte stores), warps 6-21 (ECT): page decoders;
//   * mbarrier full/empty ring, tcgen05.commit releases smem stages.
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace lsb {

// CT = true: weights arrive as ECT pages (12 KiB) in a staging ring and 16
// decoder warps expand each into the swizzled 16 KiB A tile in shared memory
// (no decoded copy of the layer in HBM, 25 % fewer weight bytes).
// TM = true (CT, BN <= 128, row-order pages): A is decoded into TMEM, so a
// stage is just a page + an activation tile and the ring is twice as deep.
template <int BN, bool CT = false, bool TM = false>
struct GemmCfg {
  static constexpr int kStages = TM ? (BN >= 128 ? 6 : 10)
                                    : CT ? (BN >= 256 ? 3 : (BN >= 128 ? 4 : 5))
                                         : (BN >= 256 ? 4 : (BN >= 192 ? 5 : (BN >= 128 ? 6 : 8)));
  static constexpr int kABytes = TM ? 0 : kTileBytes;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kPBytes = CT ? kEctPageBytes : 0;  // page staging
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAccCols = BN < 32 ? 32 : BN;     // one accumulator
  // double-buffered accumulators (+ the decoded A stages, 32 columns each, for TM)
  static_assert(!TM || (CT && 2 * (BN < 32 ? 32 : BN) + 32 * kStages <= 512), "TMEM budget");
  // tcgen05.alloc takes a power of two >= 32 columns (BN = 192: 384 -> 512)
  static constexpr int kTmemCols = TM || 2 * kAccCols > 256 ? 512 : 2 * kAccCols;
  static constexpr int kDecWarps = CT ? 16 : 0;
  static constexpr int kThreads = 192 + 32 * kDecWarps;
  static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * (kStageBytes + kPBytes) +
                                  128 * 17 * 4 + (4 * kStages + 4) * 8 + 16;
};

// Persistent: grid = min(#tiles, #SMs); CTA c takes tiles c, c+grid, ...  Tiles
// are ordered token-tile fastest, so the CTAs working on one weight m-tile at
// the same time share it through L2 (each weight byte read from HBM ~once).
// Two TMEM accumulators: the epilogue of tile i overlaps the MMAs of tile i+1.
template <int BN, int EPI, bool CT, bool TM = false>
__global__ void __launch_bounds__(GemmCfg<BN, CT, TM>::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap xmap, const GemmArgs a) {
  using Cfg = GemmCfg<BN, CT, TM>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  uint8_t* sa = smem;
  uint8_t* sb = smem + Cfg::kStages * Cfg::kABytes;
  uint8_t* spg = sb + Cfg::kStages * Cfg::kBBytes;  // ECT page staging (CT)
  float* stage_f = reinterpret_cast<float*>(spg + Cfg::kStages * Cfg::kPBytes);  // [128][17]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_f + 128 * 17);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* dec = empty + Cfg::kStages;          // CT: A tile decoded (kDecWarps arrivals)
  uint64_t* bfull = dec + Cfg::kStages;          // B (activation) tile landed
  uint64_t* acc_full = bfull + Cfg::kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kb = a.n_kb;
  const int n_nt = (a.T + BN - 1) / BN;
  const int ks = a.ks > 1 ? a.ks : 1;
  const int n_tiles = a.n_mt * n_nt * ks;  // work units: (tile, k-split)

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&dec[s], Cfg::kDecWarps > 0 ? Cfg::kDecWarps : 1);
      mbar_init(&bfull[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
    prefetch_tmap(&xmap);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TM (row-order ECT pages, EctHeader.order 1): the decoders write A straight
  // into TMEM (tcgen05.st, one row per lane) and the MMA reads it from there
  constexpr bool tm = TM;
  const uint32_t tmem_a = tmem + 2 * Cfg::kAccCols;  // A stage s at column +32 s

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      constexpr int kWBytes = CT ? kEctPageBytes : kTileBytes;
      // weights (A / ECT page, full[s]) and activations (B, bfull[s]) complete
      // on separate barriers: the first kStages weight tiles do not depend on
      // the previous kernel and are requested before pdl_wait, so they stream
      // (and, CT, get decoded) while the previous launch drains
      auto a_load = [&](int s, int mt, int kb) {
        mbar_arrive_expect_tx(&full[s], kWBytes);
        bulk_g2s(CT ? spg + s * Cfg::kPBytes : sa + s * Cfg::kABytes,
                 a.w + (static_cast<long>(mt) * n_kb + kb) * kWBytes, kWBytes, &full[s]);
      };
      int pre = 0;
#ifndef LS_GEMM_NOPRE  // diagnostic build: every weight tile after pdl_wait
      for (int t = blockIdx.x; !a.w_dep && t < n_tiles && pre < Cfg::kStages; t += gridDim.x) {
        const int tile = t / ks, sp = t % ks, mt = tile / n_nt;
        const int kb1 = (sp + 1) * n_kb / ks;
        for (int kb = sp * n_kb / ks; kb < kb1 && pre < Cfg::kStages; ++kb) a_load(pre++, mt, kb);
      }
#endif
      pdl_wait();  // activations of the previous kernel
      int s = 0, i = 0;
      uint32_t round = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int tile = t / ks, sp = t % ks;
        const int mt = tile / n_nt, n0 = (tile % n_nt) * BN;
        const int kb1 = (sp + 1) * n_kb / ks;
        for (int kb = sp * n_kb / ks; kb < kb1; ++kb, ++i) {
          if (i >= pre) {
            if (round) mbar_wait(&empty[s], (round - 1) & 1);
            a_load(s, mt, kb);
          }
          // activations in 64-row boxes (gemm_box_rows: one tensor map serves every BN)
          mbar_arrive_expect_tx(&bfull[s], Cfg::kBBytes);
#pragma unroll
          for (int q = 0; q < BN / 64; ++q)
            tma_load_2d(sb + s * Cfg::kBBytes + q * 8192, &xmap, kb * kTileCols, n0 + q * 64, &bfull[s]);
          if (++s == Cfg::kStages) {
            s = 0;
            ++round;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---- single-thread MMA issuer ----
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
      int s = 0;
      uint32_t round = 0;
      int i = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        if (i >= 2) mbar_wait(&acc_empty[b], ((i >> 1) - 1) & 1);  // epilogue drained buffer b
        tc_fence_after();
        const uint32_t acc = tmem + b * Cfg::kAccCols;
        const int sp = t % ks, kb0 = sp * n_kb / ks, kb1 = (sp + 1) * n_kb / ks;
        for (int kb = kb0; kb < kb1; ++kb) {
          if constexpr (CT) mbar_wait(&dec[s], round & 1);  // decoders waited for the page
          else mbar_wait(&full[s], round & 1);
          mbar_wait(&bfull[s], round & 1);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(sa + s * Cfg::kABytes);
          const uint64_t db = umma_desc_sw128(sb + s * Cfg::kBBytes);
          if (tm) {
#pragma unroll
            for (int k = 0; k < kTileCols / 16; ++k)  // A: 8 TMEM columns per K=16 step
              umma_bf16_ts(acc, tmem_a + s * 32 + 8 * k, db + 2ull * k, idesc, (kb > kb0 || k) ? 1u : 0u);
          } else {
#pragma unroll
            for (int k = 0; k < kTileCols / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
              umma_bf16(acc, da + 2ull * k, db + 2ull * k, idesc, (kb > kb0 || k) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
          if (++s == Cfg::kStages) {
            s = 0;
            ++round;
          }
        }
        umma_commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else if (CT && warp >= 6) {  // ---- ECT decoder warps: page -> swizzled A tile ----
    const EctHeader* h = reinterpret_cast<const EctHeader*>(a.ct_blob);
    const uint32_t e0p = (h->e0 << 7) | (h->e0 << 23);
    const uint32_t* exc_off = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_excoff) + a.ct_page0;
    const uint32_t* exc = reinterpret_cast<const uint32_t*>(a.ct_blob + h->off_exc);
    const int dt = threadIdx.x - 192;  // 0 .. 32 * kDecWarps - 1
    // u32 slots of this thread's 4 word pairs in the plain tile for fragment dt; fragment
    // dt + it * 32 * kDecWarps sits 2 * it * kDecWarps / 8 row blocks (x 32 rows) lower
    constexpr int kIts = Cfg::kDecWarps ? 1024 / (32 * Cfg::kDecWarps) : 1;
    // row-order pages reaching the shared-memory path (multi-token-tile launches
    // through the kernel API) map per fragment, not by a fixed stride
    const bool rows = h->order == 1;
    uint32_t pos[kIts][4];
#pragma unroll
    for (int it = 0; it < kIts; ++it)
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t q = (it * 32 * Cfg::kDecWarps + dt) * 8 + 2 * p;
        pos[it][p] = (rows ? ect_plain_word_rows(q) : ect_plain_word(q)) >> 1;
      }
    int s = 0;
    uint32_t round = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int tile = t / ks, sp = t % ks;
      const int mt = tile / n_nt;
      const int kb1 = (sp + 1) * n_kb / ks;
      for (int kb = sp * n_kb / ks; kb < kb1; ++kb) {
        if (round) mbar_wait(&empty[s], (round - 1) & 1);  // the MMA has released A[s]
        mbar_wait(&full[s], round & 1);
        const uint8_t* pg = spg + s * Cfg::kPBytes;
        uint32_t* ta = reinterpret_cast<uint32_t*>(sa + s * Cfg::kABytes);
        const uint32_t page = static_cast<uint32_t>(mt * n_kb + kb);
        if (tm) {
          // row r = 32 (warp % 4) + lane of the TMEM lane quarter this warp may
          // write, k-group cg = 16 k: 16 sign+mantissa bytes + 8 code bytes, one
          // tcgen05.st of 8 columns (bf16 pairs); no shared-memory A tile, no proxy fence
          const int r = 32 * (warp & 3) + lane, cg = (warp - 6) >> 2;
          const uint32_t q0 = static_cast<uint32_t>(cg * 128 + r) * 16;  // first page word
          const uint4 sm = *reinterpret_cast<const uint4*>(pg + q0);
          const uint2 nib = *reinterpret_cast<const uint2*>(pg + kEctPageWords + q0 / 2);
          uint4 w0 = ect_decode8(make_uint2(sm.x, sm.y), nib.x, e0p);
          uint4 w1 = ect_decode8(make_uint2(sm.z, sm.w), nib.y, e0p);
          if (ect_escapes(nib.x) | ect_escapes(nib.y))
            ect_patch16(w0, w1, ect_escapes(nib.x), ect_escapes(nib.y), page, q0, exc_off, exc);
          tmem_st8(tmem_a + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + s * 32 + cg * 8, w0, w1);
          tc_fence_before();  // the TMEM stores precede the arrive the MMA thread waits on
          __syncwarp();
          if (lane == 0) mbar_arrive(&dec[s]);
          if (++s == Cfg::kStages) {
            s = 0;
            ++round;
          }
          continue;
        }
#pragma unroll
        for (int it = 0; it < (Cfg::kDecWarps ? kIts : 0); ++it) {
          const uint32_t f = it * 32 * Cfg::kDecWarps + dt;  // fragment
          const uint2 sm = *reinterpret_cast<const uint2*>(pg + f * 8);
          const uint32_t nib = *reinterpret_cast<const uint32_t*>(pg + kEctPageWords + f * 4);
          uint4 w = ect_decode8(sm, nib, e0p);
          const uint32_t esc = ect_escapes(nib);
          if (esc) w = ect_patch8(w, esc, page, f * 8, exc_off, exc);
          ta[pos[it][0]] = w.x;
          ta[pos[it][1]] = w.y;
          ta[pos[it][2]] = w.z;
          ta[pos[it][3]] = w.w;
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05.mma
        __syncwarp();
        if (lane == 0) mbar_arrive(&dec[s]);
        if (++s == Cfg::kStages) {
          s = 0;
          ++round;
        }
      }
    }
  } else {  // ---- epilogue warps 2..5 ----
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int m = q * 32 + lane;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      const int tile = t / ks, sp = t % ks;
      const int mt = tile / n_nt, n0 = (tile % n_nt) * BN;
      const int f = mt * kTileRows + m;
      mbar_wait(&acc_full[b], (i >> 1) & 1);
      tc_fence_after();
      float bias = 0.f;
      if (f < a.n_valid) {
        if (a.bias) bias = a.bias[f];
        else if (a.bias_bf16) bias = bf2f(a.bias_bf16[f]);
      }
      const uint32_t acc = tmem + b * Cfg::kAccCols + (static_cast<uint32_t>(q * 32) << 16);
      if (ks == 1 && EPI == GEMM_RESID_F32) {
        // residual add, one thread per feature: all 32 old values of a chunk are
        // loaded before any store (32 independent loads in flight per thread; the
        // transposed float4 variant below measured slower here: its loads, one
        // chunk ahead, leave a round trip exposed per 16 tokens)
        float* out = static_cast<float*>(a.out);
        const bool fv = f < a.n_valid;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float old[32], v0[16], v1[16];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int tok = n0 + c0 + jj;
            old[jj] = (fv && tok < a.T) ? out[static_cast<long>(tok) * a.ldo + f] : 0.f;
          }
          tmem_ld16(acc + c0, v0);
          tmem_ld16(acc + c0 + 16, v1);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int tok = n0 + c0 + jj;
            if (fv && tok < a.T)
              out[static_cast<long>(tok) * a.ldo + f] = old[jj] + ((jj < 16 ? v0[jj] : v1[jj - 16]) + bias);
          }
        }
      } else if (ks == 1) {
        // Fused epilogue per 16-token chunk, transposed through shared memory: the
        // TMEM read gives a thread one feature x 16 tokens; after the exchange a
        // thread owns 8 (bf16) or 4 (fp32) consecutive features of one token, so a
        // store is one 16-byte access instead of 8-16 scalar ones, and every one of
        // the 128 threads computes (SiLU*up used 64) -- the per-element epilogue was
        // the bottleneck of the K = 1152 / 4096 GEMMs (gate|up 239 -> 156 us)
        const bool vec = (a.ldo % 8 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
        const bool vec4 = (a.ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          tmem_ld16(acc + c0, v);
          named_bar(2, 128);  // previous chunk's readers are done with stage_f
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) stage_f[m * 17 + jj] = EPI == GEMM_SILU_BF16 ? v[jj] : v[jj] + bias;
          named_bar(2, 128);
          if constexpr (EPI == GEMM_SILU_BF16) {
            const int jt = m & 15, fg = m >> 4;  // token, 8-feature group of the tile's 64
            const int tok = n0 + c0 + jt, g0 = mt * 64 + fg * 8;
            if (tok < a.T) {
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                o[e] = silu(stage_f[(fg * 8 + e) * 17 + jt]) * stage_f[(64 + fg * 8 + e) * 17 + jt];
              bf16* dst = static_cast<bf16*>(a.out) + static_cast<long>(tok) * a.ldo + g0;
              if (vec && g0 + 8 <= a.n_valid) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]),
                                                            pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7]));
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (g0 + e < a.n_valid) dst[e] = f2bf(o[e]);
              }
            }
          } else if constexpr (EPI == GEMM_BF16 || EPI == GEMM_BF16_GELU) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int item = m + 128 * r, jt = item & 15, fg = item >> 4;  // token, 8-feature group
              const int tok = n0 + c0 + jt, f0 = mt * kTileRows + fg * 8;
              if (tok >= a.T) continue;
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float y = stage_f[(fg * 8 + e) * 17 + jt];
                o[e] = EPI == GEMM_BF16_GELU ? gelu_tanh(y) : y;
              }
              bf16* dst = static_cast<bf16*>(a.out) + static_cast<long>(tok) * a.ldo + f0;
              if (vec) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]),
                                                            pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7]));
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) dst[e] = f2bf(o[e]);
              }
            }
          } else {  // GEMM_F32: float4 per (token, 4 features)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int item = m + 128 * r, jt = item & 15, fq = item >> 4;  // token, 4-feature group
              const int tok = n0 + c0 + jt, f0 = mt * kTileRows + fq * 4;
              if (tok >= a.T) continue;
              float4 y = make_float4(stage_f[(fq * 4) * 17 + jt], stage_f[(fq * 4 + 1) * 17 + jt],
                                     stage_f[(fq * 4 + 2) * 17 + jt], stage_f[(fq * 4 + 3) * 17 + jt]);
              float* dst = static_cast<float*>(a.out) + static_cast<long>(tok) * a.ldo + f0;
              if (vec4 && f0 + 4 <= a.n_valid) {
                *reinterpret_cast<float4*>(dst) = y;
              } else {
                const float yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (f0 + e < a.n_valid) dst[e] = yy[e];
              }
            }
          }
        }
      }
      if (ks == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        continue;
      }
      // ---- split-K: partial -> workspace (token-major, coalesced) ----
      float* part = a.sk_ws + static_cast<long>(t) * BN * kTileRows;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(acc + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) part[(c0 + j) * kTileRows + m] = v[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);  // TMEM buffer free
      // Distributed fix-up: every unit of the tile waits for all ks partials,
      // then reduces its own 1/ks of the tile's tokens (in split order, so the
      // result is deterministic) and runs the epilogue on them.  All units are
      // co-resident (grid = units <= #SMs, launch_dependents issued at entry), so
      // the wait cannot deadlock.
      __threadfence();
      named_bar(3, 128);
      if (m == 0) {
        atomicAdd(&a.sk_cnt[tile], 1);
        while (ld_acquire_gpu(&a.sk_cnt[tile]) < ks) __nanosleep(64);
      }
      named_bar(3, 128);
      __threadfence();
      const float* base = a.sk_ws + static_cast<long>(tile) * ks * BN * kTileRows + m;
      const int c_lo = sp * BN / ks, c_hi = (sp + 1) * BN / ks;
      // two tokens per round, all (<= 16) split partials of both loaded at once:
      // the reduction costs ~ceil(tokens / 2) L2 round trips, not tokens x splits
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 2) {
        const bool two = c + 1 < c_hi;
        float p0[16], p1[16];
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          p0[z] = z < ks ? __ldcg(base + (static_cast<long>(z) * BN + c) * kTileRows) : 0.f;
          p1[z] = (z < ks && two) ? __ldcg(base + (static_cast<long>(z) * BN + c + 1) * kTileRows) : 0.f;
        }
        float old0 = 0.f, old1 = 0.f;
        if constexpr (EPI == GEMM_RESID_F32) {
          if (f < a.n_valid && n0 + c < a.T) old0 = static_cast<float*>(a.out)[static_cast<long>(n0 + c) * a.ldo + f];
          if (f < a.n_valid && two && n0 + c + 1 < a.T)
            old1 = static_cast<float*>(a.out)[static_cast<long>(n0 + c + 1) * a.ldo + f];
        }
        float ys[2] = {0.f, 0.f};
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          ys[0] += p0[z];
          ys[1] += p1[z];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int tok = n0 + c + u;
          float y = ys[u];
          if constexpr (EPI == GEMM_SILU_BF16) {
            named_bar(2, 128);
            stage_f[m] = y;
            named_bar(2, 128);
            const int g = mt * 64 + m;
            if (m < 64 && tok < a.T && g < a.n_valid)
              static_cast<bf16*>(a.out)[static_cast<long>(tok) * a.ldo + g] =
                  f2bf(silu(stage_f[m]) * stage_f[m + 64]);
          } else if (tok < a.T) {
            const long o = static_cast<long>(tok) * a.ldo + f;
            y += bias;
            if constexpr (EPI == GEMM_BF16) static_cast<bf16*>(a.out)[o] = f2bf(y);
            else if constexpr (EPI == GEMM_BF16_GELU) static_cast<bf16*>(a.out)[o] = f2bf(gelu_tanh(y));
            else if constexpr (EPI == GEMM_F32) { if (f < a.n_valid) static_cast<float*>(a.out)[o] = y; }
            else if constexpr (EPI == GEMM_RESID_F32) {
              if (f < a.n_valid) static_cast<float*>(a.out)[o] = (u ? old1 : old0) + y;
            }
          }
        }
      }
      // second arrival: the last unit to leave re-arms the counter for the next launch
      named_bar(3, 128);
      if (m == 0 && atomicAdd(&a.sk_cnt[tile], 1) == 2 * ks - 1) a.sk_cnt[tile] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::kTmemCols);
  }
}

int gemm_block_n(int T) { return T <= 64 ? 64 : (T <= 256 ? 128 : 256); }

// Multi-token-tile GEMMs (T > 256) also have BN = 192: the persistent grid runs
// ceil(tiles / #SMs) waves of BN-token tiles, and 192 wins wherever it needs no
// more waves than 256 (ViT proj / fc2: 9 m-tiles x 12 token tiles = 108 tiles in
// one wave at 256, 144 in one wave at 192 -- 25 % less per CTA; ViT QKV 3 waves
// either way).  LS_DIAG_GEMM_BN192=0: off.
int gemm_block_n(int T, int n_mt, int num_sms) {
  static const bool on = [] {
    const char* v = std::getenv("LS_DIAG_GEMM_BN192");
    return !(v && std::atoi(v) == 0);
  }();
  if (T <= 256 || !on) return gemm_block_n(T);
  auto cost = [&](int bn) {
    const long tiles = static_cast<long>(n_mt) * ((T + bn - 1) / bn);
    return (tiles + num_sms - 1) / num_sms * bn;
  };
  return cost(192) < cost(256) ? 192 : 256;
}
int gemm_box_rows() { return 64; }  // activation tensor-map box: 64 token rows

int gemm_splits(int n_mt, int n_kb, int T, int num_sms, long ws_floats, int cnt_n, bool ct) {
  const int bn = ct ? gemm_block_n(T) : gemm_block_n(T, n_mt, num_sms);
  const int tiles = n_mt * ((T + bn - 1) / bn);
  // >= 4 splits or not worth the fix-up.  (ECT pages split from 2 while they were
  // decoded into shared memory; decoded into TMEM the expert QKV -- 48 tiles --
  // is faster unsplit: 14.3 vs 17-19 us in context.)
  (void)ct;
  if (tiles * 4 > num_sms || tiles > cnt_n) return 1;
  int ks = num_sms / tiles;                 // one wave of units: all co-resident (fix-up waits)
  if (ks > n_kb / 4) ks = n_kb / 4;         // >= 4 k-blocks (256 of K) per unit
  if (ks > 16) ks = 16;                     // the fix-up loads <= 16 partials per token at once
  while (ks > 1 && static_cast<long>(tiles) * ks * bn * 128 > ws_floats) --ks;
  return ks < 1 ? 1 : ks;
}

template <int BN, int EPI, bool CT, bool TM = false>
static cudaError_t launch_bn(const GemmArgs& a, const CUtensorMap& map, cudaStream_t st) {
  using Cfg = GemmCfg<BN, CT, TM>;
  static DeviceFlags attr;
  if (!attr.done()) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, EPI, CT, TM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    attr.mark();
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  GemmArgs b = a;
  b.ks = a.sk_ws ? gemm_splits(a.n_mt, a.n_kb, a.T, nsm, a.sk_ws_floats, a.sk_cnt_n, CT) : 1;
  static const int ks_cap = [] {  // LS_DIAG_GEMM_KS: split-K cap (diagnostics)
    const char* v = std::getenv("LS_DIAG_GEMM_KS");
    return v ? std::atoi(v) : 0;
  }();
  if (ks_cap > 0 && b.ks > ks_cap) b.ks = ks_cap;
  const int units = a.n_mt * ((a.T + BN - 1) / BN) * b.ks;
  dim3 grid(units < nsm ? units : nsm);
  return launch_k(gemm_kernel<BN, EPI, CT, TM>, grid, dim3(Cfg::kThreads), Cfg::kSmem, st, map, b);
}

template <int BN, bool CT, bool TM = false>
static cudaError_t launch_epi(int epi, const GemmArgs& a, const CUtensorMap& map, cudaStream_t st) {
  switch (epi) {
    case GEMM_BF16: return launch_bn<BN, GEMM_BF16, CT, TM>(a, map, st);
    case GEMM_BF16_GELU: return launch_bn<BN, GEMM_BF16_GELU, CT, TM>(a, map, st);
    case GEMM_RESID_F32: return launch_bn<BN, GEMM_RESID_F32, CT, TM>(a, map, st);
    case GEMM_SILU_BF16: return launch_bn<BN, GEMM_SILU_BF16, CT, TM>(a, map, st);
    case GEMM_F32: return launch_bn<BN, GEMM_F32, CT, TM>(a, map, st);
  }
  return cudaErrorInvalidValue;
}

template <bool CT>
static cudaError_t launch_ct(int epi, const GemmArgs& a, const CUtensorMap& map, cudaStream_t st) {
  // row-order pages on a single-token-tile launch: A decoded into TMEM
  const bool tm = CT && a.ct_order == 1 && a.T <= gemm_block_n(a.T);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  switch (CT ? gemm_block_n(a.T) : gemm_block_n(a.T, a.n_mt, nsm)) {
    case 64: return tm ? launch_epi<64, true, true>(epi, a, map, st) : launch_epi<64, CT>(epi, a, map, st);
    case 128: return tm ? launch_epi<128, true, true>(epi, a, map, st) : launch_epi<128, CT>(epi, a, map, st);
    case 192:
      if constexpr (!CT) return launch_epi<192, false>(epi, a, map, st);
      return cudaErrorInvalidValue;
    default: return launch_epi<256, CT>(epi, a, map, st);
  }
}

cudaError_t launch_gemm(int epi, const GemmArgs& a, const CUtensorMap& map, cudaStream_t st) {
  if (a.T <= 0) return cudaSuccess;
  return a.ct_blob ? launch_ct<true>(epi, a, map, st) : launch_ct<false>(epi, a, map, st);
}

// ---- tensor-map encoding through the driver entry point (no -lcuda) ----------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t ld_elems, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : static_cast<int>(r);
}

}  // namespace lsb
