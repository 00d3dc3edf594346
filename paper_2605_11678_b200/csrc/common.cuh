// common.cuh -- shared device helpers for the sm_100a kernels: bf16 packing,
// warp reductions, mbarrier / bulk-copy / TMA / tcgen05 PTX wrappers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <atomic>

// cudaFuncSetAttribute applies to the CURRENT device only, so a launcher's
// "attributes already set" flag is kept per device (bit d = done on device d).
struct DeviceFlags {
  std::atomic<uint64_t> bits{0};
  static int cur() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
  }
  bool done() const { return (bits.load(std::memory_order_acquire) >> cur()) & 1ull; }
  void mark() { bits.fetch_or(1ull << cur(), std::memory_order_release); }
};

namespace lsb {

// ---- weight tile format ------------------------------------------------------
// Every weight matrix W[N x K] (out x in, bf16) is stored "tiled": 128-row x
// 64-column tiles of 16 KiB, tile (mt, kb) at byte offset (mt*KB + kb)*16384,
// each tile already in the UMMA K-major SWIZZLE_128B image: row r occupies
// bytes [r*128, r*128+128) and logical 16-byte chunk c of that row sits at
// physical chunk c ^ (r & 7).  The same bytes feed the tcgen05 GEMM (one 1-D
// bulk copy per stage, no tensor map) and the decode GEMV.
constexpr int kTileRows = 128;
constexpr int kTileCols = 64;
constexpr int kTileBytes = kTileRows * kTileCols * 2;  // 16384

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

// generic-proxy shared-memory writes -> visible to the async proxy (TMA / tcgen05)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global -> shared (zero-filled when !valid), Ampere-style groups
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- warp-level tensor-core helpers (mma.sync m16n8k16 bf16 -> fp32) -----------
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x2_trans(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// ---- ECT page decode (kernels.h EctHeader) -------------------------------------
// 8 consecutive words of a page: sm = their sign+mantissa bytes, nib = their
// 4-bit exponent codes (word k in bits 4k..4k+3), e0p = (e0 << 7) | (e0 << 23).
// Returns the 8 BF16 words exactly as the plain tile stores them (escapes --
// code 15 -- get exponent e0 + 15 and must be patched with ect_patch8).
// Per word pair: PRMT places both sm bytes with their sign bit replicated into
// the byte above (sign lands on bit 15 / 31), one LOP3 keeps sign + mantissa
// and ORs the window base, one PRMT lines up the pair's codes, one IMAD adds
// them into the exponent fields: ~2.4 integer ops per word.  (Measured: a
// PRMT-free variant -- sm bytes pre-interleaved, codes pre-split by the encoder,
// ~3.3 ALU/FMA ops per word -- is 3 % slower in the decode GEMV; the narrow
// XU pipe PRMT issues on is not what bounds it.)
// prmt.b32 in its default mode: bit 3 of a selector nibble replicates the sign
// of the selected byte (__byte_perm ignores that bit)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t ect_pair(uint32_t sbytes, uint32_t sel_s, uint32_t lo,
                                             uint32_t hi, uint32_t sel_c, uint32_t e0p) {
  const uint32_t x = (prmt(sbytes, 0u, sel_s) & 0x807F807Fu) | e0p;
  return prmt(lo, hi, sel_c) * 128u + x;
}
__device__ __forceinline__ uint4 ect_decode8(uint2 sm, uint32_t nib, uint32_t e0p) {
  const uint32_t lo = nib & 0x0F0F0F0Fu, hi = (nib >> 4) & 0x0F0F0F0Fu;
  uint4 w;
  w.x = ect_pair(sm.x, 0x9180u, lo, hi, 0xC480u, e0p);
  w.y = ect_pair(sm.x, 0xB3A2u, lo, hi, 0xD591u, e0p);
  w.z = ect_pair(sm.y, 0x9180u, lo, hi, 0xE6A2u, e0p);
  w.w = ect_pair(sm.y, 0xB3A2u, lo, hi, 0xF7B3u, e0p);
  return w;
}
// ECT pages store words in mma.sync A-fragment order: fragment
// f = ((w * 2 + kstep / 2) * 32 + lane) * 2 + kstep % 2 holds the 8 words lane
// (g = lane / 4, t4 = lane % 4) of row block w needs for k-step `kstep` of
// m16n8k16 (rows 16 w + g [+8], k = 16 kstep + 2 t4 [+1] [+8]), i.e. registers
// a0..a3 in order; a lane's two fragments of a k-step pair are adjacent.
// Page word q -> plain (swizzled) tile word:
__device__ __forceinline__ uint32_t ect_plain_word(uint32_t q) {
  const uint32_t f = q >> 3, j = q & 7, w = f >> 7, lane = (f >> 1) & 31;
  const uint32_t ks = ((f >> 6) & 1) * 2 + (f & 1);
  const uint32_t r = 16 * w + (lane >> 2) + 8 * ((j >> 1) & 1);
  const uint32_t k = 16 * ks + 8 * (j >> 2) + 2 * (lane & 3) + (j & 1);
  return r * 64 + (((k >> 3) ^ (r & 7)) << 3) + (k & 7);
}
// Row-chunk page order (EctHeader.order 1, ect.py ORDER_ROWS): page word
// (g * 128 + r) * 16 + j is row r, k = 16 g + j of the tile.
__device__ __forceinline__ uint32_t ect_plain_word_rows(uint32_t q) {
  const uint32_t r = (q >> 4) & 127u, k = ((q >> 11) << 4) | (q & 15u);
  return r * 64 + (((k >> 3) ^ (r & 7)) << 3) + (k & 7);
}
// bit 4k set iff word k's code is 15 (escape)
__device__ __forceinline__ uint32_t ect_escapes(uint32_t nib) {
  // low 3 bits == 7 carries into bit 3; with bit 3 set the nibble is 15
  const uint32_t t = ((nib & 0x77777777u) + 0x11111111u) & nib & 0x88888888u;
  return t >> 3;
}
// Escaped words default to exponent 0 (zeros / subnormals have no exc entry).
__device__ __forceinline__ uint4 ect_zero_escapes(uint4 w, uint32_t t) {
  uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if ((t >> (4 * k)) & 1u) v[k >> 1] &= ~(0x7F80u << (16 * (k & 1)));
  return make_uint4(v[0], v[1], v[2], v[3]);
}
// Slow path: t = ect_escapes(nib) of the chunk starting at page word `word0`;
// true exponents come from the page's exception list.
static __device__ __noinline__ uint4 ect_patch8(uint4 w, uint32_t t, uint32_t page, uint32_t word0,
                                                const uint32_t* exc_off, const uint32_t* exc) {
  const uint32_t b = __ldg(exc_off + page), e = __ldg(exc_off + page + 1);
  uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // unrolled: v stays in registers
    if (!((t >> (4 * k)) & 1u)) continue;
    uint32_t ex = 0;
    for (uint32_t i = b; i < e; ++i) {
      const uint32_t x = __ldg(exc + i);
      if ((x >> 8) == word0 + k) {
        ex = x & 0xFFu;
        break;
      }
    }
    const int sh = 16 * (k & 1);
    v[k >> 1] = (v[k >> 1] & ~(0x7F80u << sh)) | ((ex << 7) << sh);
  }
  return make_uint4(v[0], v[1], v[2], v[3]);
}

// Slow path for one lane's 16 consecutive page words (two fragments from
// page word `word0`; t0 / t1 = ect_escapes of their code words): escaped words
// take exponent 0, then the page's exceptions inside [word0, word0 + 16) --
// usually none or one -- set the true exponents.
__device__ __forceinline__ void ect_patch16(uint4& w0, uint4& w1, uint32_t t0, uint32_t t1, uint32_t page,
                                            uint32_t word0, const uint32_t* exc_off, const uint32_t* exc) {
  w0 = ect_zero_escapes(w0, t0);
  w1 = ect_zero_escapes(w1, t1);
  const uint32_t b = __ldg(exc_off + page), e = __ldg(exc_off + page + 1);
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t x = __ldg(exc + i);
    const uint32_t k = (x >> 8) - word0;  // word within this lane's 16 (wraps when below)
    if (k >= 16u) continue;
    const uint32_t sh = 16u * (k & 1u), ex = ((x & 0xFFu) << 7) << sh;
    const uint32_t j = (k >> 1) & 3u;
    uint4& w = k < 8u ? w0 : w1;
    if (j == 0) w.x |= ex;
    else if (j == 1) w.y |= ex;
    else if (j == 2) w.z |= ex;
    else w.w |= ex;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// q/k RMSNorm + RoPE of one head (dim 128) for one token, one warp: lane l holds
// dims (2l, 2l+1) in xa and (64+2l, 65+2l) in xb -- the rotation pairs (d, d+64)
// stay in the lane.  w0/w1: the norm weight words of those dims; cs: (cos, sin)
// of dims 2l, 2l+1.  Shared by qk_norm_rope128_kernel and the fused GEMM
// epilogue so both round identically.
__device__ __forceinline__ uint2 qk_norm_rope128_lane(uint32_t xa, uint32_t xb, bool norm, uint32_t w0,
                                                      uint32_t w1, float4 cs, float eps) {
  const float v0 = bf16_lo(xa), v1 = bf16_hi(xa), v2 = bf16_lo(xb), v3 = bf16_hi(xb);
  float rstd = 1.0f;
  if (norm) {
    float ss = fmaf(v0, v0, 0.f);
    ss = fmaf(v1, v1, ss);
    ss = fmaf(v2, v2, ss);
    ss = fmaf(v3, v3, ss);
    rstd = rsqrtf(warp_sum(ss) / 128.f + eps);
  }
  const float n0 = v0 * rstd * bf16_lo(w0), n1 = v1 * rstd * bf16_hi(w0);
  const float n2 = v2 * rstd * bf16_lo(w1), n3 = v3 * rstd * bf16_hi(w1);
  return make_uint2(pack_bf16x2(n0 * cs.x - n2 * cs.y, n1 * cs.z - n3 * cs.w),
                    pack_bf16x2(n2 * cs.x + n0 * cs.y, n3 * cs.z + n1 * cs.w));
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// x * sigmoid(x) with the approximate divide (MUFU.RCP + one multiply, vs the
// ~10-instruction IEEE division): the SiLU*up GEMM epilogue was issue-bound on it
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }
// tanh.approx.f32: one MUFU op (max rel. error ~2^-11, far below the bf16
// rounding of the GELU output); tanhf's accurate path made the ViT fc1 GEMM
// epilogue-bound (65 us for 30 GFLOP)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * (x + k1 * x * x * x)));
}

// Order-preserving float -> uint for packed (value, index) atomicMax argmax:
// larger float -> larger key; ties resolved to the SMALLER index (torch.argmax).
__device__ __forceinline__ unsigned long long argmax_key(float v, uint32_t idx) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(b) << 32) | (0xffffffffu - idx);
}


__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- mbarrier -----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Same on a precomputed shared-memory address (hot loops: no address conversion)
__device__ __forceinline__ void mbar_arrive_u32(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---- bulk copies (TMA engine) -------------------------------------------------
// 1-D bulk global->shared copy completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same with an L2 evict-first policy: streamed weights are read exactly once.
__device__ __forceinline__ void bulk_g2s_evict_first(void* smem_dst, const void* gmem_src,
                                                     uint32_t bytes, uint64_t* bar,
                                                     uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 2-D tiled TMA load (SASS: UTMALDG).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- tcgen05 (5th-gen tensor cores, TMEM accumulators) --------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (8-row groups 1024 B apart).
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem) {
  uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= 1ull << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (1024ull >> 4) << 32;              // stride byte offset: 8 rows * 128 B
  d |= 1ull << 46;                        // descriptor version (sm_100)
  d |= 2ull << 61;                        // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::f16, BF16 x BF16 -> F32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4)                              // D format F32
         | (1u << 7)                            // A format BF16
         | (1u << 10)                           // B format BF16
         | (static_cast<uint32_t>(N >> 3) << 17)  // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24); // M / 16
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Same with the A operand in tensor memory (M = 128 rows in lanes 0..127, K
// packed two bf16 per 32-bit column): D[tmem] (+)= A[tmem_a] . B[smem desc]
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 8 consecutive 32-bit columns from registers (then wait for the stores)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint4 a, uint4 b) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(a.x),
      "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bits, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool elect_lane0() { return (threadIdx.x & 31) == 0; }

// ---- programmatic dependent launch (PDL) ----------------------------------------
// Kernels launched with programmatic stream serialisation may start while the
// previous kernel drains: everything before pdl_wait() (barrier init, TMEM
// alloc, weight prefetch) overlaps its tail; nothing that reads or writes
// activations/workspaces may precede pdl_wait().  Both are no-ops otherwise.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The executor decides per launch whether PDL is safe (never right after an
// event wait / record or a memcpy on the stream); launchers consume the flag.
void set_launch_pdl(bool on);
bool take_launch_pdl();

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = take_launch_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace lsb
