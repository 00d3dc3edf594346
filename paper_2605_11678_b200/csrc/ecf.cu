// ecf.cu -- lossless exponent-coded BF16 ("ECF") for streamed layers.
//
// The transfer engine is PCIe-bound (~55 GB/s) while HBM is ~6.5 TB/s, so
// every byte not sent over PCIe is worth ~100 bytes of on-GPU work.  BF16
// weights waste most of their 8 exponent bits (a layer uses ~20 distinct
// exponents, entropy ~2.5 bits).  ECF stores, per 1024-word unit:
//   * sign + 7 mantissa bits as one byte                      (SM plane)
//   * a 3-bit primary code: the 7 most frequent exponents, 7 = escape
//   * for escaped words, a 4-bit secondary code (next 15 exponents, 15 =
//     exception) in a nibble stream; each unit records where its nibbles start
//   * exceptions as (u32 word index, u8 exponent)
// ~11.1 bits per word on N(0, 0.02) weights (vs 16).  Decoding is bit-exact:
// one warp per unit, lane = 32 consecutive words, escape nibbles located with
// a warp prefix sum; exceptions patched by a second kernel.  It runs on the
// compute stream from the slot's tail (where the blob was DMA'd) into the
// slot's head, HBM-bound.
#include "common.cuh"
#include "kernels.h"

namespace lsb {

__global__ void __launch_bounds__(256) ecf_decode_kernel(const uint8_t* __restrict__ blob,
                                                         uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const EcfHeader* h = reinterpret_cast<const EcfHeader*>(blob);
  __shared__ uint32_t cb1[8], cb2[16];
  if (threadIdx.x < 8) cb1[threadIdx.x] = static_cast<uint32_t>(h->codebook1[threadIdx.x]) << 7;
  if (threadIdx.x < 16) cb2[threadIdx.x] = static_cast<uint32_t>(h->codebook2[threadIdx.x]) << 7;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t n_units = h->n_words / kEcfUnit;
  const uint8_t* sm_plane = blob + h->off_sm;
  const uint32_t* prim = reinterpret_cast<const uint32_t*>(blob + h->off_prim);
  const uint32_t* uoff = reinterpret_cast<const uint32_t*>(blob + h->off_uoff);
  const uint8_t* sec = blob + h->off_sec;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       u < n_units; u += warps) {
    const uint64_t w0 = u * kEcfUnit + lane * 32;
    const uint32_t* pp = prim + (u * kEcfUnit + lane * 32) * 3 / 32;
    const uint32_t p[3] = {__ldcs(pp), __ldcs(pp + 1), __ldcs(pp + 2)};
    const uint4* sp = reinterpret_cast<const uint4*>(sm_plane + w0);
    const uint4 s0 = __ldcs(sp), s1 = __ldcs(sp + 1);
    const uint32_t sb[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    // escape count of this lane's 32 codes, then exclusive warp scan
    uint32_t esc = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int b = 3 * j;
      uint32_t c = p[b >> 5] >> (b & 31);
      if ((b & 31) > 29) c |= p[(b >> 5) + 1] << (32 - (b & 31));
      esc += (c & 7) == 7;
    }
    uint32_t incl = esc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    uint32_t nib = uoff[u] + incl - esc;
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int b = 3 * j;
      uint32_t c = p[b >> 5] >> (b & 31);
      if ((b & 31) > 29) c |= p[(b >> 5) + 1] << (32 - (b & 31));
      c &= 7;
      uint32_t ex;
      if (c == 7) {
        const uint32_t byte = sec[nib >> 1];
        ex = cb2[(byte >> (4 * (nib & 1))) & 0xF];
        ++nib;
      } else {
        ex = cb1[c];
      }
      const uint32_t sbyte = (sb[j >> 2] >> (8 * (j & 3))) & 0xFF;
      const uint32_t word = ((sbyte & 0x80) << 8) | ex | (sbyte & 0x7F);
      if (j & 1) w[j >> 1] |= word << 16;
      else w[j >> 1] = word;
    }
    uint4* o = reinterpret_cast<uint4*>(out + w0);
    o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o[1] = make_uint4(w[4], w[5], w[6], w[7]);
    o[2] = make_uint4(w[8], w[9], w[10], w[11]);
    o[3] = make_uint4(w[12], w[13], w[14], w[15]);
  }
}

__global__ void __launch_bounds__(256) ecf_patch_kernel(const uint8_t* __restrict__ blob,
                                                        uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const EcfHeader* h = reinterpret_cast<const EcfHeader*>(blob);
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(blob + h->off_idx);
  const uint8_t* ex = blob + h->off_exp;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h->n_exc; i += gridDim.x * blockDim.x) {
    const uint32_t k = idx[i];
    out[k] = static_cast<uint16_t>((out[k] & 0x807F) | (static_cast<uint32_t>(ex[i]) << 7));
  }
}

cudaError_t launch_ecf_decode(const uint8_t* blob, void* out, int num_sms, cudaStream_t st) {
  cudaError_t e = launch_k(ecf_decode_kernel, dim3(4 * num_sms), dim3(256), 0, st, blob,
                           static_cast<uint16_t*>(out));
  if (e != cudaSuccess) return e;
  set_launch_pdl(true);  // the patch follows the decode kernel directly
  return launch_k(ecf_patch_kernel, dim3(64), dim3(256), 0, st, blob, static_cast<uint16_t*>(out));
}

}  // namespace lsb
