// ect.cu -- exponent-coded tiles (ECT): decode a compact layer blob into the
// plain packed layer (tiles + vectors) for the kernels that need whole tiles
// in HBM (tcgen05 GEMMs of prefill / ViT / expert).  The decode GEMV reads ECT
// pages directly (gemv.cu, ect_decode8) and never materialises them.
//
// Roofline: HBM.  Bytes per page = 12288 read + 16384 written; one thread per
// 8-word chunk (8 B sign+mantissa + 4 B codes -> one 16 B store), coalesced on
// both sides; the 16-entry exponent table lives in shared memory.  Escapes
// (~1.5e-4 of words on N(0, 0.02) weights) take a divergent slow path that
// scans the page's short exception list.
#include "common.cuh"
#include "kernels.h"

namespace lsb {

__global__ void __launch_bounds__(256) ect_decode_kernel(const uint8_t* __restrict__ blob,
                                                         uint8_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();  // `out` (the decode scratch) is read by the previous layer's kernels
  const EctHeader* h = reinterpret_cast<const EctHeader*>(blob);
  const uint32_t e0p = (h->e0 << 7) | (h->e0 << 23);
  const uint8_t* pages = blob + h->off_pages;
  const uint64_t chunks = static_cast<uint64_t>(h->n_pages) * (kEctPageWords / 8);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < chunks; i += stride) {
    const uint8_t* pg = pages + (i >> 10) * kEctPageBytes;
    const uint32_t c = static_cast<uint32_t>(i & 1023);  // fragment index in the page
    const uint2 sm = __ldcs(reinterpret_cast<const uint2*>(pg) + c);
    const uint32_t nib = __ldcs(reinterpret_cast<const uint32_t*>(pg + kEctPageWords) + c);
    const uint4 w = ect_decode8(sm, nib, e0p);
    // the 4 word pairs go back to their swizzled tile positions (4-byte stores; a
    // warp writes 16-byte runs of 8 rows, merged in L2)
    uint32_t* po = reinterpret_cast<uint32_t*>(out + (i >> 10) * 16384ull);
    po[ect_plain_word(c * 8 + 0) >> 1] = w.x;
    po[ect_plain_word(c * 8 + 2) >> 1] = w.y;
    po[ect_plain_word(c * 8 + 4) >> 1] = w.z;
    po[ect_plain_word(c * 8 + 6) >> 1] = w.w;
  }
  // raw tail (vectors), whole 16-byte chunks
  const uint64_t tail = (h->total - h->mat_bytes + 15) / 16;
  const uint4* src = reinterpret_cast<const uint4*>(blob + h->off_tail);
  uint4* dst = reinterpret_cast<uint4*>(out + h->mat_bytes);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < tail; i += stride)
    dst[i] = src[i];
}

// Escaped words: one thread per exception, page found by binary search in exc_off.
__global__ void __launch_bounds__(256) ect_patch_kernel(const uint8_t* __restrict__ blob,
                                                        uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const EctHeader* h = reinterpret_cast<const EctHeader*>(blob);
  const uint32_t* exc_off = reinterpret_cast<const uint32_t*>(blob + h->off_excoff);
  const uint32_t* exc = reinterpret_cast<const uint32_t*>(blob + h->off_exc);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h->n_exc; i += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = h->n_pages;  // largest page with exc_off[page] <= i
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (exc_off[mid] <= i) lo = mid;
      else hi = mid;
    }
    const uint32_t x = exc[i];
    const uint64_t k = static_cast<uint64_t>(lo) * kEctPageWords + ect_plain_word(x >> 8);
    out[k] = static_cast<uint16_t>((out[k] & 0x807Fu) | ((x & 0xFFu) << 7));
  }
}

cudaError_t launch_ect_decode(const uint8_t* blob, void* out, int num_sms, cudaStream_t st) {
  cudaError_t e = launch_k(ect_decode_kernel, dim3(8 * num_sms), dim3(256), 0, st, blob,
                           static_cast<uint8_t*>(out));
  if (e != cudaSuccess) return e;
  set_launch_pdl(true);  // the scatter follows the decode kernel directly
  return launch_k(ect_patch_kernel, dim3(num_sms), dim3(256), 0, st, blob, static_cast<uint16_t*>(out));
}

}  // namespace lsb
