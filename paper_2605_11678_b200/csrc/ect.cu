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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace lsb {

// Pages [page0, page0 + n_pages) -> plain tiles at out (page0 lands at out[0]);
// with_tail also copies the raw vectors after them (whole-layer decode).
__global__ void __launch_bounds__(256) ect_decode_kernel(const uint8_t* __restrict__ blob,
                                                         uint32_t page0, uint32_t n_pages,
                                                         int with_tail, uint8_t* __restrict__ out) {
  __shared__ __align__(16) uint32_t tile[kTileBytes / 4];
  pdl_trigger();
  // pages never depend on the previous kernel, but `out` (the decode scratch) is
  // read by it: the first page is loaded and decoded before griddepcontrol.wait,
  // every store comes after it
  bool waited = false;
  const EctHeader* h = reinterpret_cast<const EctHeader*>(blob);
  const uint32_t e0p = (h->e0 << 7) | (h->e0 << 23);
  const uint8_t* pages = blob + h->off_pages + static_cast<uint64_t>(page0) * kEctPageBytes;
  const uint32_t* exc_off = reinterpret_cast<const uint32_t*>(blob + h->off_excoff);
  const uint32_t* exc = reinterpret_cast<const uint32_t*>(blob + h->off_exc);
  // one page per CTA iteration: fragments decoded into the plain tile image in
  // shared memory (pair stores are bank-conflict-free thanks to the 128 B
  // swizzle), then streamed out as coalesced 16-byte stores
  // plain-tile u32 slots of this thread's word pairs (words 8 f .. 8 f + 7 of
  // fragment f = it * 256 + threadIdx.x), per page order
  const bool rows = h->order == 1;
  uint32_t pos[4][4];
#pragma unroll
  for (int it = 0; it < 4; ++it)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t q = (it * 256 + threadIdx.x) * 8 + 2 * p;
      pos[it][p] = (rows ? ect_plain_word_rows(q) : ect_plain_word(q)) >> 1;
    }
  for (uint32_t page = blockIdx.x; page < n_pages; page += gridDim.x) {
    const uint8_t* pg = pages + static_cast<uint64_t>(page) * kEctPageBytes;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const uint32_t f = it * 256 + threadIdx.x;  // fragment index in the page
      const uint2 sm = __ldcs(reinterpret_cast<const uint2*>(pg) + f);
      const uint32_t nib = __ldcs(reinterpret_cast<const uint32_t*>(pg + kEctPageWords) + f);
      uint4 w = ect_decode8(sm, nib, e0p);
      const uint32_t esc = ect_escapes(nib);
      if (esc) w = ect_zero_escapes(w, esc);  // exponent 0 unless an exc entry patches it below
      tile[pos[it][0]] = w.x;
      tile[pos[it][1]] = w.y;
      tile[pos[it][2]] = w.z;
      tile[pos[it][3]] = w.w;
    }
    __syncthreads();
    // the page's exceptions (true exponents of escaped words) patched in shared memory
    {
      const uint32_t e_lo = exc_off[page0 + page], e_hi = exc_off[page0 + page + 1];
      uint16_t* t16 = reinterpret_cast<uint16_t*>(tile);
      for (uint32_t i = e_lo + threadIdx.x; i < e_hi; i += blockDim.x) {
        const uint32_t x = exc[i];
        const uint32_t k = rows ? ect_plain_word_rows(x >> 8) : ect_plain_word(x >> 8);
        t16[k] = static_cast<uint16_t>((t16[k] & 0x807Fu) | ((x & 0xFFu) << 7));
      }
      if (e_hi > e_lo) __syncthreads();
    }
    if (!waited) {
      pdl_wait();
      waited = true;
    }
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<uint64_t>(page) * kTileBytes);
#pragma unroll
    for (int it = 0; it < 4; ++it)
      dst[it * 256 + threadIdx.x] = reinterpret_cast<const uint4*>(tile)[it * 256 + threadIdx.x];
    __syncthreads();
  }
  if (!waited) pdl_wait();
  if (!with_tail) return;
  // raw tail (vectors), whole 16-byte chunks
  const uint64_t tail = (h->total - h->mat_bytes + 15) / 16;
  const uint4* src = reinterpret_cast<const uint4*>(blob + h->off_tail);
  uint4* dst = reinterpret_cast<uint4*>(out + h->mat_bytes);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < tail; i += stride)
    dst[i] = src[i];
}

cudaError_t launch_ect_decode_pages(const uint8_t* blob, uint32_t page0, uint32_t n_pages,
                                    bool with_tail, void* out, int num_sms, cudaStream_t st) {
  static const int per_sm = [] {  // LS_DIAG_ECT_DEC_PER_SM: CTAs per SM (diagnostics)
    const char* v = std::getenv("LS_DIAG_ECT_DEC_PER_SM");
    return v ? std::atoi(v) : 8;  // 8 x 256 threads fill an SM; measured 3: +4.2 ms, 4: +2.2, 6: 0, 8: -1.1 ms
  }();
  return launch_k(ect_decode_kernel, dim3(per_sm * num_sms), dim3(256), 0, st, blob, page0, n_pages,
                  with_tail ? 1 : 0, static_cast<uint8_t*>(out));
}

cudaError_t launch_ect_decode(const uint8_t* blob, void* out, int num_sms, cudaStream_t st) {
  const EctHeader* h = nullptr;
  EctHeader hh;
  if (cudaMemcpy(&hh, blob, sizeof(hh), cudaMemcpyDefault) != cudaSuccess) return cudaErrorInvalidValue;
  h = &hh;
  return launch_ect_decode_pages(blob, 0, h->n_pages, true, out, num_sms, st);
}

}  // namespace lsb
