// capi_kernels.cu -- extern "C" kernel launchers (raw device pointers + shapes +
// cudaStream_t) used by the parity tests and by external callers.  The
// executor calls the same launch_* functions directly.
#include <mutex>
#include <string>

#include "../../include/layerswap_b200.h"
#include "kernels.h"

namespace lsb {
int set_error(int code, const char* fmt, ...);

static thread_local bool g_pdl_next = false;
void set_launch_pdl(bool on) { g_pdl_next = on; }
bool take_launch_pdl() {
  const bool v = g_pdl_next;
  g_pdl_next = false;
  return v;
}
}  // namespace lsb
using namespace lsb;

static int cuda_rc(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LS_OK;
  return set_error(LS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

extern "C" {

int ls_num_sms(int device, int32_t* out) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  *out = v;
  return cuda_rc(e, "cudaDeviceGetAttribute");
}

/* Page-locked host memory for the streamed-layer arena (one H2D per layer). */
int ls_host_alloc(uint64_t bytes, void** out) {
  *out = nullptr;
  return cuda_rc(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
}

int ls_host_free(void* p) { return cuda_rc(cudaFreeHost(p), "cudaFreeHost"); }

/* Synchronous copy between any two addresses (unified addressing). */
int ls_copy(void* dst, const void* src, uint64_t bytes) {
  return cuda_rc(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault), "cudaMemcpy");
}

int ls_gemv_plan(int32_t n_mt, int32_t n_kb, int32_t num_sms, int32_t* grid, int32_t* max_contrib) {
  *grid = gemv_grid(n_mt, n_kb, num_sms);
  *max_contrib = gemv_max_contrib(n_mt, n_kb, *grid);
  return LS_OK;
}

int ls_set_launch_pdl(int32_t on) {
  set_launch_pdl(on != 0);
  return LS_OK;
}

int ls_k_gemv(int32_t epi, const void* args, int32_t grid, void* stream) {
  return cuda_rc(launch_gemv(epi, *static_cast<const GemvArgs*>(args), grid,
                             static_cast<cudaStream_t>(stream)),
                 "ls_k_gemv");
}

int ls_k_gemm(int32_t epi, const void* w, int32_t n_mt, int32_t n_kb, const void* x, int32_t T,
              int64_t ldx, void* out, int64_t ldo, const float* bias, const void* bias_bf16,
              int32_t n_valid, void* stream) {
  CUtensorMap map;
  int rc = make_tmap_bf16(&map, x, static_cast<uint64_t>(T), static_cast<uint64_t>(n_kb) * 64,
                          static_cast<uint64_t>(ldx), static_cast<uint32_t>(gemm_box_rows()));
  if (rc) return set_error(LS_ERR_CUDA, "ls_k_gemm: cuTensorMapEncodeTiled failed (%d)", rc);
  GemmArgs a{};
  a.w = static_cast<const uint8_t*>(w);
  a.n_mt = n_mt;
  a.n_kb = n_kb;
  a.T = T;
  a.out = out;
  a.ldo = ldo;
  a.bias = bias;
  a.bias_bf16 = static_cast<const bf16*>(bias_bf16);
  a.n_valid = n_valid;
  return cuda_rc(launch_gemm(epi, a, map, static_cast<cudaStream_t>(stream)), "ls_k_gemm");
}

int ls_k_gemm_ws(int32_t epi, const void* w, int32_t n_mt, int32_t n_kb, const void* x, int32_t T,
                 int64_t ldx, void* out, int64_t ldo, const float* bias, const void* bias_bf16,
                 int32_t n_valid, float* sk_ws, int64_t sk_ws_floats, int32_t* sk_cnt,
                 int32_t sk_cnt_n, const void* ct_blob, int32_t ct_page0, void* stream) {
  CUtensorMap map;
  int rc = make_tmap_bf16(&map, x, static_cast<uint64_t>(T), static_cast<uint64_t>(n_kb) * 64,
                          static_cast<uint64_t>(ldx), static_cast<uint32_t>(gemm_box_rows()));
  if (rc) return set_error(LS_ERR_CUDA, "ls_k_gemm_ws: cuTensorMapEncodeTiled failed (%d)", rc);
  GemmArgs a{};
  a.w = static_cast<const uint8_t*>(w);
  a.n_mt = n_mt;
  a.n_kb = n_kb;
  a.T = T;
  a.out = out;
  a.ldo = ldo;
  a.bias = bias;
  a.bias_bf16 = static_cast<const bf16*>(bias_bf16);
  a.n_valid = n_valid;
  a.sk_ws = sk_ws;
  a.sk_ws_floats = sk_ws_floats;
  a.sk_cnt = sk_cnt;
  a.sk_cnt_n = sk_cnt_n;
  a.ct_blob = static_cast<const uint8_t*>(ct_blob);
  a.ct_page0 = ct_page0;
  if (ct_blob) {
    a.w = static_cast<const uint8_t*>(ct_blob) + sizeof(EctHeader) + static_cast<long>(ct_page0) * kEctPageBytes;
    EctHeader h;  // kernel-API entry point (tests / tools): the page order from the device header
    if (cudaMemcpy(&h, ct_blob, sizeof(h), cudaMemcpyDefault) != cudaSuccess)
      return set_error(LS_ERR_CUDA, "ls_k_gemm_ws: cannot read the ECT header");
    a.ct_order = static_cast<int>(h.order);
  }
  return cuda_rc(launch_gemm(epi, a, map, static_cast<cudaStream_t>(stream)), "ls_k_gemm_ws");
}

int ls_gemm_splits(int32_t n_mt, int32_t n_kb, int32_t T, int32_t num_sms, int64_t ws_floats,
                   int32_t cnt_n) {
  return gemm_splits(n_mt, n_kb, T, num_sms, ws_floats, cnt_n);
}

int ls_probe_bulk_stream(const void* src, uint64_t per_cta, int32_t stage_bytes, int32_t stages,
                         int32_t grid, void* sink, void* stream) {
  return cuda_rc(launch_bulk_stream(src, per_cta, stage_bytes, stages, grid, static_cast<uint32_t*>(sink),
                                    static_cast<cudaStream_t>(stream)),
                 "ls_probe_bulk_stream");
}

int ls_k_ect_decode(const void* blob, void* out, void* stream) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  return cuda_rc(launch_ect_decode(static_cast<const uint8_t*>(blob), out, nsm,
                                   static_cast<cudaStream_t>(stream)),
                 "ls_k_ect_decode");
}

int64_t ls_k_args_size(int32_t kind) {
  switch (kind) {
    case 0: return sizeof(GemvArgs);
    case 1: return sizeof(DecodeAttnArgs);
    case 2: return sizeof(FlashArgs);
    default: return -1;
  }
}

int ls_k_decode_attention(const void* args, void* stream) {
  return cuda_rc(launch_decode_attention(*static_cast<const DecodeAttnArgs*>(args),
                                         static_cast<cudaStream_t>(stream)),
                 "ls_k_decode_attention");
}

int ls_k_flash_attention(const void* args, void* stream) {
  return cuda_rc(launch_flash_attention(*static_cast<const FlashArgs*>(args),
                                        static_cast<cudaStream_t>(stream)),
                 "ls_k_flash_attention");
}

int ls_k_rmsnorm_rows(const float* x, const void* w, void* out, int32_t T, int32_t D, float eps,
                      void* stream) {
  return cuda_rc(launch_rmsnorm_rows(x, static_cast<const bf16*>(w), static_cast<bf16*>(out), T, D,
                                     eps, static_cast<cudaStream_t>(stream)),
                 "ls_k_rmsnorm_rows");
}

int ls_k_layernorm_rows(const float* x, const void* w, const void* b, void* out, int32_t T,
                        int32_t D, int64_t ld_out, float eps, void* stream) {
  return cuda_rc(launch_layernorm_rows(x, static_cast<const bf16*>(w), static_cast<const bf16*>(b),
                                       static_cast<bf16*>(out), T, D, ld_out, eps,
                                       static_cast<cudaStream_t>(stream)),
                 "ls_k_layernorm_rows");
}

int ls_k_qk_norm_rope(const void* qkv, int32_t T, int32_t hq, int32_t hkv, int32_t hd,
                      const void* qn_w, const void* kn_w, float eps, const void* rope, int32_t pos0,
                      void* q_out, void* k_cache, void* v_cache, int32_t cache_head_stride,
                      void* stream) {
  return cuda_rc(launch_qk_norm_rope(static_cast<const bf16*>(qkv), T, hq, hkv, hd,
                                     static_cast<const bf16*>(qn_w), static_cast<const bf16*>(kn_w),
                                     eps, static_cast<const float2*>(rope), pos0,
                                     static_cast<bf16*>(q_out), static_cast<bf16*>(k_cache),
                                     static_cast<bf16*>(v_cache), cache_head_stride,
                                     static_cast<cudaStream_t>(stream)),
                 "ls_k_qk_norm_rope");
}

}  // extern "C"
