// kernels.h -- host-side launch interface of the sm_100a kernels (shared by the
// executor and the C-ABI test launchers).  Plain POD argument blocks; every
// launcher enqueues on the given stream and returns cudaError_t.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lsb {

typedef __nv_bfloat16 bf16;

// Programmatic dependent launch for the NEXT launch_* call on this thread.
void set_launch_pdl(bool on);

// ---------------- decode GEMV (batch 1) over tiled weights --------------------
enum GemvEpi : int {
  GEMV_F32 = 0,     // out[row] = y
  GEMV_RESID = 1,   // out[row] += y           (fp32 residual stream)
  GEMV_SILU = 2,    // out[g*64+i] = silu(y_gate) * y_up (gate/up interleaved per 64 rows)
  GEMV_QKV = 3,     // per-head RMSNorm (q,k) + RoPE + q out + K/V cache append
  GEMV_ARGMAX = 4,  // logits out + packed (value, index) atomicMax
};

struct GemvArgs {
  const uint8_t* w;        // tiled weights, n_mt * n_kb tiles of 16 KiB
  int n_mt, n_kb;          // 128-row tiles, 64-column k-blocks
  const float* x;          // input vector, fp32 [n_kb*64]
  const bf16* norm_w;      // fused RMSNorm weight over x (nullptr: none)
  float eps;
  float* ws;               // stream-K partials [n_mt][max_contrib][128]
  int* counters;           // [n_mt], zero between launches (self-cleaning)
  int max_contrib;
  float* out;              // F32 / RESID / SILU / ARGMAX(logits)
  const float* bias;       // optional per-row bias (F32/RESID)
  int n_valid;             // rows that are real (vocab / padding guard)
  // QKV epilogue
  int hq, hkv, hd, pos;
  const bf16* qn_w;        // q RMSNorm weight [hd] (nullptr: no q/k norm)
  const bf16* kn_w;
  const float2* rope;      // (cos, sin) table [max_pos][hd/2]
  float* q_out;            // [hq*hd]
  bf16* k_cache;           // [hkv][max_ctx][hd]
  bf16* v_cache;
  int cache_head_stride;   // max_ctx * hd
  unsigned long long* amax;  // ARGMAX packed key
  // ECT (compact) weights: w points at this matrix's first 12 KiB page inside
  // the blob whose header is ct_blob; tile t of the matrix is page ct_page0 + t.
  // nullptr: plain 16 KiB tiles.
  const uint8_t* ct_blob;
  int ct_page0;
  int key_row0;            // ARGMAX: global index of row 0 (vocab-parallel lm-head shard)
  // ECT: cap on the page-ring slots (0: as many as fit, <= LS_GEMV_SLOTS); fewer
  // slots leave shared memory for a decode-attention CTA on the same SM
  int max_slots;
};

int gemv_max_contrib(int n_mt, int n_kb, int grid);
int gemv_grid(int n_mt, int n_kb, int num_sms);
cudaError_t launch_gemv(int epi, const GemvArgs& a, int grid, cudaStream_t st);
// ECT pages (a.ct_blob set): gemv_ect.cu; launch_gemv dispatches there
cudaError_t launch_gemv_ect(int epi, const GemvArgs& a, int grid, cudaStream_t st);

// ---------------- tcgen05 GEMM: Y[T x N] = X[T x K] * W^T ---------------------
enum GemmEpi : int {
  GEMM_BF16 = 0,       // out_bf16 = acc (+bias)
  GEMM_BF16_GELU = 1,  // out_bf16 = gelu_tanh(acc + bias)
  GEMM_RESID_F32 = 2,  // out_f32 += acc (+bias)
  GEMM_SILU_BF16 = 3,  // out_bf16[t, g*64+i] = silu(gate) * up
  GEMM_F32 = 4,        // out_f32 = acc (+bias)
};

struct GemmArgs {
  const uint8_t* w;   // tiled weights (n_mt x n_kb tiles)
  int n_mt, n_kb;
  int T;              // tokens (rows of X)
  const CUtensorMap* x_map;  // X [T x n_kb*64] bf16 row-major, SWIZZLE_128B box {64, 64} (gemm_box_rows)
  void* out;
  long ldo;           // elements between consecutive tokens in out
  const float* bias;  // per output feature (optional)
  const bf16* bias_bf16;  // alternative bf16 bias (optional)
  int n_valid;        // features < n_valid are real (bias / store guard)
  // split-K for skinny GEMMs (few output tiles, e.g. the 64-token expert):
  // each (tile, k-range) unit stores fp32 partials; the last unit of a tile
  // sums them in split order and runs the epilogue.  sk_ws == nullptr: off.
  float* sk_ws;       // partials [tiles * ks][BN tokens][128 features]
  long sk_ws_floats;  // capacity
  int* sk_cnt;        // [tiles] arrival counters, zero between launches
  int sk_cnt_n;
  int ks;             // set by launch_gemm (callers leave 0)
  // ECT weights (see GemvArgs): w = the matrix's first page, tile t = page ct_page0 + t
  const uint8_t* ct_blob;
  int ct_page0;
  // 1: w was written by the previous kernel (ECT decode scratch) -- no weight
  // tile is requested before griddepcontrol.wait
  int w_dep;
  int ct_order;  // EctHeader.order of ct_blob (1: row order -> A decoded into TMEM)
};

int gemm_block_n(int T);
int gemm_block_n(int T, int n_mt, int num_sms);  // plain weights, T > 256: 192 or 256 by waves
int gemm_box_rows();  // rows of the activation tensor-map box (the kernels load BN/64 boxes per stage)
// split factor launch_gemm picks for a shape (1 = no split)
int gemm_splits(int n_mt, int n_kb, int T, int num_sms, long ws_floats, int cnt_n, bool ct = false);
cudaError_t launch_gemm(int epi, const GemmArgs& a, const CUtensorMap& map, cudaStream_t st);
// Encode a row-major bf16 [rows x cols] tensor map with box {64, box_rows}, SWIZZLE_128B.
int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t ld_elems, uint32_t box_rows);

// ---------------- attention --------------------------------------------------
struct DecodeAttnArgs {
  const float* q;          // [hq*hd]
  const bf16* k_cache;     // [hkv][max_ctx][hd]
  const bf16* v_cache;
  int cache_head_stride;
  int hq, hkv, hd, n_ctx;
  float scale;
  float* out;              // [hq*hd]
  float* ws;               // unused (splits merge over DSMEM); kept for ABI stability
  int* counters;           // unused
  int n_split;
};
cudaError_t launch_decode_attention(const DecodeAttnArgs& a, cudaStream_t st);
// splits (one cluster of <= 16 CTAs per KV head, <= 128 positions per CTA)
int decode_attn_splits(int n_ctx);
int decode_attn_max_ctx();  // positions one decode-attention launch covers

struct FlashArgs {
  const bf16* q;  long q_tok_stride, q_head_stride;   // q[t, h, d]
  const bf16* k1; const bf16* v1; long k1_tok_stride, k1_head_stride; int len1;  // segment 1
  const bf16* k2; const bf16* v2; long k2_tok_stride, k2_head_stride; int len2;  // segment 2
  bf16* out;      long o_tok_stride, o_head_stride;
  int Tq, hq, hkv, hd;
  int causal;      // key j visible to query i iff j <= i + q_offset
  int q_offset;
  int seg_len;     // >0: block-diagonal attention over segments of seg_len tokens (ViT images)
  float scale;
  // split-KV (few query tiles, long KV: the 64-token expert over the LM cache):
  // grid.z = kv_splits (<= 8) CTAs per (q tile, head), one thread-block cluster,
  // each reduce a contiguous key range; partials are merged over DSMEM in split
  // order.  ws / counters: unused (kept for ABI stability).
  int kv_splits;   // <= 1: off
  float* ws;
  int* counters;
  // 1: segment 1 was not written by the previous kernel (the expert reading the
  // VLM cache) -- its first K/V block is requested before griddepcontrol.wait
  int k1_ready;
  // 2: GQA packing -- one CTA per (q tile, 2 query heads of one KV head), 8 warps;
  // hd 128, (hq / hkv) % 2 == 0; kv_splits counts CTAs per (q tile, head pair)
  int g_pack;
};
cudaError_t launch_flash_attention(const FlashArgs& a, cudaStream_t st);
// kv_splits the launcher will use for (Tq, hq, keys) given num_sms, and the
// workspace floats / counters it then needs
int flash_kv_splits(int Tq, int hq, int n_keys, int num_sms);
long flash_ws_floats(int Tq, int hq, int hd, int kv_splits);

// ---------------- elementwise / norms ------------------------------------------
cudaError_t launch_rmsnorm_rows(const float* x, const bf16* w, bf16* out, int T, int D, float eps,
                                cudaStream_t st);
cudaError_t launch_layernorm_rows(const float* x, const bf16* w, const bf16* b, bf16* out, int T,
                                  int D, long ld_out, float eps, cudaStream_t st);
cudaError_t launch_qk_norm_rope(const bf16* qkv, int T, int hq, int hkv, int hd, const bf16* qn_w,
                                const bf16* kn_w, float eps, const float2* rope, int pos0,
                                bf16* q_out, bf16* k_cache, bf16* v_cache, int cache_head_stride,
                                cudaStream_t st);
cudaError_t launch_embed_rows(const bf16* table, const int* ids, int n, int D, float* out,
                              long ld_out, cudaStream_t st);
cudaError_t launch_add_rows_bf16(float* x, const bf16* add, int T, int D, long period,
                                 cudaStream_t st);
cudaError_t launch_silu_inplace(float* x, int n, cudaStream_t st);
cudaError_t launch_add_f32(float* x, const float* y, long n, cudaStream_t st);  // x += y
cudaError_t launch_cast_f32_bf16(const float* x, bf16* out, long n, cudaStream_t st);
cudaError_t launch_argmax_to_token(const unsigned long long* key, int* token_out, int* history,
                                   int step, unsigned long long* key_reset, cudaStream_t st);
cudaError_t launch_action_in(const float* actions, const bf16* w_in, const bf16* b_in,
                             const float* temb, int n_tok, int a_dim, int D, float* out,
                             cudaStream_t st);
cudaError_t launch_time_embed(const float* t_scalar_table, int step, int dim, float* out,
                              cudaStream_t st);
cudaError_t launch_action_out_euler(const float* h, const bf16* norm_w, float eps,
                                    const bf16* w_out, const bf16* b_out, int n_tok, int D,
                                    int a_dim, float dt, float* actions, float* velocity,
                                    cudaStream_t st);
cudaError_t launch_fill_u64(unsigned long long* p, unsigned long long v, int n, cudaStream_t st);

// ---------------- ECT: exponent-coded tiles (compact resident / streamed layers) --
// Fixed-rate: every 16 KiB weight tile (page) is 12 KiB = 8192 sign+mantissa
// bytes then 4096 bytes of 4-bit exponent codes (word 2i in the low nibble of
// byte i).  Code c < 15 is exponent e0 + c (codebook[c] = e0 + c); 15 = escape,
// whose exponent is the low byte of the page's exc entry with (word index <<
// 8).  ect.py has the format.
constexpr int kEctPageBytes = 12288;
constexpr int kEctPageWords = 8192;
struct EctHeader {
  uint32_t magic;  // 'ECT1'
  uint32_t n_pages;
  uint64_t total;      // plain layer bytes
  uint64_t mat_bytes;  // = n_pages * 16 KiB (the layer's tiled matrices)
  uint64_t off_pages, off_tail, off_excoff, off_exc;
  uint32_t n_exc, e0;
  uint8_t codebook[16];
  // per page u32: bit r set <=> page words [256 r, 256 r + 256) hold an escape
  // (code 15); 0 = section absent (decoders then test every code)
  uint64_t off_escmask;
  // page word order: 0 = mma.sync A-fragment order (decode GEMV), 1 = row-chunk
  // order (skinny tcgen05 GEMM decoding into TMEM; ect.py ORDER_ROWS)
  uint32_t order;
  uint8_t _pad[36];
};
static_assert(sizeof(EctHeader) == 128, "ECT header is 128 bytes");
// blob -> plain layer bytes (whole 16-byte chunks: out needs a16(total) bytes);
// one kernel (exceptions patched per page in shared memory).  Reads the header
// synchronously (test / tool entry point).
cudaError_t launch_ect_decode(const uint8_t* blob, void* out, int num_sms, cudaStream_t st);
// pages [page0, page0 + n_pages) of a device blob -> plain tiles at out (+ the
// raw vectors when with_tail, for a whole-layer decode)
cudaError_t launch_ect_decode_pages(const uint8_t* blob, uint32_t page0, uint32_t n_pages,
                                    bool with_tail, void* out, int num_sms, cudaStream_t st);

// diagnostic (probe.cu): `grid` CTAs each stream `per_cta` bytes of src through a
// `stages` x `stage_bytes` bulk-copy ring, no compute
cudaError_t launch_bulk_stream(const void* src, uint64_t per_cta, int stage_bytes, int stages, int grid,
                               uint32_t* sink, cudaStream_t st);

}  // namespace lsb
