// executor.cu -- the Double-Flat-Buffer (DFB) transfer engine and the native
// executor of the Alpamayo-R1-10B-shaped stack.
//
// DFB protocol (schedule rules dfbsim.py:11-37):
//   * one device arena of `cap` bytes emulates the VRAM budget; it holds the
//     slot ring (n_slots x largest layer), always-resident tensors, KV cache,
//     activations and the planner's resident layers -- nothing else is
//     allocated on the device, so the budget is enforced, not just reported;
//   * every streamed layer is ONE cudaMemcpyAsync from its flat pinned host
//     buffer into slot (streamed_seq mod slots) on a dedicated copy stream;
//   * dma_done[slot] (copy -> compute) and compute_done[slot] (compute ->
//     copy) events implement the two-event hand-off; resident layers run on
//     the compute stream with no transfer;
//   * per-invocation barrier (copy stream waits for the invocation's last
//     EXE) unless cross-invocation prefetch; SEQUENTIAL mode makes every DMA
//     wait for the previous EXE;
//   * optional timing events around every DMA and EXE produce a Timeline in
//     the dfbsim event schema (module -> phase -> invocation -> layer order).
// The host thread only enqueues: the whole inference (ViT -> merger -> LM
// prefill -> greedy decode -> flow-matching expert) is issued without a
// single host synchronisation; greedy tokens stay on the device.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/layerswap_b200.h"
#include "kernels.h"

namespace lsb {
int set_error(int code, const char* fmt, ...);
}
using namespace lsb;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      return set_error(LS_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__,     \
                       __LINE__);                                                               \
  } while (0)

// Launch a kernel and count it (gpu_launches evidence for the bench).
// PDL only between two kernels: any event record/wait or memcpy on the
// compute stream clears pdl_ok, so the next kernel launches fully serialised.
#define KL(x)                                     \
  do {                                            \
    set_launch_pdl(e->use_pdl && e->pdl_ok);      \
    CK(x);                                        \
    e->pdl_ok = true;                             \
    ++e->launches;                                \
  } while (0)
#define SSOP(x)            \
  do {                     \
    CK(x);                 \
    e->pdl_ok = false;     \
  } while (0)

namespace {

// NCCL is resolved at run time (torch's bundled libnccl.so.2 is already mapped
// in-process), so the library has no link-time NCCL dependency.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
      api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.all_gather &&
               api.comm_destroy &&
               api.error_string;
    }
  }
  return api;
}

uint64_t tiled_bytes(int n, int k) {
  return static_cast<uint64_t>((n + 127) / 128) * static_cast<uint64_t>((k + 63) / 64) * 16384ull;
}
int n_mt(int n) { return (n + 127) / 128; }
int n_kb(int k) { return (k + 63) / 64; }
uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

void layout_push(ls_layer_layout* L, uint64_t bytes) {
  uint64_t off = L->n_parts ? align_up(L->offset[L->n_parts - 1] + L->bytes[L->n_parts - 1], 16) : 0;
  L->offset[L->n_parts] = off;
  L->bytes[L->n_parts] = bytes;
  L->n_parts++;
  L->total = off + bytes;
}

// LM / expert decoder layer: 0 qkv, 1 o, 2 gate|up (64-row interleave), 3 down,
// 4 attn_norm, 5 mlp_norm, 6 q_norm, 7 k_norm.
void layout_decoder(int d, int hq, int hkv, int hd, int ffn, ls_layer_layout* L) {
  std::memset(L, 0, sizeof(*L));
  layout_push(L, tiled_bytes((hq + 2 * hkv) * hd, d));
  layout_push(L, tiled_bytes(d, hq * hd));
  layout_push(L, tiled_bytes(2 * ffn, d));
  layout_push(L, tiled_bytes(d, ffn));
  layout_push(L, 2ull * d);
  layout_push(L, 2ull * d);
  layout_push(L, 2ull * hd);
  layout_push(L, 2ull * hd);
}

// ViT block: 0 qkv, 1 proj, 2 fc1, 3 fc2, 4 qkv_b, 5 proj_b, 6 fc1_b, 7 fc2_b,
// 8 ln1_w, 9 ln1_b, 10 ln2_w, 11 ln2_b.
void layout_vit(int d, int h, int hd, int ffn, ls_layer_layout* L) {
  std::memset(L, 0, sizeof(*L));
  layout_push(L, tiled_bytes(3 * h * hd, d));
  layout_push(L, tiled_bytes(d, h * hd));
  layout_push(L, tiled_bytes(ffn, d));
  layout_push(L, tiled_bytes(d, ffn));
  layout_push(L, 2ull * 3 * h * hd);
  layout_push(L, 2ull * d);
  layout_push(L, 2ull * ffn);
  layout_push(L, 2ull * d);
  for (int i = 0; i < 4; ++i) layout_push(L, 2ull * d);
}

int vis_tokens(const ls_dims& d) {
  return d.has_vit ? d.vit_images * d.vit_tokens_per_image / 4 : 0;
}
int prompt_len(const ls_dims& d) { return d.prompt_prefix + vis_tokens(d) + d.prompt_suffix; }
int ctx_len(const ls_dims& d) { return prompt_len(d) + d.decode_steps; }
int rope_rows(const ls_dims& d) { return ctx_len(d) + 1 + (d.has_expert ? d.ex_tokens : 0); }
// lm-head rows this rank holds: vocab-parallel under tensor parallelism (rank r
// owns rows [r*head_rows, (r+1)*head_rows) of the vocabulary, zero padded)
int head_rows(const ls_dims& d) {
  return d.tp_world > 1 ? (d.vocab + d.tp_world - 1) / d.tp_world : d.vocab;
}
int head_row0(const ls_dims& d) { return d.tp_world > 1 ? d.tp_rank * head_rows(d) : 0; }
int head_valid(const ls_dims& d) { return std::min(head_rows(d), d.vocab - head_row0(d)); }

uint64_t global_bytes(const ls_dims& d, int id) {
  const bool v = d.has_vit, x = d.has_expert;
  const uint64_t vd = d.vit_d, md = 4ull * d.vit_d;
  switch (id) {
    case 0: return d.embed_on_host ? 0 : 2ull * d.vocab * d.lm_d;  // embed (row-major)
    case 1: return tiled_bytes(head_rows(d), d.lm_d);             // lm_head (this rank's rows)
    case 2: return 2ull * d.lm_d;                                 // final norm
    case 3: return 8ull * rope_rows(d) * (d.lm_hd / 2);           // rope (cos, sin)
    case 4: return v ? tiled_bytes(d.vit_d, d.vit_patch_dim) : 0; // patch embed
    case 5: return v ? 2 * vd : 0;
    case 6: return v ? 2ull * d.vit_tokens_per_image * vd : 0;    // pos embed
    case 7: case 8: return v ? 2 * vd : 0;                        // merger LN
    case 9: return v ? tiled_bytes(static_cast<int>(md), static_cast<int>(md)) : 0;
    case 10: return v ? 2 * md : 0;
    case 11: return v ? tiled_bytes(d.lm_d, static_cast<int>(md)) : 0;
    case 12: return v ? 2ull * d.lm_d : 0;
    case 13: return x ? tiled_bytes(d.ex_d, d.time_dim) : 0;      // time MLP
    case 14: return x ? 4ull * d.ex_d : 0;
    case 15: return x ? tiled_bytes(d.ex_d, d.ex_d) : 0;
    case 16: return x ? 4ull * d.ex_d : 0;
    case 17: return x ? 2ull * d.ex_d * d.action_dim : 0;         // action in
    case 18: return x ? 2ull * d.ex_d : 0;
    case 19: return x ? 2ull * d.action_dim * d.ex_d : 0;         // action out
    case 20: return x ? 2ull * d.action_dim : 0;
    case 21: return x ? 2ull * d.ex_d : 0;                        // expert final norm
    case 22: return x ? 4ull * d.euler_steps : 0;                 // flow-time schedule
  }
  return 0;
}

struct Arena {
  char* base = nullptr;
  uint64_t cap = 0, used = 0, high = 0;
  char* alloc(uint64_t bytes, uint64_t align = 1024) {
    uint64_t off = align_up(used, align);
    if (off + bytes > cap) return nullptr;
    used = off + bytes;
    if (used > high) high = used;
    return base + off;
  }
};

struct GemvPlan {
  int n, k, grid, max_contrib;
  int slots = 0;  // GemvArgs.max_slots
};

// one DMA / EXE (or invocation span) timestamp pair of a run
struct RunRec {
  int engine, module, phase, inv, layer, ev0, ev1;
};

struct Module {
  int kind;
  int layers;
  ls_layer_layout lay;
  std::vector<const char*> host;
  std::vector<char*> resident;  // nullptr: streamed
  std::vector<int> phase_reps;
  // ECT (exponent-coded tiles): the module lives in compact form everywhere --
  // host arena, DFB slots and resident blocks hold ECT blobs; EXE decodes
  // (or the decode GEMV reads pages directly)
  bool ct = false;
  int ct_order = 0;  // EctHeader.order of the module's blobs (1: expert, A decoded into TMEM)
  std::vector<const char*> host_ct;
  std::vector<uint64_t> ct_bytes;
  uint64_t ct_stride = 0;  // resident footprint per layer (largest blob, 256-aligned)
  const char* host_of(int l) const { return ct ? host_ct[l] : host[l]; }
};

}  // namespace

struct ls_exec {
  ls_dims d;
  int dev = 0, nsm = 148;
  Arena ar;
  cudaStream_t cs = nullptr, ss = nullptr;  // copy engine stream, compute stream
  int n_slots = 2;
  uint64_t slot_bytes = 0;
  std::vector<char*> slots;
  std::vector<cudaEvent_t> dma_done, comp_done;
  cudaEvent_t inv_done = nullptr, exe_done = nullptr, ev_begin = nullptr, ev_t0 = nullptr,
              ev_t1 = nullptr, ev_end = nullptr;
  std::vector<cudaEvent_t> tev;  // timing event pool
  std::vector<Module> mods;
  char* g[LS_N_GLOBAL] = {};
  uint64_t bytes_slots = 0, bytes_always = 0, bytes_overhead = 0, mark = 0;
  uint64_t mark0 = 0;            // arena offset where the slot ring starts (after overhead)
  char* scratch = nullptr;       // decoded ECT layer (counted as overhead)
  bool ct_fused = true;          // kernels read ECT pages (else decode each layer to the scratch)
  uint64_t scratch_bytes = 0;
  int S = 0, ctx = 0, Tv = 0, Te = 0, vit_ffn_pad = 0;
  // activations
  float *vit_h = nullptr, *lm_h = nullptr, *dec_h = nullptr, *dec_q = nullptr, *dec_attn = nullptr,
        *dec_mlp = nullptr, *logits = nullptr, *gemv_ws = nullptr,
        *ex_h = nullptr, *temb_in = nullptr, *temb_mid = nullptr, *temb = nullptr,
        *actions = nullptr, *velocity = nullptr, *noise = nullptr;
  bf16 *patches = nullptr, *vit_ln = nullptr, *vit_qkv = nullptr, *vit_attn = nullptr,
       *vit_fc1 = nullptr, *merger_mid = nullptr, *lm_norm = nullptr, *lm_qkv = nullptr,
       *lm_q = nullptr, *lm_attn = nullptr, *lm_mlp = nullptr, *kv = nullptr, *ex_norm = nullptr,
       *ex_qkv = nullptr, *ex_q = nullptr, *ex_kv = nullptr, *ex_attn = nullptr, *ex_mlp = nullptr;
  int *text_ids = nullptr, *token = nullptr, *hist = nullptr,
      *gemv_cnt = nullptr, *flash_cnt = nullptr;
  float* flash_ws = nullptr;  // split-KV partials of the expert's joint attention
  float* gemm_ws = nullptr;   // split-K partials of skinny GEMMs (expert, T = 64)
  int* gemm_cnt = nullptr;
  long gemm_ws_floats = 0;
  int gemm_cnt_n = 0;
  int ex_kv_splits = 1;
  int ex_g_pack = 1;  // expert flash GQA packing (query heads per CTA)
  unsigned long long* amax = nullptr;
  CUtensorMap m_patches, m_vit_ln, m_vit_attn, m_vit_fc1, m_merge_in, m_merger_mid, m_lm_norm,
      m_lm_attn, m_lm_mlp, m_ex_norm, m_ex_attn, m_ex_mlp;
  GemvPlan gp_qkv{}, gp_o{}, gp_gu{}, gp_down{}, gp_head{}, gp_t1{}, gp_t2{};
  bool use_pdl = true, pdl_ok = false;
  // tensor parallelism: row-parallel outputs are summed in place in the
  // residual stream by NCCL on the compute stream (resid_gemm / resid_gemv);
  // the lm-head is vocab-parallel (argmax key MAX-reduced across ranks)
  int tp_world = 1, tp_rank = 0;
  bool tp_on = false;
  ncclComm_t comm = nullptr;
  int64_t launches = 0, h2d_copies = 0;
  double enqueue_us = 0.0;  // host time to enqueue the last run (before its final sync)
  // Untimed runs are captured once into a CUDA graph (both streams, events,
  // copies, PDL edges) and replayed: ~8k kernel launches per inference cost
  // ~20 us of host time each when enqueued one by one.  Any change of the
  // placement / layout / IO pointers / schedule config re-captures.
  bool use_graph = true;
  uint64_t gen = 0;  // bumped whenever resident pointers or the layout change
  cudaGraphExec_t gexec = nullptr;
  uint64_t gkey[12] = {};
  // diagnostics only (tools/layer_breakdown.py): kernels of the expert /
  // LM decode layer to leave out -- results are wrong, the timing difference is the cost
  uint32_t diag_skip = 0;
  int diag_dec_splits = 0;  // LS_DIAG_DEC_SPLITS: decode-attention split count override
  std::vector<RunRec> grecs;  // invocation-span records of the captured run
  cudaEvent_t join_ev = nullptr, fork_ev = nullptr;
  uint64_t h2d_bytes = 0;

  bf16* kc(int l) { return kv + static_cast<long>(l) * 2 * d.lm_hkv * (ctx + 1) * d.lm_hd; }
  bf16* vc(int l) { return kc(l) + static_cast<long>(d.lm_hkv) * (ctx + 1) * d.lm_hd; }
  int cache_stride() const { return (ctx + 1) * d.lm_hd; }
};

namespace {

GemvPlan plan_gemv(int n, int k, int nsm) {
  GemvPlan p{n, k, 0, 0};
  p.grid = gemv_grid(n_mt(n), n_kb(k), nsm);
  p.max_contrib = gemv_max_contrib(n_mt(n), n_kb(k), p.grid);
  return p;
}

int alloc_into(ls_exec* e, void* dst_ptr, uint64_t bytes, uint64_t* counter) {
  const uint64_t before = e->ar.used;
  char* p = e->ar.alloc(bytes ? bytes : 16);
  if (!p)
    return set_error(LS_ERR_CAP,
                     "emulated VRAM cap exceeded: need %llu more bytes (used %llu of %llu)",
                     static_cast<unsigned long long>(bytes),
                     static_cast<unsigned long long>(e->ar.used),
                     static_cast<unsigned long long>(e->ar.cap));
  *static_cast<char**>(dst_ptr) = p;
  // count what the arena actually consumed (alignment padding included), so the
  // profile's always-resident / overhead terms match the arena exactly
  if (counter) *counter += e->ar.used - before;
  return LS_OK;
}

#define ALLOC(field, bytes, counter)                                      \
  do {                                                                    \
    int rc_ = alloc_into(e, &e->field, (bytes), &e->counter);             \
    if (rc_) return rc_;                                                  \
  } while (0)

int tmap(CUtensorMap* m, const void* base, int rows, int cols, int ld) {
  if (rows <= 0) return LS_OK;
  int r = make_tmap_bf16(m, base, static_cast<uint64_t>(rows), static_cast<uint64_t>(cols),
                         static_cast<uint64_t>(ld), static_cast<uint32_t>(gemm_box_rows()));
  if (r) return set_error(LS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", r);
  return LS_OK;
}

// ---------------------------- launch helpers -----------------------------------

// Compact (ECT) view of a layer blob: where part i of the plain layout lives.
struct CtView {
  const char* blob = nullptr;  // nullptr: plain layer
  uint64_t mat = 0, tail = 0;
  int order = 0;  // EctHeader.order of the module's blobs
  CtView() = default;
  CtView(const char* b, const ls_layer_layout& L, int o = 0) : blob(b), order(o) {
    mat = L.offset[3] + L.bytes[3];
    tail = align_up(sizeof(EctHeader) + mat / 16384 * kEctPageBytes, 16);
  }
  // matrices (parts 0..3): first page; vectors: raw tail
  const char* part(const ls_layer_layout& L, int i) const {
    return i < 4 ? blob + sizeof(EctHeader) + L.offset[i] / 16384 * kEctPageBytes
                 : blob + tail + (L.offset[i] - mat);
  }
  int page0(const ls_layer_layout& L, int i) const { return static_cast<int>(L.offset[i] / 16384); }
};

int gemm(ls_exec* e, int epi, const char* w, int n, int k, int T, const CUtensorMap& map, void* out,
         long ldo, const void* bias_bf16 = nullptr, int n_valid = -1, const char* ct_blob = nullptr,
         int ct_page0 = 0, int ct_order = 0) {
  GemmArgs a{};
  a.ct_order = ct_order;
  if (ct_blob && (T + gemm_block_n(T) - 1) / gemm_block_n(T) > 1) {
    // several token tiles would each re-decode every page inside the GEMM: expand
    // this matrix's pages once into the decode scratch and run the plain GEMM on it
    // (the GEMM then must not prefetch weights before the decode has finished)
    if (!(e->diag_skip & (1u << 12)))
      KL(launch_ect_decode_pages(reinterpret_cast<const uint8_t*>(ct_blob), static_cast<uint32_t>(ct_page0),
                                 static_cast<uint32_t>(n_mt(n)) * static_cast<uint32_t>(n_kb(k)), false,
                                 e->scratch, e->nsm, e->ss));
    a.w_dep = 1;  // PDL-chained after the decode, weights only after griddepcontrol.wait
    w = e->scratch;
    ct_blob = nullptr;
  }
  a.w = reinterpret_cast<const uint8_t*>(w);
  a.ct_blob = reinterpret_cast<const uint8_t*>(ct_blob);
  a.ct_page0 = ct_page0;
  a.n_mt = n_mt(n);
  a.n_kb = n_kb(k);
  a.T = T;
  a.out = out;
  a.ldo = ldo;
  a.bias_bf16 = static_cast<const bf16*>(bias_bf16);
  a.n_valid = n_valid < 0 ? n : n_valid;
  a.sk_ws = e->gemm_ws;
  a.sk_ws_floats = e->gemm_ws_floats;
  a.sk_cnt = e->gemm_cnt;
  a.sk_cnt_n = e->gemm_cnt_n;
  KL(launch_gemm(epi, a, map, e->ss));
  return LS_OK;
}

int gemv(ls_exec* e, int epi, const GemvPlan& p, const char* w, const float* x, float* out,
         const void* norm_w, const float* bias = nullptr, int n_valid = -1, GemvArgs* extra = nullptr,
         const char* ct_blob = nullptr, int ct_page0 = 0) {
  GemvArgs a = extra ? *extra : GemvArgs{};
  a.w = reinterpret_cast<const uint8_t*>(w);
  a.ct_blob = reinterpret_cast<const uint8_t*>(ct_blob);
  a.ct_page0 = ct_page0;
  a.n_mt = n_mt(p.n);
  a.n_kb = n_kb(p.k);
  a.x = x;
  a.norm_w = static_cast<const bf16*>(norm_w);
  a.eps = e->d.lm_eps;
  a.ws = e->gemv_ws;
  a.counters = e->gemv_cnt;
  a.max_contrib = p.max_contrib;
  a.out = out;
  a.bias = bias;
  a.n_valid = n_valid < 0 ? p.n : n_valid;
  a.amax = e->amax;
  a.max_slots = p.slots;
  KL(launch_gemv(epi, a, p.grid, e->ss));
  return LS_OK;
}

FlashArgs flash_base(int Tq, int hq, int hkv, int hd) {
  FlashArgs f{};
  f.Tq = Tq;
  f.hq = hq;
  f.hkv = hkv;
  f.hd = hd;
  f.scale = 1.0f / std::sqrt(static_cast<float>(hd));
  return f;
}

#define RC(x)                \
  do {                       \
    int rc_ = (x);           \
    if (rc_) return rc_;     \
  } while (0)

// Row-parallel projections (o-proj, down-proj, ViT proj / fc2) into the fp32
// residual stream dst[T x n]: the fused RESID epilogue on one GPU.  Under tensor
// parallelism every rank holds the same residual; rank 0 writes residual +
// its partial product (the same RESID epilogue), every other rank overwrites
// its copy with its bare partial, and one in-place NCCL all-reduce (fp32 sum)
// over dst leaves residual + sum of partials on every rank -- no staging
// buffer and no separate add kernel.  At world size 1 this is the fused path
// exactly (an all-reduce over one rank is the identity).
int tp_allreduce_inplace(ls_exec* e, float* dst, long count) {
  NcclApi& api = nccl_api();
  ncclResult_t r = api.all_reduce(dst, dst, static_cast<size_t>(count), ncclFloat32, ncclSum,
                                  e->comm, e->ss);
  if (r != ncclSuccess) return set_error(LS_ERR_NCCL, "ncclAllReduce: %s", api.error_string(r));
  e->pdl_ok = false;  // no programmatic launch edge across the NCCL kernel
  return LS_OK;
}

int resid_gemm(ls_exec* e, const char* w, int n, int k, int T, const CUtensorMap& map, float* dst,
               const void* bias_bf16 = nullptr, const char* ct_blob = nullptr, int ct_page0 = 0,
               int ct_order = 0) {
  const int epi = (!e->tp_on || e->tp_rank == 0) ? GEMM_RESID_F32 : GEMM_F32;
  RC(gemm(e, epi, w, n, k, T, map, dst, n, bias_bf16, -1, ct_blob, ct_page0, ct_order));
  return e->tp_on ? tp_allreduce_inplace(e, dst, static_cast<long>(T) * n) : LS_OK;
}

int resid_gemv(ls_exec* e, const GemvPlan& p, const char* w, const float* x, float* dst,
               const char* ct_blob = nullptr, int ct_page0 = 0) {
  const int epi = (!e->tp_on || e->tp_rank == 0) ? GEMV_RESID : GEMV_F32;
  RC(gemv(e, epi, p, w, x, dst, nullptr, nullptr, -1, nullptr, ct_blob, ct_page0));
  return e->tp_on ? tp_allreduce_inplace(e, dst, p.n) : LS_OK;
}

int vit_layer(ls_exec* e, const char* w, const ls_layer_layout& L, const CtView& ct = CtView()) {
  const ls_dims& d = e->d;
  const int T = e->Tv, D = d.vit_d, H = d.vit_heads * d.vit_hd, F = d.vit_ffn;
  auto part = [&](int i) { return ct.blob ? ct.part(L, i) : w + L.offset[i]; };
  const char* cb = ct.blob;
  auto pg = [&](int i) { return cb ? ct.page0(L, i) : 0; };
  const uint32_t skip = e->diag_skip;
  if (!(skip & (1u << 18)))
    KL(launch_layernorm_rows(e->vit_h, (const bf16*)part(8), (const bf16*)part(9), e->vit_ln, T, D, D,
                             d.vit_eps, e->ss));
  if (!(skip & (1u << 19))) RC(gemm(e, GEMM_BF16, part(0), 3 * H, D, T, e->m_vit_ln, e->vit_qkv, 3 * H, part(4), -1, cb, pg(0)));
  FlashArgs f = flash_base(T, d.vit_heads, d.vit_heads, d.vit_hd);
  f.q = e->vit_qkv;
  f.q_tok_stride = 3 * H;
  f.q_head_stride = d.vit_hd;
  f.k1 = e->vit_qkv + H;
  f.v1 = e->vit_qkv + 2 * H;
  f.k1_tok_stride = 3 * H;
  f.k1_head_stride = d.vit_hd;
  f.len1 = T;
  f.out = e->vit_attn;
  f.o_tok_stride = H;
  f.o_head_stride = d.vit_hd;
  f.seg_len = d.vit_tokens_per_image;
  if (!(skip & (1u << 20))) KL(launch_flash_attention(f, e->ss));
  if (!(skip & (1u << 21))) RC(resid_gemm(e, part(1), D, H, T, e->m_vit_attn, e->vit_h, part(5), cb, pg(1)));
  if (!(skip & (1u << 18)))
    KL(launch_layernorm_rows(e->vit_h, (const bf16*)part(10), (const bf16*)part(11), e->vit_ln, T, D,
                             D, d.vit_eps, e->ss));
  if (!(skip & (1u << 22)))
    RC(gemm(e, GEMM_BF16_GELU, part(2), F, D, T, e->m_vit_ln, e->vit_fc1, e->vit_ffn_pad, part(6), F, cb,
            pg(2)));
  if (!(skip & (1u << 23))) RC(resid_gemm(e, part(3), D, e->vit_ffn_pad, T, e->m_vit_fc1, e->vit_h, part(7), cb, pg(3)));
  return LS_OK;
}

int lm_prefill_layer(ls_exec* e, const char* w, const ls_layer_layout& L, int l,
                     const CtView& ct = CtView()) {
  const ls_dims& d = e->d;
  const int S = e->S, D = d.lm_d, QN = (d.lm_hq + 2 * d.lm_hkv) * d.lm_hd, AH = d.lm_hq * d.lm_hd;
  auto part = [&](int i) { return ct.blob ? ct.part(L, i) : w + L.offset[i]; };
  const char* cb = ct.blob;
  auto pg = [&](int i) { return cb ? ct.page0(L, i) : 0; };
  KL(launch_rmsnorm_rows(e->lm_h, (const bf16*)part(4), e->lm_norm, S, D, d.lm_eps, e->ss));
  const uint32_t skip = e->diag_skip;
  if (!(skip & (1u << 14))) RC(gemm(e, GEMM_BF16, part(0), QN, D, S, e->m_lm_norm, e->lm_qkv, QN, nullptr, -1, cb, pg(0)));
  KL(launch_qk_norm_rope(e->lm_qkv, S, d.lm_hq, d.lm_hkv, d.lm_hd, (const bf16*)part(6),
                         (const bf16*)part(7), d.lm_eps, (const float2*)e->g[3], 0, e->lm_q,
                         e->kc(l), e->vc(l), e->cache_stride(), e->ss));
  FlashArgs f = flash_base(S, d.lm_hq, d.lm_hkv, d.lm_hd);
  f.q = e->lm_q;
  f.q_tok_stride = AH;
  f.q_head_stride = d.lm_hd;
  f.k1 = e->kc(l);
  f.v1 = e->vc(l);
  f.k1_tok_stride = d.lm_hd;
  f.k1_head_stride = e->cache_stride();
  f.len1 = S;
  f.out = e->lm_attn;
  f.o_tok_stride = AH;
  f.o_head_stride = d.lm_hd;
  f.causal = 1;
  if (!(skip & (1u << 13))) KL(launch_flash_attention(f, e->ss));
  if (!(skip & (1u << 15))) RC(resid_gemm(e, part(1), D, AH, S, e->m_lm_attn, e->lm_h, nullptr, cb, pg(1)));
  KL(launch_rmsnorm_rows(e->lm_h, (const bf16*)part(5), e->lm_norm, S, D, d.lm_eps, e->ss));
  if (!(skip & (1u << 16)))
    RC(gemm(e, GEMM_SILU_BF16, part(2), 2 * d.lm_ffn, D, S, e->m_lm_norm, e->lm_mlp, d.lm_ffn,
            nullptr, d.lm_ffn, cb, pg(2)));
  if (!(skip & (1u << 17))) RC(resid_gemm(e, part(3), D, d.lm_ffn, S, e->m_lm_mlp, e->lm_h, nullptr, cb, pg(3)));
  return LS_OK;
}

// ct.blob != nullptr: the layer is an ECT blob and the four GEMVs decode its
// pages in registers (no decoded copy of the layer is ever written).
int lm_decode_layer(ls_exec* e, const char* w, const ls_layer_layout& L, int l, int pos,
                    const CtView& ct = CtView()) {
  const ls_dims& d = e->d;
  auto part = [&](int i) { return ct.blob ? ct.part(L, i) : w + L.offset[i]; };
  const char* cb = ct.blob;
  auto pg = [&](int i) { return cb ? ct.page0(L, i) : 0; };
  GemvArgs q{};
  q.hq = d.lm_hq;
  q.hkv = d.lm_hkv;
  q.hd = d.lm_hd;
  q.pos = pos;
  q.qn_w = (const bf16*)part(6);
  q.kn_w = (const bf16*)part(7);
  q.rope = (const float2*)e->g[3];
  q.q_out = e->dec_q;
  q.k_cache = e->kc(l);
  q.v_cache = e->vc(l);
  q.cache_head_stride = e->cache_stride();
  const uint32_t skip = e->diag_skip;
  if (!(skip & 256)) RC(gemv(e, GEMV_QKV, e->gp_qkv, part(0), e->dec_h, e->dec_q, part(4), nullptr, -1, &q, cb, pg(0)));
  DecodeAttnArgs a{};
  a.q = e->dec_q;
  a.k_cache = e->kc(l);
  a.v_cache = e->vc(l);
  a.cache_head_stride = e->cache_stride();
  a.hq = d.lm_hq;
  a.hkv = d.lm_hkv;
  a.hd = d.lm_hd;
  a.n_ctx = pos + 1;
  a.scale = 1.0f / std::sqrt(static_cast<float>(d.lm_hd));
  a.out = e->dec_attn;
  a.n_split = decode_attn_splits(pos + 1);  // one cluster of <= 16 CTAs, merged over DSMEM
  if (e->diag_dec_splits > a.n_split && e->diag_dec_splits <= 16) a.n_split = e->diag_dec_splits;
  if (!(skip & 128)) KL(launch_decode_attention(a, e->ss));
  if (!(skip & 512)) RC(resid_gemv(e, e->gp_o, part(1), e->dec_attn, e->dec_h, cb, pg(1)));
  if (!(skip & 1024))
    RC(gemv(e, GEMV_SILU, e->gp_gu, part(2), e->dec_h, e->dec_mlp, part(5), nullptr, d.lm_ffn, nullptr,
            cb, pg(2)));
  if (!(skip & 2048)) RC(resid_gemv(e, e->gp_down, part(3), e->dec_mlp, e->dec_h, cb, pg(3)));
  return LS_OK;
}

int expert_layer(ls_exec* e, const char* w, const ls_layer_layout& L, int l,
                 const CtView& ct = CtView()) {
  const ls_dims& d = e->d;
  const int T = e->Te, D = d.ex_d, QN = (d.ex_hq + 2 * d.ex_hkv) * d.ex_hd, AH = d.ex_hq * d.ex_hd;
  auto part = [&](int i) { return ct.blob ? ct.part(L, i) : w + L.offset[i]; };
  const char* cb = ct.blob;
  auto pg = [&](int i) { return cb ? ct.page0(L, i) : 0; };
  bf16* ek = e->ex_kv;
  bf16* ev = e->ex_kv + static_cast<long>(d.ex_hkv) * T * d.ex_hd;
  const long shift = static_cast<long>(e->ctx) * d.ex_hd;  // store index t, RoPE position ctx + t
  const uint32_t skip = e->diag_skip;
  if (!(skip & 1)) KL(launch_rmsnorm_rows(e->ex_h, (const bf16*)part(4), e->ex_norm, T, D, d.lm_eps, e->ss));
  const int co = ct.order;
  if (!(skip & 8)) RC(gemm(e, GEMM_BF16, part(0), QN, D, T, e->m_ex_norm, e->ex_qkv, QN, nullptr, -1, cb, pg(0), co));
  if (!(skip & 2)) KL(launch_qk_norm_rope(e->ex_qkv, T, d.ex_hq, d.ex_hkv, d.ex_hd, (const bf16*)part(6),
                         (const bf16*)part(7), d.lm_eps, (const float2*)e->g[3], e->ctx, e->ex_q,
                         ek - shift, ev - shift, T * d.ex_hd, e->ss));
  FlashArgs f = flash_base(T, d.ex_hq, d.ex_hkv, d.ex_hd);
  f.q = e->ex_q;
  f.q_tok_stride = AH;
  f.q_head_stride = d.ex_hd;
  f.k1 = e->kc(l);
  f.v1 = e->vc(l);
  f.k1_tok_stride = d.lm_hd;
  f.k1_head_stride = e->cache_stride();
  f.len1 = e->ctx;
  f.k2 = ek;
  f.v2 = ev;
  f.k2_tok_stride = d.ex_hd;
  f.k2_head_stride = static_cast<long>(T) * d.ex_hd;
  f.len2 = T;
  f.out = e->ex_attn;
  f.o_tok_stride = AH;
  f.o_head_stride = d.ex_hd;
  f.kv_splits = e->ex_kv_splits;
  f.k1_ready = 1;  // the VLM cache was written before the expert runs
  f.g_pack = e->ex_g_pack;
  f.ws = e->flash_ws;
  f.counters = e->flash_cnt;
  if (!(skip & 4)) KL(launch_flash_attention(f, e->ss));
  if (!(skip & 16)) RC(resid_gemm(e, part(1), D, AH, T, e->m_ex_attn, e->ex_h, nullptr, cb, pg(1), co));
  if (!(skip & 1)) KL(launch_rmsnorm_rows(e->ex_h, (const bf16*)part(5), e->ex_norm, T, D, d.lm_eps, e->ss));
  if (!(skip & 32))
    RC(gemm(e, GEMM_SILU_BF16, part(2), 2 * d.ex_ffn, D, T, e->m_ex_norm, e->ex_mlp, d.ex_ffn,
            nullptr, d.ex_ffn, cb, pg(2), co));
  if (!(skip & 64)) RC(resid_gemm(e, part(3), D, d.ex_ffn, T, e->m_ex_mlp, e->ex_h, nullptr, cb, pg(3), co));
  return LS_OK;
}

// Work before / after each invocation (phase sweep) that is not a layer:
// embeddings, merger, lm head + greedy argmax, flow-time MLP, Euler step.
int pre_invocation(ls_exec* e, int kind, int phase, int inv, const ls_run_io* io) {
  const ls_dims& d = e->d;
  if (kind == LS_KIND_VIT) {
    RC(gemm(e, GEMM_F32, e->g[4], d.vit_d, d.vit_patch_dim, e->Tv, e->m_patches, e->vit_h, d.vit_d,
            e->g[5]));
    KL(launch_add_rows_bf16(e->vit_h, (const bf16*)e->g[6], e->Tv, d.vit_d, d.vit_tokens_per_image,
                            e->ss));
  } else if (kind == LS_KIND_LM) {
    if (phase == 0) {
      KL(launch_embed_rows((const bf16*)e->g[0], e->text_ids, d.prompt_prefix, d.lm_d, e->lm_h,
                           d.lm_d, e->ss));
      KL(launch_embed_rows((const bf16*)e->g[0], e->text_ids + d.prompt_prefix, d.prompt_suffix,
                           d.lm_d, e->lm_h + static_cast<long>(d.prompt_prefix + vis_tokens(d)) * d.lm_d,
                           d.lm_d, e->ss));
    } else {
      KL(launch_embed_rows((const bf16*)e->g[0], e->token, 1, d.lm_d, e->dec_h, d.lm_d, e->ss));
    }
  } else {
    if (inv == 0)
      SSOP(cudaMemcpyAsync(e->actions, e->noise, 4ull * d.ex_tokens * d.action_dim,
                         cudaMemcpyDeviceToDevice, e->ss));
    KL(launch_time_embed((const float*)e->g[22], inv, d.time_dim, e->temb_in, e->ss));
    RC(gemv(e, GEMV_F32, e->gp_t1, e->g[13], e->temb_in, e->temb_mid, nullptr, (const float*)e->g[14]));
    KL(launch_silu_inplace(e->temb_mid, d.ex_d, e->ss));
    RC(gemv(e, GEMV_F32, e->gp_t2, e->g[15], e->temb_mid, e->temb, nullptr, (const float*)e->g[16]));
    KL(launch_action_in(e->actions, (const bf16*)e->g[17], (const bf16*)e->g[18], e->temb, e->Te,
                        d.action_dim, d.ex_d, e->ex_h, e->ss));
  }
  (void)io;
  return LS_OK;
}

int post_invocation(ls_exec* e, int kind, int phase, int inv, const ls_run_io* io) {
  const ls_dims& d = e->d;
  if (kind == LS_KIND_VIT) {
    const int T4 = e->Tv / 4, MD = 4 * d.vit_d;
    KL(launch_layernorm_rows(e->vit_h, (const bf16*)e->g[7], (const bf16*)e->g[8], e->vit_ln, e->Tv,
                             d.vit_d, d.vit_d, d.vit_eps, e->ss));
    RC(gemm(e, GEMM_BF16_GELU, e->g[9], MD, MD, T4, e->m_merge_in, e->merger_mid, MD, e->g[10]));
    RC(gemm(e, GEMM_F32, e->g[11], d.lm_d, MD, T4, e->m_merger_mid,
            e->lm_h + static_cast<long>(d.prompt_prefix) * d.lm_d, d.lm_d, e->g[12]));
  } else if (kind == LS_KIND_LM) {
    const int step = phase == 0 ? 0 : inv + 1;
    const float* x = phase == 0 ? e->lm_h + static_cast<long>(e->S - 1) * d.lm_d : e->dec_h;
    // vocab-parallel under TP: this rank scores its rows, its packed argmax key
    // carries the GLOBAL row index (GemvArgs.key_row0), and a MAX all-reduce of
    // the 8-byte key picks the global winner (ties -> lowest index, as on one GPU)
    GemvArgs head{};
    head.key_row0 = head_row0(d);
    RC(gemv(e, GEMV_ARGMAX, e->gp_head, e->g[1], x, e->logits + head_row0(d), e->g[2], nullptr,
            head_valid(d), &head));
    if (e->tp_on) {
      NcclApi& api = nccl_api();
      ncclResult_t r = api.all_reduce(e->amax, e->amax, 1, ncclUint64, ncclMax, e->comm, e->ss);
      if (r != ncclSuccess) return set_error(LS_ERR_NCCL, "ncclAllReduce(argmax): %s", api.error_string(r));
      if (io->logits_out) {  // tests: gather every rank's logits slice in place
        r = api.all_gather(e->logits + head_row0(d), e->logits, static_cast<size_t>(head_rows(d)),
                           ncclFloat32, e->comm, e->ss);
        if (r != ncclSuccess) return set_error(LS_ERR_NCCL, "ncclAllGather(logits): %s", api.error_string(r));
      }
      e->pdl_ok = false;
    }
    KL(launch_argmax_to_token(e->amax, e->token, e->hist, step, e->amax, e->ss));
    if (io->logits_out)
      SSOP(cudaMemcpyAsync(io->logits_out + static_cast<long>(step) * d.vocab, e->logits,
                         4ull * d.vocab, cudaMemcpyDeviceToDevice, e->ss));
  } else {
    KL(launch_action_out_euler(e->ex_h, (const bf16*)e->g[21], d.lm_eps, (const bf16*)e->g[19],
                               (const bf16*)e->g[20], e->Te, d.ex_d, d.action_dim,
                               -1.0f / d.euler_steps, e->actions, e->velocity, e->ss));
  }
  return LS_OK;
}

int run_layer(ls_exec* e, const Module& m, int phase, int inv, int l, const char* w,
              const CtView& ct = CtView()) {
  switch (m.kind) {
    case LS_KIND_VIT: return vit_layer(e, w, m.lay, ct);
    case LS_KIND_LM:
      return phase == 0 ? lm_prefill_layer(e, w, m.lay, l, ct)
                        : lm_decode_layer(e, w, m.lay, l, e->S + inv, ct);
    default: return expert_layer(e, w, m.lay, l, ct);
  }
}

// Slot ring + ECT decode scratch after the fixed allocations.  Slot = the
// largest staged layer (plain bytes, or the largest ECT blob of a compact
// module), so the reference's buffer term slots x max(layer_mem) holds with
// layer_mem = what a resident layer occupies.  Drops resident layers (the
// next ls_exec_set_placement re-creates them).
int finalize_layout(ls_exec* e) {
  ++e->gen;
  e->ar.used = e->mark0;
  e->bytes_slots = 0;
  e->slot_bytes = 0;
  uint64_t scratch = 0;
  for (auto& m : e->mods) {
    e->slot_bytes = std::max(e->slot_bytes, m.ct ? m.ct_stride : m.lay.total);
    if (m.ct && !e->ct_fused) scratch = std::max(scratch, align_up(m.lay.total, 256) + 256);
    // fused mode: multi-token-tile GEMMs (ViT, LM prefill) expand one matrix at a time
    if (m.ct && e->ct_fused)
      for (int i = 0; i < 4; ++i) scratch = std::max(scratch, align_up(m.lay.bytes[i], 256));
    std::fill(m.resident.begin(), m.resident.end(), nullptr);
  }
  for (int s = 0; s < e->n_slots; ++s)
    if (int rc = alloc_into(e, &e->slots[s], e->slot_bytes, &e->bytes_slots)) return rc;
  e->scratch = nullptr;
  e->scratch_bytes = 0;
  if (scratch) {
    if (int rc = alloc_into(e, &e->scratch, scratch, &e->scratch_bytes)) return rc;
  }
  e->mark = e->ar.used;
  return LS_OK;
}

}  // namespace

extern "C" {

int ls_layer_layout_of(const ls_dims* d, int32_t kind, ls_layer_layout* out) {
  if (kind == LS_KIND_VIT) layout_vit(d->vit_d, d->vit_heads, d->vit_hd, d->vit_ffn, out);
  else if (kind == LS_KIND_LM) layout_decoder(d->lm_d, d->lm_hq, d->lm_hkv, d->lm_hd, d->lm_ffn, out);
  else if (kind == LS_KIND_EXPERT) layout_decoder(d->ex_d, d->ex_hq, d->ex_hkv, d->ex_hd, d->ex_ffn, out);
  else return set_error(LS_ERR_VALUE, "unknown module kind %d", kind);
  return LS_OK;
}

int ls_global_size(const ls_dims* d, int32_t id, uint64_t* bytes) {
  if (id < 0 || id >= LS_N_GLOBAL) return set_error(LS_ERR_VALUE, "bad global id %d", id);
  *bytes = global_bytes(*d, id);
  return LS_OK;
}

int ls_exec_create(const ls_dims* dims, int32_t device, uint64_t cap_bytes, int32_t n_slots,
                   ls_exec** out) {
  ls_exec* e = new ls_exec();
  e->d = *dims;
  const ls_dims& d = e->d;
  e->dev = device;
  e->n_slots = n_slots < 1 ? 1 : n_slots;
  auto fail = [&](int rc) {
    ls_exec_destroy(e);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return fail(set_error(LS_ERR_CUDA, "cudaSetDevice(%d) failed", device));
  cudaDeviceGetAttribute(&e->nsm, cudaDevAttrMultiProcessorCount, device);
  if (d.lm_hd != (d.has_expert ? d.ex_hd : d.lm_hd) || (d.has_expert && d.ex_hkv != d.lm_hkv))
    return fail(set_error(LS_ERR_VALUE, "expert KV heads must match the LM's (joint attention)"));
  e->S = prompt_len(d);
  e->ctx = ctx_len(d);
  if (e->ctx > decode_attn_max_ctx())
    return fail(set_error(LS_ERR_VALUE,
                          "context of %d tokens (prompt %d + %d decode steps) exceeds the decode "
                          "attention limit of %d positions",
                          e->ctx, e->S, d.decode_steps, decode_attn_max_ctx()));
  e->Tv = d.has_vit ? d.vit_images * d.vit_tokens_per_image : 0;
  e->Te = d.has_expert ? d.ex_tokens : 0;
  e->vit_ffn_pad = n_kb(d.vit_ffn) * 64 > n_mt(d.vit_ffn) * 128 ? n_kb(d.vit_ffn) * 64 : n_mt(d.vit_ffn) * 128;
  // modules in profile order
  if (d.has_vit) {
    Module m{LS_KIND_VIT, d.vit_layers, {}, {}, {}, {1}};
    layout_vit(d.vit_d, d.vit_heads, d.vit_hd, d.vit_ffn, &m.lay);
    e->mods.push_back(m);
  }
  {
    Module m{LS_KIND_LM, d.lm_layers, {}, {}, {}, {1, d.decode_steps}};
    layout_decoder(d.lm_d, d.lm_hq, d.lm_hkv, d.lm_hd, d.lm_ffn, &m.lay);
    e->mods.push_back(m);
  }
  if (d.has_expert) {
    Module m{LS_KIND_EXPERT, d.ex_layers, {}, {}, {}, {d.euler_steps}};
    layout_decoder(d.ex_d, d.ex_hq, d.ex_hkv, d.ex_hd, d.ex_ffn, &m.lay);
    e->mods.push_back(m);
  }
  for (auto& m : e->mods) {
    m.host.assign(m.layers, nullptr);
    m.resident.assign(m.layers, nullptr);
    if (m.lay.total > e->slot_bytes) e->slot_bytes = m.lay.total;
  }
  if (cudaMalloc(&e->ar.base, cap_bytes) != cudaSuccess)
    return fail(set_error(LS_ERR_CUDA, "cudaMalloc of the %llu-byte VRAM arena failed",
                          static_cast<unsigned long long>(cap_bytes)));
  e->ar.cap = cap_bytes;
  if (cudaStreamCreateWithFlags(&e->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->ss, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_error(LS_ERR_CUDA, "stream creation failed"));
  // 1. DFB slot ring: events now, buffers in finalize_layout (slot size depends
  //    on which modules are stored compact)
  e->slots.assign(static_cast<size_t>(e->n_slots), nullptr);
  for (int s = 0; s < e->n_slots; ++s) {
    cudaEvent_t a, b;
    cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    e->dma_done.push_back(a);
    e->comp_done.push_back(b);
  }
  // 2. always-resident tensors
  for (int i = 0; i < LS_N_GLOBAL; ++i) {
    uint64_t b = global_bytes(d, i);
    if (!b) continue;
    if (int rc = alloc_into(e, &e->g[i], b, &e->bytes_always)) return fail(rc);
  }
  // 3. overhead: KV cache, activations, workspaces
  {
    const long S = e->S, Tv = e->Tv, Te = e->Te;
    const int QN = (d.lm_hq + 2 * d.lm_hkv) * d.lm_hd, AH = d.lm_hq * d.lm_hd;
    auto A = [&](void* dst, uint64_t bytes) { return alloc_into(e, dst, bytes, &e->bytes_overhead); };
#define OV(field, bytes) \
  if (int rc = A(&e->field, (bytes))) return fail(rc)
    // Phase scratch: ViT (0), LM prefill (1) and expert (2) activations are never
    // live at the same time, so they share one region sized for the largest set.
    std::vector<std::pair<char**, uint64_t>> sets[3], alias;
#define SC(set, field, bytes) sets[set].push_back({reinterpret_cast<char**>(&e->field), (bytes)})
    OV(kv, 2ull * d.lm_layers * 2 * d.lm_hkv * (e->ctx + 1) * d.lm_hd);
    OV(lm_h, 4ull * S * d.lm_d);
    SC(1, lm_norm, 2ull * S * d.lm_d);
    SC(1, lm_qkv, 2ull * S * QN);
    SC(1, lm_q, 2ull * S * AH);
    SC(1, lm_attn, 2ull * S * AH);
    SC(1, lm_mlp, 2ull * S * d.lm_ffn);
    OV(text_ids, 4ull * (d.prompt_prefix + d.prompt_suffix + 1));
    OV(dec_h, 4ull * d.lm_d);
    OV(dec_q, 4ull * AH);
    OV(dec_attn, 4ull * AH);
    OV(dec_mlp, 4ull * d.lm_ffn);
    OV(logits, 4ull * std::max<uint64_t>(d.vocab, static_cast<uint64_t>(head_rows(d)) *
                                                  std::max(1, d.tp_world)));
    OV(amax, 16);
    OV(token, 16);
    OV(hist, 4ull * (d.decode_steps + 1));
    // QKV and O (the short GEMVs, followed by attention / the gate|up GEMV) leave
    // 1/8 of the SMs free so the next kernel's CTAs start and prefetch while they
    // drain: measured in context, 128 of 148 SMs saves ~1 ms per inference (112: none)
    // LS_DIAG_GEMV_SMS="q,o,gu,down": per-GEMV grid override (diagnostics)
    const int small = e->nsm >= 16 ? e->nsm * 128 / 148 : e->nsm;  // 148 -> 128
    int gs[4] = {small, small, e->nsm, e->nsm};
    if (const char* ov = std::getenv("LS_DIAG_GEMV_SMS"))
      std::sscanf(ov, "%d,%d,%d,%d", &gs[0], &gs[1], &gs[2], &gs[3]);
    e->gp_qkv = plan_gemv(QN, d.lm_d, gs[0]);
    e->gp_o = plan_gemv(d.lm_d, AH, gs[1]);
    // QKV / O page rings capped at 3 slots (162 KiB): measured -0.4 ms per
    // inference against 4 (LS_DIAG_QO_SLOTS overrides)
    e->gp_qkv.slots = e->gp_o.slots = 3;
    e->gp_gu = plan_gemv(2 * d.lm_ffn, d.lm_d, gs[2]);
    e->gp_down = plan_gemv(d.lm_d, d.lm_ffn, gs[3]);
    e->gp_head = plan_gemv(head_rows(d), d.lm_d, e->nsm);
    std::vector<GemvPlan> plans = {e->gp_qkv, e->gp_o, e->gp_gu, e->gp_down, e->gp_head};
    if (d.has_expert) {
      e->gp_t1 = plan_gemv(d.ex_d, d.time_dim, e->nsm);
      e->gp_t2 = plan_gemv(d.ex_d, d.ex_d, e->nsm);
      plans.push_back(e->gp_t1);
      plans.push_back(e->gp_t2);
    }
    uint64_t ws = 0, cnt = 0;
    for (auto& p : plans) {
      ws = std::max<uint64_t>(ws, 4ull * n_mt(p.n) * p.max_contrib * 128);
      cnt = std::max<uint64_t>(cnt, 4ull * n_mt(p.n));
    }
    OV(gemv_ws, ws);
    OV(gemv_cnt, cnt);
    if (d.has_vit) {
      const int H = d.vit_heads * d.vit_hd;
      SC(0, vit_h, 4ull * Tv * d.vit_d);
      SC(0, vit_ln, 2ull * Tv * d.vit_d);
      SC(0, vit_qkv, 2ull * Tv * 3 * H);
      SC(0, vit_attn, 2ull * Tv * H);
      // dead-by-then buffers alias the qkv|attn pair: patches (before layer 0),
      // fc1 output (after proj consumed attn), merger hidden (after the last layer)
      alias.push_back({reinterpret_cast<char**>(&e->patches), 2ull * Tv * d.vit_patch_dim});
      alias.push_back({reinterpret_cast<char**>(&e->vit_fc1), 2ull * Tv * e->vit_ffn_pad});
      alias.push_back({reinterpret_cast<char**>(&e->merger_mid), 2ull * (Tv / 4) * 4 * d.vit_d});
    }
    if (d.has_expert) {
      const int EQN = (d.ex_hq + 2 * d.ex_hkv) * d.ex_hd, EAH = d.ex_hq * d.ex_hd;
      SC(2, ex_h, 4ull * Te * d.ex_d);
      SC(2, ex_norm, 2ull * Te * d.ex_d);
      SC(2, ex_qkv, 2ull * Te * EQN);
      SC(2, ex_q, 2ull * Te * EAH);
      SC(2, ex_kv, 2ull * 2 * d.ex_hkv * Te * d.ex_hd);
      SC(2, ex_attn, 2ull * Te * EAH);
      SC(2, ex_mlp, 2ull * Te * d.ex_ffn);
      OV(temb_in, 4ull * d.time_dim);
      OV(temb_mid, 4ull * d.ex_d);
      OV(temb, 4ull * d.ex_d);
      OV(actions, 4ull * Te * d.action_dim);
      OV(velocity, 4ull * Te * d.action_dim);
      OV(noise, 4ull * Te * d.action_dim);
      // split-K partials: one wave of 128 x 64 fp32 units
      e->gemm_ws_floats = static_cast<long>(e->nsm) * 128 * 64;
      e->gemm_cnt_n = e->nsm;
      OV(gemm_ws, 4ull * e->gemm_ws_floats);
      OV(gemm_cnt, 4ull * e->gemm_cnt_n);
      // GQA packing (2 query heads per CTA) measured slower in context (31.8-33.5 vs
      // 22.7 us per expert layer): off unless LS_DIAG_EX_GPACK=2
      e->ex_g_pack = 1;
      if (const char* ov = std::getenv("LS_DIAG_EX_GPACK"))
        e->ex_g_pack = (std::atoi(ov) == 2 && d.ex_hd == 128 && (d.ex_hq / d.ex_hkv) % 2 == 0) ? 2 : 1;
      e->ex_kv_splits = flash_kv_splits(Te, d.ex_hq / e->ex_g_pack, e->ctx + Te, e->nsm);
      if (const char* ov = std::getenv("LS_DIAG_EX_KV_SPLITS")) e->ex_kv_splits = std::atoi(ov);  // diagnostics
      if (const char* ov = std::getenv("LS_DIAG_DEC_SPLITS")) e->diag_dec_splits = std::atoi(ov);
      if (const char* ov = std::getenv("LS_DIAG_GU_SLOTS")) e->gp_gu.slots = std::atoi(ov);
      if (const char* ov = std::getenv("LS_DIAG_DOWN_SLOTS")) e->gp_down.slots = std::atoi(ov);
      if (const char* ov = std::getenv("LS_DIAG_QO_SLOTS")) e->gp_qkv.slots = e->gp_o.slots = std::atoi(ov);
    }
    // ViT aliases start at vit_qkv (entry 2 of set 0)
    e->tp_world = std::max(1, d.tp_world);
    e->tp_rank = d.tp_rank;
    e->tp_on = e->tp_world > 1 || d.tp_force;
    uint64_t scratch = 0, alias_off = 0;
    for (int si = 0; si < 3; ++si) {
      uint64_t sz = 0;
      for (size_t i = 0; i < sets[si].size(); ++i) {
        sz = align_up(sz, 1024);
        if (si == 0 && i == 2) alias_off = sz;
        sz += sets[si][i].second;
      }
      if (si == 0)
        for (auto& f : alias) sz = std::max(sz, alias_off + f.second);
      scratch = std::max(scratch, sz);
    }
    char* base = nullptr;
    if (int rc = A(&base, scratch)) return fail(rc);
    for (auto& s : sets) {
      uint64_t off = 0;
      for (auto& f : s) {
        off = align_up(off, 1024);
        *f.first = base + off;
        off += f.second;
      }
    }
    for (auto& f : alias) *f.first = base + alias_off;
#undef SC
#undef OV
    if (cudaMemset(e->ar.base, 0, e->ar.used) != cudaSuccess)
      return fail(set_error(LS_ERR_CUDA, "arena memset failed"));
    int rc = 0;
    const int AHe = d.ex_hq * d.ex_hd;
    if ((rc = tmap(&e->m_lm_norm, e->lm_norm, S, d.lm_d, d.lm_d)) ||
        (rc = tmap(&e->m_lm_attn, e->lm_attn, S, AH, AH)) ||
        (rc = tmap(&e->m_lm_mlp, e->lm_mlp, S, d.lm_ffn, d.lm_ffn)))
      return fail(rc);
    if (d.has_vit) {
      const int H = d.vit_heads * d.vit_hd;
      if ((rc = tmap(&e->m_patches, e->patches, Tv, d.vit_patch_dim, d.vit_patch_dim)) ||
          (rc = tmap(&e->m_vit_ln, e->vit_ln, Tv, d.vit_d, d.vit_d)) ||
          (rc = tmap(&e->m_vit_attn, e->vit_attn, Tv, H, H)) ||
          (rc = tmap(&e->m_vit_fc1, e->vit_fc1, Tv, e->vit_ffn_pad, e->vit_ffn_pad)) ||
          (rc = tmap(&e->m_merge_in, e->vit_ln, Tv / 4, 4 * d.vit_d, 4 * d.vit_d)) ||
          (rc = tmap(&e->m_merger_mid, e->merger_mid, Tv / 4, 4 * d.vit_d, 4 * d.vit_d)))
        return fail(rc);
    }
    if (d.has_expert) {
      if ((rc = tmap(&e->m_ex_norm, e->ex_norm, Te, d.ex_d, d.ex_d)) ||
          (rc = tmap(&e->m_ex_attn, e->ex_attn, Te, AHe, AHe)) ||
          (rc = tmap(&e->m_ex_mlp, e->ex_mlp, Te, d.ex_ffn, d.ex_ffn)))
        return fail(rc);
    }
  }
  e->mark0 = e->ar.used;
  if (int rc = finalize_layout(e)) return fail(rc);
  cudaEvent_t* evs[] = {&e->inv_done, &e->exe_done, &e->join_ev, &e->fork_ev};
  for (auto p : evs) cudaEventCreateWithFlags(p, cudaEventDisableTiming);
  cudaEvent_t* tevs[] = {&e->ev_begin, &e->ev_t0, &e->ev_t1, &e->ev_end};
  for (auto p : tevs) cudaEventCreate(p);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(set_error(LS_ERR_CUDA, "setup failed"));
  *out = e;
  return LS_OK;
}

int ls_exec_destroy(ls_exec* e) {
  if (!e) return LS_OK;
  if (e->ss) cudaStreamSynchronize(e->ss);
  if (e->cs) cudaStreamSynchronize(e->cs);
  for (auto v : e->dma_done) cudaEventDestroy(v);
  for (auto v : e->comp_done) cudaEventDestroy(v);
  for (auto v : e->tev) cudaEventDestroy(v);
  cudaEvent_t evs[] = {e->inv_done, e->exe_done, e->ev_begin, e->ev_t0, e->ev_t1, e->ev_end};
  for (auto v : evs)
    if (v) cudaEventDestroy(v);
  if (e->gexec) cudaGraphExecDestroy(e->gexec);
  if (e->join_ev) cudaEventDestroy(e->join_ev);
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->comm && nccl_api().ok) nccl_api().comm_destroy(e->comm);
  if (e->cs) cudaStreamDestroy(e->cs);
  if (e->ss) cudaStreamDestroy(e->ss);
  if (e->ar.base) cudaFree(e->ar.base);
  delete e;
  return LS_OK;
}

int ls_exec_global_ptr(ls_exec* e, int32_t id, void** dptr) {
  if (id < 0 || id >= LS_N_GLOBAL) return set_error(LS_ERR_VALUE, "bad global id %d", id);
  *dptr = e->g[id];
  return LS_OK;
}

int ls_nccl_unique_id(uint8_t out[128]) {
  NcclApi& api = nccl_api();
  if (!api.ok) return set_error(LS_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = api.get_unique_id(&id);
  if (r != ncclSuccess) return set_error(LS_ERR_NCCL, "ncclGetUniqueId: %s", api.error_string(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, 128);
  return LS_OK;
}

int ls_exec_set_tp(ls_exec* e, const uint8_t id_bytes[128]) {
  if (!e->tp_on) return set_error(LS_ERR_VALUE, "executor was created without tensor parallelism");
  NcclApi& api = nccl_api();
  if (!api.ok) return set_error(LS_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  CK(cudaSetDevice(e->dev));
  ncclResult_t r = api.comm_init_rank(&e->comm, e->tp_world, id, e->tp_rank);
  if (r != ncclSuccess) return set_error(LS_ERR_NCCL, "ncclCommInitRank: %s", api.error_string(r));
  return LS_OK;
}

int ls_exec_set_global_host(ls_exec* e, int32_t id, void* host_ptr) {
  if (id != 0 || !e->d.embed_on_host)
    return set_error(LS_ERR_VALUE, "only the embedding table (id 0) may live on the host");
  cudaPointerAttributes attr;
  CK(cudaPointerGetAttributes(&attr, host_ptr));
  if (attr.type != cudaMemoryTypeHost)
    return set_error(LS_ERR_VALUE, "embedding table must be page-locked host memory");
  e->g[0] = static_cast<char*>(attr.devicePointer ? attr.devicePointer : host_ptr);
  return LS_OK;
}

int ls_exec_set_host_layers(ls_exec* e, int32_t kind, const void* const* host_ptrs, int32_t n) {
  for (auto& m : e->mods) {
    if (m.kind != kind) continue;
    if (n != m.layers) return set_error(LS_ERR_VALUE, "expected %d host layers, got %d", m.layers, n);
    for (int i = 0; i < n; ++i) m.host[i] = static_cast<const char*>(host_ptrs[i]);
    return LS_OK;
  }
  return set_error(LS_ERR_VALUE, "module kind %d not present", kind);
}

int ls_exec_set_host_layers_ct(ls_exec* e, int32_t kind, const void* const* host_ptrs,
                               const uint64_t* bytes, int32_t n) {
  for (auto& m : e->mods) {
    if (m.kind != kind) continue;
    if (n != m.layers) return set_error(LS_ERR_VALUE, "expected %d host layers, got %d", m.layers, n);
    CK(cudaStreamSynchronize(e->ss));
    CK(cudaStreamSynchronize(e->cs));
    uint64_t worst = 0;
    for (int i = 0; i < n; ++i) {
      if (!host_ptrs[i] || bytes[i] < sizeof(EctHeader))
        return set_error(LS_ERR_VALUE, "ECT blob %d of module kind %d is missing or truncated", i, kind);
      const EctHeader* h = static_cast<const EctHeader*>(host_ptrs[i]);
      // the kernels derive page and tail offsets from the layout: the blob must
      // cover exactly the layout's tiled matrices (parts 0..3) and its sections
      // must lie inside the blob
      const uint64_t mat = m.lay.offset[3] + m.lay.bytes[3];
      const uint64_t tail = h->total - h->mat_bytes;
      if (h->magic != 0x31544345u || h->total != m.lay.total || h->mat_bytes != mat ||
          h->mat_bytes != static_cast<uint64_t>(h->n_pages) * 16384ull ||
          h->off_pages + static_cast<uint64_t>(h->n_pages) * 12288ull > bytes[i] ||
          h->off_tail + tail > bytes[i] ||
          h->off_excoff + 4ull * (h->n_pages + 1ull) > bytes[i] ||
          h->off_exc + 4ull * h->n_exc > bytes[i] ||
          (h->off_escmask && h->off_escmask + 16ull * h->n_pages > bytes[i]))
        return set_error(LS_ERR_VALUE, "ECT blob %d of module kind %d does not match the layer layout",
                         i, kind);
      worst = std::max<uint64_t>(worst, bytes[i]);
    }
    m.host_ct.assign(n, nullptr);
    for (int i = 0; i < n; ++i) m.host_ct[i] = static_cast<const char*>(host_ptrs[i]);
    m.ct_bytes.assign(bytes, bytes + n);
    m.ct_stride = align_up(worst, 256);
    m.ct = true;
    m.ct_order = static_cast<int>(reinterpret_cast<const EctHeader*>(host_ptrs[0])->order);
    for (int i = 1; i < n; ++i)
      if (static_cast<int>(reinterpret_cast<const EctHeader*>(host_ptrs[i])->order) != m.ct_order)
        return set_error(LS_ERR_VALUE, "ECT blobs of module kind %d mix page orders", kind);
    return finalize_layout(e);
  }
  return set_error(LS_ERR_VALUE, "module kind %d not present", kind);
}

int ls_exec_set_placement(ls_exec* e, const uint8_t* mask, int64_t n) {
  int64_t total = 0;
  for (auto& m : e->mods) total += m.layers;
  if (n != total) return set_error(LS_ERR_VALUE, "placement mask has %lld entries, expected %lld",
                                   static_cast<long long>(n), static_cast<long long>(total));
  CK(cudaStreamSynchronize(e->ss));
  CK(cudaStreamSynchronize(e->cs));
  ++e->gen;  // invalidates any captured graph (it holds the old resident pointers)
  e->ar.used = e->mark;
  for (auto& m : e->mods) std::fill(m.resident.begin(), m.resident.end(), nullptr);
  // all-or-nothing: on any failure no module keeps a pointer into the rewound
  // arena and no resident copy is left in flight -- every layer is streamed
  auto fail = [&](int rc) {
    cudaStreamSynchronize(e->cs);
    for (auto& m : e->mods) std::fill(m.resident.begin(), m.resident.end(), nullptr);
    e->ar.used = e->mark;
    return rc;
  };
  int64_t off = 0;
  for (auto& m : e->mods) {
    for (int l = 0; l < m.layers; ++l) {
      if (!mask[off + l]) continue;
      if (!m.host_of(l))
        return fail(set_error(LS_ERR_VALUE, "host layer %d of module kind %d not set", l, m.kind));
      const uint64_t foot = m.ct ? m.ct_stride : m.lay.total;
      char* p = e->ar.alloc(foot, 256);
      if (!p)
        return fail(set_error(LS_ERR_CAP,
                              "resident layers exceed the emulated VRAM cap (%llu bytes used of %llu)",
                              static_cast<unsigned long long>(e->ar.used),
                              static_cast<unsigned long long>(e->ar.cap)));
      cudaError_t ce = cudaMemcpyAsync(p, m.host_of(l), m.ct ? m.ct_bytes[l] : m.lay.total,
                                       cudaMemcpyHostToDevice, e->cs);
      if (ce != cudaSuccess)
        return fail(set_error(LS_ERR_CUDA, "cudaMemcpyAsync (resident layer): %s",
                              cudaGetErrorString(ce)));
      m.resident[l] = p;
    }
    off += m.layers;
  }
  cudaError_t ce = cudaStreamSynchronize(e->cs);
  if (ce != cudaSuccess)
    return fail(set_error(LS_ERR_CUDA, "cudaStreamSynchronize: %s", cudaGetErrorString(ce)));
  return LS_OK;
}

int ls_exec_memory(ls_exec* e, uint64_t out[7]) {
  out[0] = e->ar.cap;
  out[1] = e->ar.used;
  out[2] = e->ar.high;
  out[3] = e->bytes_slots;
  out[4] = e->bytes_always;
  out[5] = e->bytes_overhead + e->scratch_bytes;
  out[6] = e->ar.used - e->mark;
  return LS_OK;
}

int ls_exec_stats(ls_exec* e, int64_t out[3]) {
  out[0] = e->launches;    // kernels launched by the last run
  out[1] = e->h2d_copies;  // streamed-layer transfers of the last run
  out[2] = static_cast<int64_t>(e->h2d_bytes);
  return LS_OK;
}

int ls_exec_set_diag_skip(ls_exec* e, uint32_t mask) {
  e->diag_skip = mask;
  ++e->gen;  // re-capture
  return LS_OK;
}

int ls_exec_enqueue_us(ls_exec* e, double* us) {
  *us = e->enqueue_us;
  return LS_OK;
}

int ls_exec_streams(ls_exec* e, void** copy_stream, void** compute_stream) {
  *copy_stream = e->cs;
  *compute_stream = e->ss;
  return LS_OK;
}

int ls_exec_run(ls_exec* e, const ls_run_io* io, const ls_run_opts* opts, ls_event* events,
                int64_t capacity, int64_t* n_events, double* total_ms, double* e2e_ms) {
  const ls_dims& d = e->d;
  const bool seq = opts->cfg.mode == LS_MODE_SEQUENTIAL;
  const bool barrier = seq || !opts->cfg.cross_invocation_prefetch;
  const int nsl = std::max(1, std::min(opts->cfg.slot_count, e->n_slots));
  // 1: per-layer DMA / EXE events (the Timeline); 2: one EXE span per invocation
  // (events only around the layer loop, so PDL chaining inside it is untouched)
  const bool coarse = opts->record_timeline == 2 && events;
  const bool timing = opts->record_timeline == 1 && events;
  if (e->tp_on && !e->comm)
    return set_error(LS_ERR_VALUE, "tensor-parallel executor has no communicator (ls_exec_set_tp)");
  for (auto& m : e->mods)
    for (int l = 0; l < m.layers; ++l)
      if (!m.resident[l] && !m.host_of(l))
        return set_error(LS_ERR_VALUE, "host layer %d of module kind %d not set", l, m.kind);
  // timing event pool
  int64_t need = 0;
  for (auto& m : e->mods)
    for (int r : m.phase_reps) need += 4ll * r * m.layers;
  if (timing || coarse) {
    if (capacity * 2 < need) return set_error(LS_ERR_VALUE, "event buffer too small");
    while (static_cast<int64_t>(e->tev.size()) < need) {
      cudaEvent_t v;
      CK(cudaEventCreate(&v));
      e->tev.push_back(v);
    }
  }
  using Rec = RunRec;
  std::vector<Rec> recs;
  if (timing || coarse) recs.reserve(static_cast<size_t>(need / 2));
  int next_ev = 0;
  bool capturing = false;
  auto tick = [&](cudaStream_t s) {
    if (capturing) cudaEventRecordWithFlags(e->tev[next_ev], s, cudaEventRecordExternal);
    else cudaEventRecord(e->tev[next_ev], s);
    if (s == e->ss) e->pdl_ok = false;
    return next_ev++;
  };

  const auto host_t0 = std::chrono::steady_clock::now();
  const bool blind = opts->blind_offload != 0;
  if (blind)
    for (auto& m : e->mods)
      if (m.ct) return set_error(LS_ERR_VALUE, "blind offload runs plain (non-compact) layers only");
  const bool graph = e->use_graph && !timing && !blind;  // NCCL calls are capturable
  const uint64_t key[12] = {reinterpret_cast<uint64_t>(io->patches), reinterpret_cast<uint64_t>(io->text_ids),
                            reinterpret_cast<uint64_t>(io->noise), reinterpret_cast<uint64_t>(io->tokens_out),
                            reinterpret_cast<uint64_t>(io->actions_out), reinterpret_cast<uint64_t>(io->logits_out),
                            static_cast<uint64_t>(io->on_host), static_cast<uint64_t>(opts->cfg.mode),
                            static_cast<uint64_t>(opts->cfg.cross_invocation_prefetch),
                            static_cast<uint64_t>(nsl), e->gen, coarse ? 2ull : 1ull};
  const bool replay = graph && e->gexec && std::memcmp(key, e->gkey, sizeof(key)) == 0;
  capturing = graph && !replay;
  // timestamps inside a capture must be external event-record nodes
  auto rec = [&](cudaEvent_t ev) {
    return capturing ? cudaEventRecordWithFlags(ev, e->ss, cudaEventRecordExternal) : cudaEventRecord(ev, e->ss);
  };
  // the whole enqueue (as a lambda so a failure during capture can end it cleanly)
  auto enqueue = [&]() -> int {
  e->launches = 0;
  e->h2d_copies = 0;
  e->h2d_bytes = 0;
  const cudaMemcpyKind kin = io->on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CK(rec(e->ev_begin));
  if (d.has_vit && io->patches)
    CK(cudaMemcpyAsync(e->patches, io->patches, 2ull * e->Tv * d.vit_patch_dim, kin, e->ss));
  if (io->text_ids)
    CK(cudaMemcpyAsync(e->text_ids, io->text_ids, 4ull * (d.prompt_prefix + d.prompt_suffix), kin, e->ss));
  if (d.has_expert && io->noise)
    CK(cudaMemcpyAsync(e->noise, io->noise, 4ull * e->Te * d.action_dim, kin, e->ss));
  CK(rec(e->ev_t0));
  e->pdl_ok = false;
  // fork the copy stream off the compute stream (a plain event: timestamp
  // records inside a capture are external and create no dependencies)
  CK(cudaEventRecord(e->fork_ev, e->ss));
  CK(cudaStreamWaitEvent(e->cs, e->fork_ev, 0));

  std::vector<bool> slot_used(static_cast<size_t>(nsl), false);
  bool exe_rec = false;
  bool pending_barrier = false;
  for (int mi = 0; mi < static_cast<int>(e->mods.size()); ++mi) {
    const Module& m = e->mods[mi];
    for (int ph = 0; ph < static_cast<int>(m.phase_reps.size()); ++ph) {
      for (int inv = 0; inv < m.phase_reps[ph]; ++inv) {
        RC(pre_invocation(e, m.kind, ph, inv, io));
        const int span0 = coarse ? tick(e->ss) : -1;
        int sseq = 0;
        for (int l = 0; l < m.layers; ++l) {
          const char* w = m.resident[l];
          int slot = -1, dma0 = -1, dma1 = -1;
          if (!w) {
            slot = sseq++ % nsl;
            if (slot_used[slot]) CK(cudaStreamWaitEvent(e->cs, e->comp_done[slot], 0));
            if (seq && exe_rec) CK(cudaStreamWaitEvent(e->cs, e->exe_done, 0));
            if (pending_barrier) {
              CK(cudaStreamWaitEvent(e->cs, e->inv_done, 0));
              pending_barrier = false;
            }
            const uint64_t nbytes = m.ct ? m.ct_bytes[l] : m.lay.total;
            char* dst = e->slots[slot];
            if (timing) dma0 = tick(e->cs);
            if (blind) {
              // the layer's compute stream is idle (device-wide sync after every layer);
              // one host-blocking copy per weight tensor
              for (int i = 0; i < m.lay.n_parts; ++i) {
                CK(cudaMemcpyAsync(dst + m.lay.offset[i], m.host[l] + m.lay.offset[i], m.lay.bytes[i],
                                   cudaMemcpyHostToDevice, e->cs));
                CK(cudaStreamSynchronize(e->cs));
              }
            } else {
            CK(cudaMemcpyAsync(dst, m.ct ? m.host_ct[l] : m.host[l], nbytes,
                               cudaMemcpyHostToDevice, e->cs));
            }
            ++e->h2d_copies;
            e->h2d_bytes += nbytes;
            if (timing) dma1 = tick(e->cs);
            CK(cudaEventRecord(e->dma_done[slot], e->cs));
            SSOP(cudaStreamWaitEvent(e->ss, e->dma_done[slot], 0));
            w = e->slots[slot];
          }
          int x0 = timing ? tick(e->ss) : -1;
          CtView ct;
          if (m.ct && e->ct_fused) {
            ct = CtView(w, m.lay, m.ct_order);  // GEMV / GEMM kernels read the blob's pages directly
          } else if (m.ct) {
            // compact layer (slot or resident block) -> plain layer in the scratch;
            // the next kernel must not start early: its weight producer reads the scratch
            KL(launch_ect_decode_pages(reinterpret_cast<const uint8_t*>(w), 0,
                                       static_cast<uint32_t>((m.lay.offset[3] + m.lay.bytes[3]) / 16384),
                                       true, e->scratch, e->nsm, e->ss));
            e->pdl_ok = false;
            w = e->scratch;
          }
          RC(run_layer(e, m, ph, inv, l, w, ct));
          int x1 = timing ? tick(e->ss) : -1;
          if (slot >= 0) {
            SSOP(cudaEventRecord(e->comp_done[slot], e->ss));
            slot_used[slot] = true;
          }
          if (seq) {
            SSOP(cudaEventRecord(e->exe_done, e->ss));
            exe_rec = true;  // (events last recorded by another run / a capture are not waited on)
          }
          if (blind && slot >= 0) {  // module deletion + empty_cache: global synchronisation
            CK(cudaDeviceSynchronize());
            e->pdl_ok = false;
          }
          if (timing) {
            if (slot >= 0) recs.push_back({0, mi, ph, inv, l, dma0, dma1});
            recs.push_back({1, mi, ph, inv, l, x0, x1});
          }
        }
        if (coarse) recs.push_back({1, mi, ph, inv, -1, span0, tick(e->ss)});
        if (barrier) {
          SSOP(cudaEventRecord(e->inv_done, e->ss));
          pending_barrier = true;
        }
        RC(post_invocation(e, m.kind, ph, inv, io));
      }
    }
  }
  CK(rec(e->ev_t1));
  const cudaMemcpyKind kout = io->on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (io->tokens_out)
    CK(cudaMemcpyAsync(io->tokens_out, e->hist, 4ull * (d.decode_steps + 1), kout, e->ss));
  if (d.has_expert && io->actions_out)
    CK(cudaMemcpyAsync(io->actions_out, e->actions, 4ull * e->Te * d.action_dim, kout, e->ss));
  CK(rec(e->ev_end));
  if (capturing) {  // join the copy stream back into the origin stream
    CK(cudaEventRecord(e->join_ev, e->cs));
    CK(cudaStreamWaitEvent(e->ss, e->join_ev, 0));
  }
  return LS_OK;
  };
  if (capturing) {
    CK(cudaStreamBeginCapture(e->ss, cudaStreamCaptureModeRelaxed));
    const int rc = enqueue();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->ss, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CK(ce);
    if (e->gexec) cudaGraphExecDestroy(e->gexec);
    e->gexec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&e->gexec, g, 0);
    cudaGraphDestroy(g);
    CK(ie);
    std::memcpy(e->gkey, key, sizeof(key));
    e->grecs = recs;
  } else if (!replay) {
    RC(enqueue());
  }
  if (replay) recs = e->grecs;
  if (graph) CK(cudaGraphLaunch(e->gexec, e->ss));
  e->enqueue_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count();
  CK(cudaStreamSynchronize(e->ss));
  CK(cudaStreamSynchronize(e->cs));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e->ev_t0, e->ev_t1));
  *total_ms = ms;
  CK(cudaEventElapsedTime(&ms, e->ev_begin, e->ev_end));
  if (e2e_ms) *e2e_ms = ms;
  int64_t n = 0;
  if (timing || coarse) {
    for (const Rec& r : recs) {
      float a = 0.f, b = 0.f;
      CK(cudaEventElapsedTime(&a, e->ev_t0, e->tev[r.ev0]));
      CK(cudaEventElapsedTime(&b, e->ev_t0, e->tev[r.ev1]));
      ls_event& x = events[n++];
      x.engine = r.engine;
      x.module = r.module;
      x.phase = r.phase;
      x._pad = 0;
      x.invocation = r.inv;
      x.layer = r.layer;
      x.start_ms = a < 0 ? 0.0 : a;
      x.end_ms = b < a ? a : b;
    }
  }
  if (n_events) *n_events = n;
  return LS_OK;
}

}  // extern "C"
