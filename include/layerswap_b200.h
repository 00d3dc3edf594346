/*
 * layerswap_b200.h -- C ABI of the B200-native Pipelined Demand Layering library
 * (liblayerswap_b200.so).
 *
 * Three groups of entry points, one per north_star subsystem:
 *
 *   1. Residency policy + performance predictor + schedule model (host code,
 *      bit-exact with the reference `layerswap` package under CPython 3.12
 *      float semantics).  Each function replaces one reference function; the
 *      reference file:line is cited beside the declaration.
 *   2. The Double-Flat-Buffer (DFB) transfer engine and the model executor
 *      (CUDA, sm_100a): pinned host arena -> N-slot HBM ring on a dedicated
 *      copy stream, event hand-off to the compute stream, emulated VRAM cap.
 *      The reference models this engine in `dfbsim.simulate`
 *      (pkg/src/layerswap/dfbsim.py:179-247) and has no executable version.
 *   3. Kernel launchers (raw device pointers + shapes + cudaStream_t) used by
 *      the executor and by the parity tests.
 *
 * Conventions: every function returns int status (LS_OK == 0); on failure
 * ls_last_error() returns a thread-local message whose wording follows the
 * reference's exception messages (tests regex-match them).  No torch types
 * cross this boundary: plain pointers, sizes and POD structs only.
 */
#ifndef LAYERSWAP_B200_H
#define LAYERSWAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
#define LS_OK 0
#define LS_ERR_VALUE 1        /* Python ValueError                               */
#define LS_ERR_INFEASIBLE 2   /* planner.InfeasibleBudgetError (planner.py:34)   */
#define LS_ERR_CUDA 3         /* CUDA runtime failure -> RuntimeError            */
#define LS_ERR_CAP 4          /* emulated VRAM cap exceeded -> MemoryError       */
#define LS_ERR_NCCL 5         /* NCCL failure -> RuntimeError                    */

const char* ls_last_error(void);
const char* ls_version(void);

/* ---- profile data model (mirror of profile.py:54-166) ---------------------- */
typedef struct ls_phase {
  const char* name;
  int64_t repetitions;     /* PhaseProfile.repetitions  (profile.py:89)  */
  double dma_ms;           /* PhaseProfile.dma_ms                        */
  double exe_ms;           /* PhaseProfile.exe_ms                        */
} ls_phase;

typedef struct ls_module {
  const char* name;
  int64_t layers;          /* ModuleProfile.layers (profile.py:107)      */
  double layer_mem_mb;     /* ModuleProfile.layer_mem_mb                 */
  int32_t n_phases;
  const ls_phase* phases;
} ls_module;

typedef struct ls_profile {
  double vram_mb;            /* HardwareProfile.vram_mb (profile.py:64)   */
  double h2d_gbps;
  double overhead_mb;
  double always_resident_mb; /* ModelProfile.always_resident_mb (:136)    */
  int32_t n_modules;
  const ls_module* modules;
} ls_profile;

/* SimConfig (dfbsim.py:106-114) */
#define LS_MODE_SEQUENTIAL 0
#define LS_MODE_PIPELINED 1
typedef struct ls_simconfig {
  int32_t mode;
  int32_t cross_invocation_prefetch;
  int32_t slot_count;
} ls_simconfig;

/* SimEvent (dfbsim.py:117-125).  engine: 0 = copy, 1 = execute. */
typedef struct ls_event {
  int32_t engine;
  int32_t module;
  int32_t phase;
  int32_t _pad;
  int64_t invocation;
  int64_t layer;
  double start_ms;
  double end_ms;
} ls_event;

/* Placement (dfbsim.py:70-103): a resident mask of sum(layers) bytes laid out
 * module after module in profile order; mask[off(m) + i] != 0 <=> layer i of
 * module m is GPU-resident. */

/* Per-layer cost overrides (dfbsim.py:57, _phase_costs :161-176).
 * costs: for (module m, phase j) with has_override[flat(m,j)] != 0, the
 * 2*layers doubles (dma0, exe0, dma1, exe1, ...) start at
 * costs[cost_offset[flat(m,j)]].  flat(m,j) = sum_{m'<m} n_phases(m') + j. */
typedef struct ls_layer_costs {
  const uint8_t* has_override;
  const int64_t* cost_offset;
  const int64_t* n_entries;   /* entries supplied per (m,j); checked == layers */
  const double* costs;
} ls_layer_costs;

/* ---- analytic.py -------------------------------------------------------- */
/* classify (profile.py:177-187): *kind = 0 exe-intensive, 1 dma-intensive */
int ls_classify(const ls_phase* ph, int32_t* kind, double* ratio);
/* phase_time_full_offload (analytic.py:71-77) */
int ls_phase_time_full_offload(const ls_phase* ph, int64_t layers, double* out);
/* module_time_full_offload (analytic.py:80-82) */
int ls_module_time_full_offload(const ls_module* m, double* out);
/* lower_bound (analytic.py:85-90): per_module[n_modules], total */
int ls_lower_bound(const ls_profile* p, double* per_module, double* total);
/* residency_benefit (analytic.py:103-117); position 0 first, 1 middle, 2 last */
int ls_residency_benefit(const ls_module* m, int32_t position, double* delta_ms,
                         double* benefit_ms_per_mb);
/* consecutive_limit (analytic.py:120-132) */
int ls_consecutive_limit(const ls_phase* ph, int64_t* out);
/* crossover_tokens (analytic.py:161-171); *out = -1 encodes None */
int ls_crossover_tokens(const ls_module* target, const ls_module* other, int64_t cap,
                        int64_t* out);

/* ---- dfbsim.py ---------------------------------------------------------- */
/* simulate (dfbsim.py:179-247).  events may be NULL (total only, the
 * simulated_total fast path dfbsim.py:250-256); otherwise capacity must be
 * >= ls_event_capacity(p). costs may be NULL. */
int64_t ls_event_capacity(const ls_profile* p);
int ls_simulate(const ls_profile* p, const uint8_t* resident_mask, const ls_simconfig* cfg,
                const ls_layer_costs* costs, ls_event* events, int64_t capacity,
                int64_t* n_events, double* total_ms);
/* vram_report (dfbsim.py:259-276): out = {buffer, resident, always, overhead, total} */
int ls_vram_report(const ls_profile* p, const uint8_t* resident_mask, int32_t slot_count,
                   double out[5], int32_t* fits);

/* ---- planner.py --------------------------------------------------------- */
/* interleaved_indices (planner.py:67-83): writes k sorted indices */
int ls_interleaved_indices(int64_t k, int64_t layers, int64_t* out);

typedef struct ls_candidate {  /* Candidate (planner.py:38-47) */
  int32_t module;
  int32_t position;            /* 0 first, 1 middle, 2 last */
  double benefit_ms_per_mb;
  double delta_ms_per_layer;
  double layer_mem_mb;
  int64_t capacity;
} ls_candidate;
/* rank_candidates (planner.py:86-116); out must hold 3*n_modules entries */
int ls_rank_candidates(const ls_profile* p, ls_candidate* out, int32_t* n_out);
/* fixed_costs_mb (planner.py:119-126) */
int ls_fixed_costs_mb(const ls_profile* p, int32_t slot_count, double* out);
/* plan_for_budget (planner.py:145-185). mask_out: sum(layers) bytes.
 * sim_total is written only when include_simulated != 0. */
int ls_plan_for_budget(const ls_profile* p, double vram_budget_mb, const ls_simconfig* cfg,
                       int32_t include_simulated, uint8_t* mask_out, double* saving_ms,
                       double vram_out[5], int32_t* fits, double* sim_total_ms);
/* sweep (planner.py:188-206) over interleaved placements of one module */
int ls_sweep(const ls_profile* p, int32_t module, const int64_t* k_values, int32_t n_k,
             const ls_simconfig* cfg, double* sim_total_ms, double* vram_total_mb);

/* ---- predictor.py ------------------------------------------------------- */
/* slope_from_profile (predictor.py:53-59) */
int ls_slope_from_profile(const ls_module* m, double* out);
/* predict (predictor.py:62-72) */
int ls_predict(double intercept_s, double slope_ms_per_layer, const int64_t* k_values,
               int32_t n, double* predicted_s);
/* validate (predictor.py:75-104).  Rows come back sorted by k (n_rows = n_pred);
 * *has_fit = 0 when fewer than two rows (fitted_slope_s is None). */
int ls_validate(const int64_t* pred_k, const double* pred_s, int32_t n_pred,
                const int64_t* meas_k, const double* meas_s, int32_t n_meas,
                int64_t* row_k, double* row_pred, double* row_meas, double* row_err,
                double* max_abs_err, int32_t* has_fit, double* fitted_slope_s);
/* resolve_intercept (predictor.py:107-112); *source = 0 measured, 1 simulated.
 * calibration_total_s < 0 encodes None. */
int ls_resolve_intercept(const ls_profile* p, double calibration_total_s,
                         const ls_simconfig* cfg, double* intercept_s, int32_t* source);

/* ==== 2. DFB transfer engine + model executor (CUDA, sm_100a) ============== */
/* No reference function: the reference models this engine in
 * dfbsim.simulate (pkg/src/layerswap/dfbsim.py:179-247) and the paper's
 * Double Flat Buffer.  ls_exec_run executes the same
 * protocol on the GPU and returns the same event schema (ls_event) with CUDA
 * event timestamps, so timelines are interchangeable with ls_simulate's. */

/* Alpamayo-R1-10B-shaped synthetic stack (shapes SURVEY 8d). */
typedef struct ls_dims {
  int32_t has_vit, has_expert;
  /* 1: the token-embedding table stays in page-locked host memory and the
   * GPU gathers the rows it needs (zero-copy over PCIe) instead of holding
   * vocab x d bf16 (1.2 GB) under the VRAM cap. */
  int32_t embed_on_host;
  /* tensor parallelism: this rank holds 1/tp_world of every layer (per-rank
   * head / FFN counts below); row-parallel outputs are all-reduced (NCCL). */
  int32_t tp_world, tp_rank;
  int32_t tp_force; /* 1: take the all-reduce path even at tp_world == 1 (tests) */
  /* ViT encoder + patch merger */
  int32_t vit_layers, vit_d, vit_heads, vit_hd, vit_ffn, vit_patch_dim, vit_images,
      vit_tokens_per_image;
  /* language model (prefill + greedy decode) */
  int32_t lm_layers, lm_d, lm_hq, lm_hkv, lm_hd, lm_ffn, vocab, prompt_prefix, prompt_suffix,
      decode_steps;
  /* flow-matching action expert */
  int32_t ex_layers, ex_d, ex_hq, ex_hkv, ex_hd, ex_ffn, ex_tokens, action_dim, euler_steps,
      time_dim;
  float lm_eps, vit_eps, rope_theta, _pad;
} ls_dims;

#define LS_KIND_VIT 0
#define LS_KIND_LM 1
#define LS_KIND_EXPERT 2
#define LS_LAYOUT_MAX 16
typedef struct ls_layer_layout {
  int32_t n_parts, _pad;
  uint64_t offset[LS_LAYOUT_MAX];
  uint64_t bytes[LS_LAYOUT_MAX];
  uint64_t total;
} ls_layer_layout;
/* Flat per-layer buffer layout (one H2D copy per streamed layer). */
int ls_layer_layout_of(const ls_dims* d, int32_t kind, ls_layer_layout* out);

#define LS_N_GLOBAL 23
/* Byte size of always-resident tensor `id` (0 when its module is absent). */
int ls_global_size(const ls_dims* d, int32_t id, uint64_t* bytes);

typedef struct ls_exec ls_exec;
/* Device arena of cap_bytes (the emulated VRAM budget) holding DFB slots,
 * always-resident tensors, KV cache, activations and resident layers. */
int ls_exec_create(const ls_dims* d, int32_t device, uint64_t cap_bytes, int32_t n_slots,
                   ls_exec** out);
int ls_exec_destroy(ls_exec* e);
int ls_exec_global_ptr(ls_exec* e, int32_t id, void** dptr);
/* NCCL communicator for tensor parallelism (dims.tp_world > 1): every rank
 * passes the 128-byte id rank 0 obtained from ls_nccl_unique_id. */
int ls_nccl_unique_id(uint8_t out[128]);
int ls_exec_set_tp(ls_exec* e, const uint8_t id[128]);
/* Point an always-resident slot at page-locked host memory (embed_on_host). */
int ls_exec_set_global_host(ls_exec* e, int32_t id, void* host_ptr);
/* Pinned host buffers of every layer of one module (streamed source). */
int ls_exec_set_host_layers(ls_exec* e, int32_t kind, const void* const* host_ptrs, int32_t n);
/* ECT-compressed host blobs (exponent-coded tiles, ect.py) of one module: the
   module is then stored compact everywhere -- DFB slots and resident blocks
   hold blobs (resident footprint = largest blob, 256-aligned).  Blob layout:
   128-byte header (magic 'ECT1', page count, section offsets, exponent window,
   off_escmask), 12 KiB pages, raw vector tail, per-page exception offsets,
   16-byte per-page escape masks, exception list.  Decode GEMVs and 64-token
   GEMMs read the pages directly; multi-token-tile GEMMs expand one matrix
   into the decode scratch first.  Re-lays out the slot ring and drops
   resident layers (call ls_exec_set_placement afterwards). */
int ls_exec_set_host_layers_ct(ls_exec* e, int32_t kind, const void* const* host_ptrs,
                               const uint64_t* bytes, int32_t n);
/* Upload resident layers for a placement mask (module order vit, lm, expert). */
int ls_exec_set_placement(ls_exec* e, const uint8_t* mask, int64_t n);
/* out: cap, used, high_water, slots, always_resident, overhead, resident (bytes) */
int ls_exec_memory(ls_exec* e, uint64_t out[7]);
int ls_exec_streams(ls_exec* e, void** copy_stream, void** compute_stream);
/* out: kernels launched, streamed-layer H2D copies, H2D bytes -- of the last run */
int ls_exec_stats(ls_exec* e, int64_t out[3]);
/* Host wall time (us) the last ls_exec_run spent enqueueing work, i.e. before
   its final stream synchronisation (enqueue-bound when close to the device time). */
int ls_exec_enqueue_us(ls_exec* e, double* us);
/* Diagnostics: leave out kernels of the expert / LM decode layer (bit mask; results are
 * wrong -- timing only, tools/layer_breakdown.py).  0 = normal. */
int ls_exec_set_diag_skip(ls_exec* e, uint32_t mask);

typedef struct ls_run_io {
  int32_t on_host;         /* 1: pointers are pinned host memory (copies inside the run) */
  int32_t _pad;
  const void* patches;     /* bf16 [images*tokens_per_image x patch_dim] */
  const int32_t* text_ids; /* [prompt_prefix + prompt_suffix] */
  const float* noise;      /* [ex_tokens x action_dim] */
  int32_t* tokens_out;     /* [decode_steps + 1] */
  float* actions_out;      /* [ex_tokens x action_dim] */
  float* logits_out;       /* optional [(decode_steps + 1) x vocab] (device only) */
} ls_run_io;

typedef struct ls_run_opts {
  ls_simconfig cfg;
  int32_t record_timeline; /* 1: per-layer CUDA event timestamps; 2: one EXE span per
                              invocation (layer = -1), PDL chaining left intact */
  int32_t blind_offload;   /* 1: Accelerate-style blind offload baseline:
                              per-tensor synchronous copies of every streamed layer, no
                              copy/compute overlap, a device-wide sync after each layer;
                              plain (non-compact) modules only */
} ls_run_opts;

/* One inference.  total_ms: device time from the first layer transfer /
 * compute to the last (events t0..t1); e2e_ms: including input/output copies. */
int ls_exec_run(ls_exec* e, const ls_run_io* io, const ls_run_opts* opts, ls_event* events,
                int64_t capacity, int64_t* n_events, double* total_ms, double* e2e_ms);

/* Page-locked host arena for streamed layers (cudaHostAlloc, portable). */
int ls_host_alloc(uint64_t bytes, void** out);
int ls_host_free(void* p);
int ls_copy(void* dst, const void* src, uint64_t bytes);

/* ==== 3. kernel launchers (raw device pointers, shapes, cudaStream_t) ====== */
int ls_num_sms(int device, int32_t* out);
int ls_gemv_plan(int32_t n_mt, int32_t n_kb, int32_t num_sms, int32_t* grid, int32_t* max_contrib);
/* args points at the GemvArgs / DecodeAttnArgs / FlashArgs blocks of csrc/kernels.h;
   ls_k_args_size(0 GemvArgs, 1 DecodeAttnArgs, 2 FlashArgs) is the size the
   library was built with (binding layout check), -1 for an unknown kind. */
int64_t ls_k_args_size(int32_t kind);
int ls_k_gemv(int32_t epi, const void* args, int32_t grid, void* stream);
/* Programmatic dependent launch for the NEXT ls_k_* launch of this thread (how the
   executor launches every in-step kernel: its prologue -- barrier init, weight
   prefetch -- overlaps the previous kernel's tail; it reads activations only
   after griddepcontrol.wait). */
int ls_set_launch_pdl(int32_t on);
int ls_k_gemm(int32_t epi, const void* w_tiled, int32_t n_mt, int32_t n_kb, const void* x,
              int32_t T, int64_t ldx, void* out, int64_t ldo, const float* bias,
              const void* bias_bf16, int32_t n_valid, void* stream);
/* Same with a split-K workspace (fp32 partials + self-cleaning tile counters):
   skinny GEMMs (few 128-feature tiles) split K across CTAs, deterministic
   reduction in split order.  ls_gemm_splits: the split factor it will use.
   ct_blob != NULL: the weights are pages ct_page0.. of that ECT blob (w_tiled
   ignored), decoded into shared memory inside the kernel. */
int ls_k_gemm_ws(int32_t epi, const void* w_tiled, int32_t n_mt, int32_t n_kb, const void* x,
                 int32_t T, int64_t ldx, void* out, int64_t ldo, const float* bias,
                 const void* bias_bf16, int32_t n_valid, float* sk_ws, int64_t sk_ws_floats,
                 int32_t* sk_cnt, int32_t sk_cnt_n, const void* ct_blob, int32_t ct_page0,
                 void* stream);
int ls_gemm_splits(int32_t n_mt, int32_t n_kb, int32_t T, int32_t num_sms, int64_t ws_floats,
                   int32_t cnt_n);
int ls_k_decode_attention(const void* args, void* stream);
/* Diagnostic: `grid` CTAs each stream `per_cta` bytes from src through a ring of
   `stages` x `stage_bytes` TMA bulk copies (per-SM streaming bandwidth probe). */
int ls_probe_bulk_stream(const void* src, uint64_t per_cta, int32_t stage_bytes, int32_t stages,
                         int32_t grid, void* sink, void* stream);
/* Exponent-coded-tiles (ECT) blob -> plain packed layer (tiles + vectors).
   out must hold the plain size rounded up to 16 bytes. */
int ls_k_ect_decode(const void* blob, void* out, void* stream);
int ls_k_flash_attention(const void* args, void* stream);
int ls_k_rmsnorm_rows(const float* x, const void* w, void* out, int32_t T, int32_t D, float eps,
                      void* stream);
int ls_k_layernorm_rows(const float* x, const void* w, const void* b, void* out, int32_t T,
                        int32_t D, int64_t ld_out, float eps, void* stream);
int ls_k_qk_norm_rope(const void* qkv, int32_t T, int32_t hq, int32_t hkv, int32_t hd,
                      const void* qn_w, const void* kn_w, float eps, const void* rope, int32_t pos0,
                      void* q_out, void* k_cache, void* v_cache, int32_t cache_head_stride,
                      void* stream);

/* ---- CPython float helpers (exported for the parity tests) ---------------- */
double ls_py_sum(const double* x, int64_t n);      /* builtins.sum, CPython 3.12 */
double ls_py_floordiv(double a, double b);         /* float.__floordiv__          */
double ls_py_fsum(const double* x, int64_t n);     /* math.fsum                   */
double ls_py_sumprod(const double* a, const double* b, int64_t n); /* math.sumprod */

#ifdef __cplusplus
}
#endif
#endif /* LAYERSWAP_B200_H */
