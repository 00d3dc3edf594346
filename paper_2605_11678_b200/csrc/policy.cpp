// policy.cpp -- residency policy, performance predictor and DFB schedule model.
//
// Native, bit-exact replacement for the reference package's analytic.py,
// dfbsim.py (simulate/vram_report), planner.py and predictor.py.  "Bit-exact"
// means: the same IEEE-754 double operations in the same order as CPython 3.12
// evaluates the reference, including builtins.sum's Neumaier compensation and
// float floor division (see pyfloat.h).  Compile with -ffp-contract=off.
//
// The schedule model is not a translation of the reference loop: it is the
// same two-engine recurrence (copy engine / execute engine / slot release
// times) written once over flat cost arrays, shared by the event-emitting and
// the totals-only entry points.
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/layerswap_b200.h"
#include "pyfloat.h"

namespace lsb {

static thread_local std::string g_err;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

namespace {

enum Kind { EXE_INT = 0, DMA_INT = 1 };
enum Pos { FIRST = 0, MIDDLE = 1, LAST = 2 };

// profile.py:177-187 -- ratio < 1 is EXE-intensive; ties are DMA-intensive.
inline Kind kind_of(double dma, double exe) { return (dma / exe < 1.0) ? EXE_INT : DMA_INT; }

// analytic.py:93-100 -- one phase's per-inference saving at a position.
inline double position_delta(int64_t reps, double dma, double exe, int pos) {
  double r = static_cast<double>(reps);
  if (kind_of(dma, exe) == EXE_INT) return pos == FIRST ? r * dma : 0.0;
  if (pos == LAST) return r * (dma - exe);
  return r * dma;
}

// analytic.py:103-117 with an optional repetition override for one phase
// (analytic.py:147-152 middle_benefit_at_tokens).
inline double module_delta(const ls_module& m, int pos, int override_phase = -1,
                           int64_t override_reps = 0) {
  PySum s;
  for (int j = 0; j < m.n_phases; ++j) {
    const ls_phase& ph = m.phases[j];
    int64_t reps = (j == override_phase) ? override_reps : ph.repetitions;
    s.add(position_delta(reps, ph.dma_ms, ph.exe_ms, pos));
  }
  return s.result();
}

inline double max_layer_mem(const ls_profile& p) {
  double best = p.modules[0].layer_mem_mb;
  for (int i = 1; i < p.n_modules; ++i) best = py_max(best, p.modules[i].layer_mem_mb);
  return best;
}

inline int64_t total_layers(const ls_profile& p) {
  int64_t n = 0;
  for (int i = 0; i < p.n_modules; ++i) n += p.modules[i].layers;
  return n;
}

int check_profile(const ls_profile* p) {
  if (!p || p->n_modules < 1 || !p->modules)
    return set_error(LS_ERR_VALUE, "modules must be nonempty");
  for (int i = 0; i < p->n_modules; ++i) {
    const ls_module& m = p->modules[i];
    if (m.layers < 1) return set_error(LS_ERR_VALUE, "layers must be >= 1");
    if (m.n_phases < 1 || !m.phases) return set_error(LS_ERR_VALUE, "phases must be nonempty");
  }
  return LS_OK;
}

// Flat per-(module, phase, layer) cost table, honouring overrides
// (dfbsim.py:161-176).
struct CostTable {
  std::vector<int64_t> base;   // per flat phase: offset into dma/exe
  std::vector<double> dma, exe;
};

int build_costs(const ls_profile& p, const ls_layer_costs* ov, CostTable& t) {
  int flat = 0;
  for (int mi = 0; mi < p.n_modules; ++mi) {
    const ls_module& m = p.modules[mi];
    for (int j = 0; j < m.n_phases; ++j, ++flat) {
      const ls_phase& ph = m.phases[j];
      t.base.push_back(static_cast<int64_t>(t.dma.size()));
      if (ov && ov->has_override && ov->has_override[flat]) {
        int64_t n = ov->n_entries[flat];
        if (n != m.layers)
          return set_error(LS_ERR_VALUE,
                           "per-layer cost override for %s/%s has %" PRId64
                           " entries, expected %" PRId64,
                           m.name ? m.name : "?", ph.name ? ph.name : "?", n, m.layers);
        const double* c = ov->costs + ov->cost_offset[flat];
        for (int64_t l = 0; l < n; ++l) {
          double d = c[2 * l], e = c[2 * l + 1];
          if (!(d > 0) || !(e > 0))
            return set_error(LS_ERR_VALUE, "per-layer cost overrides must be positive");
          t.dma.push_back(d);
          t.exe.push_back(e);
        }
      } else {
        for (int64_t l = 0; l < m.layers; ++l) {
          t.dma.push_back(ph.dma_ms);
          t.exe.push_back(ph.exe_ms);
        }
      }
    }
  }
  return LS_OK;
}

// The DFB two-engine recurrence (dfbsim.py:11-37 rules; loop :199-246).
// Emits events when `ev` is non-null.
double run_schedule(const ls_profile& p, const uint8_t* mask, const ls_simconfig& cfg,
                    const CostTable& costs, ls_event* ev, int64_t* n_ev) {
  const bool sequential = cfg.mode == LS_MODE_SEQUENTIAL;
  const bool barrier = sequential || !cfg.cross_invocation_prefetch;
  const int slots = cfg.slot_count;
  std::vector<double> slot_free(static_cast<size_t>(slots), 0.0);
  double base = 0.0, copy_free = 0.0, exe_free = 0.0, last_end = 0.0;
  bool any_event = false;
  int64_t ne = 0;
  auto emit = [&](int engine, int mi, int j, int64_t inv, int64_t layer, double s, double e) {
    if (!any_event || e > last_end) last_end = e;
    any_event = true;
    if (ev) {
      ls_event& x = ev[ne];
      x.engine = engine;
      x.module = mi;
      x.phase = j;
      x._pad = 0;
      x.invocation = inv;
      x.layer = layer;
      x.start_ms = s;
      x.end_ms = e;
    }
    ++ne;
  };
  int flat = 0;
  int64_t mask_off = 0;
  for (int mi = 0; mi < p.n_modules; ++mi) {
    const ls_module& m = p.modules[mi];
    const uint8_t* res = mask ? mask + mask_off : nullptr;
    for (int j = 0; j < m.n_phases; ++j, ++flat) {
      const double* dma = costs.dma.data() + costs.base[flat];
      const double* exe = costs.exe.data() + costs.base[flat];
      for (int64_t inv = 0; inv < m.phases[j].repetitions; ++inv) {
        int64_t seq = 0;
        for (int64_t l = 0; l < m.layers; ++l) {
          if (res && res[l]) {
            double s = exe_free;
            exe_free = s + exe[l];
            emit(1, mi, j, inv, l, base + s, base + exe_free);
            continue;
          }
          int slot = static_cast<int>(seq % slots);
          double ds = sequential ? py_max(copy_free, exe_free) : py_max(copy_free, slot_free[slot]);
          double de = ds + dma[l];
          copy_free = de;
          emit(0, mi, j, inv, l, base + ds, base + de);
          double s = py_max(exe_free, de);
          exe_free = s + exe[l];
          emit(1, mi, j, inv, l, base + s, base + exe_free);
          slot_free[slot] = exe_free;
          ++seq;
        }
        if (barrier) {
          base += exe_free;
          copy_free = 0.0;
          exe_free = 0.0;
          std::fill(slot_free.begin(), slot_free.end(), 0.0);
        }
      }
    }
    mask_off += m.layers;
  }
  if (n_ev) *n_ev = ne;
  if (barrier) return base;
  return any_event ? last_end : 0.0;
}

// Placement.resident_mb (dfbsim.py:96-97)
double resident_mb(const ls_profile& p, const uint8_t* mask) {
  PySum s;
  int64_t off = 0;
  for (int i = 0; i < p.n_modules; ++i) {
    const ls_module& m = p.modules[i];
    int64_t count = 0;
    if (mask)
      for (int64_t l = 0; l < m.layers; ++l) count += mask[off + l] ? 1 : 0;
    s.add(static_cast<double>(count) * m.layer_mem_mb);
    off += m.layers;
  }
  return s.result();
}

void vram(const ls_profile& p, const uint8_t* mask, int slot_count, double out[5], int32_t* fits) {
  double buffer = static_cast<double>(slot_count) * max_layer_mem(p);
  double res = resident_mb(p, mask);
  double total = buffer + res + p.always_resident_mb + p.overhead_mb;
  out[0] = buffer;
  out[1] = res;
  out[2] = p.always_resident_mb;
  out[3] = p.overhead_mb;
  out[4] = total;
  if (fits) *fits = total <= p.vram_mb ? 1 : 0;
}

int interleave(int64_t k, int64_t layers, int64_t* out) {
  if (layers < 2) return set_error(LS_ERR_VALUE, "interleaved placement requires layers >= 2");
  if (k < 0) return set_error(LS_ERR_VALUE, "resident count must be >= 0");
  if (k > layers - 1)
    return set_error(LS_ERR_VALUE,
                     "resident count %" PRId64 " exceeds layers-1 = %" PRId64
                     ": the last layer must stay streamed",
                     k, layers - 1);
  for (int64_t i = 0; i < k; ++i) out[i] = i * (layers - 1) / k;
  return LS_OK;
}

int check_cfg(const ls_simconfig* cfg) {
  if (!cfg || cfg->slot_count < 1) return set_error(LS_ERR_VALUE, "slot_count must be >= 1");
  return LS_OK;
}

double simulated_total(const ls_profile& p, const uint8_t* mask, const ls_simconfig& cfg) {
  CostTable t;
  build_costs(p, nullptr, t);
  return run_schedule(p, mask, cfg, t, nullptr, nullptr);
}

}  // namespace
}  // namespace lsb

using namespace lsb;

extern "C" {

const char* ls_last_error(void) { return g_err.c_str(); }

double ls_py_sum(const double* x, int64_t n) {
  PySum s;
  for (int64_t i = 0; i < n; ++i) s.add(x[i]);
  return s.result();
}
double ls_py_floordiv(double a, double b) { return py_floordiv(a, b); }
double ls_py_fsum(const double* x, int64_t n) { return py_fsum(x, n); }
double ls_py_sumprod(const double* a, const double* b, int64_t n) { return py_sumprod(a, b, n); }

int ls_classify(const ls_phase* ph, int32_t* kind, double* ratio) {
  double r = ph->dma_ms / ph->exe_ms;
  if (ratio) *ratio = r;
  if (kind) *kind = r < 1.0 ? 0 : 1;
  return LS_OK;
}

int ls_phase_time_full_offload(const ls_phase* ph, int64_t layers, double* out) {
  if (layers < 1) return set_error(LS_ERR_VALUE, "layers must be >= 1");
  double r = static_cast<double>(ph->repetitions), L = static_cast<double>(layers);
  if (kind_of(ph->dma_ms, ph->exe_ms) == EXE_INT)
    *out = r * (ph->dma_ms + L * ph->exe_ms);
  else
    *out = r * (L * ph->dma_ms + ph->exe_ms);
  return LS_OK;
}

int ls_module_time_full_offload(const ls_module* m, double* out) {
  PySum s;
  for (int j = 0; j < m->n_phases; ++j) {
    double t;
    int rc = ls_phase_time_full_offload(&m->phases[j], m->layers, &t);
    if (rc) return rc;
    s.add(t);
  }
  *out = s.result();
  return LS_OK;
}

int ls_lower_bound(const ls_profile* p, double* per_module, double* total) {
  if (int rc = check_profile(p)) return rc;
  PySum tot;
  for (int i = 0; i < p->n_modules; ++i) {
    const ls_module& m = p->modules[i];
    PySum s;
    for (int j = 0; j < m.n_phases; ++j)  // (R * L) is an exact int product first
      s.add(static_cast<double>(m.phases[j].repetitions * m.layers) * m.phases[j].exe_ms);
    double v = s.result();
    if (per_module) per_module[i] = v;
    tot.add(v);
  }
  *total = tot.result();
  return LS_OK;
}

int ls_residency_benefit(const ls_module* m, int32_t position, double* delta_ms,
                         double* benefit_ms_per_mb) {
  if (position < 0 || position > 2) return set_error(LS_ERR_VALUE, "bad position %d", position);
  double d = module_delta(*m, position);
  if (delta_ms) *delta_ms = d;
  if (benefit_ms_per_mb) *benefit_ms_per_mb = d / m->layer_mem_mb;
  return LS_OK;
}

int ls_consecutive_limit(const ls_phase* ph, int64_t* out) {
  if (kind_of(ph->dma_ms, ph->exe_ms) == EXE_INT)
    return set_error(LS_ERR_VALUE,
                     "consecutive residency limit undefined for phase '%s': transfers already "
                     "hide behind execution (ratio < 1)",
                     ph->name ? ph->name : "?");
  *out = static_cast<int64_t>(std::floor(ph->dma_ms / ph->exe_ms));
  return LS_OK;
}

int ls_crossover_tokens(const ls_module* target, const ls_module* other, int64_t cap,
                        int64_t* out) {
  double threshold = 0.0;
  for (int pos = 0; pos < 3; ++pos) {
    double b = module_delta(*other, pos) / other->layer_mem_mb;
    threshold = pos == 0 ? b : py_max(threshold, b);
  }
  *out = -1;
  for (int64_t n = 1; n <= cap; ++n) {
    int idx = -1;  // analytic.py:129-140 last DMA-intensive phase
    for (int j = target->n_phases - 1; j >= 0; --j)
      if (kind_of(target->phases[j].dma_ms, target->phases[j].exe_ms) == DMA_INT) {
        idx = j;
        break;
      }
    if (idx < 0)
      return set_error(LS_ERR_VALUE,
                       "module '%s' has no transfer-bound phase whose repetitions could "
                       "parameterize a token count",
                       target->name ? target->name : "?");
    double b = module_delta(*target, MIDDLE, idx, n) / target->layer_mem_mb;
    if (b > threshold) {
      *out = n;
      return LS_OK;
    }
  }
  return LS_OK;
}

int64_t ls_event_capacity(const ls_profile* p) {
  int64_t n = 0;
  for (int i = 0; i < p->n_modules; ++i)
    for (int j = 0; j < p->modules[i].n_phases; ++j)
      n += 2 * p->modules[i].layers * p->modules[i].phases[j].repetitions;
  return n;
}

int ls_simulate(const ls_profile* p, const uint8_t* mask, const ls_simconfig* cfg,
                const ls_layer_costs* costs, ls_event* events, int64_t capacity,
                int64_t* n_events, double* total_ms) {
  if (int rc = check_profile(p)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  if (events && capacity < ls_event_capacity(p))
    return set_error(LS_ERR_VALUE, "event buffer too small");
  CostTable t;
  if (int rc = build_costs(*p, costs, t)) return rc;
  *total_ms = run_schedule(*p, mask, *cfg, t, events, n_events);
  return LS_OK;
}

int ls_vram_report(const ls_profile* p, const uint8_t* mask, int32_t slot_count, double out[5],
                   int32_t* fits) {
  if (int rc = check_profile(p)) return rc;
  vram(*p, mask, slot_count, out, fits);
  return LS_OK;
}

int ls_interleaved_indices(int64_t k, int64_t layers, int64_t* out) {
  return interleave(k, layers, out);
}

int ls_rank_candidates(const ls_profile* p, ls_candidate* out, int32_t* n_out) {
  if (int rc = check_profile(p)) return rc;
  std::vector<ls_candidate> c;
  for (int mi = 0; mi < p->n_modules; ++mi) {
    const ls_module& m = p->modules[mi];
    int64_t caps[3] = {1, std::max<int64_t>(m.layers - 2, 0), m.layers >= 2 ? 1 : 0};
    for (int pos = 0; pos < 3; ++pos) {
      if (caps[pos] == 0) continue;
      double d = module_delta(m, pos);
      c.push_back({mi, pos, d / m.layer_mem_mb, d, m.layer_mem_mb, caps[pos]});
    }
  }
  // key (-benefit, module order, first < middle < last) -- planner.py:113-115
  std::stable_sort(c.begin(), c.end(), [](const ls_candidate& a, const ls_candidate& b) {
    double ka = -a.benefit_ms_per_mb, kb = -b.benefit_ms_per_mb;
    if (ka != kb) return ka < kb;
    if (a.module != b.module) return a.module < b.module;
    return a.position < b.position;
  });
  for (size_t i = 0; i < c.size(); ++i) out[i] = c[i];
  *n_out = static_cast<int32_t>(c.size());
  return LS_OK;
}

int ls_fixed_costs_mb(const ls_profile* p, int32_t slot_count, double* out) {
  if (int rc = check_profile(p)) return rc;
  *out = static_cast<double>(slot_count) * max_layer_mem(*p) + p->always_resident_mb +
         p->overhead_mb;
  return LS_OK;
}

int ls_plan_for_budget(const ls_profile* p, double budget, const ls_simconfig* cfg,
                       int32_t include_simulated, uint8_t* mask_out, double* saving_ms,
                       double vram_out[5], int32_t* fits, double* sim_total_ms) {
  if (int rc = check_profile(p)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  double fixed;
  ls_fixed_costs_mb(p, cfg->slot_count, &fixed);
  if (budget < fixed)
    return set_error(LS_ERR_INFEASIBLE,
                     "budget %g MB is below fixed costs %g MB (streaming buffers + "
                     "always-resident components + overhead)",
                     budget, fixed);
  std::vector<ls_candidate> cands(static_cast<size_t>(3 * p->n_modules));
  int32_t nc = 0;
  ls_rank_candidates(p, cands.data(), &nc);
  double remaining = budget - fixed;
  double saving = 0.0;
  std::vector<int64_t> picks(static_cast<size_t>(3 * p->n_modules), 0);
  for (int i = 0; i < nc; ++i) {
    const ls_candidate& c = cands[i];
    double q = py_floordiv(remaining, c.layer_mem_mb);  // int(remaining // mem)
    if (std::isnan(q)) return set_error(LS_ERR_VALUE, "cannot convert float NaN to integer");
    if (std::isinf(q)) return set_error(LS_ERR_VALUE, "cannot convert float infinity to integer");
    int64_t take;
    if (q >= static_cast<double>(c.capacity))
      take = c.capacity;
    else
      take = static_cast<int64_t>(q);  // q is integral; truncation == int()
    if (take <= 0) continue;
    remaining -= static_cast<double>(take) * c.layer_mem_mb;
    saving += static_cast<double>(take) * c.delta_ms_per_layer;
    picks[static_cast<size_t>(3 * c.module + c.position)] = take;
  }
  // _materialize (planner.py:129-142)
  int64_t off = 0;
  for (int mi = 0; mi < p->n_modules; ++mi) {
    const ls_module& m = p->modules[mi];
    uint8_t* mm = mask_out + off;
    std::memset(mm, 0, static_cast<size_t>(m.layers));
    int64_t k = picks[3 * mi + FIRST] + picks[3 * mi + MIDDLE];
    if (m.layers >= 2) {
      std::vector<int64_t> idx(static_cast<size_t>(k));
      if (int rc = interleave(k, m.layers, idx.data())) return rc;
      for (int64_t v : idx) mm[v] = 1;
    } else {
      for (int64_t l = 0; l < k; ++l) mm[l] = 1;
    }
    if (picks[3 * mi + LAST]) mm[m.layers - 1] = 1;
    off += m.layers;
  }
  *saving_ms = saving;
  vram(*p, mask_out, cfg->slot_count, vram_out, fits);
  if (include_simulated && sim_total_ms) *sim_total_ms = simulated_total(*p, mask_out, *cfg);
  return LS_OK;
}

int ls_sweep(const ls_profile* p, int32_t module, const int64_t* k_values, int32_t n_k,
             const ls_simconfig* cfg, double* sim_total_ms, double* vram_total_mb) {
  if (int rc = check_profile(p)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  if (module < 0 || module >= p->n_modules) return set_error(LS_ERR_VALUE, "no such module");
  int64_t off = 0;
  for (int i = 0; i < module; ++i) off += p->modules[i].layers;
  const int64_t L = p->modules[module].layers;
  std::vector<uint8_t> mask(static_cast<size_t>(total_layers(*p)), 0);
  CostTable t;
  build_costs(*p, nullptr, t);
  for (int32_t i = 0; i < n_k; ++i) {
    int64_t k = k_values[i];
    std::vector<int64_t> idx(static_cast<size_t>(k > 0 ? k : 0));
    if (int rc = interleave(k, L, idx.data())) return rc;
    std::fill(mask.begin(), mask.end(), 0);
    for (int64_t v : idx) mask[static_cast<size_t>(off + v)] = 1;
    sim_total_ms[i] = run_schedule(*p, mask.data(), *cfg, t, nullptr, nullptr);
    double out[5];
    vram(*p, mask.data(), cfg->slot_count, out, nullptr);
    vram_total_mb[i] = out[4];
  }
  return LS_OK;
}

int ls_slope_from_profile(const ls_module* m, double* out) {
  *out = module_delta(*m, MIDDLE);
  return LS_OK;
}

int ls_predict(double intercept_s, double slope, const int64_t* k_values, int32_t n,
               double* predicted_s) {
  if (!(intercept_s > 0)) return set_error(LS_ERR_VALUE, "intercept_s must be > 0");
  for (int32_t i = 0; i < n; ++i) {
    if (k_values[i] < 0) return set_error(LS_ERR_VALUE, "resident counts must be >= 0");
    predicted_s[i] = intercept_s - static_cast<double>(k_values[i]) * slope / 1000.0;
  }
  return LS_OK;
}

static std::string list_repr(std::vector<int64_t> v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += ", ";
    s += std::to_string(v[i]);
  }
  return s + "]";
}

// dict(...) keeps the last value for a repeated key; returns keys sorted.
static void last_wins(const int64_t* k, const double* v, int32_t n, std::vector<int64_t>& keys,
                      std::vector<double>& vals) {
  std::vector<std::pair<int64_t, double>> kv;
  for (int32_t i = 0; i < n; ++i) {
    bool found = false;
    for (auto& e : kv)
      if (e.first == k[i]) {
        e.second = v[i];
        found = true;
      }
    if (!found) kv.push_back({k[i], v[i]});
  }
  std::sort(kv.begin(), kv.end(),
            [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
              return a.first < b.first;
            });
  keys.clear();
  vals.clear();
  for (auto& e : kv) {
    keys.push_back(e.first);
    vals.push_back(e.second);
  }
}

int ls_validate(const int64_t* pred_k, const double* pred_s, int32_t n_pred, const int64_t* meas_k,
                const double* meas_s, int32_t n_meas, int64_t* row_k, double* row_pred,
                double* row_meas, double* row_err, double* max_abs_err, int32_t* has_fit,
                double* fitted_slope_s) {
  std::vector<int64_t> pk, mk;
  std::vector<double> pv, mv;
  last_wins(pred_k, pred_s, n_pred, pk, pv);
  last_wins(meas_k, meas_s, n_meas, mk, mv);
  if (pk != mk) {
    std::string a = list_repr(mk), b = list_repr(pk);
    return set_error(LS_ERR_VALUE, "measured k values %s do not match predicted k values %s",
                     a.c_str(), b.c_str());
  }
  const size_t n = pk.size();
  double best = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double meas = mv[i];
    if (!(meas > 0))
      return set_error(LS_ERR_VALUE, "measured time for k=%" PRId64 " must be > 0", pk[i]);
    double err = (pv[i] - meas) / meas * 100.0;
    row_k[i] = pk[i];
    row_pred[i] = pv[i];
    row_meas[i] = meas;
    row_err[i] = err;
    double a = std::fabs(err);
    best = i == 0 ? a : py_max(best, a);
  }
  if (n == 0) return set_error(LS_ERR_VALUE, "max() arg is an empty sequence");
  *max_abs_err = best;
  *has_fit = 0;
  if (n >= 2) {  // statistics.linear_regression (CPython 3.12)
    std::vector<double> x(n), y(n);
    for (size_t i = 0; i < n; ++i) x[i] = static_cast<double>(pk[i]);
    double xbar = py_fsum(x.data(), static_cast<int64_t>(n)) / static_cast<double>(n);
    double ybar = py_fsum(mv.data(), static_cast<int64_t>(n)) / static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) {
      x[i] = x[i] - xbar;
      y[i] = mv[i] - ybar;
    }
    double sxy = py_sumprod(x.data(), y.data(), static_cast<int64_t>(n)) + 0.0;
    double sxx = py_sumprod(x.data(), x.data(), static_cast<int64_t>(n));
    *fitted_slope_s = -(sxy / sxx);
    *has_fit = 1;
  }
  return LS_OK;
}

int ls_resolve_intercept(const ls_profile* p, double calibration_total_s, const ls_simconfig* cfg,
                         double* intercept_s, int32_t* source) {
  if (calibration_total_s >= 0) {
    *intercept_s = calibration_total_s;
    *source = 0;
    return LS_OK;
  }
  if (int rc = check_profile(p)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  *intercept_s = simulated_total(*p, nullptr, *cfg) / 1000.0;
  *source = 1;
  return LS_OK;
}

}  // extern "C"

extern "C" const char* ls_version(void) { return "0.1.0"; }
