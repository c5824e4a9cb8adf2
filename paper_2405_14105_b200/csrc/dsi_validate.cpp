// dsi_validate.cpp -- validation and tick conversion of the configs (R15), the device
// config rows, launch limits and the Eq. 1 planner helpers.
#include "dsi_host.h"

#include <algorithm>
#include <atomic>
#include <cmath>

using namespace dsih;

namespace dsih {

thread_local std::string g_create_error;

}  // namespace dsih

namespace dsi {
// ceil(2^32 / d) split into low word and bit 32 (d >= 1): divisors below 2^16 (every lookahead,
// SP and N the planner sees in practice) come from a table built once -- make_dev_cfg needs
// three per config, millions of times per update
void magic_table(uint32_t d, uint32_t &lo, uint32_t &hi) {
  static const std::vector<uint64_t> table = [] {
    std::vector<uint64_t> t(1u << 16, 0);
    for (uint32_t x = 1; x < (1u << 16); ++x) t[x] = ((1ull << 32) + x - 1) / x;
    return t;
  }();
  const uint64_t m = d < (1u << 16) ? table[d] : ((1ull << 32) + d - 1) / d;
  lo = (uint32_t)m;
  hi = (uint32_t)(m >> 32);
}
}  // namespace dsi

namespace dsih {

dsi_status to_ticks(double x, double tick, int64_t *out) { return (dsi_status)dsi::to_ticks(x, tick, out); }

// The message of convert_config's code for config i.
std::string convert_message(size_t i, int code) {
  const char *what = "invalid configuration";
  switch (code >> 8) {
    case dsi::CV_ACCEPT: what = "accept_rate must be in [0, 1]"; break;
    case dsi::CV_LOOKAHEAD: what = "lookahead must be >= 1"; break;
    case dsi::CV_SP: what = "sp_degree must be >= 1"; break;
    case dsi::CV_N: what = "n_tokens must be in [1, 32768]"; break;
    case dsi::CV_TRIALS: what = "n_trials must be in [1, 2^32]"; break;
    case dsi::CV_PATTERN_N: what = "DSI_F_PATTERN needs n_tokens <= 33"; break;
    case dsi::CV_T_TARGET: what = "t_target is not a positive whole number of ticks"; break;
    case dsi::CV_T_DRAFTER: what = "t_drafter is not a positive whole number of ticks"; break;
    case dsi::CV_ASSUMPTION2: what = "t_drafter > t_target violates Assumption 2 (P:187-189)"; break;
    case dsi::CV_TTFT_TARGET: what = "ttft_target is not 0 or a positive whole number of ticks"; break;
    case dsi::CV_TTFT_DRAFTER: what = "ttft_drafter is not 0 or a positive whole number of ticks"; break;
    case dsi::CV_ASSUMPTION2_FIRST: what = "ttft_drafter > ttft_target violates Assumption 2"; break;
    case dsi::CV_SHARED_TTFT: what = "DSI_F_SHARED_STREAMS does not support the TTFT variant"; break;
    case dsi::CV_FRESH_TTFT: what = "DSI_F_FRESH_VERIFIER does not support the TTFT variant"; break;
    case dsi::CV_BOUND: what = "N*(k*t_drafter + t_target) must stay below 2^31 ticks"; break;
    case dsi::CV_BOUND_SQ: what = "n_trials * bound^2 must stay below 2^64"; break;
    case dsi::CV_STRICT_EQ1: what = "Eq. 1 violated: ceil(t_t/(k t_d)) > SP"; break;
  }
  char buf[256];
  std::snprintf(buf, sizeof buf, "config %zu: %s", i, what);
  return buf;
}

dsi_status convert(const dsi_options &opt, const dsi_config &c, size_t i, CfgTicks &o, std::string &msg) {
  const int code = dsi::convert_config(opt.tick, opt.flags, c, o);
  if (code == 0) return DSI_OK;
  msg = convert_message(i, code);
  return (dsi_status)(code & 0xff);
}

// The sharder's cost models, in picoseconds of kernel time on one B200, fitted to measured
// launches of >= ~1 ms (profiles/r02_cost_probe_v2.jsonl, r02_cost_probe_shared_v2.jsonl: grids
// of identical-shape configs, a in {0 .. 1}, k in {1, 2, 5, 20, 200}, N in {100, 1000}).
//
// Per-config kernel, one trial of N tokens: the Philox draw dominates and is paid only when
// 0 < a < 1 (~0.6-0.75 ps per token, almost independent of a); all-reject and all-accept
// configs cost ~0.03-0.15.  A lookahead 2 <= k_eff <= 30 adds the segment walk (+0.07, most at
// a ~ 0.5-0.7); k = 1 and k_eff > 30 (the closed per-word path) do not.
double unit_cost(const CfgTicks &t, uint64_t trials) {
  const int32_t keff = std::min(t.k, t.n);
  const bool walk = keff >= 2 && keff <= 30;
  double c;
  if (t.thr == 0) c = keff == 1 ? 0.075 : (walk ? 0.13 : 0.09);  // all reject
  else if (t.thr >= (1ull << 32)) c = keff == 1 ? 0.03 : 0.06;    // all accept
  else c = 0.62 + (walk ? 0.07 + 0.2 * t.a * (1.0 - t.a) : 0.0);
  return (double)trials * (double)t.n * c;
}

// Shared-stream mode, pass 2, one trial of one config: the record scan (linear in N, more with
// a run list: 0 < a < 1), then per trial with a stored run of L > k_eff (every run of L >= 2
// for a fresh-verifier config; P = 1 - exp(-E[runs]), E[runs] = (N(1-a) + 1) a^(k+1)) a visit
// growing with the runs' length, plus a correction per run.  The two forms differ (two-pass:
// N = 100 fit, median model/measured 1.01, range 0.88-1.10; fused 128-thread form: N = 1000
// fit, 1.00, 0.75-1.26); the fused form's own stream pass is costed per slice by the caller.
double shared_eval_cost(const CfgTicks &t, bool fresh, bool two_pass) {
  const double n = t.n, a = t.a;
  const int32_t keff = (fresh && t.kd > t.t_t) ? 1 : std::min(t.k, t.n);
  const bool stream = t.thr != 0 && t.thr < (1ull << 32);
  const double runs = (t.thr == 0 || keff + 1 > t.n)
                          ? 0.0 : std::min(n / (keff + 1.0), (n * (1.0 - a) + 1.0) * std::pow(a, keff + 1.0));
  const double p_any = 1.0 - std::exp(-runs);
  const double len = a < 1.0 ? std::min(n, 1.0 / (1.0 - a)) : n;
  const bool one = keff == 1;
  if (two_pass)
    return n * (0.0040 + (stream ? 0.00011 : 0.0)) + p_any * ((one ? 1.78 : 2.43) + 0.0063 * len) +
           runs * (one ? 0.143 : 0.68);
  return n * (0.00185 + (stream ? 0.0014 : 0.0)) + p_any * ((one ? 1.155 : 0.196) + 0.0006 * len) +
         runs * (one ? 0.30 : 0.18);
}

// Validate every config into ticks; on failure h->err names the first bad config.
// Validate every config into `out`; on failure h->err names the first bad config.  With
// `prev` (dsi_sim_update), also checks what an update must keep: n_trials, and with
// DSI_F_HIST min(k, N) (the histogram layout).
dsi_status validate_all(dsi_sim *h, const dsi_config *cfg, size_t n, std::vector<CfgTicks> &out,
                        const std::vector<CfgTicks> *prev, UpdateKeys *keys) {
  std::mutex mu;
  size_t bad = n;
  dsi_status bad_s = DSI_OK;
  std::string bad_msg;
  const bool hist = h->opt.flags & DSI_F_HIST;
  // (update) which plans survive, compared in the same pass: the shared-stream plan's keys, the
  // means-only groups' keys and the heatmap cells' keys
  std::atomic<bool> plan_same{true}, groups_same{true}, cells_same{true};
  parallel_for(n, [&](size_t b, size_t e) {
    bool ps = true, gs = true, cs = true;
    for (size_t i = b; i < e; ++i) {
      std::string msg;
      dsi_status s = convert(h->opt, cfg[i], i, out[i], msg);
      if (s == DSI_OK && prev) {
        const CfgTicks &o = (*prev)[i], &t = out[i];
        if (t.trials != o.trials || (hist && std::min(t.k, t.n) != std::min(o.k, o.n))) {
          s = DSI_E_RANGE;
          msg = "config " + std::to_string(i) + ": n_trials (and, with DSI_F_HIST, min(k, N)) must not change";
        }
        const bool same_stream = t.stream_id == o.stream_id && t.thr == o.thr && t.n == o.n && t.trials == o.trials;
        const bool to = o.t_t1 != o.t_t || o.t_d1 != o.t_d, tn = t.t_t1 != t.t_t || t.t_d1 != t.t_d;
        // (shared-stream mode: a TTFT config is not shared, so the flag is a plan key too)
        ps = ps && same_stream && t.k == o.k && t.t_t == o.t_t && t.t_d == o.t_d && t.sp == o.sp && to == tn;
        gs = gs && same_stream && to == tn;
        cs = cs && t.ut == o.ut && t.ud == o.ud && t.a == o.a && t.sp == o.sp && t.n == o.n;
      }
      if (s != DSI_OK) {
        std::lock_guard<std::mutex> lock(mu);
        if (i < bad) {
          bad = i;
          bad_s = s;
          bad_msg = msg;
        }
        return;
      }
    }
    if (!ps) plan_same = false;
    if (!gs) groups_same = false;
    if (!cs) cells_same = false;
  });
  if (bad < n) return fail(h, bad_s, bad_msg);
  if (keys) {
    keys->plan_same = plan_same;
    keys->groups_same = groups_same;
    keys->cells_same = cells_same;
  }
  return DSI_OK;
}

dsi_status derive_limits(dsi_sim *h, const std::vector<CfgTicks> &ticks) {
  struct Lim {
    int32_t max_n = 1, max_keff = 1;
    bool ttft = false, fresh = false;
    double work = 0.0, work_k1 = 0.0;  // trial-tokens in all configs / in k = 1 configs without queueing
  } lim;
  std::mutex mu;
  const bool fresh = h->opt.flags & DSI_F_FRESH_VERIFIER;
  parallel_for(ticks.size(), [&](size_t b, size_t e) {
    Lim l;
    for (size_t i = b; i < e; ++i) {
      const CfgTicks &t = ticks[i];
      l.max_n = std::max(l.max_n, t.n);
      l.max_keff = std::max(l.max_keff, std::min(t.k, t.n));
      l.ttft = l.ttft || t.t_t1 != t.t_t || t.t_d1 != t.t_d;
      l.fresh = l.fresh || (fresh && t.kd > t.t_t);
      const double w = (double)t.trials * (double)t.n;
      l.work += w;
      if (std::min(t.k, t.n) == 1 && config_noqueue(t)) l.work_k1 += w;
    }
    std::lock_guard<std::mutex> lock(mu);
    lim.max_n = std::max(lim.max_n, l.max_n);
    lim.max_keff = std::max(lim.max_keff, l.max_keff);
    lim.ttft = lim.ttft || l.ttft;
    lim.fresh = lim.fresh || l.fresh;
    lim.work += l.work;
    lim.work_k1 += l.work_k1;
  });
  if (lim.ttft && lim.max_n > 4096) return fail(h, DSI_E_RANGE, "the TTFT variant supports n_tokens <= 4096");
  if (dsi::trial_kernel_smem(lim.max_n, lim.max_keff, h->opt.flags & DSI_F_HIST, lim.ttft) > 200 * 1024)
    return fail(h, DSI_E_RANGE, "DSI_F_HIST needs (64 + k + 1) * 4 bytes of shared memory <= 200 KiB");
  if (h->shared && lim.max_n > kCrnMaxN)
    return fail(h, DSI_E_RANGE, "DSI_F_SHARED_STREAMS supports n_tokens <= " + std::to_string(kCrnMaxN));
  h->max_n = lim.max_n;
  h->max_keff = lim.max_keff;
  h->any_ttft = lim.ttft;
  h->any_fresh = lim.fresh;
  // the k = 1 fast path (dsi_kernel.cu, VAR 3) pays for its extra code only when such configs carry
  // a good share of the work (measured: config 5, 86% of its configs, -14%; config 3, 0.5%, +2% if on)
  h->k1_fast = !lim.ttft && !lim.fresh && lim.work_k1 >= 0.25 * lim.work;
  if (knobs().k1_fast >= 0) h->k1_fast = !lim.ttft && !lim.fresh && knobs().k1_fast != 0;
  return DSI_OK;
}

}  // namespace dsih

extern "C" {

uint32_t dsi_abi_version(void) { return DSI_ABI_VERSION; }

const char *dsi_status_str(dsi_status s) {
  switch (s) {
    case DSI_OK: return "DSI_OK";
    case DSI_E_NULL: return "DSI_E_NULL: required pointer was NULL";
    case DSI_E_RANGE: return "DSI_E_RANGE: argument out of range";
    case DSI_E_TICK: return "DSI_E_TICK: latency is not a whole number of ticks";
    case DSI_E_OVERFLOW: return "DSI_E_OVERFLOW: tick sums would overflow";
    case DSI_E_STRICT_EQ1: return "DSI_E_STRICT_EQ1: Eq. 1 violated under DSI_F_STRICT_EQ1";
    case DSI_E_DEVICE: return "DSI_E_DEVICE: CUDA error or missing sm_100 device";
    case DSI_E_COMM: return "DSI_E_COMM: NCCL error";
    case DSI_E_STATE: return "DSI_E_STATE: call order violated";
    case DSI_E_NOMEM: return "DSI_E_NOMEM: allocation failed";
  }
  return "unknown dsi_status";
}

const char *dsi_sim_last_error(const dsi_sim *h) { return h ? h->err.c_str() : ""; }
const char *dsi_last_create_error(void) { return g_create_error.c_str(); }

dsi_status dsi_ticks(double x, double tick, int64_t *out) {
  if (!out) return DSI_E_NULL;
  if (!std::isfinite(tick) || tick <= 0.0) return DSI_E_RANGE;
  return to_ticks(x, tick, out);
}

int32_t dsi_eq1_feasible(int64_t t_t, int64_t t_d, int32_t k, int32_t sp) { return dsi::eq1_feasible(t_t, t_d, k, sp); }

int32_t dsi_min_lookahead(int64_t t_t, int64_t t_d, int32_t sp) { return dsi::min_lookahead(t_t, t_d, sp); }

int32_t dsi_required_processors(int64_t t_t, int64_t t_d, int32_t k) {
  if (t_t < 1 || t_d < 1 || k < 1) return -1;
  return (int32_t)(1 + ceil_div(t_t, (int64_t)k * t_d));
}

dsi_status dsi_shard_bounds(const double *cost, uint64_t n, int32_t parts, uint64_t *bounds) {
  if (!bounds || (!cost && n)) return DSI_E_NULL;
  if (parts < 1) return DSI_E_RANGE;
  double total = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!(cost[i] >= 0.0)) return DSI_E_RANGE;
    total += cost[i];
  }
  bounds[0] = 0;
  uint64_t i = 0;
  double run = 0.0;
  for (int32_t j = 1; j < parts; ++j) {
    const double target = total * (double)j / (double)parts;
    // advance while taking unit i keeps the prefix closer to the target
    while (i < n && run + 0.5 * cost[i] <= target) run += cost[i++];
    bounds[j] = i;
  }
  bounds[parts] = n;
  return DSI_OK;
}

}  // extern "C"

// Build identity (build.py passes -DDSI_BUILD_ID=<sha256 of the sources and flags>).
#ifndef DSI_BUILD_ID
#define DSI_BUILD_ID "unknown"
#endif
extern "C" const char *dsi_build_id(void) { return "DSI_BUILD_ID=" DSI_BUILD_ID + 13; }
