// dsi_convert.h -- the validation and tick conversion of one configuration (R15) and its
// device row (DevCfg), written once for the host (create, and the host path of update) and the
// device (dsi_stage.cu: the device path of dsi_sim_update), so both produce the same integers.
// Internal: not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/dsi_sim.h"
#include "dsi_device.h"

#define DSI_HD __host__ __device__ __forceinline__

namespace dsi {

constexpr int kMaxTokens = 32768;  // keeps every magic division exact (x * d <= 2^32)
constexpr uint64_t kMaxTrials = 1ull << 32;

// One configuration in ticks (host planning and finalize; the device path keeps only DevCfg).
struct CfgTicks {
  int64_t t_t, t_d, kd;
  int64_t t_t1, t_d1;  // first-forward latencies (TTFT variant; equal to t_t, t_d when off)
  uint64_t thr;
  int32_t k, sp, n;
  uint32_t stream_id;
  uint64_t trials;
  double a;
  double ut, ud;  // t_target, t_drafter as given (heatmap cells group on the user values)
  int32_t eq1, min_k;  // Eq. 1 holds at (k, SP); the minimal lookahead at SP
};

DSI_HD int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Eq. 1: ceil(t_t / (k t_d)) <= SP; -1 on invalid arguments
DSI_HD int32_t eq1_feasible(int64_t t_t, int64_t t_d, int32_t k, int32_t sp) {
  if (t_t < 1 || t_d < 1 || k < 1 || sp < 1) return -1;
  return ceil_div64(t_t, (int64_t)k * t_d) <= sp ? 1 : 0;
}

// smallest k with ceil(t_t/(k t_d)) <= SP  <=>  k t_d SP >= t_t; -1 on invalid
DSI_HD int32_t min_lookahead(int64_t t_t, int64_t t_d, int32_t sp) {
  if (t_t < 1 || t_d < 1 || sp < 1) return -1;
  const int64_t k = ceil_div64(t_t, t_d * (int64_t)sp);
  return (int32_t)(k > 1 ? k : 1);
}

// R15: ticks = round(x / tick) when within 1e-9 (relative) of an integer >= 1
DSI_HD int to_ticks(double x, double tick, int64_t *out) {
  if (!isfinite(x) || x <= 0.0) return DSI_E_RANGE;
  const double r = x / tick;
  if (!(r < 9.0e18)) return DSI_E_OVERFLOW;
  const int64_t t = llround(r);
  if (t < 1 || fabs(r - (double)t) > 1e-9 * fabs(r)) return DSI_E_TICK;
  *out = t;
  return DSI_OK;
}

// Which check of convert_config failed (the host turns it into the message).
enum ConvWhat : int {
  CV_OK = 0, CV_ACCEPT, CV_LOOKAHEAD, CV_SP, CV_N, CV_TRIALS, CV_PATTERN_N, CV_T_TARGET, CV_T_DRAFTER,
  CV_ASSUMPTION2, CV_TTFT_TARGET, CV_TTFT_DRAFTER, CV_ASSUMPTION2_FIRST, CV_SHARED_TTFT, CV_FRESH_TTFT,
  CV_BOUND, CV_BOUND_SQ, CV_STRICT_EQ1
};

// Validate and convert one configuration: 0, or (what << 8) | dsi_status of the first failing
// check (the order of the checks is the order of the error precedence).
DSI_HD int convert_config(double tick, uint32_t flags, const dsi_config &c, CfgTicks &o) {
#define DSI_CV_FAIL(what, st) return ((int)(what) << 8) | (int)(st)
  if (!(c.accept_rate >= 0.0 && c.accept_rate <= 1.0)) DSI_CV_FAIL(CV_ACCEPT, DSI_E_RANGE);
  if (c.lookahead < 1) DSI_CV_FAIL(CV_LOOKAHEAD, DSI_E_RANGE);
  if (c.sp_degree < 1) DSI_CV_FAIL(CV_SP, DSI_E_RANGE);
  if (c.n_tokens < 1 || c.n_tokens > kMaxTokens) DSI_CV_FAIL(CV_N, DSI_E_RANGE);
  if (c.n_trials < 1 || c.n_trials > kMaxTrials) DSI_CV_FAIL(CV_TRIALS, DSI_E_RANGE);
  if ((flags & DSI_F_PATTERN) && c.n_tokens > 33) DSI_CV_FAIL(CV_PATTERN_N, DSI_E_RANGE);
  int s = to_ticks(c.t_target, tick, &o.t_t);
  if (s != DSI_OK) DSI_CV_FAIL(CV_T_TARGET, s);
  s = to_ticks(c.t_drafter, tick, &o.t_d);
  if (s != DSI_OK) DSI_CV_FAIL(CV_T_DRAFTER, s);
  if (o.t_d > o.t_t) DSI_CV_FAIL(CV_ASSUMPTION2, DSI_E_RANGE);
  o.t_t1 = o.t_t;
  o.t_d1 = o.t_d;
  if (c.ttft_target != 0.0) {
    s = to_ticks(c.ttft_target, tick, &o.t_t1);
    if (s != DSI_OK) DSI_CV_FAIL(CV_TTFT_TARGET, s);
  }
  if (c.ttft_drafter != 0.0) {
    s = to_ticks(c.ttft_drafter, tick, &o.t_d1);
    if (s != DSI_OK) DSI_CV_FAIL(CV_TTFT_DRAFTER, s);
  }
  if (o.t_d1 > o.t_t1) DSI_CV_FAIL(CV_ASSUMPTION2_FIRST, DSI_E_RANGE);
  if ((flags & DSI_F_FRESH_VERIFIER) && (o.t_t1 != o.t_t || o.t_d1 != o.t_d)) DSI_CV_FAIL(CV_FRESH_TTFT, DSI_E_RANGE);
  // every per-trial latency is <= N (k t_d + t_t) plus the first-forward surcharges
  // (kernel overflow bound)
  const unsigned __int128 kd = (unsigned __int128)c.lookahead * (uint64_t)o.t_d;
  const unsigned __int128 bound = (unsigned __int128)c.n_tokens * (kd + (uint64_t)o.t_t) +
                                  (uint64_t)(o.t_t1 > o.t_t ? o.t_t1 - o.t_t : 0) +
                                  (uint64_t)(o.t_d1 > o.t_d ? o.t_d1 - o.t_d : 0);
  if (bound >= ((unsigned __int128)1 << 31)) DSI_CV_FAIL(CV_BOUND, DSI_E_OVERFLOW);
  if ((unsigned __int128)c.n_trials * bound * bound >= ((unsigned __int128)1 << 64))
    DSI_CV_FAIL(CV_BOUND_SQ, DSI_E_OVERFLOW);
  o.kd = (int64_t)kd;
  if ((flags & DSI_F_STRICT_EQ1) && ceil_div64(o.t_t, o.kd) > c.sp_degree) DSI_CV_FAIL(CV_STRICT_EQ1, DSI_E_STRICT_EQ1);
#undef DSI_CV_FAIL
  o.a = c.accept_rate;
  o.ut = c.t_target;
  o.ud = c.t_drafter;
  o.eq1 = eq1_feasible(o.t_t, o.t_d, c.lookahead, c.sp_degree);
  o.min_k = min_lookahead(o.t_t, o.t_d, c.sp_degree);
  o.thr = (uint64_t)(c.accept_rate * 4294967296.0);  // exact: a * 2^32, then floor
  o.k = c.lookahead;
  o.sp = c.sp_degree;
  o.n = c.n_tokens;
  o.stream_id = c.stream_id;
  o.trials = c.n_trials;
  return 0;
}

// S(b) = b k t_d for every b: Eq. 1 holds at min(SP, N), or SP >= N (no thread ever waits).
DSI_HD bool config_noqueue(const CfgTicks &t) {
  const int32_t sp_eff = t.sp < t.n ? t.sp : t.n;
  return (t.t_t <= (int64_t)sp_eff * t.kd) || sp_eff >= t.n;
}

// ceil(2^32 / d) split into low word and bit 32 (d >= 1); the host reads divisors below 2^16
// from a table (magic_table, dsi_validate.cpp), which holds the same values.
#ifndef __CUDA_ARCH__
void magic_table(uint32_t d, uint32_t &lo, uint32_t &hi);
#endif
DSI_HD void magic(uint32_t d, uint32_t &lo, uint32_t &hi) {
#ifdef __CUDA_ARCH__
  const uint64_t m = ((1ull << 32) + d - 1) / d;
  lo = (uint32_t)m;
  hi = (uint32_t)(m >> 32);
#else
  magic_table(d, lo, hi);
#endif
}

// The device row of a configuration (rec_off and si_hist_off, the test modes' prefix
// offsets, are left 0: the caller sets them).
DSI_HD DevCfg make_dev_cfg(const CfgTicks &t, bool pattern, bool fresh) {
  DevCfg d{};
  uint32_t mode = MODE_STREAM;
  if (!pattern) {
    if (t.thr >= (1ull << 32)) mode = MODE_ALL_ACCEPT;
    else if (t.thr == 0) mode = MODE_ALL_REJECT;
  }
  const int32_t k_eff = t.k < t.n ? t.k : t.n;
  const int32_t sp_eff = t.sp < t.n ? t.sp : t.n;
  const bool noqueue = config_noqueue(t);
  d.thr = (uint32_t)(t.thr < 0xffffffffull ? t.thr : 0xffffffffull);
  const bool ttft = t.t_t1 != t.t_t || t.t_d1 != t.t_d;
  // fresh-verifier variant: with k t_d <= t_t a fresh forward never finishes sooner than
  // the regular thread (R24), so only k t_d > t_t configs take its cost table
  const bool fresh_cfg = fresh && t.kd > t.t_t;
  d.flags = mode | (noqueue ? CFG_NOQUEUE : 0u) | (ttft ? CFG_TTFT : 0u) | (fresh_cfg ? CFG_FRESH : 0u);
  d.t_d = (int32_t)t.t_d;
  d.k = t.k;
  if (t.eq1 == 1) d.flags |= CFG_EQ1;
  d.nonsi = (int32_t)(t.t_t1 + (int64_t)(t.n - 1) * t.t_t);
  d.e_si = (int32_t)((t.t_d1 - t.t_d) + (t.t_t1 - t.t_t));
  d.t_t1 = (int32_t)t.t_t1;
  d.ttft_shift = (int32_t)(t.t_d1 - t.t_d);
  d.n_tokens = t.n;
  d.k_eff = k_eff;
  d.sp_eff = sp_eff;
  d.t_t = (int32_t)t.t_t;
  d.kd = (int32_t)t.kd;
  d.si_cost = (int32_t)(t.kd + t.t_t);
  // S(1) = max(k t_d, (1 mod SP) k t_d + floor(1/SP) t_t): k t_d, or max(k t_d, t_t) if SP = 1
  d.s1 = (int32_t)(t.sp >= 2 ? t.kd : (t.kd > t.t_t ? t.kd : t.t_t));
  d.stream_id = t.stream_id;
  uint32_t hi;
  magic((uint32_t)k_eff + 1u, d.m_si, hi);  // k_eff + 1 >= 2: hi == 0
  magic((uint32_t)k_eff, d.m_k_lo, d.m_k_hi);
  magic((uint32_t)sp_eff, d.m_sp_lo, d.m_sp_hi);
  d.n_trials = t.trials;
  // floor(x / t_t) for x < 2^31: l = ceil(log2 t_t), m' = floor(2^32 (2^l - t_t) / t_t) + 1
  {
    const uint64_t tt = (uint64_t)t.t_t;
    int l = 0;
    while ((1ull << l) < tt) ++l;
    d.m_tt = (uint32_t)((((1ull << 32) * ((1ull << l) - tt)) / tt + 1) & 0xffffffffull);
    d.sh_tt = l;
  }
  return d;
}

// ----------------------------------------------------------------------------- device update
enum : unsigned int {
  STAGE_TTFT = 1u,             // some config has first-forward latencies (TTFT variant)
  STAGE_FRESH = 2u,            // some config is fresh-verifier (DSI_F_FRESH_VERIFIER and k t_d > t_t)
  STAGE_PLAN_CHANGED = 4u,     // a shared-stream plan key changed (stream, a, N, T, k, t_t, t_d, SP, TTFT)
  STAGE_GROUPS_CHANGED = 8u,   // a means-only group key changed (stream, a, N, T, TTFT or not)
  STAGE_CELLS_CHANGED = 16u,   // a heatmap-cell key changed (t_target, t_drafter, a as given, SP, N)
};
struct StageStatus {
  unsigned long long first_bad;  // smallest index failing validation or changing n_trials, else ~0
  unsigned int flags;            // STAGE_*
  int max_n, max_keff;           // launch limits of the new configs
  int pad;
  double work, work_k1;          // trial-tokens in all configs / in k = 1 configs without queueing
};
struct StageParams {
  const dsi_config *raw;   // the new configurations (device copy, as given)
  const dsi_config *prev;  // the handle's current configurations (device)
  DevCfg *out;             // the spare device table
  uint64_t n;
  double tick;
  uint32_t flags;          // dsi_options.flags
  StageStatus *st;         // initialised by the host: first_bad = ~0, maxima 1, the rest 0
};
int launch_stage_kernel(const StageParams &p, void *stream);

}  // namespace dsi
