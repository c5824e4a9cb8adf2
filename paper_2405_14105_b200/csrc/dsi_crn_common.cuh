// dsi_crn_common.cuh -- what the shared-stream kernels (dsi_crn.cu, dsi_crn2.cu) share:
// the per-config constants of phase 2 and the long-run correction of the closed form.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_device.h"

namespace dsi {

struct CfgLite {  // what phase 2 needs of a config (shared memory, 48 B)
  int32_t t_t, s1, si_cost, k_eff;
  uint32_t m_si, m_k_lo, m_k_hi, m_sp_lo;
  uint32_t m_sp_hi;
  int32_t kd, nonsi;
  int16_t sp_eff, noqueue;  // noqueue: S(b) = b k t_d (CFG_NOQUEUE)
};
static_assert(sizeof(CfgLite) == 48, "CfgLite layout");

// The fresh-verifier constants of a config (CFG_FRESH: k t_d > t_t, R24), kept apart
// from CfgLite so launches without such a config (template FRESH = false) pay neither the
// shared memory nor the registers.
struct CfgFr {
  int32_t t_d;
  uint32_t m_tt;  // floor(x / t_t) magic (divu31)
  int32_t sh_tt;
  int32_t fresh;
};
static_assert(sizeof(CfgFr) == 16, "CfgFr layout");

// Fresh-verifier saving of a segment of L >= 1 accepted drafts (fresh_saving_L); a segment of
// L = 1 (g = 2) saves k t_d - t_t (one fresh forward settles its one draft, t_d <= t_t).
__device__ __forceinline__ int fresh_saving_lite(int L, const CfgLite &l, const CfgFr &f) {
  return fresh_saving_L(L, l.k_eff, l.m_k_lo, l.m_k_hi, l.kd, l.t_t, f.t_d, f.m_tt, f.sh_tt);
}

// Extra costs of a segment with L = g - 1 >= k + 1 accepted drafts (seg_long of the
// per-config kernel): x = floor(L/(k+1)) SI iterations, y = S(ceil(L/k)) - S(1).
__device__ __forceinline__ void long_run(int L, const CfgLite &l, int &ai, int &ay) {
  const uint32_t x = magic_div((uint32_t)L, l.m_si, 0u);
  const uint32_t b = magic_div((uint32_t)L + (uint32_t)l.k_eff - 1u, l.m_k_lo, l.m_k_hi);
  const uint32_t qq = magic_div(b, l.m_sp_lo, l.m_sp_hi);
  const int rr = (int)b - (int)qq * l.sp_eff;
  const int S = max((int)b * l.kd, rr * l.kd + (int)qq * l.t_t);
  ai += (int)x;
  ay += S - l.s1;
}

// The phase-2 constants of config j of a unit (an empty slot beyond the unit's count gets
// k_eff = 2^20: no run is ever long for it).
__device__ __forceinline__ CfgLite load_cfglite(const DevCfg *cfgs, const uint32_t *perm, const CrnUnit &un,
                                                int j, int N) {
  CfgLite l{};
  if (j < (int)un.count) {
    const DevCfg c = cfgs[perm[un.begin + j]];
    l.t_t = c.t_t;
    l.s1 = c.s1;
    l.si_cost = c.si_cost;
    l.k_eff = c.k_eff;
    l.m_si = c.m_si;
    l.m_k_lo = c.m_k_lo;
    l.m_k_hi = c.m_k_hi;
    l.m_sp_lo = c.m_sp_lo;
    l.m_sp_hi = c.m_sp_hi;
    l.kd = c.kd;
    l.sp_eff = (int16_t)c.sp_eff;
    l.noqueue = (c.flags & CFG_NOQUEUE) ? 1 : 0;
    l.nonsi = N * c.t_t;
  } else {
    l.k_eff = 1 << 20;
    l.m_sp_lo = 1u;
  }
  return l;
}

// The fresh-verifier constants of config j of a unit (zero, i.e. not fresh, beyond its count).
__device__ __forceinline__ CfgFr load_cfgfr(const DevCfg *cfgs, const uint32_t *perm, const CrnUnit &un, int j) {
  CfgFr f{};
  if (j < (int)un.count) {
    const DevCfg &c = cfgs[perm[un.begin + j]];
    f.t_d = c.t_d;
    f.m_tt = c.m_tt;
    f.sh_tt = c.sh_tt;
    f.fresh = (c.flags & CFG_FRESH) ? 1 : 0;
  }
  return f;
}

}  // namespace dsi
