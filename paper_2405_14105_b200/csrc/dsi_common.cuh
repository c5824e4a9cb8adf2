// dsi_common.cuh -- device helpers shared by the trial kernels (dsi_kernel.cu,
// dsi_crn.cu): Philox4x32-10 with rounds 0-1 split into a per-trial and a
// per-counter half, the Bernoulli pack, magic-number divisions and the
// per-segment DSI/SI costs of the closed form.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_device.h"

namespace dsi {

constexpr uint32_t PHILOX_M0 = 0xD2511F53u;
constexpr uint32_t PHILOX_M1 = 0xCD9E8D57u;

struct Word4 {
  uint32_t x, y, z, w;
};

// Philox rounds 2..9 from the round-1 output (c0, c1, c2, c3).
__device__ __forceinline__ Word4 philox_rounds_2_9(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   const Keys &K) {
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    const uint64_t a = (uint64_t)PHILOX_M0 * c0;
    const uint64_t b = (uint64_t)PHILOX_M1 * c2;
    const uint32_t n0 = (uint32_t)(b >> 32) ^ c1 ^ K.k0[r];
    const uint32_t n2 = (uint32_t)(a >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)b;
    c3 = (uint32_t)a;
    c0 = n0;
    c2 = n2;
  }
  return Word4{c0, c1, c2, c3};
}

// Per-q half of rounds 0-1 for counter (q, 0, trial, stream):
//   round 0: n2 = hi(M0 q) ^ stream ^ k1[0], n3 = lo(M0 q)
//   round 1: (hi(M1 n2) ^ k0[1], lo(M1 n2), n3 ^ k1[1])
__device__ __forceinline__ uint4 philox_q_half(uint32_t q, uint32_t stream, const Keys &K) {
  const uint64_t p = (uint64_t)PHILOX_M0 * q;
  const uint32_t n2 = (uint32_t)(p >> 32) ^ stream ^ K.k1[0];
  const uint64_t b = (uint64_t)PHILOX_M1 * n2;
  return make_uint4((uint32_t)(b >> 32) ^ K.k0[1], (uint32_t)b, (uint32_t)p ^ K.k1[1], 0u);
}

// Per-trial half of rounds 0-1: n0 = hi(M1 trial) ^ k0[0], n1 = lo(M1 trial),
// then a = M0 n0 gives (hi(a), lo(a)).
struct TrialHalf {
  uint32_t n1, ha, la;
};
__device__ __forceinline__ TrialHalf philox_trial_half(uint32_t trial, const Keys &K) {
  const uint64_t p = (uint64_t)PHILOX_M1 * trial;
  const uint32_t n0 = (uint32_t)(p >> 32) ^ K.k0[0];
  const uint64_t a = (uint64_t)PHILOX_M0 * n0;
  return TrialHalf{(uint32_t)p, (uint32_t)(a >> 32), (uint32_t)a};
}

// Full Philox4x32-10 output for (q, 0, trial, stream) from the two halves.
__device__ __forceinline__ Word4 philox_call(const uint4 &u, const TrialHalf &t, const Keys &K) {
  return philox_rounds_2_9(u.x ^ t.n1, u.y, t.ha ^ u.z, t.la, K);
}

// rej = (rej << 4) | [w >= thr] << 3 | [z >= thr] << 2 | [y >= thr] << 1 | [x >= thr]
// from the carries of u + (2^32 - thr) (thr >= 1): 2 instructions per bit (IADD3 + IMAD.X).
__device__ __forceinline__ uint32_t pack4(uint32_t rej, const Word4 &u, uint32_t nthr) {
  // (measured, profiles/r01_ab_pack.jsonl: compare + select packing was 6% slower; the
  //  carry as the majority bit of (u, n, u + n) funnel-shifted in, all on the ALU pipe, 16%
  //  slower for 4 bits and 8% for 2 of the 4: the IMAD.X half of addc is the cheaper pipe)
  asm("{\n\t"
      ".reg .u32 t;\n\t"
      "add.cc.u32 t, %1, %5;\n\t"
      "addc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %2, %5;\n\t"
      "addc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %3, %5;\n\t"
      "addc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %4, %5;\n\t"
      "addc.u32 %0, %0, %0;\n\t"
      "}"
      : "+r"(rej)
      : "r"(u.w), "r"(u.z), "r"(u.y), "r"(u.x), "r"(nthr));
  return rej;
}

// floor(x / d) for x * d <= 2^32 with M = ceil(2^32 / d) = lo + hi * 2^32.
__device__ __forceinline__ uint32_t magic_div(uint32_t x, uint32_t lo, uint32_t hi) {
  return __umulhi(x, lo) + x * hi;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct SegCtx {
  uint32_t k_eff, m_si, m_k_lo, m_k_hi, m_sp_lo, m_sp_hi;
  int32_t sp_eff, kd, t_t, n_tokens, s1;
};

// Segment costs beyond those of a length-1 segment: (ceil(g/(k+1)) - 1, S(ceil((g-1)/k))).
__device__ __forceinline__ uint2 seg_extra(int g, const SegCtx &s) {
  const uint32_t M = magic_div((uint32_t)g + s.k_eff, s.m_si, 0u);              // ceil(g/(k+1))
  const uint32_t b = magic_div((uint32_t)g + s.k_eff - 2u, s.m_k_lo, s.m_k_hi);  // ceil((g-1)/k)
  const uint32_t qq = magic_div(b, s.m_sp_lo, s.m_sp_hi);
  const int rr = (int)b - (int)qq * s.sp_eff;
  int S = max((int)b * s.kd, rr * s.kd + (int)qq * s.t_t);
#ifdef DSI_MUTANT_CG
  S += 1;  // mutation-test build only (libdsi_sim_mutant.so): C(g) one tick too large
#endif
  return make_uint2(M - 1u, (uint32_t)S);
}

// Costs of a long segment (g >= k+2) beyond those of a short one (2 <= g <= k+1,
// which always costs (0 extra SI iterations, S(1))): seg_extra(g) - (0, S(1)).
__device__ __forceinline__ uint2 seg_long(int g, const SegCtx &s) {
  const uint2 e = seg_extra(g, s);
  return make_uint2(e.x, e.y - (uint32_t)s.s1);
}

// Fresh-verifier variant (R24) with k t_d > t_t, where no task ever queues
// (S(b) = b k t_d): a segment of length g >= 2 ends at offset j = g-1-(b-1)k of block
// b = ceil((g-1)/k), which the chain of fresh forwards started at F_{b-1}, F_{b-1} + t_t,
// ... settles at F_{b-1} + min(k t_d, t_t ceil(j t_d / t_t)) instead of F_b = F_{b-1} + k t_d.
// Returns the saving k t_d - min(k t_d, t_t ceil(j t_d / t_t)) (< 2^31: j t_d <= k t_d).
__device__ __forceinline__ uint32_t fresh_saving(int g, const SegCtx &s, int t_d) {
  const uint32_t b = magic_div((uint32_t)g + s.k_eff - 2u, s.m_k_lo, s.m_k_hi);  // ceil((g-1)/k)
  const int j = g - 1 - ((int)b - 1) * (int)s.k_eff;
  const int v = s.t_t * ((j * t_d + s.t_t - 1) / s.t_t);
  return (uint32_t)max(0, s.kd - v);
}

// floor(x / d) for 0 <= x < 2^31 and a divisor d with magic (m, sh) from the host
// (Granlund-Montgomery: m = floor(2^32 (2^sh - d) / d) + 1, sh = ceil(log2 d)); the sum
// umulhi(x, m) + x < 2^32 because x < 2^31.
__device__ __forceinline__ uint32_t divu31(uint32_t x, uint32_t m, int sh) {
  return (__umulhi(x, m) + x) >> sh;
}

// Fresh-verifier saving (as fresh_saving) of a segment of L = g - 1 >= 1 accepted drafts, from
// per-config constants only (no integer division): b = ceil(L/k), j = L - (b-1) k,
// saving = k t_d - min(k t_d, t_t ceil(j t_d / t_t)).  Only for k t_d > t_t (CFG_FRESH).
__device__ __forceinline__ int fresh_saving_L(int L, int k_eff, uint32_t m_k_lo, uint32_t m_k_hi, int kd, int t_t,
                                              int t_d, uint32_t m_tt, int sh_tt) {
  const uint32_t b = magic_div((uint32_t)(L + k_eff - 1), m_k_lo, m_k_hi);  // ceil(L / k)
  const int j = L - ((int)b - 1) * k_eff;
  const int v = t_t * (int)divu31((uint32_t)(j * t_d + t_t - 1), m_tt, sh_tt);
  return kd - min(kd, v);
}

// Bits i of x such that bits i-n+1 .. i are all ones (runs of at least n ones),
// by log-doubling: y_s marks runs >= s, then y_s & (y_s << (n - s)) for s <= n < 2s.
__device__ __forceinline__ uint32_t runs_at_least(uint32_t x, int n) {
  uint32_t y = x;
  int sh = 1;
  while (2 * sh <= n) {
    y &= y << sh;
    sh <<= 1;
  }
  if (sh < n) y &= y << (n - sh);
  return y;
}

__device__ __forceinline__ SegCtx make_segctx(const DevCfg &cfg) {
  SegCtx s;
  s.k_eff = (uint32_t)cfg.k_eff;
  s.m_si = cfg.m_si;
  s.m_k_lo = cfg.m_k_lo;
  s.m_k_hi = cfg.m_k_hi;
  s.m_sp_lo = cfg.m_sp_lo;
  s.m_sp_hi = cfg.m_sp_hi;
  s.sp_eff = cfg.sp_eff;
  s.kd = cfg.kd;
  s.t_t = cfg.t_t;
  s.n_tokens = cfg.n_tokens;
  s.s1 = cfg.s1;
  return s;
}

}  // namespace dsi
