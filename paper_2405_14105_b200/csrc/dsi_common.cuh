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

// ---- Halves layout (DSI_F_RNG_HALVES, R26) ----------------------------------------
// Call q = (p-1) >> 3 of counter (q, 0, trial, stream) serves positions 8q+1 .. 8q+8: offset
// j = (p-1) & 7 reads v_j = the high 16 bits of word j (j < 4; words x, y, z, w) or the low 16
// bits of word j-4.  With thr = T 2^16 + R: A_p = [v < T], and on a tie (v == T, probability
// 2^-16) A_p = [w < R], w the same half of the same word of the tie-break call (q, 1, trial,
// stream) -- i.e. A_p = [v 2^16 + w < thr]: the 32-bit layout's law with half its Philox calls.
// The rejection mask keeps its meaning (bit i of word W = position 32W + i + 1); word W holds
// calls 4W .. 4W+3, call 4W + c in bits 8c .. 8c+7.

struct HalvesCtx {
  uint32_t C;       // (2^16 - T) << 16 mod 2^32: the carry of (v << 16) + C is [v >= T] (T >= 1)
  uint32_t TT;      // T in both halves (the tie test)
  uint32_t orall;   // T == 0: every v >= T (no carry ever comes), so all bits are set
  uint32_t thr;     // threshold (mode MODE_STREAM: 1 <= thr < 2^32)
  uint32_t stream;  // counter word 3
  bool direct;      // T is not an f16 NaN pattern: ties by u == TT as f16x2
};

__device__ __forceinline__ HalvesCtx make_halves(uint32_t thr, uint32_t stream) {
  HalvesCtx h;
  const uint32_t T = thr >> 16;
  h.C = (0x10000u - T) << 16;
  h.TT = T | (T << 16);
  h.orall = T == 0u ? 0xffffffffu : 0u;
  h.thr = thr;
  h.stream = stream;
  h.direct = !((T & 0x7C00u) == 0x7C00u && (T & 0x3FFu) != 0u);
  return h;
}

// rej = (rej << 8) | [lo(w) >= T] << 7 | ... | [lo(x) >= T] << 4 | [hi(w) >= T] << 3 | ... | [hi(x) >= T]
// (ties counted as rejections; the caller fixes them): 1 shift/LEA + IADD3 + IMAD.X per bit.
__device__ __forceinline__ uint32_t pack8(uint32_t rej, const Word4 &u, uint32_t C) {
  asm("{\n\t"
      ".reg .u32 t, l;\n\t"
      "shl.b32 l, %4, 16;\n\tadd.cc.u32 t, l, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "shl.b32 l, %3, 16;\n\tadd.cc.u32 t, l, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "shl.b32 l, %2, 16;\n\tadd.cc.u32 t, l, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "shl.b32 l, %1, 16;\n\tadd.cc.u32 t, l, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %4, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %3, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %2, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %1, %5;\n\taddc.u32 %0, %0, %0;\n\t"
      "}"
      : "+r"(rej)
      : "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w), "r"(C));
  return rej;
}

// Per-half equality as f16x2 (HSET2: lanes 0xFFFF where equal).  +0 and -0 compare equal and
// NaN never does, so: DIRECT (u == TT, T not a NaN pattern) flags every tie, plus lanes 0x0000 /
// 0x8000 when T is -0 / +0; the XOR form (u ^ TT == 0) flags every tie plus lanes 0x8000 of
// u ^ TT.  Flags are a superset of the ties: the fix re-decides exactly.
__device__ __forceinline__ uint32_t heq2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("set.eq.u32.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <bool DIRECT>
__device__ __forceinline__ uint32_t tie_flags(const Word4 &u, uint32_t TT, uint32_t acc) {
  if (DIRECT) return acc | heq2(u.x, TT) | heq2(u.y, TT) | heq2(u.z, TT) | heq2(u.w, TT);
  return acc | heq2(u.x ^ TT, 0u) | heq2(u.y ^ TT, 0u) | heq2(u.z ^ TT, 0u) | heq2(u.w ^ TT, 0u);
}

__device__ __forceinline__ uint32_t half_of(const Word4 &o, int j) {
  const int i = j & 3;
  const uint32_t x = i == 0 ? o.x : i == 1 ? o.y : i == 2 ? o.z : o.w;
  return j < 4 ? x >> 16 : x & 0xFFFFu;
}

// Rounds 2-9 as a loop (few registers: the rare tie paths run it, and a callee's register count is
// what its caller must save around the call).
__device__ __forceinline__ Word4 philox_call_rolled(const uint4 &u, const TrialHalf &t, const Keys &K) {
  uint32_t c0 = u.x ^ t.n1, c1 = u.y, c2 = t.ha ^ u.z, c3 = t.la;
#pragma unroll 1
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

// The trial half of rounds 0-1 for the tie-break counter (q, 1, trial, stream): counter word 1
// enters round 0 only through n0 = hi(M1 trial) ^ c1 ^ k0[0], so the tie-break call shares the
// main call's per-counter half U[q].
__device__ __forceinline__ TrialHalf tiebreak_trial_half(uint32_t trial, const Keys &K) {
  const uint64_t p = (uint64_t)PHILOX_M1 * trial;
  const uint32_t n0 = (uint32_t)(p >> 32) ^ 1u ^ K.k0[0];
  const uint64_t a = (uint64_t)PHILOX_M0 * n0;
  return TrialHalf{(uint32_t)p, (uint32_t)(a >> 32), (uint32_t)a};
}

// Exact decisions of every tied position among calls 4w .. 4w + ncalls - 1 (bits 8c + j of R):
// rejected iff w >= R_low, w from the tie-break call.  For the last (partial) word of a trial; full
// words fix their ties inline (gen_word_halves_t).  The calls are regenerated one by one, and the
// arguments are few scalars (the trial half is recomputed): a reference to a caller's local would
// force it to the stack, and every argument is one more value the hot loop keeps around the call.
template <bool TABLE>
static __device__ __noinline__ uint32_t halves_fix(uint32_t R, int w, int ncalls, const uint4 *U, uint32_t trial,
                                                   uint32_t stream, uint32_t thr, const Keys &K) {
  const uint32_t T = thr >> 16, Rl = thr & 0xFFFFu;
  const TrialHalf th = philox_trial_half(trial, K);
  const TrialHalf tb_half = tiebreak_trial_half(trial, K);
  for (int c = 0; c < ncalls; ++c) {
    const int q = 4 * w + c;
    const uint4 u = TABLE ? U[q] : philox_q_half((uint32_t)q, stream, K);
    const Word4 o = philox_call_rolled(u, th, K);
    bool have = false;
    Word4 tb{0u, 0u, 0u, 0u};
    for (int j = 0; j < 8; ++j) {
      if (half_of(o, j) != T) continue;
      if (!have) {
        tb = philox_call_rolled(u, tb_half, K);
        have = true;
      }
      const uint32_t bit = 1u << (8 * c + j);
      R = half_of(tb, j) >= Rl ? (R | bit) : (R & ~bit);
    }
  }
  return R;
}

// Rejection mask of word w in the halves layout: calls 4w .. 4w + ncalls - 1 (ncalls = min(4,
// nq - 4w), nq = ceil((N-1)/8)), U[q] the per-counter half of rounds 0-1 (TABLE) or computed.
template <bool DIRECT, bool TABLE>
__device__ __forceinline__ uint32_t gen_word_halves_t(int w, int nq, const uint4 *U, const TrialHalf &th,
                                                      uint32_t trial, const HalvesCtx &h, const Keys &K) {
  uint32_t R = 0u, tf = 0u;
  const int ncalls = min(4, nq - 4 * w);
  if (ncalls == 4) {
    Word4 o[4];
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      DSI_CHECK(4 * w + j < nq);
      const uint4 u = TABLE ? U[4 * w + j] : philox_q_half((uint32_t)(4 * w + j), h.stream, K);
      o[j] = philox_call(u, th, K);
      R = pack8(R, o[j], h.C);
      tf = tie_flags<DIRECT>(o[j], h.TT, tf);
    }
    R |= h.orall;
    // rare (~1.6% of warp-words): the word's outputs are still in registers, so only the tie-break
    // calls are computed (inline: 187.1 ms vs 188.0 with halves_fix's regeneration; guarding it
    // with a warp vote 195.8 ms -- profiles/r02c_ab_halves_inl.jsonl, r02c_ab_halves_vote.jsonl)
#ifdef DSI_MUTANT_TIES
    tf = 0u;  // mutation probe only: ties left as rejections (the tie-break dropped)
#endif
    if (tf) {
      const uint32_t T = h.thr >> 16, Rl = h.thr & 0xFFFFu;
      const TrialHalf tb_half = tiebreak_trial_half(trial, K);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t m = 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) m |= (half_of(o[c], j) == T ? 1u : 0u) << j;
        if (m) {
          const int q = 4 * w + c;
          const uint4 u = TABLE ? U[q] : philox_q_half((uint32_t)q, h.stream, K);
          const Word4 tb = philox_call_rolled(u, tb_half, K);
          for (int j = 0; j < 8; ++j)
            if ((m >> j) & 1u) {
              const uint32_t bit = 1u << (8 * c + j);
              R = half_of(tb, j) >= Rl ? (R | bit) : (R & ~bit);
            }
        }
      }
    }
    return R;
  } else {
    // the last word: 1 to 3 calls, unrolled with warp-uniform guards (cfg3 sample 187.1 -> 184.8 ms
    // against a loop, profiles/r02e_ab_halves_tail.jsonl)
#pragma unroll
    for (int j = 2; j >= 0; --j) {
      if (j >= ncalls) continue;
      DSI_CHECK(4 * w + j < nq);
      const uint4 u = TABLE ? U[4 * w + j] : philox_q_half((uint32_t)(4 * w + j), h.stream, K);
      const Word4 o = philox_call(u, th, K);
      R = pack8(R, o, h.C);
      tf = tie_flags<DIRECT>(o, h.TT, tf);
    }
  }
  R |= h.orall;
#ifdef DSI_MUTANT_TIES
  tf = 0u;
#endif
  if (tf) R = halves_fix<TABLE>(R, w, ncalls, U, trial, h.stream, h.thr, K);
  return R;
}
template <bool TABLE>
__device__ __forceinline__ uint32_t gen_word_halves(int w, int nq, const uint4 *U, const TrialHalf &th, uint32_t trial,
                                                    const HalvesCtx &h, const Keys &K) {
  return h.direct ? gen_word_halves_t<true, TABLE>(w, nq, U, th, trial, h, K)
                  : gen_word_halves_t<false, TABLE>(w, nq, U, th, trial, h, K);
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
