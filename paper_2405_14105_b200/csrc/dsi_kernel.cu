// dsi_kernel.cu -- sm_100a trial kernel of the DSI Monte Carlo latency simulator.
//
// One thread simulates one trial at a time.  A block owns one work unit
// (configuration c, tile of up to tile_trials consecutive trials); its threads
// stride over the tile.  Per trial:
//   1. Philox4x32-10 in registers, 8 calls per 32 positions; A_p = [u < thr] for
//      p = 1..N-1 is packed as a rejection mask (bit i of word w = position 32w+i+1,
//      set when A_p = 0) with a carry chain (add.cc/addc: 2 instructions per bit).
//   2. The zeros of the mask cut the trial into segments g_1..g_m (sum g = N).
//      Every segment starts with all servers free (a rejection terminates every
//      thread, Alg. 1 lines 8/10), so its costs depend on g only:
//        SI: ceil(g/(k+1)) iterations of k t_d + t_t
//        DSI (Alg. 1 P:112-142 + App. D): C(g) = t_t + S(ceil((g-1)/k)),
//            S(b) = max(b k t_d, (b mod SP) k t_d + floor(b/SP) t_t)  (FIFO, R7)
//      A segment of length 1 costs exactly (1 SI iteration, t_t), one with
//      2 <= g <= k+1 exactly (1, t_t + S(1)), so
//        I = m + sum_long x(g),  L_DSI = m t_t + n2 S(1) + sum_long y(g),
//      with n2 = popc(zeros preceded by an accepted draft, E = R & ~(R << 1 | carry))
//      and only the "long" segments (runs of >= k+1 accepted drafts) walked, found by
//      a log-doubling run detector (walk_word).  The fresh-verifier variant walks every
//      segment with g >= 2 (Lk = 1); HIST walks every zero.
//   3. Integer moments are reduced with warp shuffles and added to the
//      per-config accumulators with 64-bit integer atomics (exact, order-free).
//
// Where the time goes (ncu): Philox's 32x32->64 multiplies (IMAD.WIDE,
// ~4 cycles of the fmaheavy pipe each) bound the kernel.  So
//   - rounds 0 and 1 carry no multiply that depends on both the trial and the
//     counter q: the trial half is hoisted per trial, the q half (uniform across
//     the warp) is precomputed per block into shared memory (U table);
//   - the per-segment divisions become a shared-memory table T[g] = (ceil(g/(k+1))-1,
//     S(ceil((g-1)/k))) read with LDS, keeping the walk off the fmaheavy pipe.
// Nothing here is a contraction: no tensor cores, and HBM traffic is the config table
// and the per-config moment accumulators.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

constexpr int TABLE_MAX_N = 4096;
// Launch bounds: blocks of at most 128 threads, at least 5 per SM -- a register budget of
// ~100 per thread, of which ptxas takes 91 with the pipelined walk (78 before it); round 2: a
// minimum of 6 blocks (80 registers) 1.8% slower, of 4 the same (profiles/r02_ab_minb*.jsonl).  Measured (profiles/r01_ab_lb.jsonl, cfg3): 78
// registers 244.1 ms, 84 (bounds (256, 1)) 246.0 ms, 58 (bounds (256), no minimum) 251.3 ms,
// 70 / 64 / 48 registers 248.5 / 250.0 / 257.5 ms: more registers than the occupancy
// heuristic picks keep more independent Philox calls in flight.
#ifndef DSI_TRIAL_MINB
#define DSI_TRIAL_MINB 5
#endif
#ifndef DSI_TRIAL_MINB_HALVES
#define DSI_TRIAL_MINB_HALVES 4  // halves layout: min 4 blocks 1.3% faster than 5, 6 1.0% slower
#endif                           // (profiles/r02c_ab_halves_minb.jsonl)
#ifndef DSI_PIPE_WALK
#define DSI_PIPE_WALK 1  // (cfg3 sample 243.16 -> 242.38 ms, profiles/r02_ab_pipewalk.jsonl)
#endif
#ifndef DSI_TRIAL_MAXT
#define DSI_TRIAL_MAXT 128
#endif  // larger N: arithmetic segment costs, per-call rounds 0-1

// Test-mode (DSI_F_HIST) accounting of one segment into the block histograms.
__device__ __forceinline__ void seg_hist(int g, int seg_start, const SegCtx &s, unsigned int *sh_seg,
                                         unsigned int *sh_si) {
  atomicAdd(&sh_seg[g < 63 ? g : 63], 1u);
  // the first M-1 SI iterations of a segment accept k drafts each; the last
  // accepts r-1 and is counted only if its k-draft window ends before N
  const int kk = (int)s.k_eff;
  const int M = (int)magic_div((uint32_t)g + s.k_eff, s.m_si, 0u);
  DSI_CHECK(g >= 1 && g <= s.n_tokens);
  if (M > 1) atomicAdd(&sh_si[kk], (unsigned)(M - 1));
  const int last_start = seg_start + (M - 1) * (kk + 1);
  const int r = g - (M - 1) * (kk + 1);
  DSI_CHECK(r >= 1 && r - 1 <= kk);
  if (last_start + kk + 1 <= s.n_tokens) atomicAdd(&sh_si[r - 1], 1u);
}

// Production accounting of one word of the rejection mask R (bit i = position
// base+i, nv valid bits, bits >= nv are zero).  Segments with g >= 2 end at a zero
// whose predecessor is a one (mask E) and each costs (0, S(1)) unless its run of
// ones is long (L = g-1 >= Lk = k+1); long segments add T[g] = seg_long(g).
// FRESH (the fresh-verifier variant, k t_d > t_t, Lk = 1): every segment with g >= 2 is walked
// and its cost is lowered by the fresh forwards' saving (the table already holds it).
template <bool TABLE, bool FRESH>
__device__ __forceinline__ uint2 long_cost(int g, const uint2 *T, const SegCtx &s, int t_d) {
  if (TABLE) {
    DSI_CHECK(g >= 0 && g <= s.n_tokens);
    return T[g];
  }
  uint2 e = seg_long(g, s);
  if (FRESH) e.y -= fresh_saving(g, s, t_d);
  return e;
}

template <bool TABLE, bool FRESH>
__device__ __forceinline__ void walk_word(uint32_t R, int nv, int Lk, const uint2 *T, const SegCtx &s, int t_d,
                                          int &run, int &n2, uint32_t &ai, uint32_t &ay) {
  if (R == 0) {
    run += nv;  // the run of accepted drafts continues through the word
    return;
  }
  const uint32_t E = R & ~((R << 1) | (run == 0 ? 1u : 0u));
  n2 += __popc(E);
  const int z0 = __ffs(R) - 1;  // the first zero closes the run carried in
  if (run + z0 >= Lk) {
    const uint2 e = long_cost<TABLE, FRESH>(run + z0 + 1, T, s, t_d);
    ai += e.x;
    ay += e.y;
  }
  if (Lk <= 30) {
    // runs of >= Lk ones strictly inside the word (between two zeros)
    const uint32_t V = nv >= 32 ? 0xffffffffu : (1u << nv) - 1u;
    const uint32_t y = runs_at_least(~R & V & ~((2u << z0) - 1u), Lk);
    uint32_t El = R & (y << 1);
    while (El) {
      const int zb = 31 - __clz(El);
      El ^= 1u << zb;
      const int g = zb - (31 - __clz(R & ((1u << zb) - 1u)));
      const uint2 e = long_cost<TABLE, FRESH>(g, T, s, t_d);
      ai += e.x;
      ay += e.y;
    }
  }
  run = nv - 1 - (31 - __clz(R));  // ones above the last zero
}

// walk_word for a full word (32 valid positions) when no run strictly inside a word can be long
// (Lk > 30): branch-free, so the compiler can schedule it among the next word's Philox calls.
// T[0] = (0, 0) absorbs the common "no long run" case.
__device__ __forceinline__ void walk_full_word_nb(uint32_t R, int Lk, const uint2 *T, int &run, int &n2, uint32_t &ai,
                                                  uint32_t &ay, int n) {
  const uint32_t E = R & ~((R << 1) | (run == 0 ? 1u : 0u));
  n2 += __popc(E);
  const int z0 = __ffs(R) - 1;  // -1 when R == 0
  const bool lng = (R != 0u) & (run + z0 >= Lk);
  DSI_CHECK(!lng || run + z0 + 1 <= n);
  const uint2 e = T[lng ? run + z0 + 1 : 0];
  ai += e.x;
  ay += e.y;
  run = R ? (int)__clz(R) : run + 32;  // ones above the last zero
}

// Shared-memory layout of the TABLE variant for a config with N tokens.
__host__ __device__ __forceinline__ size_t t_table_bytes(int n) { return (size_t)((n + 2) & ~1) * 8; }
__host__ __device__ __forceinline__ size_t u_table_bytes(int n) { return (size_t)((n - 1 + 3) / 4 + 1) * 16; }

// VAR: 0 = default model, 1 = TTFT variant present, 2 = fresh-verifier variant present,
//      3 = default model with the k = 1 no-queue fast path compiled in (LaunchParams.k1_fast)
// HALVES: the halves layout of the indicator stream (DSI_F_RNG_HALVES, dsi_common.cuh)
template <bool PER_TRIAL, bool HIST, bool PATTERN, bool TABLE, int VAR, bool HALVES>
__global__ void __launch_bounds__(DSI_TRIAL_MAXT, HALVES ? DSI_TRIAL_MINB_HALVES : DSI_TRIAL_MINB)
    dsi_trial_kernel(const LaunchParams P) {
  extern __shared__ __align__(16) unsigned char smem[];

  __shared__ uint32_t s_cfg;
  const uint64_t unit = P.unit_begin + blockIdx.x;
  if (threadIdx.x == 0) {
    // config owning this unit: largest c with tile_prefix[c] <= unit
    uint32_t lo = 0, hi = P.n_cfg;  // invariant: prefix[lo] <= unit < prefix[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&P.tile_prefix[mid]) <= unit) lo = mid; else hi = mid;
    }
    s_cfg = lo;
  }
  __syncthreads();
  // (A/B measured, profiles/r01_ab.jsonl: balanced tiles, a direct unit -> config
  //  division and a host-built unit -> config map were each 1-5% slower than this)
  const uint32_t c = s_cfg;
  DSI_CHECK(c < P.n_cfg);
  const DevCfg cfg = P.cfg[c];
  const uint64_t t0 = (unit - __ldg(&P.tile_prefix[c])) * P.tile_trials;
  const uint64_t t1 = min(t0 + P.tile_trials, cfg.n_trials);

  const uint32_t mode = cfg.flags & 0xffu;
  const int N = cfg.n_tokens;
  const int npos = N - 1;  // positions carrying an indicator
  const int nwords = (npos + 31) >> 5;
  const int nq = HALVES ? (npos + 7) >> 3 : (npos + 3) >> 2;  // Philox calls per trial
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
  s.n_tokens = N;
  s.s1 = cfg.s1;
  const uint32_t nthr = 0u - cfg.thr;  // carry of u + nthr <=> u >= thr (thr >= 1 in stream mode)
  const bool stream = !PATTERN && mode == MODE_STREAM;
  // fresh-verifier variant (k t_d > t_t, R24): every segment with g >= 2 costs
  // C_fresh(g) != C(g), so the production walk visits all of them (Lk = 1, "long" = g >= 2)
  // with the saving folded into the table
  const bool fresh = VAR == 2 && (cfg.flags & CFG_FRESH) != 0;
  const bool walk_all = HIST;
  const int Lk = fresh ? 1 : cfg.k_eff + 1;  // a run of >= Lk accepted drafts is walked
  // k = 1 without queueing (Eq. 1 holds at k = 1: most of config 5): C(g) = t_t + (g-1) t_d, so
  // L_DSI = m t_t + (N-m) t_d, and I = sum ceil(g/2) = (N + #odd segments)/2, where a segment is odd
  // iff its two ends (consecutive zeros, or N) differ in parity: counted per word with bit
  // operations instead of walking the runs (block-uniform choice)
  const bool fast1 = VAR == 3 && !walk_all && cfg.k_eff == 1 && (cfg.flags & CFG_NOQUEUE) != 0;
  const int t_d = cfg.t_d;
  const HalvesCtx hc = make_halves(cfg.thr, cfg.stream_id);

  // shared memory: TABLE -> T[g] (g = 0..N) then U[q] (q < nq); HIST -> histograms
  uint2 *T = reinterpret_cast<uint2 *>(smem);
  uint4 *U = reinterpret_cast<uint4 *>(smem + t_table_bytes(N));
  unsigned int *sh_seg = reinterpret_cast<unsigned int *>(smem);
  unsigned int *sh_si = sh_seg + 64;
  if (TABLE) {
    for (int g = threadIdx.x; g <= N; g += blockDim.x) {
      uint2 e = make_uint2(0u, 0u);
      if (g >= 2) {
        e = HIST ? seg_extra(g, s) : seg_long(g, s);
        if (fresh) e.y -= fresh_saving(g, s, t_d);  // may wrap: sums are read as int32
      }
      T[g] = e;
    }
    if (stream)
      for (int q = threadIdx.x; q < nq; q += blockDim.x) U[q] = philox_q_half((uint32_t)q, cfg.stream_id, P.keys);
  }
  if (HIST)
    for (int i = threadIdx.x; i < 64 + cfg.k_eff + 1; i += blockDim.x) sh_seg[i] = 0u;
  // TTFT variant: first-segment correction D1[g] = C1(g) - C(g) (R23).  Thread 0
  // runs the FIFO schedule of the first segment in O(B): thread 0 (the target's first
  // forward, t_t1) holds one server; threads b >= 1 arrive at t_d1 + (b k - 1) t_d with
  // service t_t and take the earliest free server -- a never-used one (free at 0), thread
  // 0's server (free at t_t1) or the one of the earliest earlier thread still holding one
  // (finish times of threads b >= 1 are nondecreasing, so they form a FIFO queue: F[h]).
  // (a template parameter: launches without a TTFT config compile the variant out)
  const bool ttft = VAR == 1 && (cfg.flags & CFG_TTFT) != 0;
  int *F = reinterpret_cast<int *>(smem + (HIST ? (size_t)(64 + P.max_keff + 1) * 4
                                                : t_table_bytes(N) + u_table_bytes(N)));
  int *D1 = F + (N + 2);
  if (ttft) {
    if (TABLE || HIST) __syncthreads();
    if (threadIdx.x == 0) {
      const int B = N > 1 ? (N - 2) / cfg.k_eff + 1 : 0;  // ceil((N-1)/k)
      int zero_servers = cfg.sp_eff - 1, h = 1;
      bool first_unused = true;
      F[0] = cfg.t_t1;
      for (int b = 1; b <= B; ++b) {
        const int r = cfg.ttft_shift + b * cfg.kd;  // t_d1 + (b k - 1) t_d
        int free_at;
        if (zero_servers > 0) {
          free_at = 0;
          --zero_servers;
        } else if (first_unused && (h >= b || cfg.t_t1 <= F[h])) {
          free_at = cfg.t_t1;
          first_unused = false;
        } else {
          free_at = F[h++];
        }
        F[b] = max(r, free_at) + cfg.t_t;
      }
      for (int b = 1; b <= B; ++b) F[b] = max(F[b], F[b - 1]);  // positions settle in order
    }
    __syncthreads();
    for (int g = threadIdx.x; g <= N; g += blockDim.x) {
      if (g == 0) {
        D1[0] = 0;
        continue;
      }
      const uint32_t b = magic_div((uint32_t)g + s.k_eff - 2u, s.m_k_lo, s.m_k_hi);  // ceil((g-1)/k)
      const int S = (int)seg_extra(g, s).y;  // S(b) of the closed form (0 for g = 1)
      D1[g] = F[b] - (cfg.t_t + (g >= 2 ? S : 0));
    }
  }
  if (TABLE || HIST || ttft) __syncthreads();

  unsigned long long a_m = 0, a_i = 0, a_i2 = 0, a_dsi = 0, a_dsi2 = 0, a_gtn = 0, a_gts = 0,
                     a_trials = 0;
  const int64_t nonsi = cfg.nonsi;  // t_t1 + (N-1) t_t

  for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const uint32_t trial = (uint32_t)t;
    const TrialHalf th = philox_trial_half(trial, P.keys);

    int nz = 0;        // zeros (rejections) among positions 1..N-1
    int g1 = 0;        // TTFT variant: length of the first segment (position of the first zero)
    int n2 = 0;        // segments with g >= 2 (production walk)
    int run = 0;       // accepted drafts since the last zero (production walk)
    int lastz = 0;     // HIST walk: position of the last zero (0 = sentinel before position 1)
    uint32_t cin = 1;  // HIST walk: position 32w is a zero (the sentinel for w = 0)
    uint32_t ai = 0, ay = 0;  // summed extra costs (HIST: seg_extra of every g >= 2 segment;
                              // production: seg_long of every segment with g >= k+2)
    int odd = 0;       // fast1: segments of odd length so far
    uint32_t lzp = 0;  // fast1: parity of the last zero's position (the sentinel 0 is even)
    int w_start = 0;
#if DSI_PIPE_WALK
    if (VAR == 0 && TABLE && !HIST && !PATTERN && stream && Lk > 30) {
      // full words with the walk of word w-1 after the generation of word w, one straight-line block
      auto gen_word = [&](int w) {
        if (HALVES) return gen_word_halves<true>(w, nq, U, th, trial, hc, P.keys);
        uint32_t R = 0u;
#pragma unroll
        for (int j = 7; j >= 0; --j) R = pack4(R, philox_call(U[8 * w + j], th, P.keys), nthr);
        return R;
      };
      const int nfull = npos >> 5;
      if (nfull >= 1) {
        uint32_t Rp = gen_word(0);
        nz += __popc(Rp);
        for (int w = 1; w < nfull; ++w) {
          const uint32_t R = gen_word(w);
          walk_full_word_nb(Rp, Lk, T, run, n2, ai, ay, N);
          nz += __popc(R);
          Rp = R;
        }
        walk_full_word_nb(Rp, Lk, T, run, n2, ai, ay, N);
        w_start = nfull;
      }
    }
#endif
    for (int w = w_start; w < nwords; ++w) {
      uint32_t R;
      if (PATTERN) {
        R = ~trial;  // N <= 33: one word, A_p = bit p-1 of the trial index
      } else if (mode == MODE_STREAM && HALVES) {
        R = gen_word_halves<TABLE>(w, nq, U, th, trial, hc, P.keys);
      } else if (mode == MODE_STREAM) {
        R = 0u;
        const int ncalls = min(8, nq - 8 * w);
        if (ncalls == 8) {
#pragma unroll
          for (int j = 7; j >= 0; --j) {
            DSI_CHECK(8 * w + j < nq);
            const uint4 u = TABLE ? U[8 * w + j] : philox_q_half((uint32_t)(8 * w + j), cfg.stream_id, P.keys);
            R = pack4(R, philox_call(u, th, P.keys), nthr);
          }
        } else {
          // (a loop: unrolled with warp-uniform guards it was 1% slower on cfg3, equal on cfg5,
          //  profiles/r02e_ab_words_tail*.jsonl -- unlike the halves layout's last word)
          for (int j = ncalls - 1; j >= 0; --j) {
            DSI_CHECK(8 * w + j < nq);
            const uint4 u = TABLE ? U[8 * w + j] : philox_q_half((uint32_t)(8 * w + j), cfg.stream_id, P.keys);
            R = pack4(R, philox_call(u, th, P.keys), nthr);
          }
        }
      } else {
        R = (mode == MODE_ALL_REJECT) ? 0xffffffffu : 0u;
      }
      const int base = 32 * w + 1;  // position of bit 0
      const int rem = npos - 32 * w;
      if (rem < 32) R &= (1u << rem) - 1u;
      nz += __popc(R);
      if (ttft && g1 == 0 && R) g1 = 32 * w + __ffs(R);
      if (walk_all) {
        // test mode (HIST): walk every zero
        uint32_t Z = R;
        while (Z) {
          const int z = base + __ffs(Z) - 1;
          Z &= Z - 1u;
          const int g = z - lastz;
          if (HIST) seg_hist(g, lastz, s, sh_seg, sh_si);
          if (g >= 2) {
            DSI_CHECK(g >= 2 && g <= N);
            uint2 e = TABLE ? T[g] : seg_extra(g, s);
            if (!TABLE && VAR == 2 && fresh) e.y -= fresh_saving(g, s, t_d);
            ai += e.x;
            ay += e.y;
          }
          lastz = z;
        }
      } else if (fast1) {
        // bit i is position 32w + i + 1: odd positions at even i
        const uint32_t Eo = R & 0x55555555u, Ee = R & 0xAAAAAAAAu, NR = ~R;
        // bits after each odd (even) zero up to and including the next zero of this word
        const uint32_t Fo = (NR + (Eo << 1)) ^ NR, Fe = (NR + (Ee << 1)) ^ NR;
        odd += __popc(Fo & Ee) + __popc(Fe & Eo);  // consecutive zeros of different parity
        if (R) {
          const uint32_t first_odd = (R & (0u - R) & 0x55555555u) != 0u;  // first zero of the word
          odd += (int)(first_odd ^ lzp);
          lzp = ((31 - __clz(R)) & 1) ^ 1u;  // the word's last zero: bit b is odd iff b even
        }
      } else if (VAR == 2 && fresh) {
        walk_word<TABLE, true>(R, rem >= 32 ? 32 : rem, Lk, T, s, t_d, run, n2, ai, ay);
      } else {
        walk_word<TABLE, false>(R, rem >= 32 ? 32 : rem, Lk, T, s, t_d, run, n2, ai, ay);
      }
      if (HIST) cin = R >> 31;
    }
    int gl;
    if (walk_all) {
      gl = N - lastz;  // the final segment ends at N
      if (HIST) seg_hist(gl, lastz, s, sh_seg, sh_si);
      if (gl >= 2) {
        DSI_CHECK(gl >= 2 && gl <= N);
        uint2 e = TABLE ? T[gl] : seg_extra(gl, s);
        if (!TABLE && VAR == 2 && fresh) e.y -= fresh_saving(gl, s, t_d);
        ai += e.x;
        ay += e.y;
      }
    } else {
      gl = run + 1;  // the final segment: the trailing run of ones, then position N
      n2 += gl >= 2;
      if (run >= Lk) {
        DSI_CHECK(gl <= N);
        const uint2 e = (VAR == 2 && fresh) ? long_cost<TABLE, true>(gl, T, s, t_d) : long_cost<TABLE, false>(gl, T, s, t_d);
        ai += e.x;
        ay += e.y;
      }
    }

    const int m = nz + 1;
    int iters = m + (int)ai;
    // Every per-trial latency is < 2^31 ticks (create's overflow bound), so L_DSI and L_SI are
    // formed in 32-bit modular arithmetic -- exact, whatever the partial sums -- and squared with one
    // 32x32->64 multiply each.  (ay is a sum of signed 32-bit terms: fresh savings may exceed
    // S(b) - S(1).)
    uint32_t dsi = (uint32_t)m * (uint32_t)cfg.t_t + (uint32_t)n2 * (uint32_t)cfg.s1 + ay;
    if (fast1) {  // the final segment ends at N
      odd += (int)(((uint32_t)N & 1u) ^ lzp);
      iters = (N + odd) >> 1;
      dsi = (uint32_t)m * (uint32_t)cfg.t_t + (uint32_t)(N - m) * (uint32_t)cfg.kd;
    }
    uint32_t si = (uint32_t)iters * (uint32_t)cfg.si_cost;
    if (ttft) {  // first forwards: SI's first iteration and DSI's first segment
      DSI_CHECK(g1 >= 0 && g1 <= N);
      dsi += (uint32_t)D1[g1 ? g1 : N];
      si += (uint32_t)cfg.e_si;
    }
    a_m += (unsigned)m;
    a_i += (unsigned)iters;
    a_i2 += (unsigned long long)((uint32_t)iters * (uint32_t)iters);  // I <= N: I^2 < 2^32
    a_dsi += dsi;
    a_dsi2 += (unsigned long long)dsi * dsi;
    a_gtn += dsi > (uint32_t)nonsi;
    a_gts += dsi > si;
    a_trials += 1;
    if (PER_TRIAL) {
      const uint64_t r = cfg.rec_off + t;
      DSI_CHECK(t < cfg.n_trials);
      P.rec_acc[r] = npos - nz;
      P.rec_m[r] = m;
      P.rec_iters[r] = iters;
      P.rec_si[r] = (int32_t)si;
      P.rec_dsi[r] = (int32_t)dsi;
    }
  }

  // warp shuffle reduction, then one 64-bit integer atomic per field per warp
  a_m = warp_sum(a_m);
  a_i = warp_sum(a_i);
  a_i2 = warp_sum(a_i2);
  a_dsi = warp_sum(a_dsi);
  a_dsi2 = warp_sum(a_dsi2);
  a_gtn = warp_sum(a_gtn);
  a_gts = warp_sum(a_gts);
  a_trials = warp_sum(a_trials);
  if ((threadIdx.x & 31) == 0 && a_trials) {
    unsigned long long *acc = P.acc + (size_t)c * NF;
    atomicAdd(acc + F_M, a_m);
    atomicAdd(acc + F_I, a_i);
    atomicAdd(acc + F_I2, a_i2);
    atomicAdd(acc + F_DSI, a_dsi);
    atomicAdd(acc + F_DSI2, a_dsi2);
    if (a_gtn) atomicAdd(acc + F_GT_NONSI, a_gtn);
    if (a_gts) atomicAdd(acc + F_GT_SI, a_gts);
    atomicAdd(acc + F_TRIALS, a_trials);
  }
  if (HIST) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64; i += blockDim.x)
      if (sh_seg[i]) atomicAdd(P.seg_hist + (size_t)c * 64 + i, (unsigned long long)sh_seg[i]);
    for (int i = threadIdx.x; i <= cfg.k_eff; i += blockDim.x)
      if (sh_si[i]) atomicAdd(P.si_hist + cfg.si_hist_off + i, (unsigned long long)sh_si[i]);
  }
}

template <bool A, bool B, bool C, bool D, int E, bool H>
int launch_variant_h(const LaunchParams &p, uint64_t n_units, int threads, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(dsi_trial_kernel<A, B, C, D, E, H>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const uint64_t max_grid = 0x7fffffffull;
  LaunchParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < max_grid ? (n_units - done) : max_grid;
    q.unit_begin = p.unit_begin + done;
    dsi_trial_kernel<A, B, C, D, E, H><<<(unsigned)n, threads, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

// the halves layout is instantiated only where the stream is read (not in PATTERN launches)
template <bool A, bool B, bool C, bool D, int E>
int launch_variant_t(const LaunchParams &p, uint64_t n_units, int threads, size_t smem, cudaStream_t st) {
  if constexpr (!C) {
    if (p.halves) return launch_variant_h<A, B, C, D, E, true>(p, n_units, threads, smem, st);
  }
  return launch_variant_h<A, B, C, D, E, false>(p, n_units, threads, smem, st);
}

template <bool A, bool B, bool C, bool D>
int launch_variant(const LaunchParams &p, uint64_t n_units, int threads, size_t smem, cudaStream_t st) {
  if (p.any_fresh) return launch_variant_t<A, B, C, D, 2>(p, n_units, threads, smem, st);
  if (p.any_ttft) return launch_variant_t<A, B, C, D, 1>(p, n_units, threads, smem, st);
  if (p.k1_fast) return launch_variant_t<A, B, C, D, 3>(p, n_units, threads, smem, st);
  return launch_variant_t<A, B, C, D, 0>(p, n_units, threads, smem, st);
}

}  // namespace

size_t trial_kernel_smem(int max_n, int max_keff, bool hist, bool ttft) {
  const size_t first = ttft ? (size_t)2 * (max_n + 2) * sizeof(int) : 0;  // F and D1
  if (hist) return (size_t)(64 + max_keff + 1) * sizeof(unsigned int) + first;
  if (max_n > TABLE_MAX_N) return first;
  return t_table_bytes(max_n) + u_table_bytes(max_n) + first;
}

int launch_trial_kernel(const LaunchParams &p, uint64_t n_units, int block_threads, bool per_trial,
                        bool hist, bool pattern, void *stream) {
  if (n_units == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = trial_kernel_smem(p.max_n, p.max_keff, hist, p.any_ttft != 0);
  const int code = (per_trial ? 2 : 0) | (pattern ? 1 : 0);
  if (hist) {
    // histograms occupy shared memory: segment costs come from arithmetic
    switch (code) {
      case 0: return launch_variant<false, true, false, false>(p, n_units, block_threads, smem, st);
      case 1: return launch_variant<false, true, true, false>(p, n_units, block_threads, smem, st);
      case 2: return launch_variant<true, true, false, false>(p, n_units, block_threads, smem, st);
      default: return launch_variant<true, true, true, false>(p, n_units, block_threads, smem, st);
    }
  }
  if (p.max_n <= TABLE_MAX_N) {
    switch (code) {
      case 0: return launch_variant<false, false, false, true>(p, n_units, block_threads, smem, st);
      case 1: return launch_variant<false, false, true, true>(p, n_units, block_threads, smem, st);
      case 2: return launch_variant<true, false, false, true>(p, n_units, block_threads, smem, st);
      default: return launch_variant<true, false, true, true>(p, n_units, block_threads, smem, st);
    }
  }
  switch (code) {
    case 0: return launch_variant<false, false, false, false>(p, n_units, block_threads, smem, st);
    case 1: return launch_variant<false, false, true, false>(p, n_units, block_threads, smem, st);
    case 2: return launch_variant<true, false, false, false>(p, n_units, block_threads, smem, st);
    default: return launch_variant<true, false, true, false>(p, n_units, block_threads, smem, st);
  }
}

}  // namespace dsi
