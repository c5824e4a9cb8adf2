// dsi_crn.cu -- shared-stream (common random numbers) trial kernel, DSI_F_SHARED_STREAMS.
//
// By the random-number contract, configurations with equal (stream_id, threshold,
// N, n_trials) draw identical indicators for every trial index.  A group of such
// configurations (e.g. the 20 000 (t_d, k) points of one acceptance rate of the
// heatmap) therefore needs ONE Philox pass per trial.  This kernel:
//   block = (group, slice of <= TH configs of the group), loops over the group's
//   trials in tiles of TH (128, or 256 for large groups -- which the two-pass form in
//   dsi_crn2.cu usually takes instead):
//   phase 1 (one trial per thread): Philox + Bernoulli mask exactly as dsi_kernel.cu,
//     then the trial's summary m = #zeros + 1, n2 = #segments with g >= 2 and the list
//     of run lengths L of accepted drafts (a segment of length g has L = g - 1) that are
//     long for at least one of the block's configs (L > min k_eff), into shared memory;
//   phase 2 (each thread owns CPT configs, the tile's trials in lockstep):
//     I = m + sum_{L >= k+1} floor(L/(k+1)),
//     L_DSI = m t_t + n2 S(1) + sum_{L >= k+1} (S(ceil(L/k)) - S(1))
//     -- the closed form of DESIGN.md section 2 with short segments (2 <= g <= k+1)
//     costing (0, S(1)) -- then the per-config integer moments, in registers.
//   SUMS variant (sums-only units, every config k_eff = 1 without queueing): no run lists
//   at all, the corrections come from per-trial sums (see plan_shared).
// Per-trial latencies, and so every sum, are bit-identical to the per-config kernel.
// Bounds used for 32-bit arithmetic: L_DSI, L_SI < 2^31 (create validates
// N (k t_d + t_t) < 2^31), I <= N <= 2048 so I^2 * 256 trials < 2^32.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_crn_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

// An explicit minimum of 1 block per SM lets ptxas use 96 registers (80 with plain
// __launch_bounds__(TH)): cfg5 142.5 -> 136.0 ms, cfg4 1.15 -> 1.11 ms, cfg2 0.94 -> 1.10 ms
// (profiles/r01_ab_crn_regs.jsonl).
#ifndef DSI_CRN_MINB
#define DSI_CRN_MINB 1
#endif

// TH threads per block = trials per tile = configs per block (CPT = 1: 2 or 4 configs per
// thread measured slower, profiles/r01_ab_crn_cpt_unroll.jsonl)
// SUMS: a sums-only unit (CrnUnit::kind 1, every config k_eff = 1 without queueing): no
// run lists -- the corrections come from the per-trial sums alone (plan_shared)
// FRESH: the launch holds a fresh-verifier config (R24): its constants (CfgFr) are staged and
// its corrections compiled in; launches without one compile them out
template <int TH, int CPT, bool SUMS, bool FRESH>
__global__ void __launch_bounds__(TH, DSI_CRN_MINB) dsi_crn_kernel(const CrnParams P) {
  constexpr int CRN_THREADS = TH;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_bsum[5];
  const CrnUnit un = P.units[P.unit_begin + blockIdx.x];
  const CrnGroup G = P.groups[un.group];
  const int N = G.n_tokens;
  const int npos = N - 1;
  const int nwords = (npos + 31) >> 5;
  const bool halves = P.halves != 0;
  const int nq = halves ? (npos + 7) >> 3 : (npos + 3) >> 2;
  const uint32_t mode = G.mode;
  const uint32_t nthr = 0u - G.thr;
  const HalvesCtx hc = make_halves(G.thr, G.stream_id);

  // shared memory layout
  unsigned char *sp = smem;
  uint4 *U = reinterpret_cast<uint4 *>(sp);
  sp += (size_t)P.max_nq * sizeof(uint4);
  CfgLite *cl = reinterpret_cast<CfgLite *>(sp);
  sp += (size_t)CPT * CRN_THREADS * sizeof(CfgLite);
  CfgFr *cf = reinterpret_cast<CfgFr *>(sp);
  if (FRESH) sp += (size_t)CPT * CRN_THREADS * sizeof(CfgFr);
  // per trial slot: (m, n2, max stored L, nr | sum ceil(L/kmin) << 10 | sum floor(L/(kmin+1)) << 21)
  // (nr <= N/3 + 2 < 2^10, both sums <= N - 1 < 2^11: N <= 2048)
  uint4 *summ = reinterpret_cast<uint4 *>(sp);
  sp += (size_t)CRN_THREADS * sizeof(uint4);
  uint16_t *runs = reinterpret_cast<uint16_t *>(sp);  // runs[i * CRN_THREADS + slot]

  __shared__ int s_kmin, s_nfast, s_fresh;
  if (threadIdx.x < 5) s_bsum[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) {
    s_kmin = 1 << 30;
    s_nfast = 0;
    s_fresh = 0;
  }
  __syncthreads();
  if (mode == MODE_STREAM)
    for (int q = threadIdx.x; q < nq; q += CRN_THREADS) U[q] = philox_q_half((uint32_t)q, G.stream_id, P.keys);
  for (int j = threadIdx.x; j < CPT * CRN_THREADS; j += CRN_THREADS) {
    const CfgLite l = load_cfglite(P.cfg, P.perm, un, j, N);
    cl[j] = l;
    if (FRESH) cf[j] = load_cfgfr(P.cfg, P.perm, un, j);
    if (j < (int)un.count) {
      atomicMin(&s_kmin, l.k_eff);
      if (FRESH && cf[j].fresh) s_fresh = 1;
    }
  }
  __syncthreads();
  // a run of L accepted drafts is long for a config iff L > k_eff: runs of at most the
  // block's smallest k_eff are long for none of its configs and are not stored.  Configs
  // with k_eff == kmin (most of a block: configs are sorted by k) and no queueing take
  // every stored run, and their corrections are linear in per-trial sums over the runs:
  //   ai = sum floor(L/(k+1)),  ay = sum (S(ceil(L/k)) - S(1)) = kd sum ceil(L/k) - nr S(1)
  const int kmin = s_kmin;
  // fresh-verifier configs (k t_d > t_t) correct every segment with g >= 2: a block holding one
  // stores every run of L >= 2 (runs of L = 1 are counted as n2 - nr)
  const bool any_fresh = FRESH && s_fresh != 0;
  const int store_min = any_fresh ? 1 : kmin;
  for (int j = threadIdx.x; j < (int)un.count; j += CRN_THREADS)
    if (cl[j].noqueue && cl[j].k_eff == kmin) atomicAdd(&s_nfast, 1);
  __syncthreads();
  // the per-trial sums cost two divisions per stored run in phase 1: worth it only when
  // enough of the block's configs use them
  const bool sums = !any_fresh && s_nfast * 8 >= (int)un.count;
  const uint32_t mk_lo = (uint32_t)((0x100000000ull + (unsigned)kmin - 1) / (unsigned)kmin);
  const uint32_t mk_hi = kmin == 1 ? 1u : 0u;  // ceil(2^32 / kmin) = lo + hi 2^32
  const uint32_t mk1 = (uint32_t)((0x100000000ull + (unsigned)kmin) / (unsigned)(kmin + 1));

  // Per-trial latencies split into a config-independent part and long-run corrections:
  //   I = m + ai,  L_DSI = m t_t + n2 S(1) + ay   (ai = ay = 0 unless a run exceeds k)
  // so the moments are polynomials in sums the whole block shares -- Sm, Sn, Smm, Snn,
  // Smn over its trials -- plus per-config sums of ai, ai^2, m ai, ay, ay^2, m ay, n2 ay
  // that are only touched on trials with a long run.  The threshold counters need the
  // per-trial latency and are counted per (trial, config).
  // per owned config (registers): sums of ai, ai^2, m ai, ay, ay^2 and ay * (m t_t + n2 S(1))
  unsigned long long c_ai[CPT], c_ai2[CPT], c_mai[CPT], c_ay[CPT], c_ay2[CPT], c_ydl[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) c_ai[c] = c_ai2[c] = c_mai[c] = c_ay[c] = c_ay2[c] = c_ydl[c] = 0ull;
  unsigned long long a_gtn[CPT], a_gts[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) a_gtn[c] = a_gts[c] = 0ull;
  unsigned long long my_m = 0ull, my_n = 0ull, my_mm = 0ull, my_nn = 0ull, my_mn = 0ull;

  static_assert(CPT == 1, "one config per thread (replicas cover short slices)");
  const int C = (int)un.count;
  const int R = C >= CRN_THREADS ? 1 : CRN_THREADS / C;
  const int my_c = (int)threadIdx.x % C, my_r = (int)threadIdx.x / C;
  const bool active = (int)threadIdx.x < C * R;
  const uint64_t T = un.t1;  // this unit's trials: [un.t0, un.t1)
  for (uint64_t tile0 = un.t0; tile0 < T; tile0 += CRN_THREADS) {
    // ---------------- phase 1: one trial per thread -> summary + sorted long-run list
    const uint64_t t = tile0 + threadIdx.x;
    if (t < T) {
      const uint32_t trial = (uint32_t)t;
      const TrialHalf th = philox_trial_half(trial, P.keys);
      uint16_t *myruns = runs + threadIdx.x;
      int nz = 0, n2 = 0, run = 0, lastz = 0, nr = 0, maxL = 0;
      uint32_t sumb = 0, sumx = 0;  // sum ceil(L/kmin), sum floor(L/(kmin+1)) over stored runs
      for (int w = 0; w < nwords; ++w) {
        uint32_t Rw;
        if (mode == MODE_STREAM && halves) {
          Rw = gen_word_halves<true>(w, nq, U, th, trial, hc, P.keys);
        } else if (mode == MODE_STREAM) {
          Rw = 0u;
          const int ncalls = min(8, nq - 8 * w);
          if (ncalls == 8) {
#pragma unroll
            for (int j = 7; j >= 0; --j) Rw = pack4(Rw, philox_call(U[8 * w + j], th, P.keys), nthr);
          } else {
            DSI_CHECK(8 * w + ncalls <= nq && nq <= P.max_nq);
            for (int j = ncalls - 1; j >= 0; --j) Rw = pack4(Rw, philox_call(U[8 * w + j], th, P.keys), nthr);
          }
        } else {
          Rw = (mode == MODE_ALL_REJECT) ? 0xffffffffu : 0u;
        }
        const int base = 32 * w + 1;
        const int rem = npos - 32 * w;
        const int nv = rem >= 32 ? 32 : rem;
        if (rem < 32) Rw &= (1u << rem) - 1u;
        nz += __popc(Rw);
        if (Rw == 0) {
          run += nv;
          continue;
        }
        uint32_t E = Rw & ~((Rw << 1) | (run == 0 ? 1u : 0u));  // zeros preceded by a one
        n2 += __popc(E);
        while (E) {
          const int zb = 31 - __clz(E);
          E ^= 1u << zb;
          const uint32_t below = Rw & ((1u << zb) - 1u);
          const int prev = below ? base + 31 - __clz(below) : lastz;
          const int L = base + zb - prev - 1;  // accepted drafts in this segment
          if (L > store_min) {
            DSI_CHECK(SUMS || nr < P.max_runs);
            if (!SUMS) myruns[nr * CRN_THREADS] = (uint16_t)L;
            ++nr;
            maxL = max(maxL, L);
            if (sums) {
              sumb += magic_div((uint32_t)(L + kmin - 1), mk_lo, mk_hi);
              sumx += magic_div((uint32_t)L, mk1, 0u);
            }
          }
        }
        lastz = base + 31 - __clz(Rw);
        run = nv - 1 - (31 - __clz(Rw));
      }
      n2 += run >= 1;  // the final segment (the trailing run, then position N)
      if (run > store_min) {
        DSI_CHECK(SUMS || nr < P.max_runs);
        if (!SUMS) myruns[nr * CRN_THREADS] = (uint16_t)run;
        ++nr;
        maxL = max(maxL, run);
        if (sums) {
          sumb += magic_div((uint32_t)(run + kmin - 1), mk_lo, mk_hi);
          sumx += magic_div((uint32_t)run, mk1, 0u);
        }
      }

      const uint32_t m = (uint32_t)(nz + 1);
      summ[threadIdx.x] = make_uint4(m, (uint32_t)n2, (uint32_t)maxL, (uint32_t)nr | (sumb << 10) | (sumx << 21));
      my_m += m;
      my_n += (unsigned)n2;
      my_mm += m * m;
      my_nn += (unsigned)(n2 * n2);
      my_mn += m * (unsigned)n2;
    }
    __syncthreads();
    // ---------------- phase 2: R replicas of each of the unit's C configs (R = TH / C when
    // the slice is short: a group of 3 configs, or the k >= 2 remainder of a sums-only
    // split, still keeps every warp busy); replica r takes the tile's trials r, r+R, ...
    const int ntr = (int)min((uint64_t)CRN_THREADS, T - tile0);
    if (active) {
      const CfgLite l = cl[my_c];
      CfgFr f{};
      if (FRESH) f = cf[my_c];
      const bool fresh = FRESH && f.fresh != 0;
      // per-tile 32-bit partial sums (ai <= N/2, m <= N <= 2048, <= 256 trials: no overflow)
      uint32_t p_gtn = 0, p_gts = 0, p_ai = 0, p_ai2 = 0, p_mai = 0;
      auto visit = [&](const uint4 v, const int s) {
        const int m = (int)v.x, n2 = (int)v.y, maxL = (int)v.z;
        int dsi = m * l.t_t + n2 * l.s1;
        int si = m * l.si_cost;
        // corrections: a run long for this config, or (fresh variant) any segment with g >= 2
        if (maxL > l.k_eff || (!SUMS && fresh && n2 > 0)) {
          const int nr = (int)(v.w & 0x3ffu);
          int ai = 0, ay = 0;
          if (SUMS || (sums && l.noqueue && l.k_eff == kmin)) {  // every stored run, S linear in b
            ai = (int)(v.w >> 21);
            ay = (int)((v.w >> 10) & 0x7ffu) * l.kd - nr * l.s1;
          } else {
            for (int r = 0; r < nr; ++r) {  // the stored runs, in trial order
              const int L = runs[r * CRN_THREADS + s];
              if (L > l.k_eff) long_run(L, l, ai, ay);
              if (fresh) ay -= fresh_saving_lite(L, l, f);
            }
            if (fresh) ay -= (n2 - nr) * (l.kd - l.t_t);  // the runs of L = 1 (not stored)
          }
          p_ai += (unsigned)ai;
          p_ai2 += (unsigned)(ai * ai);
          p_mai += (unsigned)(m * ai);
          // ay may be negative (fresh savings): signed products, wrapped into the u64 sums
          c_ay[0] += (unsigned long long)(long long)ay;
          c_ay2[0] += (unsigned long long)((long long)ay * ay);
          c_ydl[0] += (unsigned long long)((long long)ay * dsi);
          dsi += ay;
          si += ai * l.si_cost;
        }
        // dsi, si, nonsi < 2^31: the sign bit of the difference is the comparison
        p_gtn += (uint32_t)(l.nonsi - dsi) >> 31;
        p_gts += (uint32_t)(si - dsi) >> 31;
      };
      int s = my_r;
      for (; s + R < ntr; s += 2 * R) {  // two trials per iteration: half the loop overhead
        const uint4 v0 = summ[s], v1 = summ[s + R];
        visit(v0, s);
        visit(v1, s + R);
      }
      if (s < ntr) visit(summ[s], s);
      a_gtn[0] += p_gtn;
      a_gts[0] += p_gts;
      c_ai[0] += p_ai;
      c_ai2[0] += p_ai2;
      c_mai[0] += p_mai;
    }
    __syncthreads();
  }
  // block sums of the config-independent terms
  for (int o = 16; o > 0; o >>= 1) {
    my_m += __shfl_xor_sync(0xffffffffu, my_m, o);
    my_n += __shfl_xor_sync(0xffffffffu, my_n, o);
    my_mm += __shfl_xor_sync(0xffffffffu, my_mm, o);
    my_nn += __shfl_xor_sync(0xffffffffu, my_nn, o);
    my_mn += __shfl_xor_sync(0xffffffffu, my_mn, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_bsum[0], my_m);
    atomicAdd(&s_bsum[1], my_n);
    atomicAdd(&s_bsum[2], my_mm);
    atomicAdd(&s_bsum[3], my_nn);
    atomicAdd(&s_bsum[4], my_mn);
  }
  __syncthreads();
  const unsigned long long Sm = s_bsum[0], Sn = s_bsum[1], Smm = s_bsum[2], Snn = s_bsum[3], Smn = s_bsum[4];
  // per config: assemble the moments (exact u64 arithmetic) and add them with 64-bit
  // integer atomics (exact and order-free); replica 0 adds the block-sum terms, every
  // replica its own trials' corrections and counters
  if (!active) return;
  const CfgLite &l = cl[my_c];
  const unsigned long long tt = (unsigned)l.t_t, ss = (unsigned)l.s1;
  const bool first = my_r == 0;
  unsigned long long *dst = P.acc + (size_t)P.perm[un.begin + my_c] * NF;
  const unsigned long long sum_i = (first ? Sm : 0ull) + c_ai[0];
  const unsigned long long sum_i2 = (first ? Smm : 0ull) + 2ull * c_mai[0] + c_ai2[0];
  const unsigned long long sum_dsi = (first ? tt * Sm + ss * Sn : 0ull) + c_ay[0];
  // sum (m t + n2 s + ay)^2 = t^2 Smm + s^2 Snn + 2 t s Smn + 2 sum ay (m t + n2 s) + sum ay^2
  const unsigned long long sum_dsi2 =
      (first ? tt * tt * Smm + ss * ss * Snn + 2ull * tt * ss * Smn : 0ull) + 2ull * c_ydl[0] + c_ay2[0];
  if (first) {
    atomicAdd(dst + F_M, Sm);
    atomicAdd(dst + F_TRIALS, (unsigned long long)(un.t1 - un.t0));
  }
  if (sum_i) atomicAdd(dst + F_I, sum_i);
  if (sum_i2) atomicAdd(dst + F_I2, sum_i2);
  if (sum_dsi) atomicAdd(dst + F_DSI, sum_dsi);
  if (sum_dsi2) atomicAdd(dst + F_DSI2, sum_dsi2);
  if (a_gtn[0]) atomicAdd(dst + F_GT_NONSI, a_gtn[0]);
  if (a_gts[0]) atomicAdd(dst + F_GT_SI, a_gts[0]);
}

template <int TH, bool SUMS, bool FRESH>
int launch_th(const CrnParams &p, uint64_t n_units, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(dsi_crn_kernel<TH, 1, SUMS, FRESH>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const uint64_t max_grid = 0x7fffffffull;
  CrnParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < max_grid ? (n_units - done) : max_grid;
    q.unit_begin = p.unit_begin + done;
    dsi_crn_kernel<TH, 1, SUMS, FRESH><<<(unsigned)n, TH, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

}  // namespace

size_t crn_kernel_smem(int max_n, int block_threads, int cfg_per_block, int max_runs, bool fresh) {
  const int max_nq = (max_n - 1 + 3) / 4 + 1;
  const size_t runs = ((size_t)block_threads * max_runs * sizeof(uint16_t) + 7) & ~(size_t)7;
  return (size_t)max_nq * sizeof(uint4) + (size_t)cfg_per_block * (sizeof(CfgLite) + (fresh ? sizeof(CfgFr) : 0)) +
         (size_t)block_threads * sizeof(uint4) + runs;
}

int launch_crn_kernel(const CrnParams &p, uint64_t n_units, int block_threads, void *stream, bool sums_only) {
  if (n_units == 0) return 0;
  if (p.cfg_per_block != block_threads) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  const bool fresh = p.any_fresh != 0;
  const size_t smem = crn_kernel_smem(p.max_n, block_threads, p.cfg_per_block, sums_only ? 0 : p.max_runs, fresh);
  // (sums-only units have every config k_eff = 1 without queueing: never fresh, k t_d <= t_t)
  if (block_threads != 128 && block_threads != 256) return (int)cudaErrorInvalidValue;
  if (sums_only)
    return block_threads == 128 ? launch_th<128, true, false>(p, n_units, smem, st)
                                : launch_th<256, true, false>(p, n_units, smem, st);
  if (fresh)
    return block_threads == 128 ? launch_th<128, false, true>(p, n_units, smem, st)
                                : launch_th<256, false, true>(p, n_units, smem, st);
  return block_threads == 128 ? launch_th<128, false, false>(p, n_units, smem, st)
                              : launch_th<256, false, false>(p, n_units, smem, st);
}

}  // namespace dsi
