// dsi_crn2.cu -- two-pass form of the shared-stream mode (DSI_F_SHARED_STREAMS) for
// large groups (the heatmap: 101 groups of 20 000 configs).
//
// The fused kernel (dsi_crn.cu) regenerates a trial's Philox stream once per block, i.e.
// once per slice of 256 configs: 79 times per trial of a heatmap group.  Here
//   pass 1, dsi_crn_stream_kernel: one block per (group, tile of TH trials), one trial per
//     thread: Philox + Bernoulli + segment walk exactly as dsi_kernel.cu, then the trial's
//     record -- summary (m, n2, longest run, run count | sum L | sum floor(L/2)) and its runs
//     of >= 2 accepted drafts sorted in decreasing order -- written once to global memory;
//   pass 2, dsi_crn_eval_kernel: one block per (group, slice of TH configs, trial range);
//     the tile records stream into shared memory with bulk asynchronous copies
//     (cp.async.bulk, completion on an mbarrier, two buffers so the copy of tile i+1
//     overlaps the evaluation of tile i), and each thread evaluates its config on the
//     tile's trials: the same closed form and moment algebra as the fused kernel, the long
//     runs walked in decreasing order until L <= k, and configs with k = 1 and no queueing
//     taking the per-trial sums (O(1)).
// Records are tile-major: [TH x uint4 summaries][FRESH: TH x uint2 short-run counts][max_runs x TH
// uint16 runs, run-major], so one tile is one contiguous copy of rec_bytes (a multiple of 16).
// FRESH (a launch with fresh-verifier configs, R24, which correct every segment): pass 1
// also counts each trial's runs of L = 2..kShortL accepted drafts (6-bit fields; a trial has at
// most max_runs <= 63 stored runs), and pass 2 prices them with kShortL - 1 per-config savings
// instead of walking them (cfg3 under R24: 211.5 -> 94.0 ms, profiles/r02_ab_freshcnt*.jsonl).
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "dsi_common.cuh"
#include "dsi_crn_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

// (an explicit minimum of 1 block per SM: 72 registers instead of 64, cfg3 unchanged)
#ifndef DSI_EVAL_MINB
#define DSI_EVAL_MINB 1
#endif

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// arm the barrier for `bytes` of incoming bulk-copy data, then start the copy
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t"
      "}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kShortL = 11;  // FRESH: runs of L = 2..kShortL accepted drafts are counted, not walked

template <int TH, bool FRESH>
__global__ void __launch_bounds__(TH) dsi_crn_stream_kernel(const CrnParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const CrnTile tile = P.tiles[P.tile_begin + blockIdx.x];
  const CrnGroup G = P.groups[tile.group];
  const int N = G.n_tokens;
  const int npos = N - 1;
  const int nwords = (npos + 31) >> 5;
  const bool halves = P.halves != 0;
  const int nq = halves ? (npos + 7) >> 3 : (npos + 3) >> 2;
  const uint32_t mode = G.mode;
  const uint32_t nthr = 0u - G.thr;
  const HalvesCtx hc = make_halves(G.thr, G.stream_id);
  uint4 *U = reinterpret_cast<uint4 *>(smem);
  uint16_t *runs_s = reinterpret_cast<uint16_t *>(smem + (size_t)P.max_nq * sizeof(uint4));  // [r * TH + tid]
  if (mode == MODE_STREAM)
    for (int q = threadIdx.x; q < nq; q += TH) U[q] = philox_q_half((uint32_t)q, G.stream_id, P.keys);
  __syncthreads();

  unsigned char *rec = P.records + (P.group_tile0[tile.group] + tile.tile) * (uint64_t)P.rec_bytes;
  uint4 *summ = reinterpret_cast<uint4 *>(rec);
  uint2 *cnts = reinterpret_cast<uint2 *>(rec + (size_t)TH * sizeof(uint4));
  uint16_t *runs = reinterpret_cast<uint16_t *>(rec + (size_t)TH * (sizeof(uint4) + (FRESH ? sizeof(uint2) : 0)));
  const uint64_t t = (uint64_t)tile.tile * TH + threadIdx.x;
  if (t >= G.n_trials) return;
  const TrialHalf th = philox_trial_half((uint32_t)t, P.keys);
  uint16_t *my = runs_s + threadIdx.x;
  int nz = 0, n2 = 0, run = 0, lastz = 0, nr = 0;
  uint32_t sum_l = 0, sum_half = 0;  // sum L, sum floor(L/2) over the runs (k = 1 corrections)
  uint64_t short_cnt = 0;            // FRESH: 6-bit counts of the runs with L = 2..kShortL
  auto push = [&](int L) {         // insertion into my[0..nr) kept in decreasing order
    if (FRESH && L <= kShortL) short_cnt += 1ull << (6 * (L - 2));
    DSI_CHECK(nr < P.max_runs);
    int i = nr++;
    while (i > 0) {
      const int prev = my[(i - 1) * TH];
      if (prev >= L) break;
      my[i * TH] = (uint16_t)prev;
      --i;
    }
    my[i * TH] = (uint16_t)L;
    sum_l += (uint32_t)L;
    sum_half += (uint32_t)L >> 1;
  };
  for (int w = 0; w < nwords; ++w) {
    uint32_t Rw;
    if (mode == MODE_STREAM && halves) {
      Rw = gen_word_halves<true>(w, nq, U, th, (uint32_t)t, hc, P.keys);
    } else if (mode == MODE_STREAM) {
      Rw = 0u;
      const int ncalls = min(8, nq - 8 * w);
      if (ncalls == 8) {
#pragma unroll
        for (int j = 7; j >= 0; --j) Rw = pack4(Rw, philox_call(U[8 * w + j], th, P.keys), nthr);
      } else {
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
      if (L >= 2) push(L);
    }
    lastz = base + 31 - __clz(Rw);
    run = nv - 1 - (31 - __clz(Rw));
  }
  n2 += run >= 1;  // the final segment (the trailing run, then position N)
  if (run >= 2) push(run);
  const uint32_t maxL = nr ? my[0] : 0u;
  summ[threadIdx.x] = make_uint4((uint32_t)(nz + 1), (uint32_t)n2, maxL,
                                 (uint32_t)nr | (sum_l << 10) | (sum_half << 21));
  if (FRESH) cnts[threadIdx.x] = make_uint2((uint32_t)short_cnt, (uint32_t)(short_cnt >> 32));
  for (int r = 0; r < nr; ++r) runs[r * TH + threadIdx.x] = my[r * TH];
}

// FRESH: the launch holds a fresh-verifier config (R24); compiled out otherwise (88 registers
// against 72 without: 2 blocks per SM instead of 3)
template <int TH, bool FRESH>
__global__ void __launch_bounds__(TH, DSI_EVAL_MINB) dsi_crn_eval_kernel(const CrnParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_bsum[5];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_kmin, s_nlong, s_wcnt[TH / 32];
  __shared__ uint16_t s_long[TH];  // (non-FRESH) the tile's trials with a run longer than s_kmin
  const CrnUnit un = P.units[P.unit_begin + blockIdx.x];
  const CrnGroup G = P.groups[un.group];
  const int N = G.n_tokens;
  // buffer b of the two tile buffers is smem + b * rec_bytes (computed from the shared array
  // itself, so the loads stay shared-memory loads)
  if (threadIdx.x < 5) s_bsum[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) {
    s_kmin = 1 << 30;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // each thread's own config, straight into registers
  const CfgLite l = load_cfglite(P.cfg, P.perm, un, threadIdx.x, N);
  CfgFr f{};
  if (FRESH) f = load_cfgfr(P.cfg, P.perm, un, threadIdx.x);
  const bool fresh = FRESH && f.fresh != 0;
  // FRESH: the savings of runs of L = 2..kShortL accepted drafts, this config's (0 if not fresh)
  int sv_short[kShortL - 1];
#pragma unroll
  for (int i = 0; i < kShortL - 1; ++i) sv_short[i] = fresh ? fresh_saving_lite(i + 2, l, f) : 0;
  __syncthreads();
  if (!FRESH && (int)threadIdx.x < (int)un.count) atomicMin(&s_kmin, l.k_eff);
  __syncthreads();
  const int kmin = s_kmin;  // the block's smallest lookahead: shorter runs are long for none of it

  const uint64_t tile_a = un.t0 / TH, tile_b = (un.t1 + TH - 1) / TH;  // un.t0 is tile-aligned
  const unsigned char *rec0 = P.records + (P.group_tile0[un.group] + tile_a) * (uint64_t)P.rec_bytes;
  if (threadIdx.x == 0) bulk_load(smem, rec0, P.rec_bytes, &bar[0]);

  const bool fast = l.noqueue && l.k_eff == 1;  // every run is long; S(b) = b k t_d
  // the lanes of a warp share k (lookahead-major order) and differ in t_d: where none of
  // them queues, the long-run loop needs no SP division (warp-uniform, so no divergence)
  const bool warp_noqueue = __all_sync(0xffffffffu, l.noqueue != 0);
  // without a long run L_DSI - L_SI = n2 S(1) - m k t_d <= m (S(1) - k t_d) (n2 <= m): where no
  // lane of the warp has S(1) > k t_d (SP >= 2 always), the L_DSI > L_SI counter can only move
  // on trials with a long run -- the short path skips it (a warp-uniform choice of loop)
  const bool warp_gts_long_only = __all_sync(0xffffffffu, l.s1 <= l.kd);
  unsigned long long c_ai = 0, c_ai2 = 0, c_mai = 0, c_ay = 0, c_ay2 = 0, c_ydl = 0, a_gtn = 0, a_gts = 0;
  unsigned long long my_m = 0, my_n = 0, my_mm = 0, my_nn = 0, my_mn = 0;
  for (uint64_t ti = tile_a; ti < tile_b; ++ti) {
    const int cur = (int)((ti - tile_a) & 1);
    if (threadIdx.x == 0 && ti + 1 < tile_b) {
      // the other buffer was last read in the previous iteration (ended by __syncthreads)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(smem + (size_t)(cur ^ 1) * P.rec_bytes, rec0 + (ti + 1 - tile_a) * (uint64_t)P.rec_bytes,
                P.rec_bytes, &bar[cur ^ 1]);
    }
    mbar_wait(&bar[cur], (uint32_t)(((ti - tile_a) >> 1) & 1));
    const unsigned char *bufc = smem + (size_t)cur * P.rec_bytes;
    const uint4 *summ = reinterpret_cast<const uint4 *>(bufc);
    const uint2 *cnts = reinterpret_cast<const uint2 *>(bufc + (size_t)TH * sizeof(uint4));
    const uint16_t *runs =
        reinterpret_cast<const uint16_t *>(bufc + (size_t)TH * (sizeof(uint4) + (FRESH ? sizeof(uint2) : 0)));
    const uint64_t tile0 = ti * TH;
    const int ntr = (int)(min(un.t1, tile0 + TH) - tile0);
    bool has_long = false;
    if ((int)threadIdx.x < ntr) {  // the config-independent block sums, one trial per thread
      const uint4 v = summ[threadIdx.x];
      my_m += v.x;
      my_n += v.y;
      my_mm += v.x * v.x;
      my_nn += v.y * v.y;
      my_mn += v.x * v.y;
      has_long = (int)v.z > kmin;
    }
    if (!FRESH) {  // compact the trials that need a correction for some config of the block
      const unsigned bal = __ballot_sync(0xffffffffu, has_long);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < TH / 32; ++w) {
        off += w < warp ? s_wcnt[w] : 0;
        tot += s_wcnt[w];
      }
      if (has_long) s_long[off + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)threadIdx.x;
      if (threadIdx.x == 0) s_nlong = tot;
      __syncthreads();
    }
    // per-tile 32-bit partial sums (ai <= N/2, m <= N <= 2048, 256 trials: no overflow)
    uint32_t p_gtn = 0, p_gts = 0, p_ai = 0, p_ai2 = 0, p_mai = 0;
    auto visit = [&](const uint4 v, const int s, auto gts_long_only) {
      const int m = (int)v.x, n2 = (int)v.y, maxL = (int)v.z;
      int dsi = m * l.t_t + n2 * l.s1;
      int si = m * l.si_cost;
      // corrections: some run is long for this config, or (fresh-verifier variant) some
      // segment has g >= 2 -- every one of them saves time (R24)
      if (maxL > l.k_eff || (fresh && n2 > 0)) {
        const int nr = (int)(v.w & 0x3ffu);
        int ai = 0, ay = 0;
        if (fast) {  // k = 1: ai = sum floor(L/2), ay = k t_d sum L - nr S(1)
          ai = (int)(v.w >> 21);
          ay = (int)((v.w >> 10) & 0x7ffu) * l.kd - nr * l.s1;
        } else if (warp_noqueue) {  // S(b) = b k t_d: ay = k t_d sum ceil(L/k) - n S(1)
          int sb = 0, cnt = 0, sv = 0;
          for (int r = 0; r < nr; ++r) {  // runs in decreasing order: stop at the first short one
            const int L = runs[r * TH + s];
            // (fresh: every run saves; those of L <= kShortL are priced from their counts below)
            if (L <= l.k_eff && (!fresh || L <= kShortL)) break;
            if (L > l.k_eff) {
              ai += (int)magic_div((uint32_t)L, l.m_si, 0u);
              sb += (int)magic_div((uint32_t)L + (uint32_t)l.k_eff - 1u, l.m_k_lo, l.m_k_hi);
              ++cnt;
            }
            if (fresh && L > kShortL) sv += fresh_saving_lite(L, l, f);
          }
          ay = sb * l.kd - cnt * l.s1 - sv;
        } else {
          for (int r = 0; r < nr; ++r) {
            const int L = runs[r * TH + s];
            if (L <= l.k_eff && (!fresh || L <= kShortL)) break;
            if (L > l.k_eff) long_run(L, l, ai, ay);
            if (fresh && L > kShortL) ay -= fresh_saving_lite(L, l, f);
          }
        }
        if (fresh) {
          ay -= (n2 - nr) * (l.kd - l.t_t);  // the runs of L = 1 (not stored)
          const uint2 c = cnts[s];
          const uint64_t c64 = (uint64_t)c.x | ((uint64_t)c.y << 32);
#pragma unroll
          for (int i = 0; i < kShortL - 1; ++i) ay -= (int)((c64 >> (6 * i)) & 63u) * sv_short[i];
        }
        p_ai += (unsigned)ai;
        p_ai2 += (unsigned)(ai * ai);
        p_mai += (unsigned)(m * ai);
        // ay may be negative (fresh savings): signed products, wrapped into the u64 sums
        c_ay += (unsigned long long)(long long)ay;
        c_ay2 += (unsigned long long)((long long)ay * ay);
        c_ydl += (unsigned long long)((long long)ay * dsi);
        dsi += ay;
        si += ai * l.si_cost;
        if (decltype(gts_long_only)::value) p_gts += (uint32_t)(si - dsi) >> 31;
      }
      // dsi, si, nonsi < 2^31: the sign bit of the difference is the comparison
      p_gtn += (uint32_t)(l.nonsi - dsi) >> 31;
      if (!decltype(gts_long_only)::value) p_gts += (uint32_t)(si - dsi) >> 31;
    };
    auto trials = [&](auto gts_long_only) {
      int s = 0;
      for (; s + 1 < ntr; s += 2) {
        const uint4 v0 = summ[s], v1 = summ[s + 1];
        visit(v0, s, gts_long_only);
        visit(v1, s + 1, gts_long_only);
      }
      if (s < ntr) visit(summ[s], s, gts_long_only);
    };
    // non-FRESH: a branch-free pass over every trial with the uncorrected latencies, then the
    // corrections over the compacted trials with a run longer than the block's smallest k (the
    // threshold counters re-decided there); the same integers as visit()
    auto base = [&](const uint4 v, auto gts_long_only) {
      const int dsi = (int)v.x * l.t_t + (int)v.y * l.s1;
      p_gtn += (uint32_t)(l.nonsi - dsi) >> 31;
      if (!decltype(gts_long_only)::value) p_gts += (uint32_t)(dsi > (int)v.x * l.si_cost);
    };
    auto split = [&](auto gts_long_only) {
      int s = 0;
      for (; s + 1 < ntr; s += 2) {
        const uint4 v0 = summ[s], v1 = summ[s + 1];
        base(v0, gts_long_only);
        base(v1, gts_long_only);
      }
      if (s < ntr) base(summ[s], gts_long_only);
      const int nl = s_nlong;
      for (int j = 0; j < nl; ++j) {
        const int s2 = s_long[j];
        const uint4 v = summ[s2];
        if ((int)v.z <= l.k_eff) continue;  // no run is long for this config
        const int m = (int)v.x, n2 = (int)v.y;
        const int dsi0 = m * l.t_t + n2 * l.s1, si0 = m * l.si_cost;
        const uint32_t g0n = (uint32_t)(l.nonsi - dsi0) >> 31, g0s = (uint32_t)(si0 - dsi0) >> 31;
        visit(v, s2, gts_long_only);  // adds the corrections and the corrected counters ...
        p_gtn -= g0n;                 // ... the base pass counted the uncorrected ones
        if (!decltype(gts_long_only)::value) p_gts -= g0s;
      }
    };
    if (FRESH) {
      if (warp_gts_long_only) trials(std::true_type{});
      else trials(std::false_type{});
    } else {
      if (warp_gts_long_only) split(std::true_type{});
      else split(std::false_type{});
    }
    a_gtn += p_gtn;
    a_gts += p_gts;
    c_ai += p_ai;
    c_ai2 += p_ai2;
    c_mai += p_mai;
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
  if ((int)threadIdx.x >= (int)un.count) return;
  const unsigned long long Sm = s_bsum[0], Sn = s_bsum[1], Smm = s_bsum[2], Snn = s_bsum[3], Smn = s_bsum[4];
  const unsigned long long tt = (unsigned)l.t_t, ss = (unsigned)l.s1;
  unsigned long long *dst = P.acc + (size_t)P.perm[un.begin + threadIdx.x] * NF;
  atomicAdd(dst + F_M, Sm);
  atomicAdd(dst + F_I, Sm + c_ai);
  atomicAdd(dst + F_I2, Smm + 2ull * c_mai + c_ai2);
  atomicAdd(dst + F_DSI, tt * Sm + ss * Sn + c_ay);
  // sum (m t + n2 s + ay)^2 = t^2 Smm + s^2 Snn + 2 t s Smn + 2 sum ay (m t + n2 s) + sum ay^2
  atomicAdd(dst + F_DSI2, tt * tt * Smm + ss * ss * Snn + 2ull * tt * ss * Smn + 2ull * c_ydl + c_ay2);
  if (a_gtn) atomicAdd(dst + F_GT_NONSI, a_gtn);
  if (a_gts) atomicAdd(dst + F_GT_SI, a_gts);
  atomicAdd(dst + F_TRIALS, (unsigned long long)(un.t1 - un.t0));
}

template <class K>
int launch_grid(K kernel, const CrnParams &p, uint64_t n_blocks, int threads, size_t smem, cudaStream_t st,
                bool tiles) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const uint64_t max_grid = 0x7fffffffull;
  CrnParams q = p;
  for (uint64_t done = 0; done < n_blocks;) {
    const uint64_t n = (n_blocks - done) < max_grid ? (n_blocks - done) : max_grid;
    if (tiles) q.tile_begin = p.tile_begin + done;
    else q.unit_begin = p.unit_begin + done;
    kernel<<<(unsigned)n, threads, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

}  // namespace

size_t crn_record_bytes(int max_runs, int threads, bool fresh) {
  return ((size_t)threads * (sizeof(uint4) + (fresh ? sizeof(uint2) : 0)) + (size_t)max_runs * threads * sizeof(uint16_t) +
          15) &
         ~(size_t)15;
}

size_t crn_eval_smem(int max_runs, int threads, bool fresh) { return 2 * crn_record_bytes(max_runs, threads, fresh); }

int launch_crn_two_pass(const CrnParams &p, uint64_t n_tiles, uint64_t n_units, int threads, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (threads != 256) return (int)cudaErrorInvalidValue;
  if (n_tiles) {
    const size_t smem = (size_t)p.max_nq * sizeof(uint4) + (size_t)p.max_runs * threads * sizeof(uint16_t);
    const int e = p.any_fresh ? launch_grid(dsi_crn_stream_kernel<256, true>, p, n_tiles, threads, smem, st, true)
                              : launch_grid(dsi_crn_stream_kernel<256, false>, p, n_tiles, threads, smem, st, true);
    if (e) return e;
  }
  if (n_units) {
    const size_t smem = crn_eval_smem(p.max_runs, threads, p.any_fresh != 0);
    return p.any_fresh ? launch_grid(dsi_crn_eval_kernel<256, true>, p, n_units, threads, smem, st, false)
                       : launch_grid(dsi_crn_eval_kernel<256, false>, p, n_units, threads, smem, st, false);
  }
  return 0;
}

}  // namespace dsi
