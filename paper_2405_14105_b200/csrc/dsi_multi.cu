// dsi_multi.cu -- sm_100a kernel of multi-drafter DSI (include/dsi_sim.h
// dsi_multi_simulate): Algorithm 1 with m = D+1 models, lookahead 1, unbounded threads
// (P:112-142).  Per trial the run takes L_DSI = t_m + sum_{p=1}^{N-1} t_{j*(p)} (P:418,
// j_N = m), j*(p) the smallest drafter whose token at p equals the target's, else m.
//
// One thread simulates one trial at a time; a block owns one unit (config, tile of
// trials).  Positions come in quads (one Philox call = 4 positions): drafter 1's call
// settles the positions it accepts, drafter 2's call is made only if some position of the
// quad is still open, and so on (A_{j,p} of the other drafters is never needed there).
// Drafter j draws Philox4x32-10 at counter (q, j-1, trial, stream): round 0's
// per-trial product M1*trial is shared by all drafters (c1 = j-1 enters by xor), round 1's
// per-trial product M0*n0 is hoisted per (trial, drafter), and the per-q half (rounds 0-1
// of the (q, stream) words) is staged per block in shared memory when N <= 4096.  Counts
// per drafter live in registers (D is a template parameter), moments are reduced with warp
// shuffles and added with 64-bit integer atomics (exact, order-free).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

constexpr int MULTI_TABLE_MAX_N = 4096;


// 4 acceptance bits of a quad: bit i = [word i < thr] (thr < 2^32)
__device__ __forceinline__ uint32_t accept4(const Word4 &w, uint32_t thr) {
  return (uint32_t)(w.x < thr) | (uint32_t)(w.y < thr) << 1 | (uint32_t)(w.z < thr) << 2 |
         (uint32_t)(w.w < thr) << 3;
}

// acceptance bits of one drafter's call for quad u (rounds 0-1 halves: u per q, ha/la per
// (trial, drafter), n1 per trial)
__device__ __forceinline__ uint32_t call4(const uint4 &u, uint32_t n1, uint32_t ha, uint32_t la, uint32_t thr,
                                          const Keys &K) {
  return accept4(philox_rounds_2_9(u.x ^ n1, u.y, ha ^ u.z, la, K), thr);
}

// The halves layout (DSI_F_RNG_HALVES, R26) for drafter j (0-based): the call at counter
// (q, 2j, trial, stream) gives 8 acceptance bits (bit i = position 8q + i + 1), a tie decided by
// the call at (q, 2j + 1, ...): its trial half of rounds 0-1 differs only through c1 (n0 ^ (2j+1)).
// Drafter 0 draws exactly the single-drafter halves stream (counter words 1 = 0 and 1).
__device__ __forceinline__ uint32_t call8(const uint4 &u, uint32_t n1, uint32_t ha, uint32_t la, uint32_t thr,
                                          const Keys &K, uint32_t pt_hi, uint32_t c1) {
  const Word4 o = philox_rounds_2_9(u.x ^ n1, u.y, ha ^ u.z, la, K);
  const uint32_t T = thr >> 16;
  const uint32_t TT = T | (T << 16);
  uint32_t rej = pack8(0u, o, (0x10000u - T) << 16) | (T == 0u ? 0xFFu : 0u);
  if (tie_flags<false>(o, TT, 0u)) {  // rare: exact decisions of the tied positions
    const uint32_t n0 = pt_hi ^ (c1 + 1u) ^ K.k0[0];
    const uint64_t a = (uint64_t)PHILOX_M0 * n0;
    const TrialHalf tb_half{n1, (uint32_t)(a >> 32), (uint32_t)a};
    const Word4 tb = philox_call_rolled(u, tb_half, K);
    const uint32_t Rl = thr & 0xFFFFu;
    for (int j = 0; j < 8; ++j)
      if (half_of(o, j) == T) rej = half_of(tb, j) >= Rl ? (rej | 1u << j) : (rej & ~(1u << j));
  }
  return ~rej & 0xFFu;
}

template <bool HALVES>
__device__ __forceinline__ uint32_t callw(const uint4 &u, uint32_t n1, uint32_t ha, uint32_t la, uint32_t thr,
                                          const Keys &K, uint32_t pt_hi, uint32_t c1) {
  if (HALVES) return call8(u, n1, ha, la, thr, K, pt_hi, c1);
  return call4(u, n1, ha, la, thr, K);
}

// HALVES: positions come in octets (one call = 8 positions) instead of quads.
template <int D, bool PATTERN, bool TABLE, bool HALVES>
__global__ void __launch_bounds__(128) dsi_multi_kernel(const MultiParams P) {
  constexpr int W = HALVES ? 8 : 4;                  // positions per call
  constexpr uint32_t FULL = HALVES ? 0xFFu : 0xFu;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_cfg;
  const uint64_t unit = P.unit_begin + blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = P.n_cfg;  // prefix[lo] <= unit < prefix[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&P.tile_prefix[mid]) <= unit) lo = mid; else hi = mid;
    }
    s_cfg = lo;
  }
  __syncthreads();
  const uint32_t c = s_cfg;
  const MultiCfg cfg = P.cfg[c];
  const uint64_t t0 = (unit - __ldg(&P.tile_prefix[c])) * P.tile_trials;
  const uint64_t t1 = min(t0 + P.tile_trials, cfg.n_trials);
  const int nd = cfg.n_drafters;
  const int npos = cfg.n_tokens - 1;
  const int nq = (npos + W - 1) / W;
  const uint32_t tail = npos % W ? (1u << (npos % W)) - 1u : FULL;  // open bits of the last call

  uint4 *U = reinterpret_cast<uint4 *>(smem);
  if (TABLE && !PATTERN) {
    for (int q = threadIdx.x; q < nq; q += blockDim.x)
      U[q] = philox_q_half((uint32_t)q, cfg.stream_id, P.keys);
    __syncthreads();
  }

  unsigned long long a_dsi = 0, a_dsi2 = 0, a_gt = 0, a_trials = 0;
  unsigned long long a_set[D];
#pragma unroll
  for (int j = 0; j < D; ++j) a_set[j] = 0;

  for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    uint32_t cnt[D];
#pragma unroll
    for (int j = 0; j < D; ++j) cnt[j] = 0;
    if (PATTERN) {
      // digit p-1 of the trial index in base m is j*(p) - 1
      uint64_t x = t;
      const uint32_t m = (uint32_t)nd + 1u;
      for (int p = 1; p <= npos; ++p) {
        const uint32_t d = (uint32_t)(x % m);
        x /= m;
#pragma unroll
        for (int j = 0; j < D; ++j) cnt[j] += (d == (uint32_t)j && j < nd);
      }
    } else {
      // per-trial halves of rounds 0-1, one per drafter (counter word 1 = j)
      const uint64_t pt = (uint64_t)PHILOX_M1 * (uint32_t)t;
      const uint32_t n1 = (uint32_t)pt;
      const uint32_t pt_hi = (uint32_t)(pt >> 32);
      uint32_t ha[D], la[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const uint32_t n0 = pt_hi ^ (uint32_t)(HALVES ? 2 * j : j) ^ P.keys.k0[0];
        const uint64_t a = (uint64_t)PHILOX_M0 * n0;
        ha[j] = (uint32_t)(a >> 32);
        la[j] = (uint32_t)a;
      }
      // Quads in groups of 4 (16 positions): drafter 1's four calls are independent chains
      // the scheduler interleaves.  A later drafter j is called per group, per pair or per
      // quad (cfg.width[j]: 4, 2, 1) for the quads with an open position -- the host picks
      // the widest grouping whose extra calls are rare (P(quad open) high).
      int q = 0;
      for (; q + 3 < nq; q += 4) {
        uint4 u[4];
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          u[i] = TABLE ? U[q + i] : philox_q_half((uint32_t)(q + i), cfg.stream_id, P.keys);
          o[i] = q + i == nq - 1 ? tail : FULL;
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (j < nd && (o[0] | o[1] | o[2] | o[3])) {
            uint32_t c[4] = {0u, 0u, 0u, 0u};
            if (cfg.mode[j] != MODE_STREAM) {
#pragma unroll
              for (int i = 0; i < 4; ++i) c[i] = cfg.mode[j] == MODE_ALL_ACCEPT ? o[i] : 0u;
            } else if (j == 0 || cfg.width[j] == 4) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                c[i] = callw<HALVES>(u[i], n1, ha[j], la[j], cfg.thr[j], P.keys, pt_hi, 2 * j) & o[i];
            } else if (cfg.width[j] == 2) {
#pragma unroll
              for (int i = 0; i < 4; i += 2)
                if (o[i] | o[i + 1]) {
                  c[i] = callw<HALVES>(u[i], n1, ha[j], la[j], cfg.thr[j], P.keys, pt_hi, 2 * j) & o[i];
                  c[i + 1] = callw<HALVES>(u[i + 1], n1, ha[j], la[j], cfg.thr[j], P.keys, pt_hi, 2 * j) & o[i + 1];
                }
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (o[i]) c[i] = callw<HALVES>(u[i], n1, ha[j], la[j], cfg.thr[j], P.keys, pt_hi, 2 * j) & o[i];
            }
            cnt[j] += __popc(c[0] | c[1] << W | c[2] << (2 * W) | c[3] << (3 * W));
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] &= ~c[i];
          }
        }
      }
      for (; q < nq; ++q) {  // the last nq mod 4 quads one at a time
        const uint4 uq = TABLE ? U[q] : philox_q_half((uint32_t)q, cfg.stream_id, P.keys);
        uint32_t open = q == nq - 1 ? tail : FULL;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (j < nd && open) {
            uint32_t acc;
            if (cfg.mode[j] == MODE_STREAM) {
              acc = callw<HALVES>(uq, n1, ha[j], la[j], cfg.thr[j], P.keys, pt_hi, 2 * j) & open;
            } else {
              acc = cfg.mode[j] == MODE_ALL_ACCEPT ? open : 0u;
            }
            cnt[j] += __popc(acc);
            open &= ~acc;
          }
        }
      }
    }
    uint32_t by_drafters = 0;
    int64_t dsi = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      by_drafters += cnt[j];
      dsi += (int64_t)cnt[j] * cfg.t_d[j];
      a_set[j] += cnt[j];
    }
    const uint32_t by_target = (uint32_t)npos - by_drafters;
    dsi += (int64_t)cfg.t_t * (1 + by_target);  // position N always comes from the target
    a_dsi += (unsigned long long)dsi;
    a_dsi2 += (unsigned long long)dsi * (unsigned long long)dsi;
    a_gt += dsi > (int64_t)cfg.t_t * cfg.n_tokens;
    a_trials += 1;
    if (P.rec_dsi) P.rec_dsi[cfg.rec_off + t] = (int32_t)dsi;
    if (P.rec_settled) {
      int32_t *r = P.rec_settled + (cfg.rec_off + t) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int32_t v = 0;
        if (j < D && j < nd) v = (int32_t)cnt[j < D ? j : 0];
        if (j == nd) v = (int32_t)by_target;
        r[j] = v;
      }
    }
  }

  a_dsi = warp_sum(a_dsi);
  a_dsi2 = warp_sum(a_dsi2);
  a_gt = warp_sum(a_gt);
  a_trials = warp_sum(a_trials);
#pragma unroll
  for (int j = 0; j < D; ++j) a_set[j] = warp_sum(a_set[j]);
  if ((threadIdx.x & 31) == 0 && a_trials) {
    unsigned long long *acc = P.acc + (size_t)c * MF;
    atomicAdd(acc + MF_DSI, a_dsi);
    atomicAdd(acc + MF_DSI2, a_dsi2);
    if (a_gt) atomicAdd(acc + MF_GT_NONSI, a_gt);
    atomicAdd(acc + MF_TRIALS, a_trials);
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (a_set[j]) atomicAdd(acc + MF_SETTLED + j, a_set[j]);
  }
}

template <int D, bool PATTERN, bool TABLE, bool HALVES>
int launch_multi_t(const MultiParams &p, uint64_t n_units, cudaStream_t st) {
  const size_t smem = TABLE && !PATTERN ? (size_t)((p.max_n - 1 + 3) / 4 + 1) * sizeof(uint4) : 0;
  const uint64_t max_grid = 0x7fffffffull;
  MultiParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < max_grid ? (n_units - done) : max_grid;
    q.unit_begin = p.unit_begin + done;
    dsi_multi_kernel<D, PATTERN, TABLE, HALVES><<<(unsigned)n, 128, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

template <int D>
int launch_multi_d(const MultiParams &p, uint64_t n_units, bool pattern, cudaStream_t st) {
  if (pattern) return launch_multi_t<D, true, false, false>(p, n_units, st);
  if (p.halves) {
    if (p.max_n <= MULTI_TABLE_MAX_N) return launch_multi_t<D, false, true, true>(p, n_units, st);
    return launch_multi_t<D, false, false, true>(p, n_units, st);
  }
  if (p.max_n <= MULTI_TABLE_MAX_N) return launch_multi_t<D, false, true, false>(p, n_units, st);
  return launch_multi_t<D, false, false, false>(p, n_units, st);
}

}  // namespace

int launch_multi_kernel(const MultiParams &p, uint64_t n_units, bool pattern, void *stream) {
  if (n_units == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  // the drafter loop is unrolled to D; configs with fewer drafters skip the rest
  if (p.max_drafters <= 1) return launch_multi_d<1>(p, n_units, pattern, st);
  if (p.max_drafters <= 2) return launch_multi_d<2>(p, n_units, pattern, st);
  if (p.max_drafters <= 4) return launch_multi_d<4>(p, n_units, pattern, st);
  return launch_multi_d<7>(p, n_units, pattern, st);
}

}  // namespace dsi
