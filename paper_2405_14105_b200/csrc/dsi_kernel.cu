// dsi_kernel.cu -- sm_100a trial kernel of the DSI Monte Carlo latency simulator.
//
// One thread simulates one trial at a time.  A block owns one work unit
// (configuration c, tile of up to tile_trials consecutive trials); its threads
// stride over the tile.  Per trial:
//   1. Philox4x32-10 in registers, 8 calls per 32 positions (4 words per call);
//      A_p = [u < thr] for p = 1..N-1 is packed as a rejection mask (bit = A_p == 0).
//   2. The zeros of the mask cut the trial into segments g_1..g_m (sum g = N).
//      Every segment starts with all servers free (a rejection terminates every
//      thread, Alg. 1 lines 8/10), so its costs depend on g only:
//        SI: ceil(g/(k+1)) iterations of k t_d + t_t
//        DSI (Alg. 1 P:112-142 + App. D): C(g) = t_t + S(ceil((g-1)/k)),
//            S(b) = max(b k t_d, (b mod SP) k t_d + floor(b/SP) t_t)  (FIFO, R7)
//   3. Integer moments are reduced with warp shuffles and added to the
//      per-config accumulators with 64-bit integer atomics (exact, order-free).
// Nothing here is a contraction: the kernel is bound by the SM issue rate
// (Philox is ~10 integer instructions per trial-token), not by HBM or tensor cores.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_device.h"

namespace dsi {
namespace {

constexpr uint32_t PHILOX_M0 = 0xD2511F53u;
constexpr uint32_t PHILOX_M1 = 0xCD9E8D57u;

struct Word4 {
  uint32_t x, y, z, w;
};

// Philox4x32-10 for counter (q, 0, trial, stream).  Round 0 depends on q only
// through M0*q; its trial half (M1*trial) is hoisted per trial by the caller:
//   r0_c0 = hi(M1*trial) ^ 0 ^ k0[0],  r0_c1 = lo(M1*trial),  sk1 = stream ^ k1[0].
__device__ __forceinline__ Word4 philox_q(uint32_t q, uint32_t r0_c0, uint32_t r0_c1, uint32_t sk1,
                                          const Keys &K) {
  uint64_t p0 = (uint64_t)PHILOX_M0 * q;
  uint32_t c0 = r0_c0;
  uint32_t c1 = r0_c1;
  uint32_t c2 = (uint32_t)(p0 >> 32) ^ sk1;
  uint32_t c3 = (uint32_t)p0;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    uint64_t a = (uint64_t)PHILOX_M0 * c0;
    uint64_t b = (uint64_t)PHILOX_M1 * c2;
    uint32_t n0 = (uint32_t)(b >> 32) ^ c1 ^ K.k0[r];
    uint32_t n2 = (uint32_t)(a >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)b;
    c3 = (uint32_t)a;
    c0 = n0;
    c2 = n2;
  }
  return Word4{c0, c1, c2, c3};
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
  int32_t sp_eff, kd, t_t, n_tokens;
  bool noqueue;
};

template <bool HIST>
__device__ __forceinline__ void segment(int g, int seg_start, const SegCtx &s, int &iters,
                                        int &sum_b, int &sum_s, unsigned int *sh_seg,
                                        unsigned int *sh_si) {
  // SI iterations in this segment: ceil(g / (k+1)) = floor((g + k) / (k+1))
  uint32_t M = magic_div((uint32_t)g + s.k_eff, s.m_si, 0u);
  iters += (int)M;
  // DSI: the last position of the segment is settled by thread b = ceil((g-1)/k)
  uint32_t b = magic_div((uint32_t)g + s.k_eff - 2u, s.m_k_lo, s.m_k_hi);
  if (s.noqueue) {
    sum_b += (int)b;  // S(b) = b k t_d
  } else {
    uint32_t qq = magic_div(b, s.m_sp_lo, s.m_sp_hi);
    int rr = (int)b - (int)qq * s.sp_eff;
    sum_s += max((int)b * s.kd, rr * s.kd + (int)qq * s.t_t);
  }
  if (HIST) {
    atomicAdd(&sh_seg[g < 63 ? g : 63], 1u);
    // the first M-1 SI iterations of a segment accept k drafts each; the last
    // accepts r-1 and is counted only if its k-draft window ends before N
    int kk = (int)s.k_eff;
    if (M > 1) atomicAdd(&sh_si[kk], M - 1u);
    int last_start = seg_start + ((int)M - 1) * (kk + 1);
    int r = g - ((int)M - 1) * (kk + 1);
    if (last_start + kk + 1 <= s.n_tokens) atomicAdd(&sh_si[r - 1], 1u);
  }
}

template <bool PER_TRIAL, bool HIST, bool PATTERN>
__global__ void __launch_bounds__(256) dsi_trial_kernel(const LaunchParams P) {
  extern __shared__ unsigned int sh_hist[];  // HIST only: 64 segment bins + k_eff+1 SI bins
  __shared__ uint32_t s_cfg;

  const uint64_t unit = P.unit_begin + blockIdx.x;
  if (threadIdx.x == 0) {
    // config owning this unit: largest c with tile_prefix[c] <= unit
    uint32_t lo = 0, hi = P.n_cfg;  // invariant: prefix[lo] <= unit < prefix[hi]
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&P.tile_prefix[mid]) <= unit) lo = mid; else hi = mid;
    }
    s_cfg = lo;
  }
  __syncthreads();
  const uint32_t c = s_cfg;
  const DevCfg cfg = P.cfg[c];
  const uint64_t tile = unit - __ldg(&P.tile_prefix[c]);
  const uint64_t t0 = tile * P.tile_trials;
  const uint64_t t1 = min(t0 + P.tile_trials, cfg.n_trials);

  const uint32_t mode = cfg.flags & 0xffu;
  const int N = cfg.n_tokens;
  const int npos = N - 1;  // positions carrying an indicator
  const int nwords = (npos + 31) >> 5;
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
  s.noqueue = (cfg.flags & CFG_NOQUEUE) != 0;
  const uint32_t thr = cfg.thr;
  const uint32_t sk1 = cfg.stream_id ^ P.keys.k1[0];
  const int64_t nonsi = (int64_t)N * cfg.t_t;

  unsigned int *sh_seg = sh_hist;
  unsigned int *sh_si = sh_hist + 64;
  if (HIST) {
    for (int i = threadIdx.x; i < 64 + cfg.k_eff + 1; i += blockDim.x) sh_hist[i] = 0u;
    __syncthreads();
  }

  unsigned long long a_m = 0, a_i = 0, a_i2 = 0, a_dsi = 0, a_dsi2 = 0, a_gtn = 0, a_gts = 0,
                     a_trials = 0;

  for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const uint32_t trial = (uint32_t)t;
    const uint64_t pt = (uint64_t)PHILOX_M1 * trial;
    const uint32_t r0_c0 = (uint32_t)(pt >> 32) ^ P.keys.k0[0];
    const uint32_t r0_c1 = (uint32_t)pt;

    int prev = 0, nz = 0, iters = 0, sum_b = 0, sum_s = 0;
    for (int w = 0; w < nwords; ++w) {
      uint32_t rej;
      if (PATTERN) {
        rej = ~trial;  // N <= 33: one word, A_p = bit p-1 of the trial index
      } else if (mode == MODE_STREAM) {
        rej = 0u;
        const int ncalls = min(8, (npos - 32 * w + 3) >> 2);
        if (ncalls == 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            Word4 u = philox_q((uint32_t)(8 * w + j), r0_c0, r0_c1, sk1, P.keys);
            rej |= ((uint32_t)(u.x >= thr) | ((uint32_t)(u.y >= thr) << 1) |
                    ((uint32_t)(u.z >= thr) << 2) | ((uint32_t)(u.w >= thr) << 3))
                   << (4 * j);
          }
        } else {
          for (int j = 0; j < ncalls; ++j) {
            Word4 u = philox_q((uint32_t)(8 * w + j), r0_c0, r0_c1, sk1, P.keys);
            rej |= ((uint32_t)(u.x >= thr) | ((uint32_t)(u.y >= thr) << 1) |
                    ((uint32_t)(u.z >= thr) << 2) | ((uint32_t)(u.w >= thr) << 3))
                   << (4 * j);
          }
        }
      } else {
        rej = (mode == MODE_ALL_REJECT) ? 0xffffffffu : 0u;
      }
      const int rem = npos - 32 * w;  // positions 32w+1 .. 32w+32 map to bits 0..31
      if (rem < 32) rej &= (1u << rem) - 1u;
      nz += __popc(rej);
      while (rej) {
        const int z = 32 * w + __ffs(rej);  // position of the next rejection
        rej &= rej - 1u;
        segment<HIST>(z - prev, prev, s, iters, sum_b, sum_s, sh_seg, sh_si);
        prev = z;
      }
    }
    segment<HIST>(N - prev, prev, s, iters, sum_b, sum_s, sh_seg, sh_si);  // final segment ends at N

    const int m = nz + 1;
    const int64_t dsi = (int64_t)m * cfg.t_t + (s.noqueue ? (int64_t)sum_b * cfg.kd : (int64_t)sum_s);
    const int64_t si = (int64_t)iters * cfg.si_cost;
    a_m += (unsigned)m;
    a_i += (unsigned)iters;
    a_i2 += (unsigned long long)iters * (unsigned long long)iters;
    a_dsi += (unsigned long long)dsi;
    a_dsi2 += (unsigned long long)dsi * (unsigned long long)dsi;
    a_gtn += dsi > nonsi;
    a_gts += dsi > si;
    a_trials += 1;
    if (PER_TRIAL) {
      const uint64_t r = cfg.rec_off + t;
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

template <bool A, bool B, bool C>
int launch_variant(const LaunchParams &p, uint64_t n_units, int threads, size_t smem,
                   cudaStream_t st) {
  const uint64_t max_grid = 0x7fffffffull;
  LaunchParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < max_grid ? (n_units - done) : max_grid;
    q.unit_begin = p.unit_begin + done;
    dsi_trial_kernel<A, B, C><<<(unsigned)n, threads, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

}  // namespace

int launch_trial_kernel(const LaunchParams &p, uint64_t n_units, int block_threads, bool per_trial,
                        bool hist, bool pattern, size_t hist_smem, void *stream) {
  if (n_units == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = hist ? hist_smem : 0;
  if (hist && smem > 48 * 1024) {
    // the attribute is per device; setting it before every launch is cheap
    cudaFuncSetAttribute(dsi_trial_kernel<false, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dsi_trial_kernel<true, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dsi_trial_kernel<false, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dsi_trial_kernel<true, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int code = (per_trial ? 4 : 0) | (hist ? 2 : 0) | (pattern ? 1 : 0);
  switch (code) {
    case 0: return launch_variant<false, false, false>(p, n_units, block_threads, smem, st);
    case 1: return launch_variant<false, false, true>(p, n_units, block_threads, smem, st);
    case 2: return launch_variant<false, true, false>(p, n_units, block_threads, smem, st);
    case 3: return launch_variant<false, true, true>(p, n_units, block_threads, smem, st);
    case 4: return launch_variant<true, false, false>(p, n_units, block_threads, smem, st);
    case 5: return launch_variant<true, false, true>(p, n_units, block_threads, smem, st);
    case 6: return launch_variant<true, true, false>(p, n_units, block_threads, smem, st);
    default: return launch_variant<true, true, true>(p, n_units, block_threads, smem, st);
  }
}

}  // namespace dsi
