// dsi_crn.cu -- shared-stream (common random numbers) trial kernel, DSI_F_SHARED_STREAMS.
//
// By the random-number contract, configurations with equal (stream_id, threshold,
// N, n_trials) draw identical indicators for every trial index.  A group of such
// configurations (e.g. the 20 000 (t_d, k) points of one acceptance rate of the
// heatmap) therefore needs ONE Philox pass per trial.  This kernel:
//   block = (group, slice of <= cfg_per_block configs of the group), loops over the
//   group's trials in tiles of blockDim:
//   phase 1 (one trial per thread): Philox + Bernoulli mask exactly as dsi_kernel.cu,
//     then the trial's summary m = #zeros + 1, n2 = #segments with g >= 2 and the list
//     of run lengths L >= 2 of accepted drafts (a segment of length g has L = g - 1),
//     sorted in decreasing order, into shared memory;
//   phase 2 (configs across threads, trials in lockstep): for each config,
//     I = m + sum_{L >= k+1} floor(L/(k+1)),  L_DSI = m t_t + n2 S(1) + sum_{L >= k+1} (S(ceil(L/k)) - S(1))
//     -- the closed form of DESIGN.md section 2 with short segments (2 <= g <= k+1)
//     costing (0, S(1)) -- then the per-config integer moments.
// Per-trial latencies, and so every sum, are bit-identical to the per-config kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

struct CfgLite {  // what phase 2 needs of a config (shared memory)
  int32_t t_t, s1, si_cost, k_eff;
  uint32_t m_si, m_k_lo, m_k_hi, m_sp_lo;
  uint32_t m_sp_hi;
  int32_t kd, sp_eff, pad;
};

__device__ __forceinline__ void insert_desc(uint16_t *runs, int stride, int &nr, int L) {
  // insertion into runs[0..nr) kept in decreasing order (slot-interleaved layout)
  int i = nr++;
  while (i > 0) {
    const int prev = runs[(i - 1) * stride];
    if (prev >= L) break;
    runs[i * stride] = (uint16_t)prev;
    --i;
  }
  runs[i * stride] = (uint16_t)L;
}

__global__ void __launch_bounds__(128) dsi_crn_kernel(const CrnParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const CrnUnit un = P.units[P.unit_begin + blockIdx.x];
  const CrnGroup G = P.groups[un.group];
  const int TT = blockDim.x;  // trials per tile (one per thread in phase 1)
  const int N = G.n_tokens;
  const int npos = N - 1;
  const int nwords = (npos + 31) >> 5;
  const int nq = (npos + 3) >> 2;
  const uint32_t mode = G.mode;
  const uint32_t nthr = 0u - G.thr;

  // shared memory layout
  unsigned char *sp = smem;
  uint4 *U = reinterpret_cast<uint4 *>(sp);
  sp += (size_t)P.max_nq * sizeof(uint4);
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(sp);  // [cfg][NF]
  sp += (size_t)P.cfg_per_block * NF * sizeof(unsigned long long);
  CfgLite *cl = reinterpret_cast<CfgLite *>(sp);
  sp += (size_t)P.cfg_per_block * sizeof(CfgLite);
  uint2 *summ = reinterpret_cast<uint2 *>(sp);  // per trial slot: (m | n2 << 16, nruns)
  sp += (size_t)TT * sizeof(uint2);
  uint16_t *runs = reinterpret_cast<uint16_t *>(sp);  // runs[i * TT + slot]

  if (mode == MODE_STREAM)
    for (int q = threadIdx.x; q < nq; q += TT) U[q] = philox_q_half((uint32_t)q, G.stream_id, P.keys);
  for (int j = threadIdx.x; j < (int)un.count; j += TT) {
    const DevCfg c = P.cfg[P.perm[un.begin + j]];
    CfgLite l;
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
    l.sp_eff = c.sp_eff;
    l.pad = 0;
    cl[j] = l;
    for (int f = 0; f < NF; ++f) acc[j * NF + f] = 0ull;
  }
  __syncthreads();

  const uint64_t T = G.n_trials;
  for (uint64_t tile0 = 0; tile0 < T; tile0 += TT) {
    // ---------------- phase 1: one trial per thread -> summary + sorted long-run list
    const uint64_t t = tile0 + threadIdx.x;
    if (t < T) {
      const uint32_t trial = (uint32_t)t;
      const TrialHalf th = philox_trial_half(trial, P.keys);
      uint16_t *myruns = runs + threadIdx.x;
      int nz = 0, n2 = 0, run = 0, lastz = 0, nr = 0;
      for (int w = 0; w < nwords; ++w) {
        uint32_t Rw;
        if (mode == MODE_STREAM) {
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
          if (L >= 2) insert_desc(myruns, TT, nr, L);
        }
        lastz = base + 31 - __clz(Rw);
        run = nv - 1 - (31 - __clz(Rw));
      }
      n2 += run >= 1;  // the final segment (the trailing run, then position N)
      if (run >= 2) insert_desc(myruns, TT, nr, run);
      summ[threadIdx.x] = make_uint2((uint32_t)(nz + 1) | ((uint32_t)n2 << 16), (uint32_t)nr);
    }
    __syncthreads();
    // ---------------- phase 2: configs across threads, this tile's trials in lockstep
    const int ntr = (int)min((uint64_t)TT, T - tile0);
    for (int j = threadIdx.x; j < (int)un.count; j += TT) {
      const CfgLite l = cl[j];
      const int Lk = l.k_eff + 1;
      const int64_t nonsi = (int64_t)N * l.t_t;
      unsigned long long a_i = 0, a_i2 = 0, a_dsi = 0, a_dsi2 = 0, a_gtn = 0, a_gts = 0, a_m = 0;
      for (int s = 0; s < ntr; ++s) {
        const uint2 sm = summ[s];
        const int m = (int)(sm.x & 0xffffu), n2 = (int)(sm.x >> 16), nr = (int)sm.y;
        int ai = 0, ay = 0;
        for (int r = 0; r < nr; ++r) {
          const int L = runs[r * TT + s];
          if (L < Lk) break;
          // a segment of g = L + 1: ceil(g/(k+1)) - 1 = floor(L/(k+1)) extra SI iterations,
          // thread b = ceil((g-1)/k) = ceil(L/k) settles its last position
          const uint32_t x = magic_div((uint32_t)L, l.m_si, 0u);
          const uint32_t b = magic_div((uint32_t)L + (uint32_t)l.k_eff - 1u, l.m_k_lo, l.m_k_hi);
          const uint32_t qq = magic_div(b, l.m_sp_lo, l.m_sp_hi);
          const int rr = (int)b - (int)qq * l.sp_eff;
          const int S = max((int)b * l.kd, rr * l.kd + (int)qq * l.t_t);
          ai += (int)x;
          ay += S - l.s1;
        }
        const int iters = m + ai;
        const int64_t dsi = (int64_t)m * l.t_t + (int64_t)n2 * l.s1 + ay;
        const int64_t si = (int64_t)iters * l.si_cost;
        a_m += (unsigned)m;
        a_i += (unsigned)iters;
        a_i2 += (unsigned long long)iters * (unsigned long long)iters;
        a_dsi += (unsigned long long)dsi;
        a_dsi2 += (unsigned long long)dsi * (unsigned long long)dsi;
        a_gtn += dsi > nonsi;
        a_gts += dsi > si;
      }
      unsigned long long *a = acc + (size_t)j * NF;
      a[F_M] += a_m;
      a[F_I] += a_i;
      a[F_I2] += a_i2;
      a[F_DSI] += a_dsi;
      a[F_DSI2] += a_dsi2;
      a[F_GT_NONSI] += a_gtn;
      a[F_GT_SI] += a_gts;
      a[F_TRIALS] += (unsigned long long)ntr;
    }
    __syncthreads();
  }
  // every config of the slice is owned by this block: plain stores of its moments
  for (int j = threadIdx.x; j < (int)un.count; j += TT) {
    unsigned long long *dst = P.acc + (size_t)P.perm[un.begin + j] * NF;
    for (int f = 0; f < NF; ++f) dst[f] = acc[j * NF + f];
  }
}

}  // namespace

size_t crn_kernel_smem(int max_n, int block_threads, int cfg_per_block, int max_runs) {
  const int max_nq = (max_n - 1 + 3) / 4 + 1;
  return (size_t)max_nq * sizeof(uint4) + (size_t)cfg_per_block * NF * sizeof(unsigned long long) +
         (size_t)cfg_per_block * sizeof(CfgLite) + (size_t)block_threads * sizeof(uint2) +
         (size_t)block_threads * max_runs * sizeof(uint16_t);
}

int launch_crn_kernel(const CrnParams &p, uint64_t n_units, int block_threads, void *stream) {
  if (n_units == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = crn_kernel_smem(p.max_n, block_threads, p.cfg_per_block, p.max_runs);
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(dsi_crn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const uint64_t max_grid = 0x7fffffffull;
  CrnParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < max_grid ? (n_units - done) : max_grid;
    q.unit_begin = p.unit_begin + done;
    dsi_crn_kernel<<<(unsigned)n, block_threads, smem, st>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

}  // namespace dsi
