// dsi_reduce_dev.cu -- device side of dsi_sim_reduce (the partition check) and the
// on-device heatmap product (Fig. 3 / Fig. 5 of the
// paper): per (drafter latency, acceptance) cell, the argmin over
// the lookaheads of the mean SI latency, and over the Eq.-1-feasible lookaheads of the
// mean DSI latency (ties to the smallest k), plus the four ratio panels.
//
// One warp per cell; lanes stride over the cell's configs and reduce (value, k)
// lexicographically with shuffles.  It reads 3 of the 8 accumulator words of each
// config and writes 64 B per cell, so only the cells cross PCIe instead of every
// config's moments.  The arithmetic is the host finalize's, operation for operation
// (integer sums, then ((double)sum / (double)T) * tick), so the cells are bit-identical
// to dsi_heatmap over dsi_sim_reduce's results.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "dsi_device.h"

namespace dsi {
namespace {

__device__ __forceinline__ bool better(double v, int k, double bv, int bk) {
  return v < bv || (v == bv && k < bk);
}

__global__ void __launch_bounds__(256) dsi_heatmap_kernel(const HeatParams P) {
  const uint32_t slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= P.n_cells) return;  // warp-uniform
  const uint32_t cell = P.idx ? P.idx[slot] : slot;  // (cell-local heatmap: this rank's cells)
  const HeatCell c = P.cells[cell];
  double si_v = INFINITY, dsi_v = INFINITY;
  int si_k = 0x7fffffff, dsi_k = 0x7fffffff;
  bool bad = false;
  for (uint64_t i = c.first + lane; i < c.first + c.count; i += 32) {
    const DevCfg &g = P.cfg[i];
    const unsigned long long *a = P.acc + i * NF;
    const uint64_t T = g.n_trials;
    bad |= a[F_TRIALS] != T;
    // L_SI = I (k t_d + t_t) + e per trial (e: TTFT surcharge); sums < 2^63 (create's bound)
    const int64_t sum_si = (int64_t)g.si_cost * (int64_t)a[F_I] + (int64_t)T * (int64_t)g.e_si;
    const double Td = (double)T;
    const double si = ((double)sum_si / Td) * P.tick;
    const double dsi = ((double)(int64_t)a[F_DSI] / Td) * P.tick;
    if (better(si, g.k, si_v, si_k)) {
      si_v = si;
      si_k = g.k;
    }
    if ((g.flags & CFG_EQ1) && better(dsi, g.k, dsi_v, dsi_k)) {
      dsi_v = dsi;
      dsi_k = g.k;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double sv = __shfl_xor_sync(0xffffffffu, si_v, o);
    const int sk = __shfl_xor_sync(0xffffffffu, si_k, o);
    const double dv = __shfl_xor_sync(0xffffffffu, dsi_v, o);
    const int dk = __shfl_xor_sync(0xffffffffu, dsi_k, o);
    if (better(sv, sk, si_v, si_k)) {
      si_v = sv;
      si_k = sk;
    }
    if (better(dv, dk, dsi_v, dsi_k)) {
      dsi_v = dv;
      dsi_k = dk;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(P.bad, 1u);
  if (lane != 0) return;
  HeatOut o;
  o.nonsi = (double)P.cfg[c.first].nonsi * P.tick;
  o.si = si_v;
  o.si_k = si_k;
  if (dsi_k == 0x7fffffff) {
    o.dsi = NAN;
    o.dsi_k = -1;
  } else {
    o.dsi = dsi_v;
    o.dsi_k = dsi_k;
  }
  // "X/Y plots the ratio between the run time of algorithm X and the run time of Y"
  o.r_nonsi_si = o.nonsi / o.si;
  o.r_si_dsi = o.si / o.dsi;
  o.r_nonsi_dsi = o.nonsi / o.dsi;
  o.r_min_dsi = fmin(o.si, o.nonsi) / o.dsi;
  P.out[cell] = o;
}

// dsi_sim_reduce's partition check: every config's trial counter equals n_trials (each
// trial simulated exactly once), read on the device so the host never scans the sums.
__global__ void __launch_bounds__(256) dsi_check_trials_kernel(const DevCfg *cfg,
                                                               const unsigned long long *acc, uint64_t n,
                                                               unsigned int *bad) {
  bool b = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b |= acc[i * NF + F_TRIALS] != cfg[i].n_trials;
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

}  // namespace

int launch_check_trials(const DevCfg *cfg, const unsigned long long *acc, uint64_t n, unsigned int *bad,
                        void *stream) {
  if (n == 0) return 0;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 8);
  dsi_check_trials_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(cfg, acc, n, bad);
  return (int)cudaGetLastError();
}

int launch_heatmap_kernel(const HeatParams &p, void *stream) {
  if (p.n_cells == 0) return 0;
  const unsigned threads = 256;
  const unsigned blocks = (unsigned)(((uint64_t)p.n_cells * 32 + threads - 1) / threads);
  dsi_heatmap_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

}  // namespace dsi
