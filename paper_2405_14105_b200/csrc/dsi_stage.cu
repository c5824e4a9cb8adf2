// dsi_stage.cu -- the device path of dsi_sim_update: the new configurations, copied to the GPU as
// given, are validated and converted to device rows on the GPU (dsi_convert.h: the very functions
// the host path runs), into the spare table; the kernel also reports what decides whether the
// handle's plans survive -- the first failing configuration, the launch limits and whether the
// shared-stream / means-only / heatmap-cell keys changed (compared with the current
// configurations, kept on the device).  The host commits (swaps the tables) only when nothing
// failed and nothing needs a new plan; otherwise it runs the host path, which reproduces every
// error message and re-plans.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_convert.h"
#include "dsi_device.h"

namespace dsi {
namespace {

__device__ __forceinline__ bool ttft_of(const CfgTicks &t) { return t.t_t1 != t.t_t || t.t_d1 != t.t_d; }

__global__ void __launch_bounds__(256) dsi_stage_kernel(const StageParams P) {
  int max_n = 1, max_keff = 1;
  unsigned int flags = 0;  // STAGE_* bits
  double work = 0.0, work_k1 = 0.0;
  const bool fresh_opt = (P.flags & DSI_F_FRESH_VERIFIER) != 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const dsi_config c = P.raw[i];
    CfgTicks t, o;
    const int code = convert_config(P.tick, P.flags, c, t);
    convert_config(P.tick, P.flags, P.prev[i], o);  // (validated when it was committed)
    if (code != 0 || t.trials != o.trials) {  // the host path reports it (n_trials must not change)
      atomicMin(&P.st->first_bad, (unsigned long long)i);
      continue;
    }
    DevCfg d = make_dev_cfg(t, false, fresh_opt);
    P.out[i] = d;
    max_n = max(max_n, t.n);
    max_keff = max(max_keff, min(t.k, t.n));
    if (ttft_of(t)) flags |= STAGE_TTFT;
    if (fresh_opt && t.kd > t.t_t) flags |= STAGE_FRESH;
    const double w = (double)t.trials * (double)t.n;
    work += w;
    if (min(t.k, t.n) == 1 && config_noqueue(t)) work_k1 += w;
    // the keys dsi_sim_update compares on the host path (validate_all's UpdateKeys)
    const bool same_stream = t.stream_id == o.stream_id && t.thr == o.thr && t.n == o.n && t.trials == o.trials;
    if (!(same_stream && t.k == o.k && t.t_t == o.t_t && t.t_d == o.t_d && t.sp == o.sp && ttft_of(t) == ttft_of(o)))
      flags |= STAGE_PLAN_CHANGED;
    if (!(same_stream && ttft_of(t) == ttft_of(o))) flags |= STAGE_GROUPS_CHANGED;
    if (!(t.ut == o.ut && t.ud == o.ud && t.a == o.a && t.sp == o.sp && t.n == o.n)) flags |= STAGE_CELLS_CHANGED;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    max_n = max(max_n, __shfl_xor_sync(0xffffffffu, max_n, off));
    max_keff = max(max_keff, __shfl_xor_sync(0xffffffffu, max_keff, off));
    flags |= __shfl_xor_sync(0xffffffffu, flags, off);
    work += __shfl_xor_sync(0xffffffffu, work, off);
    work_k1 += __shfl_xor_sync(0xffffffffu, work_k1, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&P.st->max_n, max_n);
    atomicMax(&P.st->max_keff, max_keff);
    if (flags) atomicOr(&P.st->flags, flags);
    // (work sums only choose a kernel variant, never a result: their summation order is free)
    atomicAdd(&P.st->work, work);
    atomicAdd(&P.st->work_k1, work_k1);
  }
}

}  // namespace

int launch_stage_kernel(const StageParams &p, void *stream) {
  if (p.n == 0) return 0;
  const unsigned threads = 256;
  const uint64_t want = (p.n + threads - 1) / threads;
  const unsigned blocks = (unsigned)(want < 148ull * 16 ? want : 148ull * 16);
  dsi_stage_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

}  // namespace dsi
