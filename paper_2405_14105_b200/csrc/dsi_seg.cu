// dsi_seg.cu -- means-only mode (DSI_F_MEANS_ONLY, SURVEY 8(f) N3's "aggregate H[g]"):
// per group of configs drawing identical indicators (equal stream_id, floor(a 2^32), N, T),
// one pass over the group's trials builds the histogram H[g] of segment lengths g = 1..N
// (H[0] counts the trials); then every config's sums follow by linearity over segments,
//   sum_trials L_DSI = sum_g H[g] C(g),  sum_trials I = sum_g H[g] ceil(g/(k+1)),
//   sum_trials m = sum_g H[g],
// the same integers the per-trial kernels add up (L_DSI and I are sums over segments,
// DESIGN.md section 2), so means are bit-identical to the default mode.  Second moments and
// the per-trial counters need per-trial values and are not produced.
//
// Pass 1 (dsi_seg_hist_kernel): one block per unit (group, tile of trials); per trial the
// Philox stream and rejection mask exactly as dsi_kernel.cu, then its segments: g = 1
// segments (a zero preceded by a zero, or position 1) are counted with bit operations in a
// register, longer ones with shared-memory atomics into the block's H, flushed to the
// group's H with 64-bit atomics.  Pass 2 (dsi_seg_eval_kernel): one thread per config,
// an O(N) dot product of H with the config's segment costs (H read by every lane of a
// warp at once: a broadcast).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsi_common.cuh"
#include "dsi_device.h"

namespace dsi {
namespace {

constexpr int SEG_SMEM_MAX_N = 8192;  // 8(N+1) + 16 N/4 bytes = 96 KB of shared memory

// SMEM: the block's histogram and q halves in shared memory (N <= 8192); else segments go to
// the group's histogram in global memory with 64-bit atomics and the q halves are per call.
template <bool SMEM>
__global__ void __launch_bounds__(128) dsi_seg_hist_kernel(const SegParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_grp;
  const uint64_t unit = P.unit_begin + blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = P.n_groups;  // prefix[lo] <= unit < prefix[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&P.unit_prefix[mid]) <= unit) lo = mid; else hi = mid;
    }
    s_grp = lo;
  }
  __syncthreads();
  const uint32_t gi = s_grp;
  const SegGroup G = P.groups[gi];
  const uint64_t t0 = (unit - __ldg(&P.unit_prefix[gi])) * P.tile_trials;
  const uint64_t t1 = min(t0 + P.tile_trials, G.n_trials);
  const int N = G.n_tokens;
  const int npos = N - 1;
  const int nwords = (npos + 31) >> 5;
  const bool halves = P.halves != 0;
  const int nq = halves ? (npos + 7) >> 3 : (npos + 3) >> 2;
  const uint32_t nthr = 0u - G.thr;
  const HalvesCtx hc = make_halves(G.thr, G.stream_id);

  uint32_t *H = reinterpret_cast<uint32_t *>(smem);           // N + 1 bins
  uint4 *U = reinterpret_cast<uint4 *>(smem + (((size_t)(N + 1) * 4 + 15) & ~(size_t)15));
  uint32_t *H1 = reinterpret_cast<uint32_t *>(U + nq + 1);     // TTFT: first-segment lengths
  unsigned long long *out = P.hist + G.hist_off;
  unsigned long long *out1 = P.hist1 ? P.hist1 + G.hist_off : nullptr;
  auto add1 = [&](int g) {  // the trial's first segment has length g
    if (!out1) return;
    DSI_CHECK(g >= 1 && g <= N);
    if (SMEM) atomicAdd(&H1[g], 1u);
    else atomicAdd(out1 + g, 1ull);
  };
  auto add = [&](int g) {
    DSI_CHECK(g >= 1 && g <= N);
    if (SMEM) atomicAdd(&H[g], 1u);
    else atomicAdd(out + g, 1ull);
  };
  if (SMEM) {
    for (int g = threadIdx.x; g <= N; g += blockDim.x) H[g] = 0u;
    if (out1)
      for (int g = threadIdx.x; g <= N; g += blockDim.x) H1[g] = 0u;
    if (G.mode == MODE_STREAM)
      for (int q = threadIdx.x; q < nq; q += blockDim.x) U[q] = philox_q_half((uint32_t)q, G.stream_id, P.keys);
    __syncthreads();
  }

  uint32_t ones = 0;  // segments of length 1 counted by this thread
  for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    if (G.mode != MODE_STREAM) {  // a = 0: N segments of 1; a = 1: one segment of N
      if (G.mode == MODE_ALL_REJECT) ones += (uint32_t)N;
      else if (N == 1) ones += 1u;
      else add(N);
      add1(G.mode == MODE_ALL_REJECT ? 1 : N);
      continue;
    }
    const TrialHalf th = philox_trial_half((uint32_t)t, P.keys);
    int lastz = 0;     // position of the last zero (0: the sentinel before position 1)
    int g1 = 0;        // TTFT: the first zero's position = the first segment's length
    uint32_t cin = 1;  // position 32w is a zero (the sentinel for w = 0)
    for (int w = 0; w < nwords; ++w) {
      uint32_t R = 0u;
      const int ncalls = halves ? 0 : min(8, nq - 8 * w);
      if (halves) {
        R = gen_word_halves<SMEM>(w, nq, U, th, (uint32_t)t, hc, P.keys);
      } else if (ncalls == 8) {
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          const uint4 u = SMEM ? U[8 * w + j] : philox_q_half((uint32_t)(8 * w + j), G.stream_id, P.keys);
          R = pack4(R, philox_call(u, th, P.keys), nthr);
        }
      } else {
        for (int j = ncalls - 1; j >= 0; --j) {
          const uint4 u = SMEM ? U[8 * w + j] : philox_q_half((uint32_t)(8 * w + j), G.stream_id, P.keys);
          R = pack4(R, philox_call(u, th, P.keys), nthr);
        }
      }
      const int rem = npos - 32 * w;
      if (rem < 32) R &= (1u << rem) - 1u;
      // a zero whose predecessor is a zero ends a segment of length 1
      const uint32_t single = R & ((R << 1) | cin);
      ones += __popc(single);
      uint32_t Z = R & ~single;  // zeros ending a segment of length >= 2
      while (Z) {
        const int b = __ffs(Z) - 1;  // bit b is position 32w + b + 1
        Z &= Z - 1u;
        const uint32_t below = R & ((1u << b) - 1u);
        const int prev = below ? 32 * w + 32 - __clz(below) : lastz;  // the previous zero
        add(32 * w + b + 1 - prev);
      }
      if (g1 == 0 && R) g1 = 32 * w + __ffs(R);
      if (R) lastz = 32 * w + 32 - __clz(R);
      cin = R >> 31;
    }
    add1(g1 ? g1 : N);
    const int gl = N - lastz;  // the final segment ends at N
    if (gl == 1) ones += 1u;
    else add(gl);
  }
  // the g = 1 count: warp sums, one shared atomic per warp
  unsigned long long o = warp_sum((unsigned long long)ones);
  if (!SMEM) {
    if ((threadIdx.x & 31) == 0 && o) atomicAdd(out + 1, o);
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    return;
  }
  if ((threadIdx.x & 31) == 0 && o) atomicAdd(&H[1], (uint32_t)o);
  __syncthreads();
  for (int g = threadIdx.x; g <= N; g += blockDim.x) {
    const uint32_t v = g == 0 ? (uint32_t)(t1 - t0) : H[g];
    if (v) atomicAdd(out + g, (unsigned long long)v);
    if (out1 && g > 0 && H1[g]) atomicAdd(out1 + g, (unsigned long long)H1[g]);
  }
}

// TTFT variant (R23, 6.4): L_DSI gains D1(g1) = C1(g1) - C(g1) where g1 is the trial's
// first segment, so a config's sum gains sum_g H1[g] D1(g).  One block per TTFT config: thread 0
// runs the first segment's FIFO schedule exactly as dsi_kernel.cu (F[b]: completion of thread b
// with the target's first forward t_t1 and drafts late by t_d1 - t_d), then the block sums.
__global__ void __launch_bounds__(128) dsi_seg_ttft_kernel(const SegParams P, uint64_t begin) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t c = P.ttft_cfgs[begin + blockIdx.x];
  const DevCfg cfg = P.cfg[c];
  const SegGroup G = P.groups[P.cfg_group[c]];
  const unsigned long long *H1 = P.hist1 + G.hist_off;
  const SegCtx s = make_segctx(cfg);
  const int N = cfg.n_tokens;
  int *F = reinterpret_cast<int *>(smem);
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
  long long part = 0;
  for (int g = 1 + threadIdx.x; g <= N; g += blockDim.x) {
    const unsigned long long h1 = H1[g];
    if (!h1) continue;
    const uint32_t b = magic_div((uint32_t)g + s.k_eff - 2u, s.m_k_lo, s.m_k_hi);  // ceil((g-1)/k)
    const int S = g >= 2 ? (int)seg_extra(g, s).y : 0;
    part += (long long)h1 * (long long)(F[b] - (cfg.t_t + S));
  }
  __shared__ long long red[4];
  part = (long long)warp_sum((unsigned long long)part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    P.acc[(size_t)c * NF + F_DSI] += (unsigned long long)t;  // one block per config: no race
  }
}

// P[g] = H[1] + ... + H[g] (P[0] = 0) per group, for the bucketed evaluation below: one block
// per group, each thread scans a contiguous chunk, chunk totals scanned across the block.
__global__ void __launch_bounds__(128) dsi_seg_prefix_kernel(const SegParams P) {
  __shared__ unsigned long long warp_tot[4];
  const SegGroup G = P.groups[blockIdx.x];
  const unsigned long long *H = P.hist + G.hist_off;
  unsigned long long *pre = P.pre + G.hist_off;
  const int N = G.n_tokens;
  const int per = (N + blockDim.x - 1) / blockDim.x;  // bins 1..N in chunks
  const int lo = 1 + (int)threadIdx.x * per, hi = min(lo + per - 1, N);
  unsigned long long sum = 0;
  for (int g = lo; g <= hi; ++g) sum += H[g];
  // inclusive scan of the chunk sums: within the warp, then across the four warps
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned long long inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (unsigned)o) inc += v;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  unsigned long long base = 0;
  for (unsigned w = 0; w < warp; ++w) base += warp_tot[w];
  unsigned long long run = base + inc - sum;  // exclusive prefix of this chunk
  if (threadIdx.x == 0) pre[0] = 0;
  for (int g = lo; g <= hi; ++g) {
    run += H[g];
    pre[g] = run;
  }
}

// S(b) of the closed form (FIFO start of thread b), as seg_extra computes it.
__device__ __forceinline__ uint32_t seg_S(uint32_t b, const SegCtx &s) {
  const uint32_t qq = magic_div(b, s.m_sp_lo, s.m_sp_hi);
  const int rr = (int)b - (int)qq * s.sp_eff;
  return (uint32_t)max((int)b * s.kd, rr * s.kd + (int)qq * s.t_t);
}

__global__ void __launch_bounds__(128) dsi_seg_eval_kernel(const SegParams P) {
  const uint64_t c = P.cfg_begin + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P.cfg_end) return;
  const DevCfg cfg = P.cfg[c];
  const SegGroup G = P.groups[P.cfg_group[c]];
  const unsigned long long *H = P.hist + G.hist_off;
  const SegCtx s = make_segctx(cfg);
  const bool fresh = (cfg.flags & CFG_FRESH) != 0;
  const int N = cfg.n_tokens;
  unsigned long long sm = 0, si = 0, sd = 0;
  const int k = cfg.k_eff;
  if (k >= 2 && !fresh) {
    // bucketed: ceil(g/(k+1)) and ceil((g-1)/k) are constant on runs of g, so each run costs one
    // difference of the prefix sums P (O(N/k) per config instead of O(N))
    const unsigned long long *pre = P.pre + G.hist_off;
    sm = pre[N];
    for (int lo = 0, M = 1; lo < N; lo += k + 1, ++M) {  // g in (lo, lo + k + 1]: M iterations
      const int hi = min(lo + k + 1, N);
      si += (unsigned long long)M * (pre[hi] - pre[lo]);
    }
    sd = (unsigned long long)(uint32_t)cfg.t_t * sm;  // every segment pays t_t; g >= 2 adds S(b)
    for (int b = 1, lo = 2; lo <= N; ++b, lo += k) {     // g in [(b-1)k + 2, bk + 1]: thread b
      const int hi = min(lo + k - 1, N);
      sd += (unsigned long long)seg_S((uint32_t)b, s) * (pre[hi] - pre[lo - 1]);
    }
  } else
  for (int g = 1; g <= N; ++g) {
    const unsigned long long h = __ldg(H + g);
    if (!h) continue;
    uint32_t M = 1u, S = 0u;  // SI iterations ceil(g/(k+1)) and S(ceil((g-1)/k)) of C(g)
    if (g >= 2) {
      const uint2 e = seg_extra(g, s);
      M = e.x + 1u;
      S = e.y;
      if (fresh) S -= fresh_saving(g, s, cfg.t_d);
    }
    sm += h;
    si += h * M;
    sd += h * (unsigned long long)((uint32_t)cfg.t_t + S);
  }
  unsigned long long *acc = P.acc + c * NF;
  acc[F_M] = sm;
  acc[F_I] = si;
  acc[F_DSI] = sd;
  acc[F_TRIALS] = __ldg(H);
}

}  // namespace

size_t seg_hist_smem(int max_n) {  // H, U and (TTFT) H1
  return (((size_t)(max_n + 1) * 4 + 15) & ~(size_t)15) + (size_t)((max_n - 1 + 3) / 4 + 1) * sizeof(uint4) +
         (size_t)(max_n + 1) * 4;
}

int launch_seg_ttft(const SegParams &p, uint64_t begin, uint64_t end, void *stream) {
  if (end <= begin) return 0;
  const size_t smem = (size_t)(p.max_n + 2) * sizeof(int);
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(dsi_seg_ttft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  dsi_seg_ttft_kernel<<<(unsigned)(end - begin), 128, smem, (cudaStream_t)stream>>>(p, begin);
  return (int)cudaGetLastError();
}

int launch_seg_hist(const SegParams &p, uint64_t n_units, void *stream) {
  if (n_units == 0) return 0;
  const bool use_smem = p.max_n <= SEG_SMEM_MAX_N;
  const size_t smem = use_smem ? seg_hist_smem(p.max_n) : 0;
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(dsi_seg_hist_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  SegParams q = p;
  for (uint64_t done = 0; done < n_units;) {
    const uint64_t n = (n_units - done) < 0x7fffffffull ? (n_units - done) : 0x7fffffffull;
    q.unit_begin = p.unit_begin + done;
    if (use_smem)
      dsi_seg_hist_kernel<true><<<(unsigned)n, 128, smem, (cudaStream_t)stream>>>(q);
    else
      dsi_seg_hist_kernel<false><<<(unsigned)n, 128, 0, (cudaStream_t)stream>>>(q);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    done += n;
  }
  return 0;
}

int launch_seg_prefix(const SegParams &p, void *stream) {
  if (p.n_groups == 0) return 0;
  dsi_seg_prefix_kernel<<<p.n_groups, 128, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

int launch_seg_eval(const SegParams &p, void *stream) {
  if (p.cfg_end <= p.cfg_begin) return 0;
  const uint64_t blocks = (p.cfg_end - p.cfg_begin + 127) / 128;
  dsi_seg_eval_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

}  // namespace dsi
