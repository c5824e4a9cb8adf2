// philox_ceiling.cu -- practical ceiling of the Philox4x32-10 + Bernoulli part of the
// trial kernel on this GPU (measurement tool, not product code).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o philox_ceiling profiles/philox_ceiling.cu
//   ./philox_ceiling
// Variant 0: mul-wide (IMAD.WIDE.U32) rounds; variant 1: mulhi + mullo (IMAD.HI + IMAD).
// Each thread runs `trials` trials of N = 100 positions (25 calls), packs the rejection
// bits and accumulates their popcount (so nothing is dead code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ void round_(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3,
                                       uint32_t k0, uint32_t k1) {
  uint32_t hi0, lo0, hi1, lo1;
  if (V == 0) {
    uint64_t a = (uint64_t)0xD2511F53u * c0, b = (uint64_t)0xCD9E8D57u * c2;
    hi0 = a >> 32; lo0 = (uint32_t)a; hi1 = b >> 32; lo1 = (uint32_t)b;
  } else {
    hi0 = __umulhi(0xD2511F53u, c0); lo0 = 0xD2511F53u * c0;
    hi1 = __umulhi(0xCD9E8D57u, c2); lo1 = 0xCD9E8D57u * c2;
  }
  uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

template <int V>
__global__ void __launch_bounds__(128) ceiling(uint32_t seed, int trials, uint32_t thr,
                                               unsigned long long *out) {
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const uint32_t trial = tid * trials + t;
    for (int w = 0; w < 4; ++w) {
      uint32_t rej = 0;
      const int nc = w < 3 ? 8 : 1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nc) {
          uint32_t c0 = 8 * w + j, c1 = 0, c2 = trial, c3 = 7;
          uint32_t k0 = seed, k1 = seed ^ 0x1234;
#pragma unroll
          for (int r = 0; r < 10; ++r) {
            round_<V>(c0, c1, c2, c3, k0, k1);
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
          }
          rej |= ((uint32_t)(c0 >= thr) | ((uint32_t)(c1 >= thr) << 1) | ((uint32_t)(c2 >= thr) << 2) |
                  ((uint32_t)(c3 >= thr) << 3)) << (4 * j);
        }
      }
      acc += __popc(rej);
    }
  }
  atomicAdd(out, (unsigned long long)acc);
}

int main() {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int trials = 64;
  for (int v = 0; v < 2; ++v) {
    for (int bps : {4, 8, 16}) {
      const int blocks = sms * bps * 8;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(d, 0, 8);
        cudaEventRecord(a);
        if (v == 0) ceiling<0><<<blocks, 128>>>(2405141050u, trials, 0x80000000u, d);
        else ceiling<1><<<blocks, 128>>>(2405141050u, trials, 0x80000000u, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double tt = (double)blocks * 128 * trials * 100;  // N = 100 trial-tokens
        if (rep == 2)
          printf("variant %d (%s) blocks %d: %.3f ms, %.3e trial-tokens/s (%.3e Philox calls/s)\n", v,
                 v == 0 ? "IMAD.WIDE" : "IMAD.HI+IMAD", blocks, ms, tt / (ms * 1e-3),
                 (double)blocks * 128 * trials * 25 / (ms * 1e-3));
      }
    }
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d kHz\n", sms, clk);
  return 0;
}
