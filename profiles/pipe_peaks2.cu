// pipe_peaks2.cu -- issue rates of the remaining ALU instructions the pack alternatives use
// (LEA.HI, SHF.L.W funnel, ISETP+SEL, PRMT, POPC, FLO), measured like pipe_peaks.cu.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pp2 profiles/pipe_peaks2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int UNROLL = 32;

template <int OP>
__device__ __forceinline__ void step(uint32_t (&r)[CH], uint32_t k) {
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint32_t o = r[(c + 1) % CH];
    if (OP == 0) r[c] = (o >> 1) - r[c];                 // LEA.HI
    else if (OP == 1) r[c] = __funnelshift_l(o, r[c], 1);  // SHF.L.W
    else if (OP == 2) r[c] = __popc(o) + r[c];            // POPC (+ add)
    else if (OP == 3) r[c] = __byte_perm(o, r[c], 0x5410); // PRMT
    else if (OP == 4) r[c] = __clz(o) ^ r[c];             // FLO (+ lop)
    else if (OP == 5) r[c] = (o >= k ? 2u : 1u) + r[c];   // ISETP + SEL (+ add)
    else if (OP == 6) r[c] = r[c] << 1 | o >> 31;         // shift/or (ptxas: SHF or LEA)
    else if (OP == 7) r[c] = r[(c + 1) % CH] + 0x9E3779B9u;  // add immediate (VIADD?)
    else if (OP == 8) r[c] = (r[c] ^ o) + 0x3C6EF372u;       // LOP3 + add immediate
  }
}

template <int OP>
__global__ void __launch_bounds__(128) peak(int iters, uint32_t seed, unsigned long long *sink) {
  uint32_t r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = seed ^ (threadIdx.x * 977u + c * 131u + blockIdx.x);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) step<OP>(r, seed + i);
  }
  uint64_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc += r[c];
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <int OP>
void run(const char *name, int sms, double mhz) {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 16, threads = 128, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    peak<OP><<<blocks, threads>>>(iters, 12345u, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = ms < best ? ms : best;
  }
  const double steps = (double)blocks * threads * iters * UNROLL * CH;  // C-level steps
  const double warp_steps_per_clk_smsp = steps / 32.0 / (4.0 * sms) / (best * 1e-3 * mhz * 1e6);
  printf("{\"op\": \"%s\", \"cycles_per_warp_step\": %.3f, \"ms\": %.3f}\n", name, 1.0 / warp_steps_per_clk_smsp, best);
  cudaFree(d);
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double mhz = khz / 1000.0;
  run<0>("(o >> 1) - r: LEA.HI", sms, mhz);
  run<1>("funnelshift_l: SHF.L.W", sms, mhz);
  run<2>("popc + add", sms, mhz);
  run<3>("byte_perm: PRMT", sms, mhz);
  run<4>("clz ^ r: FLO + LOP3", sms, mhz);
  run<5>("(o >= k ? 2 : 1) + r: ISETP + SEL + add", sms, mhz);
  run<6>("r << 1 | o >> 31", sms, mhz);
  run<7>("o + imm: VIADD?", sms, mhz);
  run<8>("(r ^ o) + imm", sms, mhz);
  return 0;
}
