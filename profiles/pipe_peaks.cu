// pipe_peaks.cu -- measured issue rates of the integer instructions the trial kernel is made of
// ("commit an IMAD.WIDE-only microbenchmark that measures the fmaheavy peak
// directly").  Measurement tool, not product code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_peaks profiles/pipe_peaks.cu
//   /tmp/pipe_peaks            (prints one JSON line per instruction mix)
// Each thread runs CH independent dependency chains (ILP) of one PTX instruction, unrolled, so
// the SASS of the loop body is that instruction only (checked with cuobjdump -sass: see
// profiles/r02_pipe_peaks_sass.txt).  Rates are reported per SMSP per SM clock: warp-instr /
// clk / SMSP = thread-ops / (32 x 4 x 148 x cycles), with the SM cycles and the wall time taken
// inside the kernel (clock64 and %globaltimer of each block), so the clock is measured, not assumed.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent chains per thread
constexpr int UNROLL = 32;  // chain steps per loop iteration
constexpr uint32_t M0 = 0xD2511F53u;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int OP>
__device__ __forceinline__ void step(uint32_t (&r)[CH], uint64_t (&w)[CH], uint32_t k) {
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (OP == 0) {  // mad.wide with a 64-bit addend: ptxas emits IMAD.WIDE (RZ) + a 64-bit IADD3 pair
      asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w[c]) : "r"((uint32_t)(w[c] >> 32)), "n"(M0), "l"(w[(c + 1) % CH]));
    } else if (OP == 1) {  // IMAD.HI.U32
      asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(r[c]) : "n"(M0));
    } else if (OP == 2) {  // IMAD (low word); the addend from the next chain stops ptxas folding steps
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[c]) : "n"(M0), "r"(r[(c + 1) % CH]));
    } else if (OP == 3) {  // LOP3 (three-input xor, the Philox key mix)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[c]) : "r"(r[(c + 1) % CH]), "r"(k));
    } else if (OP == 4) {  // add.u32 (ptxas spreads these over IADD3 and IMAD.IADD)
      asm volatile("add.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(r[(c + 1) % CH]));
    } else if (OP == 5) {  // IMAD.X (addc with the carry of an add.cc: the pack's two instructions)
      asm volatile("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
                   : "+r"(r[c]) : "r"(r[(c + 1) % CH]), "r"(k));
    } else if (OP == 6) {  // one Philox-like half round: IMAD.WIDE + LOP3 (hi ^ lo ^ k keeps both
                           // halves live, so this is the only way to get IMAD.WIDE.U32 alone on
                           // the fma pipe; the LOP3 goes to the ALU pipe)
      asm volatile("mad.wide.u32 %0, %1, %2, 0;" : "=l"(w[c]) : "r"(r[c]), "n"(M0));
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r[c]) : "r"((uint32_t)(w[c] >> 32)), "r"((uint32_t)w[c]), "r"(k));
    }
  }
}

template <int OP>
__global__ void __launch_bounds__(128) peak(int iters, uint32_t seed, unsigned long long *sink,
                                            unsigned long long *cyc, unsigned long long *ns) {
  uint32_t r[CH];
  uint64_t w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    r[c] = seed ^ (threadIdx.x * 977u + c * 131u + blockIdx.x);
    w[c] = r[c];
  }
  __syncthreads();
  const uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) step<OP>(r, w, seed + i);
  }
  __syncthreads();
  const uint64_t c1 = clock64(), t1 = gtimer();
  uint64_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc += r[c] + w[c];
  if (acc == 0x123456789ull) sink[0] = acc;  // keeps the chains live
  if (threadIdx.x == 0) {
    atomicAdd(cyc, c1 - c0);
    atomicAdd(ns, t1 - t0);
  }
}

template <int OP>
void run(const char *name, int ops_per_step, int sms) {
  unsigned long long *d;
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  const int blocks = sms * 16, threads = 128;  // 16 x 4 warps per SM: 16 warps per SMSP
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 3 * sizeof(unsigned long long));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    peak<OP><<<blocks, threads>>>(iters, 12345u, d, d + 1, d + 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[3];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    if (rep == 1) {
      const double ops = (double)blocks * threads * iters * UNROLL * CH * ops_per_step;
      const double cyc_per_block = (double)h[1] / blocks, ns_per_block = (double)h[2] / blocks;
      const double mhz = cyc_per_block / ns_per_block * 1e3;
      // blocks run in waves; per SM the measured cycles of all its blocks add up when they run
      // one after another, so use the grid's wall time x the measured clock
      const double cycles = ms * 1e-3 * mhz * 1e6;
      const double per_smsp_clk = ops / 32.0 / (4.0 * sms) / cycles;  // warp-instr / clk / SMSP
      printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_smsp\": %.4f, \"cycles_per_warp_instr\": %.3f, "
             "\"thread_ops_per_s\": %.4e, \"sm_mhz_measured\": %.0f, \"ms\": %.3f}\n",
             name, per_smsp_clk, 1.0 / per_smsp_clk, ops / (ms * 1e-3), mhz, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<6>("IMAD.WIDE + LOP3 (Philox half round)", 2, sms);
  run<0>("mad.wide.u32 + 64-bit addend (IMAD.WIDE + IADD3 + IADD3.X/IMAD.X)", 1, sms);
  run<1>("IMAD.HI.U32 (imm)", 1, sms);
  run<2>("IMAD (imm, low word)", 1, sms);
  run<3>("LOP3", 1, sms);
  run<4>("IADD3", 1, sms);
  run<5>("IADD3.CC + IMAD.X/IADD3.X (add.cc + addc pair)", 2, sms);
  printf("{\"sms\": %d}\n", sms);
  return 0;
}
