// philox_variants.cu -- A/B of the Philox rounds 2-9 + Bernoulli pack of the trial kernel
// (measurement tool, not product code).  Same structure as dsi_trial_kernel: rounds 0-1
// split into a per-trial half (registers) and a per-counter half (shared-memory table), N = 100
// (25 calls per trial), the rejection mask packed 32 positions per word, popcount accumulated.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pv profiles/philox_variants.cu
// Variants of the 32x32->64 multiplies of rounds 2-9:
//   W: IMAD.WIDE.U32 (4 cycles of the fmaheavy pipe per warp, profiles/r02_pipe_peaks.jsonl)
//   D: low word by IMAD (2 cycles) and the high word from one exact DFMA on the FP64 pipe:
//      with x_d = 2^52 + x and l_d = 2^52 + lo (bit patterns 0x43300000:x, 0x43300000:lo),
//      fma((2^32 + M), x_d, -l_d) = 2^84 + (M-1) 2^52 + 2^32 (x + hi) exactly (a multiple of
//      2^32 in [2^84, 2^85) for M <= 0xFFFFE000), whose low word is x + hi + ((M-1) << 20).
// Pack variants: C = add.cc/addc carry chain (current), S = compare + shift/or.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
constexpr uint32_t THR = 0xCCCCCCCCu;  // even (a = 0.8): every pack variant is exact

struct Keys {
  uint32_t k0[10], k1[10];
};

template <bool D>
__device__ __forceinline__ void mul(uint32_t M, uint32_t x, uint32_t &hi, uint32_t &lo) {
  if (!D) {
    const uint64_t p = (uint64_t)M * x;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
  } else {
    lo = M * x;
    const double xd = __hiloint2double(0x43300000, (int)x);
    const double ld = __hiloint2double(0x43300000, (int)lo);
    const double r = __fma_rn((double)(0x100000000ull + M), xd, -ld);
    hi = (uint32_t)__double2loint(r) - x - ((M - 1u) << 20);
  }
}

// DA: the variant of the M0 multiply, DB: of the M1 multiply
template <bool DA, bool DB>
__device__ __forceinline__ uint4 rounds_2_9(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const Keys &K) {
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    uint32_t ha, la, hb, lb;
    mul<DA>(M0, c0, ha, la);
    mul<DB>(M1, c2, hb, lb);
    const uint32_t n0 = hb ^ c1 ^ K.k0[r];
    const uint32_t n2 = ha ^ c3 ^ K.k1[r];
    c1 = lb;
    c3 = la;
    c0 = n0;
    c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

template <int P>
__device__ __forceinline__ uint32_t pack4(uint32_t rej, const uint4 &u, uint32_t nthr, uint32_t thr) {
  if (P == 0) {
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %1, %5;\n\taddc.u32 %0, %0, %0;\n\t"
        "add.cc.u32 t, %2, %5;\n\taddc.u32 %0, %0, %0;\n\t"
        "add.cc.u32 t, %3, %5;\n\taddc.u32 %0, %0, %0;\n\t"
        "add.cc.u32 t, %4, %5;\n\taddc.u32 %0, %0, %0;\n\t}"
        : "+r"(rej)
        : "r"(u.w), "r"(u.z), "r"(u.y), "r"(u.x), "r"(nthr));
    return rej;
  }
  if (P == 1) {
    const uint32_t b = (uint32_t)(u.w >= thr) << 3 | (uint32_t)(u.z >= thr) << 2 | (uint32_t)(u.y >= thr) << 1 |
                       (uint32_t)(u.x >= thr);
    return (rej << 4) | b;
  }
  if (P == 2) {  // even thr = 2t: accept <=> (u >> 1) < t <=> MSB((u >> 1) - t); funnel the MSB in
    const uint32_t t = thr >> 1;  // (builds the ACCEPT mask: the caller inverts once per word)
    rej = __funnelshift_l((u.w >> 1) - t, rej, 1);
    rej = __funnelshift_l((u.z >> 1) - t, rej, 1);
    rej = __funnelshift_l((u.y >> 1) - t, rej, 1);
    return __funnelshift_l((u.x >> 1) - t, rej, 1);
  }
  if (P == 4) {  // NOT a Bernoulli pack: the cheapest dependent fold (one LOP3 per call) -- an upper
                 // bound on what any pack could gain over the carry chain
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(u.x), "r"(u.y), "r"(u.z ^ u.w));
    return (rej << 1) ^ r;
  }
  // P == 3: exact for any thr, x and y on the ALU (borrow = MSB of maj(~u, thr, d), d = u - thr),
  // z and w by the carry chain (builds the REJECT mask like P == 0)
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %1, %3;\n\taddc.u32 %0, %0, %0;\n\t"
      "add.cc.u32 t, %2, %3;\n\taddc.u32 %0, %0, %0;\n\t}"
      : "+r"(rej)
      : "r"(u.w), "r"(u.z), "r"(nthr));
  {
    const uint32_t d = u.y - thr;
    const uint32_t br = (~u.y & thr) | ((~u.y | thr) & d);  // borrow of u - thr in the MSB
    rej = __funnelshift_l(~br, rej, 1);
  }
  {
    const uint32_t d = u.x - thr;
    const uint32_t br = (~u.x & thr) | ((~u.x | thr) & d);
    rej = __funnelshift_l(~br, rej, 1);
  }
  return rej;
}

// Two words' calls (16) in one unrolled block before either is packed: more independent chains
template <int MINB>
__global__ void __launch_bounds__(128, MINB) kern2(Keys K, int trials, uint32_t thr, unsigned long long *out) {
  __shared__ uint4 U[26];
  if (threadIdx.x < 25) {
    const uint32_t q = threadIdx.x;
    const uint64_t p = (uint64_t)M0 * q;
    const uint32_t n2 = (uint32_t)(p >> 32) ^ 0u ^ K.k1[0];
    const uint64_t b = (uint64_t)M1 * n2;
    U[q] = make_uint4((uint32_t)(b >> 32) ^ K.k0[1], (uint32_t)b, (uint32_t)p ^ K.k1[1], 0u);
  }
  __syncthreads();
  const uint32_t nthr = 0u - thr;
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const uint32_t trial = tid * trials + t;
    const uint64_t p = (uint64_t)M1 * trial;
    const uint32_t n1 = (uint32_t)p, n0 = (uint32_t)(p >> 32) ^ K.k0[0];
    const uint64_t a = (uint64_t)M0 * n0;
    const uint32_t ha = (uint32_t)(a >> 32), la = (uint32_t)a;
    // words 0 and 1 together, then word 2 alone, then the last (1 call)
    {
      uint4 w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint4 u = U[j];
        w[j] = rounds_2_9<false, false>(u.x ^ n1, u.y, ha ^ u.z, la, K);
      }
      uint32_t R0 = 0, R1 = 0;
#pragma unroll
      for (int j = 7; j >= 0; --j) R0 = pack4<0>(R0, w[j], nthr, thr);
#pragma unroll
      for (int j = 15; j >= 8; --j) R1 = pack4<0>(R1, w[j], nthr, thr);
      acc += __popc(R0) + __popc(R1);
    }
    {
      uint32_t R = 0;
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        const uint4 u = U[16 + j];
        R = pack4<0>(R, rounds_2_9<false, false>(u.x ^ n1, u.y, ha ^ u.z, la, K), nthr, thr);
      }
      acc += __popc(R);
    }
    {
      const uint4 u = U[24];
      acc += __popc(pack4<0>(0, rounds_2_9<false, false>(u.x ^ n1, u.y, ha ^ u.z, la, K), nthr, thr) & 7u);
    }
  }
  atomicAdd(out, (unsigned long long)acc);
}

template <bool DA, bool DB, int P>
__global__ void __launch_bounds__(128, 5) kern(Keys K, int trials, uint32_t thr, unsigned long long *out) {
  __shared__ uint4 U[26];
  if (threadIdx.x < 25) {
    const uint32_t q = threadIdx.x;
    const uint64_t p = (uint64_t)M0 * q;
    const uint32_t n2 = (uint32_t)(p >> 32) ^ 0u ^ K.k1[0];
    const uint64_t b = (uint64_t)M1 * n2;
    U[q] = make_uint4((uint32_t)(b >> 32) ^ K.k0[1], (uint32_t)b, (uint32_t)p ^ K.k1[1], 0u);
  }
  __syncthreads();
  const uint32_t nthr = 0u - thr;
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const uint32_t trial = tid * trials + t;
    const uint64_t p = (uint64_t)M1 * trial;
    const uint32_t n1 = (uint32_t)p, n0 = (uint32_t)(p >> 32) ^ K.k0[0];
    const uint64_t a = (uint64_t)M0 * n0;
    const uint32_t ha = (uint32_t)(a >> 32), la = (uint32_t)a;
    for (int w = 0; w < 4; ++w) {
      uint32_t R = 0;
      if (w < 3) {
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          const uint4 u = U[8 * w + j];
          R = pack4<P>(R, rounds_2_9<DA, DB>(u.x ^ n1, u.y, ha ^ u.z, la, K), nthr, thr);
        }
        if (P == 2) R = ~R;
      } else {
        const uint4 u = U[24];
        R = pack4<P>(R, rounds_2_9<DA, DB>(u.x ^ n1, u.y, ha ^ u.z, la, K), nthr, thr);
        R = (P == 2 ? ~R : R) & 7u;
      }
      acc += __popc(R);
    }
  }
  atomicAdd(out, (unsigned long long)acc);
}

// host reference of one Philox4x32-10 call for the check
static void philox_host(uint32_t ctr[4], const Keys &K, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    const uint64_t a = (uint64_t)M0 * c0, b = (uint64_t)M1 * c2;
    const uint32_t n0 = (uint32_t)(b >> 32) ^ c1 ^ K.k0[r], n2 = (uint32_t)(a >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)b;
    c3 = (uint32_t)a;
    c0 = n0;
    c2 = n2;
  }
  out[0] = c0, out[1] = c1, out[2] = c2, out[3] = c3;
}

template <bool DA, bool DB, int P>
void run(const char *name, const Keys &K, unsigned long long want, int sms) {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  const int trials = 64;
  const int blocks = sms * 5 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  unsigned long long got = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(d, 0, 8);
    cudaEventRecord(a);
    kern<DA, DB, P><<<blocks, 128>>>(K, trials, THR, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = ms < best ? ms : best;
    cudaMemcpy(&got, d, 8, cudaMemcpyDeviceToHost);
  }
  const double tt = (double)blocks * 128 * trials * 100;
  printf("{\"variant\": \"%s\", \"ms\": %.3f, \"trial_tokens_per_s\": %.4e, \"popcount\": %llu, \"ok\": %s}\n", name,
         best, tt / (best * 1e-3), got, (want == 0 || got == want) ? "true" : "false");
  cudaFree(d);
}

template <int MINB>
void run2(const char *name, const Keys &K, unsigned long long want, int sms) {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  const int trials = 64, blocks = sms * 5 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  unsigned long long got = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(d, 0, 8);
    cudaEventRecord(a);
    kern2<MINB><<<blocks, 128>>>(K, trials, THR, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = ms < best ? ms : best;
    cudaMemcpy(&got, d, 8, cudaMemcpyDeviceToHost);
  }
  const double tt = (double)blocks * 128 * trials * 100;
  printf("{\"variant\": \"%s\", \"ms\": %.3f, \"trial_tokens_per_s\": %.4e, \"popcount\": %llu, \"ok\": %s}\n", name,
         best, tt / (best * 1e-3), got, (want == 0 || got == want) ? "true" : "false");
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Keys K;
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = 2405141050u + (uint32_t)r * 0x9E3779B9u;
    K.k1[r] = 0u + (uint32_t)r * 0xBB67AE85u;
  }
  // host check of the first thread's first trial (counter (q, 0, 0, 0))
  uint32_t o[4], c[4];
  int pc = 0;
  for (uint32_t q = 0; q < 25; ++q) {
    c[0] = q, c[1] = 0, c[2] = 0, c[3] = 0;
    philox_host(c, K, o);
    for (int i = 0; i < 4; ++i)
      if (4 * q + i < 99) pc += o[i] >= THR;
  }
  printf("{\"host_trial0_rejections\": %d}\n", pc);
  unsigned long long ref = 0;
  {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    kern<false, false, 0><<<sms * 40, 128>>>(K, 64, THR, d);
    cudaMemcpy(&ref, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
  }
  run<false, false, 0>("W W, carry pack (current)", K, ref, sms);
  run2<5>("W W, carry pack, two words' 16 calls before packing (min 5 blocks)", K, ref, sms);
  run2<4>("W W, carry pack, two words' 16 calls before packing (min 4 blocks)", K, ref, sms);
  run2<3>("W W, carry pack, two words' 16 calls before packing (min 3 blocks)", K, ref, sms);
  run<false, false, 2>("W W, sign-funnel pack (even threshold)", K, ref, sms);
  run<false, false, 3>("W W, 2 carry + 2 borrow-funnel bits (exact)", K, ref, sms);
  run<false, false, 1>("W W, compare pack", K, ref, sms);
  run<false, false, 4>("W W, xor fold (upper bound: not a Bernoulli pack)", K, 0, sms);
  if (getenv("PV_ALL")) {
    run<false, true, 0>("W D, carry pack", K, ref, sms);
    run<true, false, 0>("D W, carry pack", K, ref, sms);
    run<true, true, 0>("D D, carry pack", K, ref, sms);
    run<false, true, 1>("W D, compare pack", K, ref, sms);
  }
  return 0;
}
