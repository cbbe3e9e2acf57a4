// tools/pass2_probe.cu -- throughput of the fused kernel's pass-2 instruction
// mix (HSUB2, exp2 on MUFU or the FMA-pipe polynomial, PRMT, 8-chain FHADD row
// sum) as a function of warps per SMSP (profiling tool, not product code).
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;

template <int POLY_EVERY>  // 0: MUFU only; k: one pair in k on the polynomial
__global__ void pass2_kernel(uint32_t* out, int iters, uint32_t cj2) {
  uint32_t s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i)
    s[i] = h2_as_u32(__floats2half2_rn(-0.01f * (i + threadIdx.x % 7), -0.02f * i));
  float tot = 0.f;
  for (int it = 0; it < iters; ++it) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const uint32_t x = h2_as_u32(__hsub2(u32_as_h2(s[i]), u32_as_h2(cj2)));
      const uint32_t pv = (POLY_EVERY && (i % POLY_EVERY) == POLY_EVERY - 1) ? ex2_poly_f16x2(x)
                                                                             : ex2_f16x2(x);
      acc[2 * (i & 3)] = add_lo_f16(acc[2 * (i & 3)], pv);
      acc[2 * (i & 3) + 1] = add_hi_f16(acc[2 * (i & 3) + 1], pv);
      s[i] = pv ^ 0x80008000u;
    }
    tot += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  uint32_t r = __float_as_uint(tot);
#pragma unroll
  for (int i = 0; i < 64; ++i) r ^= s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, sms * 1024 * 4);
  const int iters = 2000;
  for (int poly : {0, 4, 2}) {
    for (int wps : {1, 2, 4}) {  // warps per SMSP
      const int threads = 128 * wps;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (poly == 0) pass2_kernel<0><<<sms, threads>>>(out, iters, 0x3c003c00u);
        if (poly == 4) pass2_kernel<4><<<sms, threads>>>(out, iters, 0x3c003c00u);
        if (poly == 2) pass2_kernel<2><<<sms, threads>>>(out, iters, 0x3c003c00u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double cyc = ms * 1e-3 * clk * 1e3;
      // cycles for one warp to finish one 64-pair row pass, per SMSP
      printf("poly 1/%d  warps/SMSP %d : %7.1f cycles per row-pass per warp, %6.1f per warp-slot\n",
             poly ? poly : 0, wps, cyc / iters, cyc / iters / wps);
    }
  }
  return 0;
}
