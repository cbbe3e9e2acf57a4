// tools/mufu_occ_probe.cu -- profiling tool, not product code.  The fused kernel's
// exp pass (HFMA2 argument, ex2.approx.f16x2, two FP32 FHADD accumulations per pair,
// eight chains) run by W warps per SMSP (one CTA of 32*4*W threads per SM), to see
// whether MUFU saturates with the warp count the d = 64 exp pass has (2 per SMSP).
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;

constexpr int ITERS = 512, NP = 32;

template <int POLY>
__global__ void exp_pass(uint32_t* out, uint32_t scale2, uint32_t c2) {
  uint32_t s[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) s[i] = h2_as_u32(__floats2half2_rn(-0.01f * i - threadIdx.x * 1e-4f, -0.3f));
  float tot = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const uint32_t x = h2_as_u32(__hfma2(u32_as_h2(s[i]), u32_as_h2(scale2), u32_as_h2(c2)));
      const uint32_t pv = (POLY > 0 && i % (POLY > 0 ? POLY : 1) == POLY - 1) ? ex2_poly_f16x2(x) : ex2_f16x2(x);
      acc[2 * (i & 3)] = add_lo_f16(acc[2 * (i & 3)], pv);
      acc[2 * (i & 3) + 1] = add_hi_f16(acc[2 * (i & 3) + 1], pv);
      s[i] = pv ^ 0x80008000u;
    }
    tot += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  uint32_t r = __float_as_uint(tot);
#pragma unroll
  for (int i = 0; i < NP; ++i) r ^= s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, sms * 1024 * 4 * 4);
  const uint32_t scale2 = 0x40004000u, c2 = 0x3C003C00u;  // x = 2 s + 1 (s <= -0.5ish)
  for (int poly = 0; poly <= 8; poly += 4) {
    for (int w : {1, 2, 3, 4, 8}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (poly == 0) exp_pass<0><<<sms, 128 * w>>>(out, scale2, c2);
        else if (poly == 4) exp_pass<4><<<sms, 128 * w>>>(out, scale2, c2);
        else exp_pass<8><<<sms, 128 * w>>>(out, scale2, c2);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double elems = double(sms) * 128 * w * ITERS * NP * 2;
      const double cycles = ms * 1e-3 * clk * 1e3;
      printf("poly 1/%d  %d warps/SMSP: %7.2f exp/clk/SM  (%.0f cycles per 16384-element tile-block)\n",
             poly, w, elems / cycles / sms, 16384.0 / (elems / cycles / sms));
    }
  }
  return 0;
}
