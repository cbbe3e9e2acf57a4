// tools/mufu_probe.cu -- microbenchmark of the per-element softmax building
// blocks on sm_100a (profiling tool, not product code).  Each variant runs
// ITERS x 16 independent operations per thread over one full wave of CTAs and
// reports throughput in elements per clock per SM.
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;

constexpr int ITERS = 4096;

// 2^x (x <= 0) for a half2 on the FMA/ALU pipes: x clamped to [-15, 0],
// n = round(x) via the 1039 = 1024 + 15 magic add (the low mantissa bits of t
// hold n + 15 in 0..15), f = x - n in [-0.5, 0.5], 2^f by a cubic, times 2^n
// built from the exponent field (n = -15 gives +0).
__device__ __forceinline__ uint32_t exp2_poly_h2(uint32_t xr) {
  const __half2 x = __hmax2(u32_as_h2(xr), __float2half2_rn(-15.0f));
  const __half2 magic = __float2half2_rn(1039.0f);
  const __half2 t = __hadd2(x, magic);
  const __half2 n = __hsub2(t, magic);
  const __half2 f = __hsub2(x, n);
  const __half2 c3 = __float2half2_rn(0.0555041086f), c2 = __float2half2_rn(0.2402264923f),
                c1 = __float2half2_rn(0.6931471806f), one = __float2half2_rn(1.0f);
  __half2 p = __hfma2(f, c3, c2);
  p = __hfma2(p, f, c1);
  p = __hfma2(p, f, one);
  const uint32_t e = (h2_as_u32(t) & 0x000F000Fu) << 10;  // 2^n as fp16 bits
  return h2_as_u32(__hmul2(p, u32_as_h2(e)));
}

template <int MODE>
__global__ void __launch_bounds__(256) bench_kernel(uint32_t* out, float seed) {
  uint32_t v[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = h2_as_u32(__floats2half2_rn(-(seed + i * 0.01f + threadIdx.x * 1e-4f), -0.5f - i * 0.02f));
    f[i] = -(seed + i * 0.03f);
  }
  float acc = 0.f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {  // MUFU ex2 f16x2
        v[i] = ex2_f16x2(v[i]) ^ 0x80008000u;  // keep the argument negative
      } else if (MODE == 1) {  // ex2 f32 (x2 per pair)
        f[i] = -ex2_f32(f[i]);
      } else if (MODE == 2) {  // FMA-pipe polynomial exp2 per half2
        v[i] = exp2_poly_h2(v[i]) | 0x80008000u;  // keep negative
      } else if (MODE == 3) {  // fp32 += fp16 (FHADD), two per pair
        acc = add_lo_f16(acc, v[i]);
        f[i] = add_hi_f16(f[i], v[i]);
      } else if (MODE == 4) {  // HFMA2
        v[i] = h2_as_u32(__hfma2(u32_as_h2(v[i]), u32_as_h2(v[i]), u32_as_h2(v[(i + 1) & 15])));
      } else if (MODE == 5) {  // HMNMX2
        v[i] = h2_as_u32(__hmax2(u32_as_h2(v[i]), u32_as_h2(v[(i + 3) & 15])));
      }
    }
  }
  uint32_t r = __float_as_uint(acc);
#pragma unroll
  for (int i = 0; i < 16; ++i) r ^= v[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  const int blocks = sms * 4;
  cudaMalloc(&out, blocks * 256 * 4);
  const char* names[] = {"ex2.approx.f16x2 (MUFU)", "ex2.approx.f32 (MUFU)", "exp2 poly f16x2 (FMA)",
                         "add.f32.f16 (FHADD)", "HFMA2", "HMNMX2"};
  // elements per op: f16x2 variants handle 2 elements, f32/FHADD 1 (MODE 3 does 2 FHADD = 2 elements)
  const double elems[] = {2, 1, 2, 2, 2, 2};
  for (int mode = 0; mode < 6; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: bench_kernel<0><<<blocks, 256>>>(out, 0.3f); break;
        case 1: bench_kernel<1><<<blocks, 256>>>(out, 0.3f); break;
        case 2: bench_kernel<2><<<blocks, 256>>>(out, 0.3f); break;
        case 3: bench_kernel<3><<<blocks, 256>>>(out, 0.3f); break;
        case 4: bench_kernel<4><<<blocks, 256>>>(out, 0.3f); break;
        case 5: bench_kernel<5><<<blocks, 256>>>(out, 0.3f); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = double(blocks) * 256 * ITERS * 16;
    const double cycles = ms * 1e-3 * clk * 1e3;  // at the nominal max clock
    printf("%-28s %8.3f ms  %7.2f elem/clk/SM (at %d MHz nominal)\n", names[mode], ms,
           ops * elems[mode] / cycles / sms, clk / 1000);
  }
  // accuracy of the polynomial vs exact 2^x over the softmax range
  return 0;
}
