// tools/mufu_contention_probe.cu -- profiling tool, not product code.  Two warps per SMSP
// run the fused kernel's exp pass (HFMA2 argument, ex2.approx.f16x2, two FHADD per pair)
// while two other warps per SMSP run a competing instruction stream; the exp warps time
// themselves with clock64.  Shows how much the other tile's work (max/sum pass, O update,
// TMEM/shared loads, barrier waits) slows the MUFU-bound exp pass.
#include <cuda_fp16.h>
#include <cstdio>

#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;

constexpr int ITERS = 256, NP = 32;

template <int B_MODE, bool SUM>
__global__ void __launch_bounds__(512, 1) probe(uint32_t* out, long long* cyc, uint32_t scale2, uint32_t c2) {
  __shared__ uint4 sm[1024];
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  if (warp < 8) {  // exp warps (2 per SMSP)
    uint32_t s[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) s[i] = h2_as_u32(__floats2half2_rn(-0.01f * i - threadIdx.x * 1e-4f, -0.3f));
    float tot = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        const uint32_t x = h2_as_u32(__hfma2(u32_as_h2(s[i]), u32_as_h2(scale2), u32_as_h2(c2)));
        const uint32_t pv = ex2_f16x2(x);
        if (SUM) {
          acc[2 * (i & 3)] = add_lo_f16(acc[2 * (i & 3)], pv);
          acc[2 * (i & 3) + 1] = add_hi_f16(acc[2 * (i & 3) + 1], pv);
        }
        s[i] = pv ^ 0x80008000u;
      }
      tot += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    }
    const long long t1 = clock64();
    uint32_t r = __float_as_uint(tot);
#pragma unroll
    for (int i = 0; i < NP; ++i) r ^= s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 8 + warp] = t1 - t0;
    __syncwarp();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
  } else {  // competing warps (2 per SMSP)
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 0x10001u + i;
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = 0.f;
    int n = 0;
    while (true) {
      if (B_MODE == 1) {  // ALU/FMA stream: HMNMX2 + FHADD (the max/sum pass)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] = h2_as_u32(__hmax2(u32_as_h2(v[i]), u32_as_h2(v[(i + 5) & 15])));
          f[i & 7] = add_lo_f16(f[i & 7], v[i]);
        }
      } else if (B_MODE == 2) {  // HFMA2 stream (O update)
#pragma unroll
        for (int i = 0; i < 16; ++i)
          v[i] = h2_as_u32(__hfma2(u32_as_h2(v[i]), u32_as_h2(v[(i + 3) & 15]), u32_as_h2(v[(i + 7) & 15])));
      } else if (B_MODE == 3) {  // shared-memory loads (MIO)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 x = sm[(threadIdx.x + i * 128 + n) & 1023];
          v[i] ^= x.x ^ x.y ^ x.z ^ x.w;
        }
      } else if (B_MODE == 4) {  // try_wait spin on a barrier the exp warps complete at the end
      }
      ++n;
      if (B_MODE == 0 || mbar_test_wait(smem_u32(&bar), 0)) break;
      if (B_MODE == 4) { while (!mbar_try_wait(smem_u32(&bar), 0)) {} break; }
    }
    uint32_t r = n;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= __float_as_uint(f[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8 * 8);
  long long* h = new long long[sms * 8];
  const char* names[] = {"none (exp warps alone)", "HMNMX2+FHADD stream", "HFMA2 stream", "LDS.128 stream",
                         "mbarrier try_wait spin"};
  for (int sum = 1; sum >= 0; --sum)
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: (sum ? probe<0, true> : probe<0, false>)<<<sms, 512>>>(out, cyc, 0x40004000u, 0x3C003C00u); break;
        case 1: (sum ? probe<1, true> : probe<1, false>)<<<sms, 512>>>(out, cyc, 0x40004000u, 0x3C003C00u); break;
        case 2: (sum ? probe<2, true> : probe<2, false>)<<<sms, 512>>>(out, cyc, 0x40004000u, 0x3C003C00u); break;
        case 3: (sum ? probe<3, true> : probe<3, false>)<<<sms, 512>>>(out, cyc, 0x40004000u, 0x3C003C00u); break;
        case 4: (sum ? probe<4, true> : probe<4, false>)<<<sms, 512>>>(out, cyc, 0x40004000u, 0x3C003C00u); break;
      }
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sms * 8 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms * 8; ++i) mx = h[i] > mx ? h[i] : mx;
    // per SMSP: 2 warps x 32 lanes x NP pairs x 2 elements per iteration
    const double elems = 2.0 * 32 * NP * 2 * ITERS;
    printf("sum=%d %-26s exp pass: %6.2f exp/clk/SMSP -> %5.0f cycles per 16384-exp tile-block (1024 = MUFU bound)\n",
           sum, names[mode], elems / mx, 16384.0 / (4 * elems / mx));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
