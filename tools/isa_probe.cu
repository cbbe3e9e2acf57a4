// tools/isa_probe.cu -- issue/pipe throughput of the softmax's building blocks on
// sm_100a, alone and interleaved (profiling tool, not product code).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_isa_probe tools/isa_probe.cu
//
// One CTA per SM, W warps per SMSP, each warp runs ITERS x 16 independent ops per
// mode; cycles from clock64 (slowest warp).  Prints warp-instructions per cycle per
// SMSP for the op the mode names (1.0 = one warp instruction every cycle).
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
  uint32_t r;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float fhadd_lo(float a, uint32_t p) {
  float r;
  asm volatile("{.reg .f16 l, h; mov.b32 {l, h}, %2; add.rn.f32.f16 %0, l, %1;}" : "=f"(r) : "f"(a), "r"(p));
  return r;
}
__device__ __forceinline__ float fhadd_hi(float a, uint32_t p) {
  float r;
  asm volatile("{.reg .f16 l, h; mov.b32 {l, h}, %2; add.rn.f32.f16 %0, h, %1;}" : "=f"(r) : "f"(a), "r"(p));
  return r;
}
__device__ __forceinline__ void fadd2(float& a, float& b, float c, float d) {
  uint64_t x = (uint64_t(__float_as_uint(b)) << 32) | __float_as_uint(a);
  uint64_t y = (uint64_t(__float_as_uint(d)) << 32) | __float_as_uint(c);
  uint64_t r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  a = __uint_as_float(uint32_t(r));
  b = __uint_as_float(uint32_t(r >> 32));
}

template <int MODE>
__global__ void __launch_bounds__(1024) probe(uint32_t* out, long long* cyc, float seed) {
  uint32_t v[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = h2u(__floats2half2_rn(-(seed + i * 0.01f + threadIdx.x * 1e-4f), -0.5f - i * 0.02f));
    f[i] = seed * i;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) v[i] = ex2h2(v[i]) ^ 0x80008000u;                        // MUFU pair (2 MUFU)
      if (MODE == 1) f[i] = fhadd_lo(f[i], v[i]);                             // FHADD
      if (MODE == 2) v[i] = h2u(__hfma2(u2h(v[i]), u2h(v[(i + 1) & 15]), u2h(v[(i + 5) & 15])));
      if (MODE == 3) v[i] = h2u(__hadd2(u2h(v[i]), u2h(v[(i + 3) & 15])));    // HADD2
      if (MODE == 4) f[i] = __fadd_rn(f[i], f[(i + 3) & 15]);                 // FADD
      if (MODE == 5 && (i & 1) == 0) fadd2(f[i], f[i + 1], f[(i + 2) & 15], f[(i + 3) & 15]);
      if (MODE == 6) v[i] = __byte_perm(v[i], v[(i + 1) & 15], 0x5410);       // PRMT
      if (MODE == 7) {  // one MUFU pair + 2 FHADD (the exp pass's inner pattern, no arg)
        v[i] = ex2h2(v[i]) ^ 0x80008000u;
        f[i] = fhadd_lo(f[i], v[i]);
        f[(i + 8) & 15] = fhadd_hi(f[(i + 8) & 15], v[i]);
      }
      if (MODE == 8) {  // HFMA2 + 2 FHADD
        v[i] = h2u(__hfma2(u2h(v[i]), u2h(v[(i + 1) & 15]), u2h(v[(i + 5) & 15])));
        f[i] = fhadd_lo(f[i], v[i]);
        f[(i + 8) & 15] = fhadd_hi(f[(i + 8) & 15], v[i]);
      }
      if (MODE == 9) {  // MUFU pair + HFMA2
        v[i] = ex2h2(v[i]) ^ 0x80008000u;
        v[(i + 8) & 15] = h2u(__hfma2(u2h(v[(i + 8) & 15]), u2h(v[(i + 1) & 15]), u2h(v[(i + 5) & 15])));
      }
      if (MODE == 10) {  // HFMA2 arg + MUFU pair + 2 FHADD (exp pass without PRMT/poly)
        const uint32_t x = h2u(__hfma2(u2h(v[i]), __float2half2_rn(2.f), u2h(v[(i + 5) & 15])));
        v[i] = ex2h2(x) ^ 0x80008000u;
        f[i] = fhadd_lo(f[i], v[i]);
        f[(i + 8) & 15] = fhadd_hi(f[(i + 8) & 15], v[i]);
      }
      if (MODE == 11) {  // HADD2 pair pre-sum + 1 FHADD per pair (P sum via FP16 pairs)
        v[i] = ex2h2(v[i]) ^ 0x80008000u;
        if (i & 1) {
          const uint32_t s2 = h2u(__hadd2(u2h(v[i]), u2h(v[i - 1])));
          f[i] = fhadd_lo(f[i], s2);
          f[i - 1] = fhadd_hi(f[i - 1], s2);
        }
      }
      if (MODE == 12) v[i] = h2u(__hmax2(u2h(v[i]), u2h(v[(i + 3) & 15])));   // HMNMX2
      if (MODE == 13) {  // FADD2 pair sum of cvt'd halves: cvt.f32.f16 x2 + f32x2 add
        const float a = __low2float(u2h(v[i])), b = __high2float(u2h(v[i]));
        fadd2(f[i], f[(i + 8) & 15], a, b);
        v[i] ^= 0x00010001u;
      }
    }
  }
  const long long t1 = clock64();
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r ^= v[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const char* name, double instr_per_iter, uint32_t* out, long long* cyc, int sms) {
  for (int wps : {1, 2, 4, 8}) {
    const int threads = 128 * wps;
    probe<MODE><<<sms, threads>>>(out, cyc, 0.3f);
    probe<MODE><<<sms, threads>>>(out, cyc, 0.3f);
    cudaDeviceSynchronize();
    long long h[32 * 200];
    cudaMemcpy(h, cyc, sizeof(long long) * 32 * sms, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < sms; ++b)
      for (int w = 0; w < threads / 32; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
    // warp-instructions of the named op per cycle per SMSP
    const double ops = double(ITERS) * 16 * instr_per_iter * wps;
    printf("%-40s warps/SMSP %d : %6.3f warp-op/cyc/SMSP  (%lld cyc)\n", name, wps, ops / mx, mx);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 32 * 8);
  run<0>("ex2.f16x2 (per pair = 2 MUFU)", 1, out, cyc, sms);
  run<1>("FHADD", 1, out, cyc, sms);
  run<2>("HFMA2", 1, out, cyc, sms);
  run<3>("HADD2", 1, out, cyc, sms);
  run<4>("FADD", 1, out, cyc, sms);
  run<5>("FADD2 (f32x2)", 0.5, out, cyc, sms);
  run<6>("PRMT", 1, out, cyc, sms);
  run<7>("pair: ex2.f16x2 + 2 FHADD", 1, out, cyc, sms);
  run<8>("pair: HFMA2 + 2 FHADD", 1, out, cyc, sms);
  run<9>("pair: ex2.f16x2 + HFMA2", 1, out, cyc, sms);
  run<10>("pair: HFMA2 + ex2.f16x2 + 2 FHADD", 1, out, cyc, sms);
  run<11>("pair: ex2.f16x2 + (HADD2 + 2 FHADD)/2", 1, out, cyc, sms);
  run<12>("HMNMX2", 1, out, cyc, sms);
  run<13>("pair: cvt x2 + FADD2", 1, out, cyc, sms);
  return 0;
}
