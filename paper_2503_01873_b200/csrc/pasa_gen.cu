// pasa_gen.cu -- device-side input generators.
//
// The reference draws every element as a pure function of (seed, stream,
// counter) through SplitMix64 (rng.hpp:14-27) and rounds it once to binary16
// (bench.cpp:28-48, gen_tensor :50-56).  Each thread here owns one flat index,
// so a 128K-token problem is generated in HBM in milliseconds instead of
// minutes on the host, with the reference's bits:
//   * uniform: integer hash + three double ops -> bit-exact (the ops are
//     written as __dadd_rn/__dmul_rn so nvcc cannot contract them into an FMA
//     the x86 reference does not perform);
//   * hybrid: Box-Muller uses log/cos, which CUDA evaluates within 1 ulp of
//     libm; after the single FP16 rounding the outputs agree except where a
//     double lands within an ulp of an FP16 rounding boundary (tests count it).
// The resonance generator restates oracle/pasa_oracle.c:orc_generate_resonance
// (SURVEY.md 8d config 3).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pasa_kernels.cuh"

namespace pasa_b200 {
namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t ctr) {
  const uint64_t h = splitmix(splitmix(splitmix(seed) ^ stream) ^ ctr);
  return __dmul_rn(static_cast<double>(h >> 11), 0x1.0p-53);
}

// rng.hpp:30-35: u1 in (0, 1], u2 in [0, 1).
__device__ __forceinline__ double gaussian(uint64_t seed, uint64_t stream, uint64_t i) {
  const double u1 = __dsub_rn(1.0, u01(seed, stream, 2 * i));
  const double u2 = u01(seed, stream, 2 * i + 1);
  const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
  return __dmul_rn(r, cos(__dmul_rn(2.0 * 3.14159265358979323846, u2)));
}

__global__ void gen_kernel(GenParams p, __half* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t ii = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; ii < p.n;
       ii += stride) {
    const uint64_t idx = p.start + ii;
    double v;
    if (p.kind == 0) {  // bench.cpp:30-33
      const double u = u01(p.seed, p.tensor_id, idx);
      v = __dadd_rn(__dsub_rn(p.x0, p.am), __dmul_rn(__dmul_rn(2.0, p.am), u));
    } else {  // bench.cpp:34-41
      const uint64_t base = p.tensor_id * 4;
      const double core = __dadd_rn(p.x0, gaussian(p.seed, base, idx));
      const bool gate = u01(p.seed, base + 2, idx) < p.p;
      v = gate ? __dadd_rn(core, __dmul_rn(p.am, gaussian(p.seed, base + 1, idx))) : core;
    }
    out[ii] = __double2half(v);  // one RNE rounding, f16_round (half.cpp)
  }
}

__global__ void gen_resonance_kernel(ResonanceParams p, __half* __restrict__ out) {
  const double twopi = 2.0 * 3.14159265358979323846;
  const uint64_t n = static_cast<uint64_t>(p.B) * p.H * p.S * p.d;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t ii = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; ii < n;
       ii += stride) {
    const uint64_t c = ii % p.d;
    const uint64_t s = (ii / p.d) % p.S;
    const uint64_t h = (ii / (static_cast<uint64_t>(p.d) * p.S)) % p.H;
    const double noise = __dsub_rn(__dmul_rn(2.0, u01(p.seed, p.tensor_id, ii)), 1.0);
    const double arg = __dadd_rn(
        __ddiv_rn(__dmul_rn(__dmul_rn(twopi, 3.0), static_cast<double>(c)), static_cast<double>(p.d)),
        __dmul_rn(0.3, static_cast<double>(h)));
    const double wave = cos(arg);
    double v;
    if (p.tensor_id == 0) {
      v = __dadd_rn(__dmul_rn(p.qa, wave), noise);
    } else if (p.tensor_id == 1) {
      const double sn = sin(__ddiv_rn(__dmul_rn(twopi, static_cast<double>(s)), 512.0));
      v = __dadd_rn(__dmul_rn(__dmul_rn(-p.ka, __dadd_rn(1.0, __dmul_rn(0.1, sn))), wave), noise);
    } else {
      v = noise;
    }
    out[ii] = __double2half(v);
  }
}

int grid_for(uint64_t n) {
  const int sms = current_sm_count();
  const uint64_t want = (n + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * 16;  // grid-stride beyond 16 CTAs per SM
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_generate(const GenParams& p, void* out, cudaStream_t stream) {
  if (p.n == 0) return cudaSuccess;
  gen_kernel<<<grid_for(p.n), 256, 0, stream>>>(p, static_cast<__half*>(out));
  return cudaGetLastError();
}

cudaError_t launch_generate_resonance(const ResonanceParams& p, void* out, cudaStream_t stream) {
  const uint64_t n = static_cast<uint64_t>(p.B) * p.H * p.S * p.d;
  if (n == 0) return cudaSuccess;
  gen_resonance_kernel<<<grid_for(n), 256, 0, stream>>>(p, static_cast<__half*>(out));
  return cudaGetLastError();
}

}  // namespace pasa_b200
