// tools/prep_probe.cu -- the packed kernel's per-tile pre-pass (self_prep_stage, the SVD
// temporal shape's slot width 32) alone on one CTA, no TMA / MMA / softmax around it: its
// intrinsic latency per phase, from the PASA_TRACE events (profiling tool).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_01873_b200/csrc \
//        -o tools/_prep_probe tools/prep_probe.cu -lcuda && tools/_prep_probe [ctas]
#define PASA_TRACE
#include "pasa_fwd_packed.cu"

#include <cstdio>
#include <vector>

using namespace pasa_b200;

template <int D>
__global__ void __launch_bounds__(384, 1) prep_probe(PackedParams p, int iters) {
  using Cfg = PackedCfg<D, 32>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sb = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sb - smem_u32(smem_raw));
  const uint32_t in_full = sb + Cfg::SMEM_BAR;
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + Cfg::SMEM_BAR + 8 * Cfg::NUM_BARS);
  volatile uint32_t* bad = holder + 1;
  int* c0s = reinterpret_cast<int*>(holder + 5);
  unsigned* vmx = reinterpret_cast<unsigned*>(c0s + 32);
  for (int e = threadIdx.x; e < Cfg::STAGE_BYTES / 4; e += blockDim.x) {  // halves in (-2, 2)
    const uint32_t h = (e * 2654435761u) >> 7;
    reinterpret_cast<uint32_t*>(smem)[e] = (0x3800u + (h & 0x3ffu) + ((h >> 10) & 1u) * 0x8000u) |
                                           ((0x3800u + ((h >> 11) & 0x3ffu)) << 16);
  }
  const uint32_t kdone = in_full + 8;  // (arrived on, never waited for)
  if (threadIdx.x == 0) {
    mbar_init(in_full, 1);
    mbar_init(kdone, 1);
  }
  fence_barrier_init();
  __syncthreads();
  const int nseq = p.P;
  if (threadIdx.x >= 256) {
    for (int it = 0; it < iters; ++it) {
      if (threadIdx.x == 256) {
        mbar_arrive(in_full);
        PK_TR(1, it, 5);
      }
      self_prep_stage<D, 32>(sb, p.N, p.dm, p.off, p.lscale, nseq, smem_u32(c0s), smem_u32(vmx),
                             smem_u32(const_cast<uint32_t*>(bad)), in_full, in_full, kdone, it & 1, p.trace, it, 0);
      if (threadIdx.x == 256) PK_TR(1, it, 6);
    }
  }
  __syncthreads();
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 1;
  constexpr int D = 64;
  using Cfg = PackedCfg<D, 32>;
  PackedParams p{};
  p.N = 25;
  p.W = 32;
  p.P = 4;
  p.BH = 4;
  p.self_prep = 1;
  p.dm = 0.0156f;
  p.off = -0.0156f / 128;
  p.lscale = 0.7213475f;
  long long* tr;
  cudaMalloc(&tr, 2 * 64 * 16 * 8);
  cudaMemset(tr, 0, 2 * 64 * 16 * 8);
  p.trace = tr;
  cudaFuncSetAttribute(prep_probe<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  prep_probe<D><<<ctas, 384, Cfg::SMEM_BYTES>>>(p, 64);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<long long> t(2 * 64 * 16);
  cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
    constexpr int STRIDE = 16;
  auto at = [&](int role, int it, int ev) { return t[(role * 64 + it) * STRIDE + ev]; };
  double s[4] = {0};
  int n = 0;
  for (int it = 4; it < 64; ++it, ++n) {
    s[0] += at(1, it, 8) - at(0, it, 6);   // K side (sums, K')
    s[1] += at(1, it, 10) - at(1, it, 9);  // V side: scan, atomics, barrier
    s[2] += at(1, it, 11) - at(1, it, 10); // c0, V scale, fence, barrier
    s[3] += at(1, it, 6) - at(1, it, 5);   // whole stage
  }
  printf("ctas %d, d=%d N=25 W=32 4 slots: K side %.0f  V scan %.0f  c0+fence %.0f | whole %.0f cycles\n", ctas, D,
         s[0] / n, s[1] / n, s[2] / n, s[3] / n);
  return 0;
}
