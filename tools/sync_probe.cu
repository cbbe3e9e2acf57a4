// tools/sync_probe.cu -- latency of the CTA synchronisation primitives the MMA issuer
// waits on, when the awaited event has ALREADY happened (profiling tool, not product code):
// mbarrier try_wait / test_wait on a completed phase, an acquire load of a shared-memory
// counter, and a plain volatile shared load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_sync_probe tools/sync_probe.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;

__device__ __forceinline__ uint32_t ld_acquire(uint32_t a) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_volatile(uint32_t a) {
  uint32_t v;
  asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

__global__ void probe(long long* out, int mode, int n) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t cnt;
  const uint32_t b = smem_u32(&bar), c = smem_u32(&cnt);
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    cnt = 5;
  }
  fence_barrier_init();
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(b);  // phase 0 completes
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0, off = 0;  // off is 0 but data-dependent on the previous result: a latency chain
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    uint32_t r = 0;
    if (mode == 0) r = mbar_try_wait(b + off, 0) ? 1 : 0, off = (1 - r) * 8;
    if (mode == 1) r = mbar_test_wait(b + off, 0) ? 1 : 0, off = (1 - r) * 8;
    if (mode == 2) r = ld_acquire(c + off), off = (r - 5) * 4;
    if (mode == 3) r = ld_volatile(c + off), off = (r - 5) * 4;
    if (mode == 4) { mbar_wait(b + off, 0); r = 1; }
    if (mode == 5) { asm volatile("add.u32 %0, %1, 1;" : "=r"(r) : "r"(off)); off = r - 1; }
    acc += r;
  }
  const long long t1 = clock64();
  out[0] = (t1 - t0) / n;
  out[1] = acc;
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const char* names[] = {"mbarrier.try_wait (completed)", "mbarrier.test_wait (completed)",
                         "ld.acquire.cta.shared", "ld.volatile.shared", "mbar_wait (completed)", "add.u32 chain"};
  for (int m = 0; m < 6; ++m) {
    probe<<<1, 32>>>(d, m, 1000);
    probe<<<1, 32>>>(d, m, 1000);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-34s %5lld cycles per call (dependent chain)\n", names[m], h[0]);
  }
  return 0;
}
