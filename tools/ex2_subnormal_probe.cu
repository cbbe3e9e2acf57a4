// Does MUFU ex2.approx.f16x2 produce FP16 subnormals?  (tool)
#include <cuda_fp16.h>
#include <cstdio>
#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;
__global__ void k(const float* x, float* mufu, float* poly, int n) {
  int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i >= n) return;
  // low half = x, high half = x - 0.5: both lanes checked
  uint32_t h = h2_as_u32(__floats2half2_rn(x[i], x[i] - 0.5f));
  const uint32_t m = ex2_f16x2(h), p = ex2_poly_f16x2(h);
  mufu[2 * i] = __low2float(u32_as_h2(m));
  mufu[2 * i + 1] = __high2float(u32_as_h2(m));
  poly[2 * i] = __low2float(u32_as_h2(p));
  poly[2 * i + 1] = __high2float(u32_as_h2(p));
}
int main() {
  const int n = 12;
  float hx[n] = {-1.f, -10.f, -13.9f, -14.f, -14.5f, -15.f, -16.f, -18.f, -20.f, -22.f, -24.f, -25.f};
  float *dx, *dm, *dp, hm[2 * n], hp[2 * n];
  cudaMalloc(&dx, n * 4); cudaMalloc(&dm, 2 * n * 4); cudaMalloc(&dp, 2 * n * 4);
  cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dx, dm, dp, n);
  cudaMemcpy(hm, dm, 2 * n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hp, dp, 2 * n * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i)
    printf("x=%6.2f exact lo %.4e hi %.4e | mufu lo %.4e hi %.4e | poly lo %.4e hi %.4e\n", hx[i],
           exp2((double)hx[i]), exp2((double)hx[i] - 0.5), hm[2 * i], hm[2 * i + 1], hp[2 * i], hp[2 * i + 1]);
  return 0;
}
