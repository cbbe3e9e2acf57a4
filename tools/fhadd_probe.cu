// Does add.rn.f32.f16 (FHADD) flush FP16 subnormal inputs? (tool)
#include <cuda_fp16.h>
#include <cstdio>
#include "../paper_2503_01873_b200/csrc/sm100.cuh"
using namespace pasa_b200::sm100;
__global__ void k(const float* x, float* lo, float* hi, float* cvt, int n) {
  int i = threadIdx.x;
  if (i >= n) return;
  uint32_t h = h2_as_u32(__floats2half2_rn(x[i], x[i]));
  lo[i] = add_lo_f16(0.f, h);
  hi[i] = add_hi_f16(0.f, h);
  cvt[i] = __low2float(u32_as_h2(h));
}
int main() {
  const int n = 5;
  float hx[n] = {1e-3f, 6.1035156e-05f, 3.0517578e-05f, 1e-6f, 5.9604645e-08f};
  float *dx, *a, *b, *c, ha[n], hb[n], hc[n];
  cudaMalloc(&dx, n * 4); cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4);
  cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dx, a, b, c, n);
  cudaMemcpy(ha, a, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, b, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, c, n * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("x=%.6e  half->f32=%.6e  FHADD lo=%.6e hi=%.6e\n", hx[i], hc[i], ha[i], hb[i]);
  return 0;
}
