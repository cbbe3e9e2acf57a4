// tests/cuda/umma_probe.cu -- TEST-ONLY probe of the tcgen05 building blocks
// the fused kernel uses (TMA 128B-swizzle tiles, SS UMMA with K-major A/B,
// TS UMMA with P in TMEM and MN-major V, F16/F32 TMEM accumulators, TMEM
// ld/st).  One CTA, one 128-row tile; results are checked against torch in
// tests/test_gpu_kernels.py.  Not part of the product library.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../paper_2503_01873_b200/csrc/sm100.cuh"

using namespace pasa_b200::sm100;

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int tmap_2d(CUtensorMap* m, const void* base, int d, int rows) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess)
    return -1;
  auto enc = reinterpret_cast<EncodeFn>(p);
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)d * 2 * rows};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : -2;
}

// mode 0: out[128 x 128] = A[128 x D] * B[128 x D]^T   (SS, K-major both)
// mode 1: out[128 x D]   = P[128 x 128] * V[128 x D]   (TS, P staged to TMEM, V MN-major)
template <int D>
__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ CUtensorMap ta,
                                                    const __grid_constant__ CUtensorMap tb,
                                                    const __half* P, float* out, int mode,
                                                    int f32acc) {
  constexpr int TILE = 128 * D * 2;
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * TILE);
  uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = warp_id(), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const int ncols = (mode == 0) ? 128 : D;
  if (mode == 1) {
    // stage P (row = thread) packed two halves per column at TMEM cols [0, 64)
    const __half* prow = P + threadIdx.x * 128;
    for (int c = 0; c < 4; ++c) {
      uint32_t r[16];
      for (int k = 0; k < 16; ++k)
        r[k] = h2_as_u32(__halves2half2(prow[(c * 16 + k) * 2], prow[(c * 16 + k) * 2 + 1]));
      tmem_st_16cols_b32(tbase + lane_off + c * 16, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && elect_one()) {
    const int nbox = D / 64;
    if (mode == 0) {
      mbar_expect_tx(&bars[0], 2 * TILE);
      for (int bx = 0; bx < nbox; ++bx) {
        tma_load_3d(smem + bx * 16384, &ta, &bars[0], bx * 64, 0, 0);
        tma_load_3d(smem + TILE + bx * 16384, &tb, &bars[0], bx * 64, 0, 0);
      }
    } else {
      mbar_expect_tx(&bars[0], TILE);
      for (int bx = 0; bx < nbox; ++bx) tma_load_3d(smem + TILE + bx * 16384, &tb, &bars[0], bx * 64, 0, 0);
    }
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint32_t d_tmem = tbase + 128;
    if (mode == 0) {
      const uint32_t id = idesc_f16(128, 128, f32acc, 0, 0);
      const uint32_t aa = smem_u32(smem), ba = smem_u32(smem + TILE);
      for (int s = 0; s < D / 16; ++s) {
        const uint32_t off = (s / 4) * 16384 + (s % 4) * 32;
        umma_ss(d_tmem, smem_desc_sw128(aa + off, 16, 1024), smem_desc_sw128(ba + off, 16, 1024), id, s > 0);
      }
    } else {
      const uint32_t id = idesc_f16(128, D, f32acc, 0, 1);
      const uint32_t va = smem_u32(smem + TILE);
      for (int s = 0; s < 8; ++s)
        umma_ts(d_tmem, tbase + s * 8, smem_desc_sw128(va + s * 2048, 16384, 1024), id, s > 0);
    }
    tc_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  float* orow = out + (warp * 32 + lane) * ncols;
  for (int c = 0; c < ncols; c += 32) {
    uint32_t r[16];
    if (f32acc) {
      tmem_ld_16cols_b32(tbase + lane_off + 128 + c, r);
      tmem_wait_ld();
      for (int k = 0; k < 16; ++k) orow[c + k] = __uint_as_float(r[k]);
      tmem_ld_16cols_b32(tbase + lane_off + 128 + c + 16, r);
      tmem_wait_ld();
      for (int k = 0; k < 16; ++k) orow[c + 16 + k] = __uint_as_float(r[k]);
    } else {
      tmem_ld_32cols_pack16(tbase + lane_off + 128 + c, r);
      tmem_wait_ld();
      for (int k = 0; k < 16; ++k) {
        orow[c + 2 * k] = __low2float(u32_as_h2(r[k]));
        orow[c + 2 * k + 1] = __high2float(u32_as_h2(r[k]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int probe_umma(const void* a, const void* b,
                                                                  const void* p, float* out,
                                                                  int D, int mode, int f32acc) {
  CUtensorMap ta, tb;
  if (mode == 0 && tmap_2d(&ta, a, D, 128)) return -1;
  if (tmap_2d(&tb, b, D, 128)) return -1;
  if (mode == 1) ta = tb;
  const int smem = 2 * 128 * D * 2 + 1024 + 64;
  cudaError_t e;
  if (D == 128) {
    cudaFuncSetAttribute(probe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<128><<<1, 128, smem>>>(ta, tb, static_cast<const __half*>(p), out, mode, f32acc);
  } else {
    cudaFuncSetAttribute(probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<64><<<1, 128, smem>>>(ta, tb, static_cast<const __half*>(p), out, mode, f32acc);
  }
  e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : -3;
}
