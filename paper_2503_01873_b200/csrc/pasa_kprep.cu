// pasa_kprep.cu -- the key pre-pass K'_j = K_j^T * M (reference pasa.cpp:53-56,
// driven per (b, h, j) by pasa.cpp:231-240) and max|V| per (b, kv head).
//
// Bit-exact with the reference's FP32 sequential GEMM (matrix.cpp:26-74 with
// RoundFp32): for every (t, c) the reference runs acc = fl32(acc + K[p][t] *
// M[p][c]) for p = 0..s2-1 and rounds once to FP16.  K and M are FP16 values,
// so each product is exact in FP32 and one FFMA per step reproduces it.  M
// has only two distinct entries, so the chains for all columns c share the
// prefix p < c (all `off`); a thread owns one head-dim index t and four groups
// of eight columns, carries the shared prefix upwards and runs each group's
// eight chains in lock-step from there -- half the FMAs of the dense product,
// eight-way ILP, identical bits.
//
// The K block is staged in shared memory transposed (t-major, p contiguous,
// rows padded by 16 B) so a thread reads eight consecutive p with one
// conflict-free 16-byte load.
#include <cuda_fp16.h>

#include "pasa_kernels.cuh"
#include "sm100.cuh"

namespace pasa_b200 {

template <int D>
__global__ void __launch_bounds__(D * 4) pasa_kprep_kernel(const KprepParams p) {
  constexpr int S2 = kTile;
  constexpr int ROW = S2 + 8;  // halves per transposed row (16 B pad: conflict-free 16 B loads)
  __shared__ __align__(16) __half kt[D * ROW];
  __shared__ float red[D * 4 / 32];

  const int j = blockIdx.y;    // KV block
  const int bh = blockIdx.x;   // b * Hkv + h (x: up to 2^31 - 1 kv heads)
  const int t = threadIdx.x;   // head-dim index owned by this thread
  const int y = threadIdx.y;   // column-group slot 0..3
  const int tid = y * D + t;
  const size_t base = (static_cast<size_t>(bh) * p.S2 + static_cast<size_t>(j) * S2) * D;
  const __half* kg = reinterpret_cast<const __half*>(p.k) + base;

  // Stage K_j transposed: kt[t][p] = K[p][t].
  for (int e = tid * 8; e < S2 * D; e += D * 4 * 8) {
    const uint4 w = *reinterpret_cast<const uint4*>(kg + e);
    const __half* h = reinterpret_cast<const __half*>(&w);
    const int pr = e / D, tc = e % D;
#pragma unroll
    for (int k = 0; k < 8; ++k) kt[(tc + k) * ROW + pr] = h[k];
  }
  // max |V| over this block (same element range as K).
  {
    const __half* vg = reinterpret_cast<const __half*>(p.v) + base;
    float vm = 0.f;
    for (int e = tid * 8; e < S2 * D; e += D * 4 * 8) {
      const uint4 w = *reinterpret_cast<const uint4*>(vg + e);
      const __half* h = reinterpret_cast<const __half*>(&w);
#pragma unroll
      for (int k = 0; k < 8; ++k) vm = fmaxf(vm, fabsf(__half2float(h[k])));  // NaN ignored
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
    if ((tid & 31) == 0) red[tid / 32] = vm;
  }
  __syncthreads();
  if (tid == 0) {
    float vm = 0.f;
    for (int w = 0; w < D * 4 / 32; ++w) vm = fmaxf(vm, red[w]);
    atomicMax(reinterpret_cast<int*>(p.vmax) + bh, __float_as_int(vm));  // vm >= 0
  }

  // Thread (t, y) owns the 8-column groups {y, 7-y, 8+y, 15-y} (equal work per
  // slot, increasing order).  Column c's chain is prefix(c) (all `off`), then
  // `diag` at p = c, then `off` to the end; the eight chains of a group walk the
  // same p together, so one K value feeds eight independent FFMAs.
  const __half* col = kt + t * ROW;
  __half* out = reinterpret_cast<__half*>(p.kp) + base + t;
  const float diag = p.diag, off = p.off, L = p.lscale;
  const int groups[4] = {y, 7 - y, 8 + y, 15 - y};
  float prefix = 0.f;
  int pdone = 0;
#pragma unroll 1
  for (int gi = 0; gi < 4; ++gi) {
    const int c0 = 8 * groups[gi];
    for (int q = pdone; q < c0; ++q) prefix = __fmaf_rn(__half2float(col[q]), off, prefix);
    pdone = c0;
    float acc[8];
    {
      // p = c0 .. c0+7: column c0+cc takes `diag` at p == c0+cc
      const uint4 w = *reinterpret_cast<const uint4*>(col + c0);
      const __half* h = reinterpret_cast<const __half*>(&w);
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) acc[cc] = prefix;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float kv = __half2float(h[k]);
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) acc[cc] = __fmaf_rn(kv, k == cc ? diag : off, acc[cc]);
      }
    }
#pragma unroll 2
    for (int q = c0 + 8; q < S2; q += 8) {
      const uint4 w = *reinterpret_cast<const uint4*>(col + q);
      const __half* h = reinterpret_cast<const __half*>(&w);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float kv = __half2float(h[k]);
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) acc[cc] = __fmaf_rn(kv, off, acc[cc]);
      }
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      float a = acc[cc];
      if (L != 1.0f) a = __fmul_rn(a, L);
      out[static_cast<size_t>(c0 + cc) * D] = __float2half_rn(a);
    }
  }
}

// The fused path's pre-pass (lscale != 1, no bit-parity with the reference's
// chains required): M = (diag - off) I + off J is a rank-1 update of a scaled
// identity, so K'_j[t][c] = (diag - off) K[c][t] + off * colsum_j[t] -- one FMA
// per element after an FP32 column sum, three FP32 roundings instead of the
// chain's 128, and a memory-bound kernel (the chain kernel above is kept for the
// bit-exact reference pre-pass, lscale = 1).  Also reduces max|V| per head.
//   colsum = sum_p K[p][t] (FP32, p ascending); os = fl32(off * colsum);
//   K' = fl16(fl32(fma(diag - off, K[c][t], os)) * lscale)
// restated in oracle/pasa_oracle.c (orc_preprocess_keys, p_acc = PR1).
template <int D>
__global__ void __launch_bounds__(256) pasa_kprep_rank1_kernel(const KprepParams p) {
  constexpr int S2 = kTile, NT = 256;
  __shared__ __align__(16) __half kb[S2 * D];
  __shared__ float os[D];
  __shared__ float red[NT / 32];
  const int j = blockIdx.y, bh = blockIdx.x, tid = threadIdx.x;
  sm100::pdl_trigger();  // the V scale may launch now (it waits for this grid before reading)
  const size_t base = (static_cast<size_t>(bh) * p.S2 + static_cast<size_t>(j) * S2) * D;
  // the input block: rows j S2 .. j S2 + S2 - 1 of head (b, h), row stride in_ss
  const long long ibase = (bh / p.Hkv) * p.in_bs + (bh % p.Hkv) * p.in_hs +
                          static_cast<long long>(j) * S2 * p.in_ss;
  const __half* kin0 = reinterpret_cast<const __half*>(p.k) + ibase;
  const __half* vin0 = reinterpret_cast<const __half*>(p.v) + ibase;
  float vm = 0.f;
#pragma unroll 4
  for (int e = tid; e < S2 * D / 8; e += NT) {
    const long long off = (e / (D / 8)) * p.in_ss + (e % (D / 8)) * 8;
    reinterpret_cast<uint4*>(kb)[e] = *reinterpret_cast<const uint4*>(kin0 + off);
    const uint4 w = *reinterpret_cast<const uint4*>(vin0 + off);
    const __half2* h = reinterpret_cast<const __half2*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(__habs2(h[k]));
      vm = fmaxf(vm, fmaxf(f.x, f.y));  // NaN ignored
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
  if ((tid & 31) == 0) red[tid / 32] = vm;
  __syncthreads();
  if (tid < D) {
    float cs = 0.f;
    for (int r = 0; r < S2; ++r) cs = __fadd_rn(cs, __half2float(kb[r * D + tid]));
    os[tid] = __fmul_rn(p.off, cs);
  }
  if (tid == 0) {
    float m = 0.f;
    for (int w = 0; w < NT / 32; ++w) m = fmaxf(m, red[w]);
    atomicMax(reinterpret_cast<int*>(p.vmax) + bh, __float_as_int(m));  // m >= 0
  }
  __syncthreads();
  const float dm = p.diag - p.off;  // exact: both are FP16 values
  __half2* out = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(p.kp) + base);
  const __half2* kin = reinterpret_cast<const __half2*>(kb);
#pragma unroll 4
  for (int e = tid; e < S2 * D / 2; e += NT) {
    const int t = (2 * e) % D;
    const float2 kv = __half22float2(kin[e]);
    const float a = __fmul_rn(__fmaf_rn(dm, kv.x, os[t]), p.lscale);
    const float b = __fmul_rn(__fmaf_rn(dm, kv.y, os[t + 1]), p.lscale);
    out[e] = __floats2half2_rn(a, b);
  }
}

// The same chains for a KV block of s2 < 128 keys (ragged / short sequences,
// e.g. temporal attention with S2 = 25): one thread per head-dim index, the
// block read straight from global memory (L1-resident), no column groups.
__global__ void __launch_bounds__(128) pasa_kprep_small_kernel(const KprepParams p) {
  const int j = blockIdx.y, bh = blockIdx.x, t = threadIdx.x, s2 = p.s2, D = p.D;
  const size_t base = (static_cast<size_t>(bh) * p.S2 + static_cast<size_t>(j) * s2) * D;
  const __half* kg = reinterpret_cast<const __half*>(p.k) + base;
  __half* out = reinterpret_cast<__half*>(p.kp) + base;
  __shared__ float red[4];
  float vm = 0.f;
  if (p.v) {
    const __half* vg = reinterpret_cast<const __half*>(p.v) + base;
    for (int e = t; e < s2 * D; e += blockDim.x) vm = fmaxf(vm, fabsf(__half2float(vg[e])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
  if ((t & 31) == 0) red[t / 32] = vm;
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < blockDim.x / 32; ++w) vm = fmaxf(vm, red[w]);
    atomicMax(reinterpret_cast<int*>(p.vmax) + bh, __float_as_int(vm));
  }
  if (t >= D) return;
  float prefix = 0.f;
  for (int c = 0; c < s2; ++c) {
    const float kc = __half2float(kg[c * D + t]);
    float acc = __fmaf_rn(kc, p.diag, prefix);
    for (int q = c + 1; q < s2; ++q) acc = __fmaf_rn(__half2float(kg[q * D + t]), p.off, acc);
    if (p.lscale != 1.0f) acc = __fmul_rn(acc, p.lscale);
    out[c * D + t] = __float2half_rn(acc);
    prefix = __fmaf_rn(kc, p.off, prefix);
  }
}

// The rank-1 pre-pass for KV blocks of s2 < 128 keys (ragged blocks, short sequences such
// as the temporal attention's N = 25): one warp per block, each lane owns D/64 head-dim
// pairs; FP32 column sums over the s2 keys ascending, then one FMA per element -- the same
// arithmetic as pasa_kprep_rank1_kernel (orc_preprocess_keys, p_acc = PR1) -- and max|V|.
template <int D, int MAXR>
__global__ void __launch_bounds__(256) pasa_kprep_rank1_small_kernel(const KprepParams p,
                                                                      int nblk_total) {
  constexpr int U = D / 64;  // half2 columns per lane
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int blk = blockIdx.x * 8 + warp;
  if (blk >= nblk_total) return;
  const int nkv = p.S2 / p.s2, s2 = p.s2;
  const int bh = blk / nkv, j = blk % nkv;
  const size_t base = (static_cast<size_t>(bh) * p.S2 + static_cast<size_t>(j) * s2) * D;
  const long long ibase = (bh / p.Hkv) * p.in_bs + (bh % p.Hkv) * p.in_hs +
                          static_cast<long long>(j) * s2 * p.in_ss;
  // input rows (strided by in_ss), as half2: row c at kg + c * RS2
  const __half2* kg = reinterpret_cast<const __half2*>(reinterpret_cast<const __half*>(p.k) + ibase);
  const __half2* vg = reinterpret_cast<const __half2*>(reinterpret_cast<const __half*>(p.v) + ibase);
  const long long RS2 = p.in_ss / 2;
  float2 cs[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cs[u] = make_float2(0.f, 0.f);
  float vm = 0.f;
  if (MAXR > 0 && s2 <= MAXR) {
    // short blocks (e.g. the SVD temporal N = 25): every row's K and V loads are issued
    // before the first is used (the row loop below waits a memory latency per row), and the
    // K values stay in registers for the output pass; same sums in the same order.
    __half2 kr[MAXR > 0 ? MAXR : 1][U], vr[MAXR > 0 ? MAXR : 1][U];
#pragma unroll
    for (int c = 0; c < MAXR; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        kr[c][u] = c < s2 ? kg[c * RS2 + lane + 32 * u] : __half2{};
        vr[c][u] = c < s2 ? vg[c * RS2 + lane + 32 * u] : __half2{};
      }
#pragma unroll
    for (int c = 0; c < MAXR; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c < s2) {
          const float2 k2 = __half22float2(kr[c][u]);
          cs[u].x = __fadd_rn(cs[u].x, k2.x);
          cs[u].y = __fadd_rn(cs[u].y, k2.y);
        }
        const float2 v2 = __half22float2(__habs2(vr[c][u]));  // padded rows are 0
        vm = fmaxf(vm, fmaxf(v2.x, v2.y));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
    if (lane == 0) atomicMax(reinterpret_cast<int*>(p.vmax) + bh, __float_as_int(vm));  // vm >= 0
    const float dm = p.diag - p.off;
    float2 os[U];
#pragma unroll
    for (int u = 0; u < U; ++u) os[u] = make_float2(__fmul_rn(p.off, cs[u].x), __fmul_rn(p.off, cs[u].y));
    __half2* out = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(p.kp) + base);
#pragma unroll
    for (int c = 0; c < MAXR; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c < s2) {
          const float2 k2 = __half22float2(kr[c][u]);
          const float a = __fmul_rn(__fmaf_rn(dm, k2.x, os[u].x), p.lscale);
          const float b = __fmul_rn(__fmaf_rn(dm, k2.y, os[u].y), p.lscale);
          out[c * (D / 2) + lane + 32 * u] = __floats2half2_rn(a, b);
        }
    return;
  }
  for (int c = 0; c < s2; ++c) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float2 k2 = __half22float2(kg[c * RS2 + lane + 32 * u]);
      cs[u].x = __fadd_rn(cs[u].x, k2.x);
      cs[u].y = __fadd_rn(cs[u].y, k2.y);
      const float2 v2 = __half22float2(__habs2(vg[c * RS2 + lane + 32 * u]));
      vm = fmaxf(vm, fmaxf(v2.x, v2.y));  // NaN ignored
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
  if (lane == 0) atomicMax(reinterpret_cast<int*>(p.vmax) + bh, __float_as_int(vm));  // vm >= 0
  const float dm = p.diag - p.off;  // exact: both are FP16 values
  float2 os[U];
#pragma unroll
  for (int u = 0; u < U; ++u) os[u] = make_float2(__fmul_rn(p.off, cs[u].x), __fmul_rn(p.off, cs[u].y));
  __half2* out = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(p.kp) + base);
  for (int c = 0; c < s2; ++c) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float2 k2 = __half22float2(kg[c * RS2 + lane + 32 * u]);
      const float a = __fmul_rn(__fmaf_rn(dm, k2.x, os[u].x), p.lscale);
      const float b = __fmul_rn(__fmaf_rn(dm, k2.y, os[u].y), p.lscale);
      out[c * (D / 2) + lane + 32 * u] = __floats2half2_rn(a, b);
    }
  }
}

// V' = V * 2^-c0 (exact power-of-two scaling; RNE only where V' is subnormal).  Grid
// (B Hkv, row chunks): c0 once per block, 32-bit index math within a head (a 64-bit
// division per 16 bytes held the old grid-stride form to 2.7 TB/s), four 16-byte loads
// in flight per thread before the stores.
template <int D>
__global__ void __launch_bounds__(256) pasa_vscale_kernel(const VscaleParams p) {
  constexpr int C8 = D / 8, U = 4, NT = 256;  // 16-byte words per row, per thread, threads
  const int bh = blockIdx.x;
  sm100::pdl_trigger();  // the forward may launch now (it waits for this grid before reading)
  sm100::pdl_wait();     // max|V| comes from the pre-pass grid
  const int c0 = pasa_inflation(p.S2, p.vmax[bh]);
  const __half2 sc = __half2half2(__float2half_rn(ldexpf(1.0f, -c0)));
  const int n8 = p.S2 * C8;  // 16-byte words per head
  const __half* vin = reinterpret_cast<const __half*>(p.v) + (bh / p.Hkv) * p.in_bs +
                      (bh % p.Hkv) * p.in_hs;
  uint4* out = reinterpret_cast<uint4*>(p.vp) + static_cast<size_t>(bh) * n8;
  for (int base = blockIdx.y * NT * U; base < n8; base += gridDim.y * NT * U) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * NT + threadIdx.x;
      if (i < n8)
        w[u] = *reinterpret_cast<const uint4*>(vin + static_cast<long long>(i / C8) * p.in_ss +
                                               (i % C8) * 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * NT + threadIdx.x;
      if (i < n8) {
        __half2* h = reinterpret_cast<__half2*>(&w[u]);
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __hmul2(h[k], sc);
        out[i] = w[u];
      }
    }
  }
}

// Short heads (fewer than 1024 16-byte words, e.g. the SVD temporal N = 25 with 46080
// heads): one block per head would leave most threads idle and make block scheduling the
// cost, so the words of all heads are walked flat, head = word / words-per-head.
template <int D>
__global__ void __launch_bounds__(256) pasa_vscale_flat_kernel(const VscaleParams p, int n8,
                                                               int total8) {
  constexpr int C8 = D / 8;
  sm100::pdl_trigger();
  sm100::pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total8; i += gridDim.x * blockDim.x) {
    const int bh = i / n8, r = i - bh * n8;
    const int c0 = pasa_inflation(p.S2, p.vmax[bh]);
    const __half2 sc = __half2half2(__float2half_rn(ldexpf(1.0f, -c0)));
    const __half* vin = reinterpret_cast<const __half*>(p.v) + (bh / p.Hkv) * p.in_bs +
                        (bh % p.Hkv) * p.in_hs + static_cast<long long>(r / C8) * p.in_ss +
                        (r % C8) * 8;
    uint4 w = *reinterpret_cast<const uint4*>(vin);
    __half2* h = reinterpret_cast<__half2*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __hmul2(h[k], sc);
    reinterpret_cast<uint4*>(p.vp)[i] = w;
  }
}

cudaError_t launch_vscale(const VscaleParams& p, cudaStream_t stream) {
  const long long bh = p.total / p.per_head;
  const long long chunks = (p.per_head / 8 + 1023) / 1024;
  const bool flat = p.per_head / 8 < 1024 && p.total / 8 < (1LL << 31);
  dim3 grid(static_cast<unsigned>(bh), static_cast<unsigned>(chunks < 65535 ? chunks : 65535));
  if (flat) {
    const int sms = current_sm_count();  // the launching (current) device
    const long long blocks = (p.total / 8 + 255) / 256;
    grid = dim3(static_cast<unsigned>(blocks < 16LL * sms ? blocks : 16LL * sms));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const int n8 = static_cast<int>(p.per_head / 8), total8 = static_cast<int>(p.total / 8);
  if (flat && p.D == 128) return cudaLaunchKernelEx(&cfg, pasa_vscale_flat_kernel<128>, p, n8, total8);
  if (flat && p.D == 64) return cudaLaunchKernelEx(&cfg, pasa_vscale_flat_kernel<64>, p, n8, total8);
  if (p.D == 128) return cudaLaunchKernelEx(&cfg, pasa_vscale_kernel<128>, p);
  if (p.D == 64) return cudaLaunchKernelEx(&cfg, pasa_vscale_kernel<64>, p);
  return cudaErrorInvalidValue;
}

cudaError_t launch_kprep(const KprepParams& p, int B, int Hkv, cudaStream_t stream) {
  if (p.s2 != kTile && p.rank1 && p.v && (p.D == 64 || p.D == 128)) {
    const int total = (p.S2 / p.s2) * B * Hkv;
    const int grid = (total + 7) / 8;
    if (p.D == 64) {
      if (p.s2 <= 32) pasa_kprep_rank1_small_kernel<64, 32><<<grid, 256, 0, stream>>>(p, total);
      else pasa_kprep_rank1_small_kernel<64, 0><<<grid, 256, 0, stream>>>(p, total);
    } else {
      if (p.s2 <= 32) pasa_kprep_rank1_small_kernel<128, 32><<<grid, 256, 0, stream>>>(p, total);
      else pasa_kprep_rank1_small_kernel<128, 0><<<grid, 256, 0, stream>>>(p, total);
    }
    return cudaGetLastError();
  }
  if (p.s2 != kTile) {
    pasa_kprep_small_kernel<<<dim3(B * Hkv, p.S2 / p.s2), 128, 0, stream>>>(p);
    return cudaGetLastError();
  }
  dim3 grid(B * Hkv, p.S2 / kTile);  // kv heads on x (no 65535 limit)
  if (p.rank1) {  // the fused path's pre-pass: rank-1 form, memory-bound
    if (p.D == 128) pasa_kprep_rank1_kernel<128><<<grid, 256, 0, stream>>>(p);
    else if (p.D == 64) pasa_kprep_rank1_kernel<64><<<grid, 256, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
  }
  if (p.D == 128) {
    pasa_kprep_kernel<128><<<grid, dim3(128, 4), 0, stream>>>(p);
  } else if (p.D == 64) {
    pasa_kprep_kernel<64><<<grid, dim3(64, 4), 0, stream>>>(p);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Block sums of K' for the fused kernel's pseudo-average GEMM:
// ks[(bh, 2j + r), t], r = 0: hi = fl16(sum_c K'_j[c][t]), r = 1: lo = fl16(sum - hi),
// the FP32 sum over the block's s2 keys.  One thread per head-dim index t.
__global__ void pasa_ksum_kernel(const uint16_t* __restrict__ kp, uint16_t* __restrict__ ks,
                                 int S2, int s2, int D) {
  const int j = blockIdx.y, bh = blockIdx.x, t = threadIdx.x;
  const __half* src = reinterpret_cast<const __half*>(kp) +
                      (static_cast<size_t>(bh) * S2 + static_cast<size_t>(j) * s2) * D + t;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int c = 0;
  for (; c + 4 <= s2; c += 4)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] += __half2float(src[static_cast<size_t>(c + u) * D]);
  for (; c < s2; ++c) acc[0] += __half2float(src[static_cast<size_t>(c) * D]);
  const float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  const __half hi = __float2half_rn(sum);
  const __half lo = __float2half_rn(sum - __half2float(hi));
  __half* dst = reinterpret_cast<__half*>(ks) + (static_cast<size_t>(bh) * 2 * (S2 / s2) + 2 * j) * D + t;
  dst[0] = hi;
  dst[D] = lo;
}

cudaError_t launch_ksum(const void* kp, void* ks, int BH, int S2, int s2, int D, cudaStream_t stream) {
  pasa_ksum_kernel<<<dim3(BH, S2 / s2), D, 0, stream>>>(static_cast<const uint16_t*>(kp),
                                                        static_cast<uint16_t*>(ks), S2, s2, D);
  return cudaGetLastError();
}

}  // namespace pasa_b200
