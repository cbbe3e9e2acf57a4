// pasa_kernels.cuh -- shared parameter blocks for the PASA B200 kernels.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstdint>

namespace pasa_b200 {

constexpr int kTile = 128;  // query tile rows (s1 on the device) and the KV block s2

// Key pre-pass: K'_j = K_j^T * M (reference pasa.cpp:53-56) in the kernel's
// K-major layout kp[(b, h, j*s2 + c), t] = K'_j[t][c], plus max|V| per (b, h).
struct KprepParams {
  int s2;              // KV block size (128 on the fast path)
  const uint16_t* k;   // (B, Hkv, S2, D) fp16
  const uint16_t* v;   // (B, Hkv, S2, D) fp16 (only read for vmax)
  uint16_t* kp;        // (B, Hkv, S2, D) fp16
  float* vmax;         // (B * Hkv) max |V|, zeroed by the launcher
  int S2;
  int D;
  float diag;          // fl16((1 - beta/s2)/alpha)     (pasa.cpp:26)
  float off;           // fl16(-beta/(alpha*s2))        (pasa.cpp:27)
  float lscale;        // 1 reproduces the reference; log2(e)/2 for the fused kernel
  int rank1;           // fused path: K' = (diag-off) K + off colsum (pasa_kprep_rank1_kernel)
  // input K / V element (b, h, s, t) at b in_bs + h in_hs + s in_ss + t (BHSD or BSHD; the
  // rank-1 kernels only -- the output K' is always BHSD, (b Hkv + h) S2 D + s D + t)
  int Hkv;
  long long in_bs, in_hs, in_ss;
};

// element strides (batch, head, seq) of a (B, H, S, D) tensor stored BHSD (layout 0) or BSHD
struct Strides3 {
  long long bs, hs, ss;
};
__host__ __device__ inline Strides3 layout_strides(int layout, int H, int S, int D) {
  return layout == 1 ? Strides3{static_cast<long long>(S) * H * D, D, static_cast<long long>(H) * D}
                     : Strides3{static_cast<long long>(H) * S * D, static_cast<long long>(S) * D, D};
}

// O-bounding exponent c0 >= 0: the smallest integer with
// S2 * max|V| <= 2^14 * 2^c0, computed identically on host and device.  The
// pre-pass scales V by the exact power of two 2^-c0, so T = P V and the FP16 O
// stay below 2^14 while P keeps its full (0, 1] range (no subnormal P).
// A head whose V holds an infinity (vmax = inf) gets c0 = 0: its output is non-finite
// whatever the scale, and V' = V keeps the other values intact.
__host__ __device__ inline int pasa_inflation(int S2, float vmax) {
  const float need = static_cast<float>(S2) * vmax * (1.0f / 16384.0f);
  if (!(need > 1.0f) || !(need < 3.0e38f)) return 0;
  const int e = ilogbf(need);  // floor(log2 need), exact
  return ldexpf(1.0f, e) == need ? e : e + 1;
}

// Programmatic dependent launch for the kernels that follow another of the path's kernels
// in a stream (V scale after the K' pre-pass, the forward after the pre-pass): their launch
// and prologue overlap the previous kernel's tail.  PASA_B200_NO_PDL=1 turns it off.
inline bool pdl_enabled() {
  static const bool on = std::getenv("PASA_B200_NO_PDL") == nullptr;
  return on;
}

// SM count of the CURRENT device (grid sizing), cached per device ordinal.
inline int current_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    return 148;
  if (dev < 64) cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// V' = V * 2^-c0 per (b, kv head), written by the pre-pass for the fused kernel.
struct VscaleParams {
  const uint16_t* v;   // (B, Hkv, S2, D) fp16, BHSD or BSHD (in_*: element strides)
  uint16_t* vp;        // (B, Hkv, S2, D) fp16, BHSD
  const float* vmax;   // (B * Hkv)
  long long per_head;  // S2 * D
  long long total;     // B * Hkv * S2 * D
  int S2;
  int D, Hkv;
  long long in_bs, in_hs, in_ss;
};

// Fused forward.  PASA mode: scores live in the log2 domain (K' carries log2 e).
// FA16 mode (beta == 0, pasa.cpp:212-221 -> attention.cpp:92-180): raw K, the
// 1/alpha scale is applied after the FP16 store, FP16 running max, no
// pseudo-average shift and no O inflation -- the naive FP16 FlashAttention.
enum FwdMode : int { kModePasa = 0, kModeFa16 = 1 };
// PASA mode, head dims with free TMEM columns (S' 128 + T D <= 240 of a tile's 256):
// the S' row sums come from the tensor core -- the pseudo-average GEMM G = Q K'sum_j
// (M = 128, N = 16, FP32 accumulator) against the block sums of K' (pasa_ksum_kernel)
// -- instead of 64 FP32 adds per thread and block.  At D = 128 all 512 columns are in use
// and the sums stay on the CUDA cores.
__host__ __device__ constexpr bool pasa_tc_rowsum(int D) { return 128 + D + 16 <= 256; }
struct FwdParams {
  int B, Hq, Hkv, S1, S2;
  int S2_bound;           // key count the pre-pass's O bound c0 was computed for (>= S2 when a
                          // launch covers a prefix of the keys, e.g. the host pipeline's pieces)
  int nq, nkv, group;     // ceil(S1/128), S2/s2, Hq/Hkv
  int qoff;               // causal: S2 - S1, the bottom-right alignment offset (any value)
  int s2;                 // KV block (shifting-matrix size), <= 128; < 128 masks columns
  float inv_s2;           // fl32(1/s2): the block mean S'bar = sum * inv_s2
  int q_bshd;             // Q and O stored BSHD (TMA coordinates, output address)
  int kv_bshd;            // the K / V operands stored BSHD (FA16 mode's raw K, V)
  int tiles_per_kv;       // group * (tile_hi - tile_lo): the query tiles computed per kv head
  int tile_hi;            // one past the last query tile computed (nq; less for a tile range,
                          // pasa_b200_attention_fwd_tiles: a query-row shard of the problem)
  float inva;             // beta / (1 - beta)       (pasa.cpp:85)
  float qk_scale;         // FA16 mode only: log2(e) / alpha applied after the FP16 store
  const float* vmax;      // per (b, kv head), from the pre-pass (PASA mode: V is pre-scaled)
  // (O: stored by TMA through the kernel's tm_o map, Q's shape and layout)
  void* diag;             // optional device pasa_b200_diag (RunDiagnostics); nullptr = off
  float diag_scale;       // stored score -> reference units (PASA: 2/log2(e); FA16: 1)
  long long* trace;       // PASA_TRACE builds only: clock64 timeline (see pasa_fwd.cu)
  float* gsum;            // D = 128 PASA: per-SM scratch of the prologue's S' row sums,
                          // [smid][tile][block][row] FP32 (gslots x 2 x nkv x 128)
  int gslots;             // SM-id slots in gsum (>= %nsmid of the device)
  int ks_rows;            // rows of the K'-sum TMA box (d = 64: 2 = hi, lo of one block;
                          // d = 128: blocks per prologue chunk, min(nkv, 128), per hi/lo box)
};
// D = 128 PASA, PASA_PRO_SUM=1 builds: the prologue pseudo-average (pasa_fwd.cu, kProSum);
// D = 64 uses the per-block tensor-core row sum (pasa_tc_rowsum).  Both need the K' block
// sums (pasa_ksum_kernel).  Defined here so the launcher and the kernel always agree.
#ifndef PASA_PRO_SUM
#define PASA_PRO_SUM 0
#endif
__host__ __device__ constexpr bool pasa_prologue_rowsum(int D) {
  return PASA_PRO_SUM != 0 && !pasa_tc_rowsum(D);
}

// Packed short-sequence forward (pasa_fwd_packed.cu): B*H sequences of N <= 64 rows, each
// a single KV block (S1 = S2 = s2 = N), in 16-aligned slots of W = 16 ceil(N/16) rows,
// P = 128 / W per 128-row tile; Q, K' (or K), V' (or V) and O are flat [B H N, d] rows.
struct PackedParams {
  int BH, N, W, P;
  float qk_scale;         // FA16 mode: log2(e) / alpha
  const float* vmax;      // PASA, prepped inputs: per sequence, from the pre-pass (V' = V 2^-c0)
  // (O: stored by TMA through the kernel's tm_o map)
  // PASA, self_prep = 1: the kernel reads raw K and V and runs the pre-pass per tile in shared
  // memory -- K' = fl16(fl32(fma(dm, K, fl32(off colsum))) lscale) (pasa_kprep_rank1_small
  // _kernel's arithmetic), max|V| and V' = V 2^-c0 per sequence (pasa_vscale_kernel's)
  int self_prep;
  float dm, off, lscale;  // diag - off, off (FP16 values), log2(e) / 2
  long long* trace;       // PASA_TRACE builds: clock64 timeline of CTA 0 (pasa_fwd_packed.cu)
};

// Device generators (pasa_gen.cu; bench.cpp:28-56, rng.hpp).
struct GenParams {
  int kind;            // 0 = uniform(x0 +- am), 1 = hybrid normal + Bernoulli(p) outlier
  double x0, am, p;
  uint64_t seed, tensor_id, start, n;  // flat indices [start, start + n) of tensor `tensor_id`
};
struct ResonanceParams {
  uint64_t seed;
  int tensor_id, B, H, S, d;
  double qa, ka;
};

}  // namespace pasa_b200
