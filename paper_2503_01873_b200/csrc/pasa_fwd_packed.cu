// pasa_fwd_packed.cu -- PASA forward for short sequences (one KV block per sequence:
// S1 = S2 = s2 = N <= 64, e.g. the SVD temporal attention with N = 25 frames), packed
// in 16-aligned slots, 128 / (16 ceil(N / 16)) sequences to a 128-row tensor-core tile.
//
// With a single KV block the PASA recursion (pasa.cpp:117-194) collapses: j = 1, so
// F = S'bar, both corrections are zero and m = m' -- the output is the softmax of the
// shifted scores S' = fl16(Q K'^T) of the sequence, computed exactly like the fused
// kernel's first block (pasa_fwd.cu; numerics DESIGN.md section 4): P = fl16(2^(2 S' - 2 m'))
// (K' carries log2(e)/2), T = P V' with an F16 accumulator, O = T 2^c0 / l.  The
// pseudo-average drops out of the result and is not computed.  FA16 mode (beta = 0) is
// the naive FP16 FlashAttention's single block (attention.cpp:92-180).
//
// Layout: Q, K', V' (and O) are flat [B H N, d] row matrices.  Tile i holds sequences
// [i P, i P + P), sequence s of the tile in the 16-aligned slot of rows / keys
// [s W, s W + N), W = 16 ceil(N / 16), P = 128 / W (one TMA box of N rows per sequence;
// V' gaps are zero).  Each row attends only to the N keys of its own slot (block-diagonal
// mask within the 128 x 128 S').  Because every slot starts on a 16-key boundary, the
// tensor core's F16 accumulation chunks and the row-sum chains see a sequence exactly as
// the fused kernel does when the sequence is alone: the output is bit-identical to
// pasa_fwd.cu's, whatever the packing (host pipeline pieces, multi-GPU shards).
//
// Persistent CTAs walk the tiles with a two-stage TMA ring (Q / K and V of a stage arrive on
// separate barriers, so S' can run before V has landed); the kernel is instantiated per slot
// width WS.  Warpgroups: warp 0 loads, warp 1 issues the MMAs; warps 4-7 run the softmax with
// one thread per row (TMEM lane quadrant = warp % 4) and the epilogue, whose O tile is staged
// in the stage's consumed V' buffer and leaves by TMA; warps 8-11 and 12-15 (self_prep, the
// public entry point) run the key pre-pass and the V scale of the staged tiles in shared
// memory -- K' = rank-1 form of K^T M, V' = V 2^-c0 -- warpgroup g taking stage g, so the
// kernel reads raw K, V from HBM and no workspace round trip is needed.  TMEM: S'/P at +0,
// T at +128, T_clean at +128 + D (256 columns at d = 64, so two CTAs share an SM; 512 at
// d = 128).
//
// Non-finite V: the tile's P V' also multiplies each row's zero P entries by the other
// sequences' V' rows, and 0 x Inf = NaN would leak one sequence's Inf/NaN into its
// neighbours (the unpacked kernel keeps heads apart).  So the pre-pass (or, on prepped
// inputs, the MMA warp while S' runs) finds the slots with a non-finite V' row; for such a
// tile the MMA warp issues P V' twice -- into T (the poisoned sequences read it: exactly what
// they get alone) and, after zeroing the poisoned sequences' V' rows in shared memory, into
// T_clean (everyone else reads it).  A ragged last tile first zeroes its unused slots (they
// hold an earlier tile's staged O).  Clean tiles pay nothing extra.
#include <cuda.h>
#include <cuda_fp16.h>

#include "pasa_kernels.cuh"
#include "sm100.cuh"

namespace pasa_b200 {
using namespace sm100;

// PASA_TRACE builds: CTA 0 records clock64() at fixed points of its first 64 tiles,
// p.trace[(role * 64 + it) * 16 + event]: role 0 = softmax thread 128 (0 start, 1 S' ready,
// 2 P stored, 3 O stored, 4 T ready, 5 T read) and the prep (6 Q/K landed); role 1 = MMA
// issuer (0 S' issued, 1 P ready, 2 PV committed), TMA producer (3 Q/K issued, 4 V issued),
// prep (5 start, 6 done, 8 K' written, 9 V landed, 10 max|V| in, 11 c0 and mask written)
#ifdef PASA_TRACE
#define PK_TRP(tr, role, it, ev)                                                   \
  do {                                                                             \
    if ((tr) && blockIdx.x == 0 && (it) < 64) (tr)[((role) * 64 + (it)) * 16 + (ev)] = clock64(); \
  } while (0)
#define PK_TR(role, it, ev) PK_TRP(p.trace, role, it, ev)
#else
#define PK_TRP(tr, role, it, ev) \
  do {                           \
  } while (0)
#define PK_TR(role, it, ev) \
  do {                      \
  } while (0)
#endif

namespace {

template <int D, int WS>
struct PackedCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int BOX_BYTES = kTile * 128;
  static constexpr int TILE_BYTES = NBOX * BOX_BYTES;
  static constexpr int STAGE_BYTES = 3 * TILE_BYTES;  // Q, K', V' of one tile
  static constexpr int STAGES = 2;
  static constexpr int SMEM_BAR = STAGES * STAGE_BYTES;
  // qk_full, v_full, in_empty, kprep_done, vprep_done, qk_empty, o_free [ST]; s/p/t_full,
  // t_empty, aux, mask
  static constexpr int NUM_BARS = 7 * STAGES + 6;
  // after the barriers: TMEM holder, bad-slot masks [4], slot exponents c0 [4][8], each prep
  // warpgroup's per-slot max|V| bits and non-finite slots [2][16]
  static constexpr int SMEM_BYTES = SMEM_BAR + 8 * NUM_BARS + 4 * (1 + 4 + 32 + 32) + 1024;
  // softmax pairs per thread (NPR): W = 16, 32 -> 16 (the warp's 32 rows span whole slots);
  // W = 64 -> 32; W = 48 straddles warps -> all 64
  static constexpr int NPR = WS <= 32 ? 16 : WS == 64 ? 32 : 64;
  // prep warpgroups: two, alternating stages (tile it on stage it % 2 -> warpgroup it % 2), so
  // the per-tile pre-pass -- the latency-bound step -- has two tiles' time; one at d = 64,
  // W = 48, whose all-column softmax leaves no registers for a second
  static constexpr int NPREP = (D == 64 && WS == 48) ? 1 : 2;
  // warpgroup 0: warp 0 TMA, warp 1 MMA (2, 3 idle); 1: softmax (warps 4-7 = TMEM lane
  // quadrants 0-3); 2, 3: the per-tile pre-pass (self_prep)
  static constexpr int THREADS = 256 + 128 * NPREP;
  static constexpr int CTAS = D == 64 ? 2 : 1;  // per SM (shared memory: 2 x 98 KB / 194 KB)
  // setmaxnreg split of the launch allocation (65536 / (CTAS x THREADS) registers per thread)
  static constexpr int REGS_CTL = D == 64 ? 32 : 40, REGS_PREP = D == 64 ? (NPREP == 2 ? 40 : 56) : 64,
                       REGS_SM = D == 64 ? (NPR == 16 ? 88 : NPR == 32 ? 136 : 152) : 232;
  static constexpr int REGS_LAUNCH = (65536 / (CTAS * THREADS)) & ~7;
  static_assert(128 * (REGS_CTL + NPREP * REGS_PREP + REGS_SM) <= REGS_LAUNCH * THREADS, "registers");
  static constexpr uint32_t TMEM_COLS = D == 64 ? 256 : 512;
  static constexpr uint32_t T_CLEAN = 128 + D;  // P V' over zeroed poisoned rows
};

__device__ __forceinline__ float lo_f(uint32_t u) { return __low2float(u32_as_h2(u)); }
__device__ __forceinline__ float hi_f(uint32_t u) { return __high2float(u32_as_h2(u)); }

// keep lo / hi of the pair of columns (2i, 2i + 1) that fall in [lo, hi)
__device__ __forceinline__ uint32_t range_keep(int i, int lo, int hi) {
  const uint32_t a = (2 * i >= lo && 2 * i < hi) ? 0x0000FFFFu : 0u;
  const uint32_t b = (2 * i + 1 >= lo && 2 * i + 1 < hi) ? 0xFFFF0000u : 0u;
  return a | b;
}

// One thread per row: the softmax of the row's slot over the warp's NPR column pairs
// [c0 / 2, c0 / 2 + NPR), c0 = 2 NPR floor(32 quad / (2 NPR)), read from the S' columns and
// written back as P (zeros elsewhere in [0, 64), two keys per column).  Returns the FP32
// row sum l.  Masked pairs (outside the row's sequence [lo, hi)) are -inf for the max and 0
// in P, exactly as over the full row.
template <int NPR, int MODE>
__device__ __noinline__ float row_softmax(uint32_t t_s, int quad, int lo, int hi, float qk_scale) {
  const int pb = NPR >= 64 ? 0 : NPR * ((32 * quad) / (2 * NPR));  // first pair (= P column)
  uint32_t s[NPR];
#pragma unroll
  for (int c = 0; c < NPR / 16; ++c) tmem_ld_32cols_pack16(t_s + 2 * pb + 32 * c, s + 16 * c);
  tmem_wait_ld();
  uint32_t mx = 0xFC00FC00u;
#pragma unroll
  for (int k = 0; k < NPR; ++k) {
    const uint32_t keep = range_keep(pb + k, lo, hi);
    const uint32_t vm = (s[k] & keep) | (0xFC00FC00u & ~keep);
    mx = h2_as_u32(__hmax2(u32_as_h2(mx), u32_as_h2(vm)));
  }
  const float mloc = fmaxf(lo_f(mx), hi_f(mx));
  uint32_t cj2, scale2;
  if (MODE == kModePasa) {
    // j = 1: F = S'bar, both corrections 0, c = fl16(m'); x = fl16(2 S' - 2 c), or (a row
    // of the warp with |c| > 32752) 2 fl16(S' - c)
    const __half cj = __float2half_rn(mloc);
    const bool fast2 = __all_sync(0xFFFFFFFFu, __habs(cj) <= __float2half_rn(32752.f));
    scale2 = h2_as_u32(__float2half2_rn(2.f));
    if (fast2) {
      cj2 = h2_as_u32(__half2half2(__hmul(cj, __float2half_rn(-2.f))));
    } else {
#pragma unroll
      for (int k = 0; k < NPR; ++k) s[k] = h2_as_u32(__hsub2(u32_as_h2(s[k]), __half2half2(cj)));
      cj2 = 0u;
    }
  } else {
    // naive FP16 FA: x = fl16(S s - fl16(m s)), s = log2(e) / alpha after the store
    cj2 = h2_as_u32(__half2half2(__hneg(__float2half_rn(__fmul_rn(mloc, qk_scale)))));
    scale2 = h2_as_u32(__half2half2(__float2half_rn(qk_scale)));
  }
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
  for (int k = 0; k < NPR; ++k) {
    const uint32_t x = h2_as_u32(__hfma2(u32_as_h2(s[k]), u32_as_h2(scale2), u32_as_h2(cj2)));
    const uint32_t pv = ex2_f16x2(x) & range_keep(pb + k, lo, hi);
    acc[2 * (k & 3)] = add_lo_f16(acc[2 * (k & 3)], pv);  // pb is a multiple of 4: chain k & 3
    acc[2 * (k & 3) + 1] = add_hi_f16(acc[2 * (k & 3) + 1], pv);
    s[k] = pv;
  }
  // P -> TMEM columns [pb, pb + NPR), zeros to the rest of [0, 64)
  uint32_t z[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) z[k] = 0u;
#pragma unroll
  for (int c = 0; c < NPR / 16; ++c) tmem_st_16cols_b32(t_s + pb + 16 * c, s + 16 * c);
#pragma unroll
  for (int c = 0; c < 4; ++c)  // (warp-uniform condition, constant register operands)
    if (NPR < 64 && (16 * c < pb || 16 * c >= pb + NPR)) tmem_st_16cols_b32(t_s + 16 * c, z);
  return __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                   __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
}

// Self-prepped tile (PackedParams::self_prep, PASA): the prep warpgroup turns the raw K and
// V of the stage's nseq sequences into K' and V' in place, with the pre-pass kernels'
// arithmetic (so the output is bit-identical to the prepped path): per sequence and column,
// colsum = FP32 sum over its N rows ascending, K' = fl16(fl32(fl32(fma(dm, K, fl32(off
// colsum))) lscale)); max|V| (NaN ignored), c0 = pasa_inflation(N, max|V|), V' = V x
// fl16(2^-c0) (only when c0 > 0).  Also the slots holding a non-finite V (the poisoned-tile
// mask for the MMA warp) and c0 per slot for the epilogue.  Thread e owns column pair e % (D/2)
// of slot e / (D/2); the smem tiles are SW128 (row r: 128 bytes per 64-column box, 16-byte
// chunks XOR-ed with r % 8).
//
// This runs once per tile on one warp per SMSP, so its latency sets the tile rate
// (tools/prep_probe.cu times it alone), and on a lone warp every branch costs ~20 cycles
// (predicate set + resolve + reconvergence).  So the slot width WS is a template parameter
// and the code is straight-line: the WS rows of a slot fully unrolled, rows >= N masked by
// selects / predicated stores (rows past N are the slot's gap: stale K, zero V), a thread's
// column pairs unrolled with a predicate, c0 without branches, and the one branch left is the
// rare V scale.  Shared memory through shared-space pointers (sptr): in an out-of-line
// function a generic pointer would take the slow generic path.
template <class T>
__device__ __forceinline__ T* sptr(uint32_t a) {  // a .shared address as a shared-space pointer
  extern __shared__ uint8_t smem_raw[];
  return reinterpret_cast<T*>(smem_raw + (a - smem_u32(smem_raw)));
}

// pasa_inflation without branches (same value): 0 unless 1 < need < 3e38, else ceil(log2 need)
__device__ __forceinline__ int inflation_nb(int S2, float vmax) {
  const float need = static_cast<float>(S2) * vmax * (1.0f / 16384.0f);
  const uint32_t b = __float_as_uint(need);
  const int e = static_cast<int>(b >> 23) - 127 + ((b & 0x7fffffu) != 0u);
  return (need > 1.0f && need < 3.0e38f) ? e : 0;
}

// K side of a tile, as soon as its Q and K have landed: column sums and K' in place; clears
// the max|V| words for the V side (whose atomics follow this function's last barrier).
template <int D, int WS>
__device__ __forceinline__ void self_prep_k(uint32_t stage, int N, float dm, float off_s, float lscale, int nseq,
                                            uint32_t vmx_s, uint32_t qk_full, uint32_t parity, long long* trace,
                                            int trit, int g) {
  // (the parameters as register arguments: a PackedParams reference would be read from the
  // caller's stack -- local memory -- on every call)
  constexpr int BOX = kTile * 128, TILE = (D / 64) * BOX;
  constexpr int P = 128 / WS, IPT = (P * (D / 2) + 127) / 128;  // column pairs per thread
  const uint32_t kt = stage + TILE;
  const int tid = threadIdx.x - 256 - 128 * g;  // (prep warpgroup g)
  if (tid < 9) sptr<unsigned>(vmx_s)[tid] = 0u;  // [0, 8): slot max|V| bits, [8]: non-finite slots
  mbar_wait(qk_full, parity);
  if (threadIdx.x == 256 + 128 * g) PK_TRP(trace, 0, trit, 6);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = tid + 128 * i;
    const bool live = e < nseq * (D / 2);
    // (items past the live ones still load -- straight-line code -- so their slot is clamped
    // into the tile: with P = 2 slots, threads 64-127 would otherwise read past the stage)
    const int sl = min(e / (D / 2), P - 1), cp = e % (D / 2);
    const int col = 2 * cp, ck = (col % 64) / 8;
    // row c of the slot: swizzle key c % 8 (slots start at multiples of 8): a constant offset
    const uint32_t cb = kt + (col / 64) * BOX + (col % 8) * 2 + sl * WS * 128;
    auto off = [&](int c) { return cb + static_cast<uint32_t>(c * 128 + ((ck ^ (c & 7)) << 4)); };
    // FP32 column sums, rows ascending (the pre-pass's order; add.f32.f16 converts exactly;
    // + 0 for the masked rows is exact: the sum starts at +0 and never becomes -0)
    float csx = 0.f, csy = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < WS; c0 += 8) {
      uint32_t kb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kb[u] = *sptr<uint32_t>(off(c0 + u));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t k = c0 + u < N ? kb[u] : 0u;  // (gap rows hold stale K)
        csx = add_lo_f16(csx, k);
        csy = add_hi_f16(csy, k);
      }
    }
    // K' = fl16(fl32(fma(dm, K, fl32(off colsum))) lscale), rows < N
    const float osx = __fmul_rn(off_s, csx), osy = __fmul_rn(off_s, csy);
#pragma unroll
    for (int c0 = 0; c0 < WS; c0 += 8) {
      uint32_t kb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kb[u] = *sptr<uint32_t>(off(c0 + u));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float2 k2 = __half22float2(u32_as_h2(kb[u]));
        const uint32_t kp = h2_as_u32(__floats2half2_rn(__fmul_rn(__fmaf_rn(dm, k2.x, osx), lscale),
                                                        __fmul_rn(__fmaf_rn(dm, k2.y, osy), lscale)));
        if (live && c0 + u < N) *sptr<uint32_t>(off(c0 + u)) = kp;
      }
    }
  }
  if (threadIdx.x == 256 + 128 * g) PK_TRP(trace, 1, trit, 8);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // K' for the tensor core
  named_bar_sync(1 + g, 128);
}

// V side, once V has landed: max|V| and the non-finite check per slot, c0, V' in the (rare)
// tiles that need it, the poisoned-slot mask.  (Tried on the idle warps 2-3 instead, beside
// the K side: slower -- two warps at 32-40 registers take longer than the P V' can wait.)
template <int D, int WS>
__device__ __forceinline__ void self_prep_v(uint32_t stage, int N, int nseq, uint32_t c0_s, uint32_t vmx_s,
                                            uint32_t bad_s, uint32_t v_full, uint32_t parity, long long* trace,
                                            int trit, int g) {
  constexpr int BOX = kTile * 128, TILE = (D / 64) * BOX;
  constexpr int P = 128 / WS, IPT = (P * (D / 2) + 127) / 128;
  const uint32_t vt = stage + 2 * TILE;
  unsigned* vmx = sptr<unsigned>(vmx_s);
  const int tid = threadIdx.x - 256 - 128 * g;  // (prep warpgroup g)
  mbar_wait(v_full, parity);
  if (threadIdx.x == 256 + 128 * g) PK_TRP(trace, 1, trit, 9);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = tid + 128 * i;
    const int sl = min(e / (D / 2), P - 1), cp = e % (D / 2), col = 2 * cp, ck = (col % 64) / 8;
    const uint32_t cb = vt + (col / 64) * BOX + (col % 8) * 2 + sl * WS * 128;
    __half2 vm2 = __float2half2_rn(0.f), nf2 = vm2;
#pragma unroll
    for (int c0 = 0; c0 < WS; c0 += 8) {
      uint32_t vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)  // (gap rows of V are zero)
        vb[u] = *sptr<uint32_t>(cb + static_cast<uint32_t>((c0 + u) * 128 + ((ck ^ u) << 4)));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        vm2 = __hmax2(vm2, __habs2(u32_as_h2(vb[u])));               // NaN ignored, like fmaxf
        nf2 = __hfma2(u32_as_h2(vb[u]), __float2half2_rn(0.f), nf2);  // NaN iff some V is Inf / NaN
      }
    }
    if (e < nseq * (D / 2)) {
      atomicMax(vmx + sl, __float_as_uint(fmaxf(__low2float(vm2), __high2float(vm2))));  // >= 0: bits order
      if (__hisnan(__low2half(nf2)) || __hisnan(__high2half(nf2))) atomicOr(vmx + 8, 1u << sl);
    }
  }
  named_bar_sync(1 + g, 128);  // every slot's max|V| and the non-finite slots are in
  if (threadIdx.x == 256 + 128 * g) PK_TRP(trace, 1, trit, 10);
  // V' = V fl16(2^-c0): only in the (rare) tiles where some slot needs it
  int cz[IPT];
  bool any = false;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = tid + 128 * i;
    cz[i] = e < nseq * (D / 2) ? inflation_nb(N, __uint_as_float(vmx[e / (D / 2)])) : 0;
    any |= cz[i] > 0;
  }
  if (__any_sync(0xffffffffu, any)) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int e = tid + 128 * i;
      const int sl = min(e / (D / 2), P - 1), cp = e % (D / 2), col = 2 * cp, ck = (col % 64) / 8;
      const __half2 sc = __half2half2(__float2half_rn(ldexpf(1.0f, -cz[i])));
      const uint32_t cb = vt + (col / 64) * BOX + (col % 8) * 2 + sl * WS * 128;
#pragma unroll
      for (int c = 0; c < WS; ++c) {
        uint32_t* a = sptr<uint32_t>(cb + static_cast<uint32_t>(c * 128 + ((ck ^ (c & 7)) << 4)));
        if (cz[i] > 0 && c < N) *a = h2_as_u32(__hmul2(u32_as_h2(*a), sc));
      }
    }
  }
  if (tid < 8) sptr<int>(c0_s)[tid] = tid < nseq ? inflation_nb(N, __uint_as_float(vmx[tid])) : 0;
  if (tid == 0) *sptr<uint32_t>(bad_s) = vmx[8];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // V' for the tensor core
  named_bar_sync(1 + g, 128);
  if (threadIdx.x == 256 + 128 * g) PK_TRP(trace, 1, trit, 11);
}

// One tile: the K side, kprep_done (the MMA warp may issue S'), then the V side.  (One
// out-of-line function: two consecutive out-of-line calls here make ptxas 12.9 run for hours.)
template <int D, int WS>
__device__ __noinline__ void self_prep_stage(uint32_t stage, int N, float dm, float off_s, float lscale, int nseq,
                                             uint32_t c0_s, uint32_t vmx_s, uint32_t bad_s, uint32_t qk_full,
                                             uint32_t v_full, uint32_t kprep_done, uint32_t parity,
                                             long long* trace, int trit, int g) {
  self_prep_k<D, WS>(stage, N, dm, off_s, lscale, nseq, vmx_s, qk_full, parity, trace, trit, g);
  if (threadIdx.x == 256 + 128 * g) mbar_arrive(kprep_done);
  self_prep_v<D, WS>(stage, N, nseq, c0_s, vmx_s, bad_s, v_full, parity, trace, trit, g);
}

}  // namespace

// Persistent: CTA b processes tiles b, b + gridDim.x, ...; the loads of the next tile run
// in the second stage while the current one is computed.
template <int D, int MODE, int WS>
__global__ void __launch_bounds__(PackedCfg<D, WS>::THREADS, PackedCfg<D, WS>::CTAS)
    pasa_fwd_packed_kernel(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_kp,
                           const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_o, const PackedParams p) {
  using Cfg = PackedCfg<D, WS>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sb = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sb - smem_u32(smem_raw));
  const uint32_t qk_full = sb + Cfg::SMEM_BAR;  // [ST]: the stage's Q and K (K') have landed
  const uint32_t v_full = qk_full + 8 * ST;     // [ST]: its V (V') has landed
  const uint32_t in_empty = v_full + 8 * ST;    // [ST]: the stage's MMAs are done
  const uint32_t s_full = in_empty + 8 * ST, p_full = s_full + 8, t_full = p_full + 8,
                 t_empty = t_full + 8;
  const uint32_t aux = t_empty + 8;       // the first P V' of a poisoned tile is done
  const uint32_t mask_full = aux + 8;     // the tile's poisoned-slot mask is published
  const uint32_t kprep_done = mask_full + 8;     // [ST] self_prep: the stage holds K'
  const uint32_t vprep_done = kprep_done + 8 * ST;  // [ST] self_prep: ... and V', c0, the mask
  const uint32_t qk_empty = vprep_done + 8 * ST;  // [ST]: the stage's S' MMA has read Q and K'
  // (in_empty: its P V' has read V' -- the Q / K' half of a stage refills a PV earlier)
  const uint32_t o_free = qk_empty + 8 * ST;  // [ST]: the O tile staged in its V' buffer is stored
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Cfg::SMEM_BAR + 8 * Cfg::NUM_BARS);
  // [it % 2]: bit s = slot s of tile it holds a non-finite V' row
  // per tile it, slot it & 3: written up to two tiles ahead of the epilogue that reads it
  volatile uint32_t* bad_mask = tmem_holder + 1;                 // [4]
  int* c0s = reinterpret_cast<int*>(tmem_holder + 5);            // [4][8]
  unsigned* vmx = reinterpret_cast<unsigned*>(c0s + 32);         // [NPREP][16] (prep scratch)
  const int warp = static_cast<int>(warp_id());
  const int lane = threadIdx.x & 31;
  constexpr int W = WS;                             // slot stride (rows / keys) = p.W
  const int ntiles = (p.BH + p.P - 1) / p.P;

  if (threadIdx.x == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(qk_full + 8 * st, 1);
      mbar_init(v_full + 8 * st, 1);
      mbar_init(in_empty + 8 * st, 1);
      mbar_init(qk_empty + 8 * st, 1);
      mbar_init(kprep_done + 8 * st, 1);
      mbar_init(vprep_done + 8 * st, 1);
      mbar_init(o_free + 8 * st, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(t_full, 1);
    mbar_init(t_empty, 4);
    mbar_init(aux, 1);
    mbar_init(mask_full, 1);
    fence_barrier_init();
  }
  {  // V' rows outside the sequences' N-row slots must read as zero (P = 0 there, and 0 x
     // uninitialised shared memory could be NaN); later tiles only overwrite slot rows
    for (int st = 0; st < ST; ++st) {
      uint4* z = reinterpret_cast<uint4*>(smem + st * Cfg::STAGE_BYTES + 2 * Cfg::TILE_BYTES);
      for (int e = threadIdx.x; e < Cfg::TILE_BYTES / 16; e += blockDim.x) z[e] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const bool self_prep = MODE == kModePasa && p.self_prep;
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_CTL));
  if (warp == 0) {
    // ---- TMA producer: each sequence's N rows of Q, K', V' into its slot
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_kp);
      tma_prefetch(&tm_v);
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % ST, seq0 = tile * p.P, nseq = min(p.P, p.BH - seq0);
        const uint32_t base = sb + st * Cfg::STAGE_BYTES;
        // Q and K' as soon as the stage's S' has run, V' once its P V' has
        mbar_wait(qk_empty + 8 * st, ((it / ST) & 1) ^ 1);
        mbar_expect_tx(qk_full + 8 * st, 2 * Cfg::NBOX * nseq * p.N * 128);
        for (int sl = 0; sl < nseq; ++sl) {
          const int r = (seq0 + sl) * p.N;  // flat row of the sequence
          for (int bx = 0; bx < Cfg::NBOX; ++bx) {
            const uint32_t off = bx * Cfg::BOX_BYTES + sl * W * 128;
            tma_load_3d(base + off, &tm_q, qk_full + 8 * st, bx * 64, r, 0);
            tma_load_3d(base + Cfg::TILE_BYTES + off, &tm_kp, qk_full + 8 * st, bx * 64, r, 0);
          }
        }
        PK_TR(1, it, 3);
        mbar_wait(in_empty + 8 * st, ((it / ST) & 1) ^ 1);
        mbar_wait(o_free + 8 * st, ((it / ST) & 1) ^ 1);  // the V buffer also stages O
        mbar_expect_tx(v_full + 8 * st, Cfg::NBOX * nseq * p.N * 128);
        for (int sl = 0; sl < nseq; ++sl) {
          const int r = (seq0 + sl) * p.N;
          for (int bx = 0; bx < Cfg::NBOX; ++bx)
            tma_load_3d(base + 2 * Cfg::TILE_BYTES + bx * Cfg::BOX_BYTES + sl * W * 128, &tm_v,
                        v_full + 8 * st, bx * 64, r, 0);
        }
        PK_TR(1, it, 4);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (one elected lane); the whole warp scans V' for non-finite rows
    const bool leader = elect_one();
    constexpr uint32_t kIdS = idesc_f16(128, 128, 0, 0, 0);
    constexpr uint32_t kIdPV = idesc_f16(128, D, 0, 0, 1);
    int it = 0, npois = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % ST, nseq = min(p.P, p.BH - tile * p.P);
      const uint32_t base = sb + st * Cfg::STAGE_BYTES;
      const uint32_t vbase = base + 2 * Cfg::TILE_BYTES;
      // self_prep: the prep warpgroup turns K into K' in place first (V' and the non-finite
      // slots follow, before P V'); else the stage holds the pre-pass output as loaded
      mbar_wait((self_prep ? kprep_done : qk_full) + 8 * st, (it / ST) & 1);
      tc_fence_after();
      // S' = Q K'^T (SS, F16 accumulator) into columns [0, 128); in-order after the
      // previous tile's PV, so its P columns are free
      if (leader) {
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32;
          umma_ss(tmem_base, smem_desc_sw128(base + off, 16, 1024),
                  smem_desc_sw128(base + Cfg::TILE_BYTES + off, 16, 1024), kIdS, s > 0);
        }
        tc_commit(s_full);
        tc_commit(qk_empty + 8 * st);
        PK_TR(1, it, 0);
      }
      // while S' runs: which slots' V' rows hold Inf / NaN?  0 x v is NaN exactly for a
      // non-finite v, so one HFMA2 per pair accumulates the verdict.
      uint32_t bad = 0u;
      if (!self_prep) mbar_wait(v_full + 8 * st, (it / ST) & 1);
      for (int r = lane; !self_prep && r < nseq * W; r += 32) {
        if (r % W >= p.N) continue;  // gap rows are zero
        __half2 acc = __float2half2_rn(0.f);
#pragma unroll
        for (int bx = 0; bx < Cfg::NBOX; ++bx) {
          const uint4* row = reinterpret_cast<const uint4*>(smem + (vbase - sb) + bx * Cfg::BOX_BYTES + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 x = row[c];
            acc = __hfma2(u32_as_h2(x.x), __float2half2_rn(0.f), acc);
            acc = __hfma2(u32_as_h2(x.y), __float2half2_rn(0.f), acc);
            acc = __hfma2(u32_as_h2(x.z), __float2half2_rn(0.f), acc);
            acc = __hfma2(u32_as_h2(x.w), __float2half2_rn(0.f), acc);
          }
        }
        if (__hisnan(__low2half(acc)) || __hisnan(__high2half(acc))) bad |= 1u << (r / W);
      }
      bad = __reduce_or_sync(0xffffffffu, bad);
      // T = P V' (TS: P packed in columns [0, 64), V' MN-major) into [128, 128 + D), once
      // the softmax has stored P and read the previous tile's T
      if (self_prep) {  // V' and the mask (from the prep)
        mbar_wait(vprep_done + 8 * st, (it / ST) & 1);
        tc_fence_after();
        bad = bad_mask[it & 3];
      }
      mbar_wait(p_full, it & 1);
      if (leader) PK_TR(1, it, 1);
      // publish the mask (release) only now: the softmax has finished tile it - 1 (p_full),
      // so mask_full is never two phases ahead of its reader and slot it & 1 is free
      if (leader) {
        if (!self_prep) bad_mask[it & 3] = bad;
        mbar_arrive(mask_full);
      }
      if (nseq < p.P) {
        // a ragged tile: its unused slots hold an earlier tile's staged O (possibly non-finite),
        // and P = 0 there multiplies them -- zero those V' rows first
        for (int e = lane; e < (p.P - nseq) * W * Cfg::NBOX * 8; e += 32) {
          const int r = nseq * W + e / (Cfg::NBOX * 8), bx = (e / 8) % Cfg::NBOX, c = e % 8;
          *reinterpret_cast<uint4*>(smem + (vbase - sb) + bx * Cfg::BOX_BYTES + r * 128 + c * 16) =
              make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      mbar_wait(t_empty, (it & 1) ^ 1);
      tc_fence_after();
      auto issue_pv = [&](uint32_t dcol) {
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_ts(tmem_base + dcol, tmem_base + s * 8,
                  smem_desc_sw128(vbase + s * 2048, Cfg::BOX_BYTES, 1024), kIdPV, s > 0);
      };
      if (leader) issue_pv(128);
      if (bad) {
        // the poisoned sequences keep T; the rest get T_clean over zeroed poisoned rows
        if (leader) tc_commit(aux);
        mbar_wait(aux, npois & 1);
        ++npois;
        for (int e = lane; e < nseq * W * Cfg::NBOX * 8; e += 32) {
          const int r = e / (Cfg::NBOX * 8), bx = (e / 8) % Cfg::NBOX, c = e % 8;
          if ((bad >> (r / W)) & 1u)
            *reinterpret_cast<uint4*>(smem + (vbase - sb) + bx * Cfg::BOX_BYTES + r * 128 + c * 16) =
                make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        tc_fence_after();
        if (leader) issue_pv(Cfg::T_CLEAN);
      }
      if (leader) {
        tc_commit(t_full);
        PK_TR(1, it, 2);
        tc_commit(in_empty + 8 * st);
      }
      __syncwarp();
    }
  }
  } else if (warp < 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_SM));
    // ---- softmax: one thread per row
    const int quad = warp % 4;
    const int row = quad * 32 + lane;
    const uint32_t t_s = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    const int sl = row / W, rr = row % W;            // the row's slot and row in the slot
    const int lo = sl * W, hi = lo + p.N;            // its sequence's key columns
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int seq0 = tile * p.P, nseq = min(p.P, p.BH - seq0);
      const bool row_ok = sl < nseq && rr < p.N;
      const int st = it % ST;
      const bool tr0 = threadIdx.x == 128;
      if (tr0) PK_TR(0, it, 0);
      mbar_wait(s_full, it & 1);
      if (tr0) PK_TR(0, it, 1);
      tc_fence_after();
      // Only the key columns of the warp's own slots are loaded and exponentiated (the
      // warp's 32 rows span one 32-wide slot, two 16-wide ones, or half a 64-wide one:
      // 32 or 64 columns, warp-uniform; 48-wide slots straddle warps and take all 128); the
      // rest of P is stored as zeros for the PV MMA.
      // The pair index keeps its tile position (chain i & 3, mask range_keep(i, lo, hi)),
      // so the row's sums are the same FP32 chains as over all 128 columns.
      // (W = 16, 32: 32 columns; W = 64: 64; W = 48 straddles -- all 128)
      const float l = row_softmax<Cfg::NPR, MODE>(t_s, quad, lo, hi, p.qk_scale);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (tr0) PK_TR(0, it, 2);
      // epilogue: O = T 2^c0 / l (global recovering, pasa.cpp:184-194); self_prep: c0 from the
      // prep, published with the mask
      mbar_wait(mask_full, it & 1);
      const int c0 = MODE != kModePasa || !row_ok ? 0
                     : self_prep ? c0s[8 * (it & 3) + sl] : pasa_inflation(p.N, p.vmax[seq0 + sl]);
      const float inv_l = __fmul_rn(__frcp_rn(l), ldexpf(1.0f, c0));
      const uint32_t bad = bad_mask[it & 3];
      // a poisoned tile: this row's own sequence poisoned -> T, else T_clean (warp-uniform
      // column choice per load: rows of a warp may sit in different slots)
      const bool clean = bad != 0 && !((bad >> sl) & 1u);
      mbar_wait(t_full, it & 1);
      if (tr0) PK_TR(0, it, 4);
      tc_fence_after();
      uint32_t tv[D / 2];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld_32cols_pack16(t_s + 128 + 32 * c, tv + 16 * c);
      if (__any_sync(0xffffffffu, clean)) {  // rare: 16 extra registers at a time
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t tc[16];
          tmem_ld_32cols_pack16(t_s + Cfg::T_CLEAN + 32 * c, tc);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) tv[16 * c + i] = clean ? tc[i] : tv[16 * c + i];
        }
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty);
      if (tr0) PK_TR(0, it, 5);
      // O rows staged in the stage's V' buffer (P V' has read it: t_full), SW128 like the loads
      // (slot rows start at multiples of 8, so the 16-byte chunk of row r sits at c ^ r % 8),
      // then one TMA store of N rows per sequence and 64-column box.  Gap rows and unused
      // slots are not written (the MMA warp zeroes a ragged tile's unused slots before P V').
      const uint32_t vst = sb + st * Cfg::STAGE_BYTES + 2 * Cfg::TILE_BYTES;
#pragma unroll
      for (int i = 0; i < D / 2; i += 4) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half a = __float2half_rn(__fmul_rn(lo_f(tv[i + k]), inv_l));
          const __half c = __float2half_rn(__fmul_rn(hi_f(tv[i + k]), inv_l));
          w[k] = h2_as_u32(__halves2half2(a, c));
        }
        const int col = 2 * i, chunk = (col % 64) / 8;
        const uint32_t a = vst + (col / 64) * Cfg::BOX_BYTES + row * 128 + ((chunk ^ (row & 7)) << 4);
        if (row_ok)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                       "r"(w[3]) : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // O for the TMA engine
      named_bar_sync(3, 128);
      if (tr0) {
        for (int s2 = 0; s2 < nseq; ++s2)
          for (int bx = 0; bx < Cfg::NBOX; ++bx)
            tma_store_3d(&tm_o, vst + bx * Cfg::BOX_BYTES + s2 * W * 128, bx * 64, (seq0 + s2) * p.N, 0);
        tma_store_commit_wait_read();
        mbar_arrive(o_free + 8 * st);
      }
      if (tr0) PK_TR(0, it, 3);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_PREP));
    // ---- the pre-pass of every tile (self_prep), as soon as its stage has landed: runs
    // ahead of the softmax, which it never waits for (the MMA warp waits for kprep_done before
    // S' and for vprep_done before P V').  Prep warpgroup g takes the tiles it with
    // it % NPREP == g (with two: always stage g).
    const int g = (warp - 8) / 4;
    const uint32_t lead = 256 + 128 * g;  // the warpgroup's first thread
    int it = g;
    for (int tile = blockIdx.x + g * gridDim.x; self_prep && tile < ntiles;
         tile += Cfg::NPREP * gridDim.x, it += Cfg::NPREP) {
      const int st = it % ST;
      if (threadIdx.x == lead) PK_TR(1, it, 5);
      self_prep_stage<D, WS>(sb + st * Cfg::STAGE_BYTES, p.N, p.dm, p.off, p.lscale, min(p.P, p.BH - tile * p.P),
                             smem_u32(c0s + 8 * (it & 3)), smem_u32(vmx + 16 * g),
                             smem_u32(const_cast<uint32_t*>(bad_mask) + (it & 3)), qk_full + 8 * st, v_full + 8 * st,
                             kprep_done + 8 * st, (it / ST) & 1, p.trace, it, g);
      if (threadIdx.x == lead) mbar_arrive(vprep_done + 8 * st);  // (after the prep's last barrier)
      if (threadIdx.x == lead) PK_TR(1, it, 6);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

template <int D, int MODE, int WS>
static cudaError_t launch_packed_t(const CUtensorMap& tq, const CUtensorMap& tk,
                                   const CUtensorMap& tv, const CUtensorMap& to, const PackedParams& p,
                                   cudaStream_t stream) {
  using Cfg = PackedCfg<D, WS>;
  cudaError_t e = cudaFuncSetAttribute(pasa_fwd_packed_kernel<D, MODE, WS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = (p.BH + p.P - 1) / p.P;  // p.P = 128 / p.W sequences per tile
  const int sms = current_sm_count();  // the launching (current) device
  int per_sm = Cfg::CTAS;
#ifdef PASA_TRACE
  if (getenv("PASA_PACKED_PER_SM")) per_sm = atoi(getenv("PASA_PACKED_PER_SM"));  // (profiling)
#endif
  const int grid = tiles < per_sm * sms ? tiles : per_sm * sms;
  pasa_fwd_packed_kernel<D, MODE, WS><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, stream>>>(tq, tk, tv, to, p);
  return cudaGetLastError();
}

template <int D, int MODE>
static cudaError_t launch_packed_w(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                   const CUtensorMap& to, const PackedParams& p, cudaStream_t stream) {
  switch (p.W) {  // the slot width as a compile-time row count
    case 16: return launch_packed_t<D, MODE, 16>(tq, tk, tv, to, p, stream);
    case 32: return launch_packed_t<D, MODE, 32>(tq, tk, tv, to, p, stream);
    case 48: return launch_packed_t<D, MODE, 48>(tq, tk, tv, to, p, stream);
    case 64: return launch_packed_t<D, MODE, 64>(tq, tk, tv, to, p, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fwd_packed(int D, int mode, const CUtensorMap& tq, const CUtensorMap& tk,
                              const CUtensorMap& tv, const CUtensorMap& to, const PackedParams& p,
                              cudaStream_t stream) {
  if (D == 64) return mode == kModePasa ? launch_packed_w<64, kModePasa>(tq, tk, tv, to, p, stream)
                                        : launch_packed_w<64, kModeFa16>(tq, tk, tv, to, p, stream);
  if (D == 128) return mode == kModePasa ? launch_packed_w<128, kModePasa>(tq, tk, tv, to, p, stream)
                                         : launch_packed_w<128, kModeFa16>(tq, tk, tv, to, p, stream);
  return cudaErrorInvalidValue;
}

}  // namespace pasa_b200
