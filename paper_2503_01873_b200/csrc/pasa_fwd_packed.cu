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
// Persistent CTAs walk the tiles; 6 warps: warp 0 loads (TMA, a two-stage ring, so the next
// tile's loads overlap this one's compute), warp 1 issues the MMAs, warps 2-5 run the
// softmax with one thread per row (TMEM lane quadrant = warp % 4).  TMEM: S'/P at +0, T at
// +128, T_clean at +128 + D (256 columns at d = 64, so two CTAs share an SM; 512 at d = 128).
//
// Non-finite V: the tile's P V' also multiplies each row's zero P entries by the other
// sequences' V' rows, and 0 x Inf = NaN would leak one sequence's Inf/NaN into its
// neighbours (the unpacked kernel keeps heads apart).  So the MMA warp scans the tile's V'
// rows while S' runs; for a tile with a non-finite V' row it issues P V' twice -- into T
// (the poisoned sequences read it: exactly what they get alone) and, after zeroing the
// poisoned sequences' V' rows in shared memory, into T_clean (everyone else reads it).
// The zeroed rows stay zero until TMA refills them, so the stale slots of a ragged last
// tile are clean too.  Clean tiles pay only the scan.
#include <cuda.h>
#include <cuda_fp16.h>

#include "pasa_kernels.cuh"
#include "sm100.cuh"

namespace pasa_b200 {
using namespace sm100;

// PASA_TRACE builds: CTA 0 records clock64() at fixed points of its first 64 tiles,
// p.trace[(role * 64 + it) * 8 + event] (role 0 = softmax warp 2 lane 0, 1 = MMA issuer)
#ifdef PASA_TRACE
#define PK_TR(role, it, ev)                                                        \
  do {                                                                             \
    if (p.trace && blockIdx.x == 0 && (it) < 64) p.trace[((role) * 64 + (it)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define PK_TR(role, it, ev) \
  do {                      \
  } while (0)
#endif

namespace {

template <int D>
struct PackedCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int BOX_BYTES = kTile * 128;
  static constexpr int TILE_BYTES = NBOX * BOX_BYTES;
  static constexpr int STAGE_BYTES = 3 * TILE_BYTES;  // Q, K', V' of one tile
  static constexpr int STAGES = 2;
  static constexpr int SMEM_BAR = STAGES * STAGE_BYTES;
  static constexpr int NUM_BARS = 4 * STAGES + 6;  // in_full/empty, s/p/t_full, t_empty, aux, mask, prep_done, qk_empty
  // after the barriers: TMEM holder, bad-slot masks [2], per-stage slot exponents c0 [ST][8],
  // per-slot max|V| bits [8]
  // after the barriers: TMEM holder, bad-slot masks [4], slot exponents c0 [4][8], the
  // prep's per-slot max|V| bits and non-finite slots [9]
  static constexpr int SMEM_BYTES = SMEM_BAR + 8 * NUM_BARS + 4 * (1 + 4 + 32 + 16) + 1024;
  // warpgroup 0: warp 0 TMA, warp 1 MMA (2, 3 idle); 1: softmax (warps 4-7 = TMEM lane
  // quadrants 0-3); 2: the per-tile pre-pass (self_prep)
  static constexpr int THREADS = 384;
  // setmaxnreg split of the launch allocation (d = 64: 2 CTAs per SM, 80 x 384 = 30720
  // registers each; d = 128: 1 CTA, 168 x 384)
  static constexpr int REGS_CTL = D == 64 ? 32 : 40, REGS_PREP = D == 64 ? 56 : 64,
                       REGS_SM = D == 64 ? 152 : 232;
  static_assert(128 * (REGS_CTL + REGS_PREP + REGS_SM) <= (D == 64 ? 80 : 168) * THREADS, "registers");
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

// Self-prepped tile (PackedParams::self_prep, PASA): the 128 softmax threads turn the raw
// K and V of the stage's nseq sequences into K' and V' in place, with the pre-pass kernels'
// arithmetic (so the output is bit-identical to the prepped path): per sequence and column,
// colsum = FP32 sum over its N rows ascending, K' = fl16(fl32(fl32(fma(dm, K, fl32(off
// colsum))) lscale)); max|V| (NaN ignored), c0 = pasa_inflation(N, max|V|), V' = V x
// fl16(2^-c0) (only when c0 > 0).  Also the slots holding a non-finite V (the poisoned-tile
// mask for the MMA warp) and c0 per slot for the epilogue.  Thread e owns column pair e % (D/2)
// of slot e / (D/2); the smem tiles are SW128 (row r: 128 bytes per 64-column box, 16-byte
// chunks XOR-ed with r % 8).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <int D>
__device__ __noinline__ void self_prep_stage(uint32_t stage, const PackedParams& p, int nseq, int* c0,
                                             unsigned* vmx, volatile uint32_t* bad_out, uint32_t in_full,
                                             uint32_t parity, int trit) {
  // (shared-memory addresses as 32-bit .shared offsets: through a generic pointer in this
  // out-of-line function every access would take the slow generic path)
  constexpr int BOX = kTile * 128, TILE = (D / 64) * BOX;
  const uint32_t kt = stage + TILE;
  const uint32_t vt = stage + 2 * TILE;
  // (the parameters as values: through the reference every "memory"-clobbering shared
  // access below would reload them)
  const int tid = threadIdx.x - 256, W = p.W, N = p.N;
  const float dm = p.dm, off_s = p.off, lscale = p.lscale;
  if (tid < 9) vmx[tid] = 0u;  // [0, 8): slot max|V| bits, [8]: non-finite slots
  mbar_wait(in_full, parity);
  if (threadIdx.x == 256) PK_TR(0, trit, 6);
  named_bar_sync(1, 128);  // vmx reset before any thread's atomicMax
  // Rows of a slot start at a multiple of 8 (W is), so row r0 + c of a batch of 8 (c0 % 8 == 0)
  // has swizzle key u = c % 8: within a batch every address is a constant offset from the
  // batch's base -- no per-element address arithmetic.
  uint32_t badl = 0;
  for (int e = tid; e < nseq * (D / 2); e += 128) {
    const int sl = e / (D / 2), cp = e % (D / 2), r0 = sl * W;
    const int col = 2 * cp, chunk = (col % 64) / 8;
    const uint32_t cbase = (col / 64) * BOX + (col % 8) * 2 + r0 * 128;  // + c * 128 + swizzle
    auto off = [&](int u) { return static_cast<uint32_t>(u * 128 + ((chunk ^ u) << 4)); };
    // FP32 column sums, rows ascending (the pre-pass's order; add.f32.f16 converts exactly),
    // max|V| in half2 (HMNMX2 ignores NaN like fmaxf), and 0 x V accumulated in half2: NaN
    // exactly when some V is Inf or NaN
    float csx = 0.f, csy = 0.f;
    __half2 vm2 = __float2half2_rn(0.f), nf2 = __float2half2_rn(0.f);
    auto absorb = [&](__half2 kh, __half2 vh) {
      csx = add_lo_f16(csx, h2_as_u32(kh));
      csy = add_hi_f16(csy, h2_as_u32(kh));
      vm2 = __hmax2(vm2, __habs2(vh));
      nf2 = __hfma2(vh, __float2half2_rn(0.f), nf2);
    };
    int c0 = 0;
    for (; c0 + 8 <= N; c0 += 8) {  // full batches: every load in flight before the first use
      const uint32_t b = cbase + c0 * 128;
      __half2 kb[8], vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        kb[u] = u32_as_h2(lds_u32(kt + b + off(u)));
        vb[u] = u32_as_h2(lds_u32(vt + b + off(u)));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) absorb(kb[u], vb[u]);
    }
    for (int u = 0; c0 + u < N; ++u)
      absorb(u32_as_h2(lds_u32(kt + cbase + c0 * 128 + off(u))), u32_as_h2(lds_u32(vt + cbase + c0 * 128 + off(u))));
    const float vm = fmaxf(__low2float(vm2), __high2float(vm2));
    atomicMax(vmx + sl, __float_as_uint(vm));  // vm >= 0: bit order = value order
    if (__hisnan(__low2half(nf2)) || __hisnan(__high2half(nf2))) badl |= 1u << sl;
    const float osx = __fmul_rn(off_s, csx), osy = __fmul_rn(off_s, csy);
    auto kprime = [&](uint32_t a) {
      const float2 k2 = __half22float2(u32_as_h2(lds_u32(a)));
      sts_u32(a, h2_as_u32(__floats2half2_rn(__fmul_rn(__fmaf_rn(dm, k2.x, osx), lscale),
                                             __fmul_rn(__fmaf_rn(dm, k2.y, osy), lscale))));
    };
    for (c0 = 0; c0 + 8 <= N; c0 += 8) {
      const uint32_t b = kt + cbase + c0 * 128;
      __half2 kb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kb[u] = u32_as_h2(lds_u32(b + off(u)));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float2 k2 = __half22float2(kb[u]);
        sts_u32(b + off(u), h2_as_u32(__floats2half2_rn(__fmul_rn(__fmaf_rn(dm, k2.x, osx), lscale),
                                                         __fmul_rn(__fmaf_rn(dm, k2.y, osy), lscale))));
      }
    }
    for (int u = 0; c0 + u < N; ++u) kprime(kt + cbase + c0 * 128 + off(u));
  }
  badl = __reduce_or_sync(0xffffffffu, badl);
  if ((threadIdx.x & 31) == 0 && badl) atomicOr(vmx + 8, badl);
  named_bar_sync(1, 128);  // every slot's max|V| and the non-finite slots are in
  if (threadIdx.x == 256) PK_TR(0, trit, 7);
  for (int e = tid; e < nseq * (D / 2); e += 128) {
    const int sl = e / (D / 2), cp = e % (D / 2), r0 = sl * W;
    const int cz = pasa_inflation(N, __uint_as_float(vmx[sl]));
    if (cz == 0) continue;  // (the usual case: V' = V)
    const __half2 sc = __half2half2(__float2half_rn(ldexpf(1.0f, -cz)));
    const int col = 2 * cp;
    for (int c = 0; c < N; ++c) {
      const uint32_t a = vt + (col / 64) * BOX + (r0 + c) * 128 + ((((col % 64) / 8) ^ (c & 7)) << 4) +
                         (col % 8) * 2;
      sts_u32(a, h2_as_u32(__hmul2(u32_as_h2(lds_u32(a)), sc)));
    }
  }
  if (tid < 8) c0[tid] = tid < nseq ? pasa_inflation(N, __uint_as_float(vmx[tid])) : 0;
  if (tid == 0) *bad_out = vmx[8];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // K', V' for the tensor core
  named_bar_sync(1, 128);
}

}  // namespace

// Persistent: CTA b processes tiles b, b + gridDim.x, ...; the loads of the next tile run
// in the second stage while the current one is computed.
template <int D, int MODE>
__global__ void __launch_bounds__(PackedCfg<D>::THREADS, D == 64 ? 2 : 1)
    pasa_fwd_packed_kernel(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_kp,
                           const __grid_constant__ CUtensorMap tm_v, const PackedParams p) {
  using Cfg = PackedCfg<D>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sb = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sb - smem_u32(smem_raw));
  const uint32_t in_full = sb + Cfg::SMEM_BAR;  // [ST]
  const uint32_t in_empty = in_full + 8 * ST;   // [ST]: the stage's MMAs are done
  const uint32_t s_full = in_empty + 8 * ST, p_full = s_full + 8, t_full = p_full + 8,
                 t_empty = t_full + 8;
  const uint32_t aux = t_empty + 8;       // the first P V' of a poisoned tile is done
  const uint32_t mask_full = aux + 8;     // the tile's poisoned-slot mask is published
  const uint32_t prep_done = mask_full + 8;     // [ST] self_prep: the stage holds K', V', c0, mask
  const uint32_t qk_empty = prep_done + 8 * ST;  // [ST]: the stage's S' MMA has read Q and K'
  // (in_empty: its P V' has read V' -- the Q / K' half of a stage refills a PV earlier)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Cfg::SMEM_BAR + 8 * Cfg::NUM_BARS);
  // [it % 2]: bit s = slot s of tile it holds a non-finite V' row
  // per tile it, slot it & 3: written up to two tiles ahead of the epilogue that reads it
  volatile uint32_t* bad_mask = tmem_holder + 1;                 // [4]
  int* c0s = reinterpret_cast<int*>(tmem_holder + 5);            // [4][8]
  unsigned* vmx = reinterpret_cast<unsigned*>(c0s + 32);         // [9] (prep scratch)
  const int warp = static_cast<int>(warp_id());
  const int lane = threadIdx.x & 31;
  const int W = p.W;                                // slot stride (rows / keys)
  const int ntiles = (p.BH + p.P - 1) / p.P;

  if (threadIdx.x == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(in_full + 8 * st, 1);
      mbar_init(in_empty + 8 * st, 1);
      mbar_init(qk_empty + 8 * st, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(t_full, 1);
    mbar_init(t_empty, 4);
    mbar_init(aux, 1);
    mbar_init(mask_full, 1);
    for (int st = 0; st < ST; ++st) mbar_init(prep_done + 8 * st, 1);
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
        mbar_expect_tx(in_full + 8 * st, 3 * Cfg::NBOX * nseq * p.N * 128);
        for (int sl = 0; sl < nseq; ++sl) {
          const int r = (seq0 + sl) * p.N;  // flat row of the sequence
          for (int bx = 0; bx < Cfg::NBOX; ++bx) {
            const uint32_t off = bx * Cfg::BOX_BYTES + sl * W * 128;
            tma_load_3d(base + off, &tm_q, in_full + 8 * st, bx * 64, r, 0);
            tma_load_3d(base + Cfg::TILE_BYTES + off, &tm_kp, in_full + 8 * st, bx * 64, r, 0);
          }
        }
        mbar_wait(in_empty + 8 * st, ((it / ST) & 1) ^ 1);
        for (int sl = 0; sl < nseq; ++sl) {
          const int r = (seq0 + sl) * p.N;
          for (int bx = 0; bx < Cfg::NBOX; ++bx)
            tma_load_3d(base + 2 * Cfg::TILE_BYTES + bx * Cfg::BOX_BYTES + sl * W * 128, &tm_v,
                        in_full + 8 * st, bx * 64, r, 0);
        }
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
      // self_prep: the softmax warps turn K, V into K', V' in place first (and find the
      // non-finite slots); else the stage holds the pre-pass output as loaded
      if (self_prep) mbar_wait(prep_done + 8 * st, (it / ST) & 1);
      else mbar_wait(in_full + 8 * st, (it / ST) & 1);
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
      uint32_t bad = self_prep ? bad_mask[it & 3] : 0u;  // (self_prep: from the prep)
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
      mbar_wait(p_full, it & 1);
      if (leader) PK_TR(1, it, 1);
      // publish the mask (release) only now: the softmax has finished tile it - 1 (p_full),
      // so mask_full is never two phases ahead of its reader and slot it & 1 is free
      if (leader) {
        if (!self_prep) bad_mask[it & 3] = bad;
        mbar_arrive(mask_full);
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
      const float l = W <= 32  ? row_softmax<16, MODE>(t_s, quad, lo, hi, p.qk_scale)
                      : W == 64 ? row_softmax<32, MODE>(t_s, quad, lo, hi, p.qk_scale)
                                : row_softmax<64, MODE>(t_s, quad, lo, hi, p.qk_scale);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (tr0) PK_TR(0, it, 2);
      if (tr0) PK_TR(0, it, 3);
      // epilogue: O = T 2^c0 / l (global recovering, pasa.cpp:184-194)
      const int c0 = MODE != kModePasa || !row_ok ? 0
                     : self_prep ? c0s[8 * (it & 3) + sl] : pasa_inflation(p.N, p.vmax[seq0 + sl]);
      const float inv_l = __fmul_rn(__frcp_rn(l), ldexpf(1.0f, c0));
      mbar_wait(mask_full, it & 1);
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
      uint16_t* dst = p.out + (static_cast<long long>(seq0 + sl) * p.N + rr) * D;
#pragma unroll
      for (int i = 0; i < D / 2; i += 4) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half a = __float2half_rn(__fmul_rn(lo_f(tv[i + k]), inv_l));
          const __half c = __float2half_rn(__fmul_rn(hi_f(tv[i + k]), inv_l));
          w[k] = h2_as_u32(__halves2half2(a, c));
        }
        if (row_ok) *reinterpret_cast<uint4*>(dst + 2 * i) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_PREP));
    // ---- the pre-pass of every tile (self_prep), as soon as its stage has landed: runs
    // ahead of the softmax, which it never waits for (the MMA warp waits for prep_done)
    int it = 0;
    for (int tile = blockIdx.x; self_prep && tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % ST;
      self_prep_stage<D>(sb + st * Cfg::STAGE_BYTES, p, min(p.P, p.BH - tile * p.P), c0s + 8 * (it & 3),
                         vmx, bad_mask + (it & 3), in_full + 8 * st, (it / ST) & 1, it);
      if (threadIdx.x == 256) mbar_arrive(prep_done + 8 * st);  // (after the prep's last barrier)
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

template <int D, int MODE>
static cudaError_t launch_packed_t(const CUtensorMap& tq, const CUtensorMap& tk,
                                   const CUtensorMap& tv, const PackedParams& p,
                                   cudaStream_t stream) {
  using Cfg = PackedCfg<D>;
  cudaError_t e = cudaFuncSetAttribute(pasa_fwd_packed_kernel<D, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = (p.BH + p.P - 1) / p.P;  // p.P = 128 / p.W sequences per tile
  const int sms = current_sm_count();  // the launching (current) device
  const int per_sm = D == 64 ? 2 : 1;  // shared memory: 2 x 98 KB (d = 64), 194 KB (d = 128)
  const int grid = tiles < per_sm * sms ? tiles : per_sm * sms;
  pasa_fwd_packed_kernel<D, MODE><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_packed(int D, int mode, const CUtensorMap& tq, const CUtensorMap& tk,
                              const CUtensorMap& tv, const PackedParams& p, cudaStream_t stream) {
  if (D == 64) return mode == kModePasa ? launch_packed_t<64, kModePasa>(tq, tk, tv, p, stream)
                                        : launch_packed_t<64, kModeFa16>(tq, tk, tv, p, stream);
  if (D == 128) return mode == kModePasa ? launch_packed_t<128, kModePasa>(tq, tk, tv, p, stream)
                                         : launch_packed_t<128, kModeFa16>(tq, tk, tv, p, stream);
  return cudaErrorInvalidValue;
}

}  // namespace pasa_b200
