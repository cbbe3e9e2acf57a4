// pasa_fwd.cu -- the fused PASA forward kernel for sm_100a.
//
// One CTA owns NT = 2 query tiles of 128 rows that share one KV head (GQA
// groups and neighbouring query tiles are paired), so every K'/V tile staged
// in shared memory feeds two tensor-core tiles.  Warp roles:
//
//   warp 0      TMA producer: Q tiles once, then a K'/V ring (2 stages each)
//   warp 1      MMA issuer (one elected lane) + TMEM owner (512 columns)
//   warps 2-3   idle (warpgroup 0 gives its registers away via setmaxnreg)
//   warps 4-11  softmax/correction for tile 0: two threads per row (warps
//               4-7 hold S' columns 0-63, warps 8-11 columns 64-127)
//   warps 12-19 the same for tile 1
//
// Per KV block j and tile t (reference pasa.cpp:256-278, Algorithm 1):
//   S'_t  = Q_t K'_j^T      tcgen05.mma kind::f16, SS, F16 accumulator in TMEM
//   softmax WG: tcgen05.ld S' (packed half2), row max / FP32 row mean,
//   pseudo-average recursion, corrected max, P = 2^(2(S' - c_j)) (f16x2 MUFU;
//   S' is stored in units of log2(e)/2),
//   tcgen05.st P back over the S' columns (packed 2 x f16 per column)
//   T_t   = P V_j           tcgen05.mma kind::f16, TS (P from TMEM), F16 acc
//   softmax WG: O <- e_prev * O + T in half2 registers (HFMA2)
// Epilogue ("global recovering"): O * 2^c0 / l, fp16 store (V' = V 2^-c0).
//
// Numerics are documented in DESIGN.md section 4 and restated on the CPU in
// oracle/pasa_oracle.c:orc_model_pasa (the tight oracle for this kernel).
#include <cuda.h>
#include <cuda_fp16.h>

#include "pasa_kernels.cuh"
#include "sm100.cuh"

namespace pasa_b200 {
using namespace sm100;

// PASA_TRACE (profiling builds only): CTAs whose blockIdx.x == 0 and blockIdx.y
// < kTraceCtas record clock64() at fixed points of the first kTraceIters
// blocks -- per softmax warpgroup (warp quadrant 0, lane 0) and for the MMA
// issuer -- into p.trace[cta][role][iter][event].
// Alternate the two softmax warpgroups' exp passes (named barriers 1, 2).  Pays at
// d = 64 (+12 %: the exp passes dominate); at d = 128, with P released to the PV MMA in
// parts, letting both tiles' exp passes overlap is faster (+2-3 %, tools/variants.py).
#ifndef PASA_PINGPONG
#define PASA_PINGPONG 0
#endif
#ifndef PASA_PINGPONG_D64
#define PASA_PINGPONG_D64 1
#endif
template <int D>
constexpr bool kPingPong = (D == 64 ? PASA_PINGPONG_D64 : PASA_PINGPONG) != 0;
#ifndef PASA_DYN_ORDER
#define PASA_DYN_ORDER 1
#endif
// One exp pair in kPolyEvery on the FMA-pipe polynomial (0: MUFU only).  d = 128
// balances MUFU against issue slots at 8 (round 2, with the TMA-stored epilogue: +1-2 % over
// 6 at Qwen 16K, 10 and MUFU-only lose 2-4 %; round 1: +2-3 % over 4); at d = 64 the FMA pipe and the
// issue slots are shared with twice the softmax work per FLOP and MUFU-only wins
// (measured: tools/variants.py, +6 % at d = 64 over 1/4; 1/8 and 1/16 lose 9-10 %).
#ifndef PASA_POLY_EVERY
#define PASA_POLY_EVERY 8
#endif
#ifndef PASA_POLY_EVERY_D64
#define PASA_POLY_EVERY_D64 0
#endif
template <int D>
constexpr int kPolyEvery = D == 64 ? PASA_POLY_EVERY_D64 : PASA_POLY_EVERY;
// Pass 2 stores P in kPParts parts, each released to the PV MMA on its own mbarrier,
// so the tensor core starts PV on a part while the exp of the next part runs
// (measured, tools/variants.py: d = 128 best at 4 parts, d = 64 at 2).
#ifndef PASA_PPARTS
#define PASA_PPARTS 4
#endif
#ifndef PASA_PPARTS_D64
#define PASA_PPARTS_D64 2
#endif
template <int D>
constexpr int kPParts = D == 64 ? PASA_PPARTS_D64 : PASA_PPARTS;
static_assert(PASA_PPARTS == 1 || PASA_PPARTS == 2 || PASA_PPARTS == 4, "P parts");
static_assert(PASA_PPARTS_D64 == 1 || PASA_PPARTS_D64 == 2 || PASA_PPARTS_D64 == 4, "P parts");
// setmaxnreg split of the per-CTA register pool (640 x 96 = 61440 at launch):
// warpgroup 0 (TMA, MMA, 2 idle warps) drops to PASA_WG0_REGS, the four softmax
// warpgroups rise to PASA_SM_REGS; 128 * WG0 + 512 * SM <= 61440.
#ifndef PASA_SPLIT_ISSUE_D64
#define PASA_SPLIT_ISSUE_D64 1
#endif
#ifndef PASA_WG0_REGS
#define PASA_WG0_REGS 56
#endif
#ifndef PASA_SM_REGS
#define PASA_SM_REGS 104
#endif
static_assert(128 * PASA_WG0_REGS + 512 * PASA_SM_REGS <= 61440, "register pool");
#define PASA_STR2(x) #x
#define PASA_STR(x) PASA_STR2(x)

[[maybe_unused]] constexpr int kTraceCtas = 4, kTraceIters = 32, kTraceEvents = 10, kTraceRoles = 3;
// ... followed by a per-block row-state dump (CTA (0,0), tile 0, row kTraceRow,
// half 0): kStateIters x 8 floats {mloc, ssum, fnew, mnew, cj, ep, lsum, l_run}.
[[maybe_unused]] constexpr int kTraceRow = 2, kStateIters = 512;
[[maybe_unused]] constexpr int kTraceStateOffset =
    kTraceCtas * kTraceRoles * kTraceIters * kTraceEvents;
#ifdef PASA_TRACE
#define PASA_TR(role, it, ev)                                                                  \
  do {                                                                                        \
    if (p.trace && blockIdx.x == 0 && blockIdx.y < kTraceCtas && (it) < kTraceIters)          \
      p.trace[((blockIdx.y * kTraceRoles + (role)) * kTraceIters + (it)) * kTraceEvents + (ev)] = \
          clock64();                                                                          \
  } while (0)
#define PASA_STATE(j, k, val)                                                                \
  do {                                                                                      \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && t == 0 && h == 0 && row == kTraceRow && \
        (j) < kStateIters)                                                                  \
      reinterpret_cast<float*>(p.trace + kTraceStateOffset)[(j) * 8 + (k)] = (val);          \
  } while (0)
#else
#define PASA_STATE(j, k, val) \
  do {                        \
  } while (0)
#define PASA_TR(role, it, ev) \
  do {                        \
  } while (0)
#endif

// d = 128 (no free TMEM columns in the loop): the pseudo-average from the tensor core in a
// PROLOGUE -- G_t[r][j] = q_r . (K'sum_j hi + K'sum_j lo) as ONE GEMM over K = 2 D,
// A = [Q_t | Q_t], B row j = [hi_j | lo_j], FP32 accumulator, up to 128 blocks per GEMM
// (N <= 128) in tile t's T columns, so S'(0) runs beside it in the S' columns -- read out
// to an L2-resident scratch slot of this SM and read back one float per row and block,
// instead of 64 FP32 adds per thread and block in pass 1.  Off by default (PASA_PRO_SUM in
// pasa_kernels.cuh): the exact mean cuts the RMSE by a quarter (uniform(30, 0.5) at Qwen 16K:
// 1.07e-3 -> 7.9e-4), but the prologue's 128 KB of scratch stores per CTA cost 2-5 % of
// throughput, and the pass-1 adds it removes are not what sets the block period.
constexpr int kGChunk = 128;  // blocks per prologue GEMM (N = 128 FP32 columns = a T region)

// K'/V' pipeline stages at d = 64 (d = 128 fills shared memory at two); 3 or 4 at d = 64
// measured 1.5 % slower than 2 (tools/variants.py): the loads are not what the tiles wait on
#ifndef PASA_STAGES_D64
#define PASA_STAGES_D64 2
#endif
template <int D>
struct FwdCfg {
  static constexpr int NT = 2;
  static constexpr int KS = D == 64 ? PASA_STAGES_D64 : 2;
  static constexpr int VS = D == 64 ? PASA_STAGES_D64 : 2;
  static constexpr int NBOX = D / 64;                     // 128-byte swizzle boxes per row
  static constexpr int BOX_BYTES = kTile * 128;           // 128 rows x 64 halves
  static constexpr int TILE_BYTES = NBOX * BOX_BYTES;     // one 128 x D fp16 tile
  static constexpr int SMEM_Q = 0;
  static constexpr int SMEM_K = SMEM_Q + NT * TILE_BYTES;
  static constexpr int SMEM_V = SMEM_K + KS * TILE_BYTES;
  // PASA with the tensor-core row sum (pasa_tc_rowsum): per K' stage the block sums
  // as the N = 16 B operand of G, rows (hi, lo) of a zeroed 16-row box per 64 columns
  static constexpr bool TCSUM = pasa_tc_rowsum(D);
  static constexpr int KS_BOX = 2048;
  static constexpr int SMEM_KS = SMEM_V + VS * TILE_BYTES;
  static constexpr int SMEM_BAR = SMEM_KS + (TCSUM ? KS * NBOX * KS_BOX : 0);
  static constexpr int NUM_BARS = NT + 2 * KS + 2 * VS + (3 + kPParts<D>) * NT + 3 + NT;
  static constexpr int HALVES = 2;  // threads per row: each owns 64 S' columns, D/2 outputs
  static constexpr int SMEM_XCH = SMEM_BAR + NUM_BARS * 8 + 16;  // row max/sum exchange
  static constexpr int XCH_BYTES = 2 * NT * HALVES * kTile * 8;  // [j&1][t][half][row] float2
  static constexpr int SMEM_DIAG = SMEM_XCH + XCH_BYTES;  // RunDiagnostics: 5 words / thread
  static constexpr int DIAG_BYTES = NT * HALVES * 128 * 5 * 4;
  static constexpr int SMEM_BYTES = SMEM_DIAG + DIAG_BYTES + 1024;
  static constexpr int THREADS = 128 + NT * HALVES * 128;  // WG0: TMA, MMA, 2 idle; 4 softmax WGs
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t TMEM_TILE = 256;               // S/P at +0, T at +128
  static constexpr uint32_t TM_G = 128 + D;                // G (TCSUM): 16 free columns after T
};

namespace {

__device__ __forceinline__ float lo_f(uint32_t u) { return __low2float(u32_as_h2(u)); }
__device__ __forceinline__ float hi_f(uint32_t u) { return __high2float(u32_as_h2(u)); }

struct TileInfo {
  int valid, i, hq, nblk;
};

__device__ __forceinline__ TileInfo tile_info(const FwdParams& p, int hkv, int idx, bool causal) {
  TileInfo ti;
  ti.valid = idx < p.tiles_per_kv;
  ti.i = p.tile_hi - 1 - idx / p.group;  // longest (causal) tiles first
  ti.hq = hkv * p.group + idx % p.group;
  // causal, bottom-right aligned: query row r sees keys <= r + (S2 - S1); the tile runs the
  // blocks up to the one holding its last valid row's last key (blocks masked for every
  // row of the tile are skipped; a row may still see a block of the tile fully masked)
  const int last = min(p.S1, (ti.i + 1) * kTile) - 1;
  const int kb = p.s2 == kTile ? (last + p.qoff) / kTile : (last + p.qoff) / p.s2;
  ti.nblk = ti.valid ? (causal ? min(kb + 1, p.nkv) : p.nkv) : 0;
  return ti;
}

// Column mask: keep lo/hi of pair i when its columns are < lim (lim = row + 1
// on the causal diagonal block, s2 for a short KV block).
__device__ __forceinline__ uint32_t col_keep(int i, int lim) {
  return (2 * i + 1 < lim) ? 0xFFFFFFFFu : (2 * i < lim ? 0x0000FFFFu : 0u);
}

// Pass 1 over this thread's half of an S' row (32 packed pairs, global pair
// index pbase + i): max over unmasked columns and the FP32 sum over all of its
// columns.  Eight sum chains (pair i -> chain i % 4, lo/hi) and four max
// chains keep the dependency depth at 8; the reduction order is restated in
// oracle/pasa_oracle.c (orc_model_pasa).
template <bool DIAG, int NP, bool SUM = true>
__device__ __forceinline__ void row_max_sum(const uint32_t* s, int lim, int pbase, float& mloc,
                                            float& ssum) {
  float acc[8];
  uint32_t mx[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) mx[k] = 0xFC00FC00u;  // (-inf, -inf)
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const uint32_t v = s[i];
    if (SUM) {
      acc[2 * (i & 3)] = add_lo_f16(acc[2 * (i & 3)], v);
      acc[2 * (i & 3) + 1] = add_hi_f16(acc[2 * (i & 3) + 1], v);
    }
    uint32_t vm = v;
    if (DIAG) {
      const uint32_t keep = col_keep(pbase + i, lim);
      vm = (v & keep) | (0xFC00FC00u & ~keep);
    }
    mx[i & 3] = h2_as_u32(__hmax2(u32_as_h2(mx[i & 3]), u32_as_h2(vm)));
  }
  const uint32_t m01 = h2_as_u32(__hmax2(u32_as_h2(mx[0]), u32_as_h2(mx[1])));
  const uint32_t m23 = h2_as_u32(__hmax2(u32_as_h2(mx[2]), u32_as_h2(mx[3])));
  const uint32_t m = h2_as_u32(__hmax2(u32_as_h2(m01), u32_as_h2(m23)));
  mloc = fmaxf(lo_f(m), hi_f(m));
  ssum = __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                   __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
}

// Pass 2: P = 2^(S' - c_j) in place (masked -> 0) and its FP32 sum, same
// eight-chain order as pass 1.  Three pairs in four use MUFU ex2.approx.f16x2,
// one the FMA-pipe polynomial (sm100.cuh); both are within 1 ulp of 2^x.
template <int D, bool DIAG, int I0, int I1>
__device__ __forceinline__ void row_exp_range(uint32_t* s, int lim, int pbase, uint32_t cj2,
                                              uint32_t scale2, float* acc) {
#pragma unroll
  for (int i = I0; i < I1; ++i) {
    // x = fl16(S * scale - c) in one HFMA2 -- FA16: scale = log2e/alpha, c = m*scale;
    // PASA: scale = 2, c = 2 c_j (scores are stored in units of log2(e)/2, so the FP16
    // store holds 0.72x the reference's scores), or -- rows with |c_j| > 32752 -- S
    // already holds fl16(S' - c_j) and c = 0: x = 2 fl16(S' - c_j), an exact doubling.
    const uint32_t x = h2_as_u32(__hfma2(u32_as_h2(s[i]), u32_as_h2(scale2), u32_as_h2(cj2)));
    // one pair in kPolyEvery on the FMA pipe, the rest on MUFU: balances MUFU time
    // (8 cycles / pair / SMSP) against issue slots (poly ~11 vs MUFU 3 per pair)
    constexpr int PE = kPolyEvery<D>;
    uint32_t pv = (PE > 0 && (i % (PE > 0 ? PE : 1)) == PE - 1)
                      ? ex2_poly_f16x2(x)
                      : ex2_f16x2(x);
    if (DIAG) pv &= col_keep(pbase + i, lim);
    acc[2 * (i & 3)] = add_lo_f16(acc[2 * (i & 3)], pv);
    acc[2 * (i & 3) + 1] = add_hi_f16(acc[2 * (i & 3) + 1], pv);
    s[i] = pv;
  }
}

// Pass 2 over a half row in kPParts parts: part(q) runs after pairs [q NP/kPParts,
// (q+1) NP/kPParts) are done -- the caller stores them to TMEM so the PV MMA can
// start on those keys while the exp continues.
template <int D, bool DIAG, int NP, int Q = 0, class Part>
__device__ __forceinline__ void row_exp_parts(uint32_t* s, int lim, int pbase, uint32_t cj2,
                                              uint32_t scale2, float* acc, Part&& part) {
  constexpr int W = NP / kPParts<D>;
  row_exp_range<D, DIAG, Q * W, (Q + 1) * W>(s, lim, pbase, cj2, scale2, acc);
  part(Q);
  if constexpr (Q + 1 < kPParts<D>)
    row_exp_parts<D, DIAG, NP, Q + 1>(s, lim, pbase, cj2, scale2, acc, part);
}
template <int D, bool DIAG, int NP, class Part>
__device__ __forceinline__ float row_exp_sum(uint32_t* s, int lim, int pbase, uint32_t cj2,
                                             uint32_t scale2, Part&& part) {
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  row_exp_parts<D, DIAG, NP>(s, lim, pbase, cj2, scale2, acc, part);
  return __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                   __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
}

// RunDiagnostics (attention.cpp:25-36, track_store) over this thread's stored
// scores of one block (masked columns excluded), merged into its shared-memory slot
// {finite min, finite max, +inf, -inf, NaN}.  Diagnostic mode only.
template <int NP>
__device__ __forceinline__ void track_store_block(const uint32_t* s, int lim, int pbase, bool masked,
                                               float* slot) {
  float mn = slot[0], mx = slot[1];
  uint32_t pinf = __float_as_uint(slot[2]), ninf = __float_as_uint(slot[3]),
           nan = __float_as_uint(slot[4]);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      if (masked && 2 * (pbase + i) + half >= lim) continue;
      const float v = half ? hi_f(s[i]) : lo_f(s[i]);
      if (isnan(v)) ++nan;
      else if (isinf(v)) (v > 0.f ? ++pinf : ++ninf);
      else { mn = fminf(mn, v); mx = fmaxf(mx, v); }
    }
  }
  slot[0] = mn; slot[1] = mx;
  slot[2] = __uint_as_float(pinf); slot[3] = __uint_as_float(ninf); slot[4] = __uint_as_float(nan);
}

__device__ __forceinline__ void atomic_min_f(float* a, float v) {
  if (v >= 0.f) atomicMin(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMax(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_f(float* a, float v) {
  if (v >= 0.f) atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMin(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}

// Device-side RunDiagnostics accumulator (the layout of pasa_b200_diag).
struct DiagAccum {
  unsigned long long out_nonfinite, out_total, store_pos_inf, store_neg_inf, store_nan;
  float store_finite_min, store_finite_max;
};

}  // namespace

template <int D, bool CAUSAL, int MODE, bool DIAGNOSE>
__global__ void __launch_bounds__(FwdCfg<D>::THREADS, 1)
    pasa_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_kp,
                    const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_ks,
                    const __grid_constant__ CUtensorMap tm_o, const FwdParams p) {
  constexpr bool kTcSum = FwdCfg<D>::TCSUM && MODE == kModePasa;
  constexpr bool kProSum = pasa_prologue_rowsum(D) && MODE == kModePasa;
  // MMA issue: one warp for both tiles (PV of the first-ready tile, then its S'(j+1);
  // best at D = 128, where an S' MMA queued ahead of the other tile's PV stalls it) or,
  // at D = 64, one warp per tile (+5 %, tools/variants.py).
  constexpr bool kSplitIssue = PASA_SPLIT_ISSUE_D64 && D == 64;
  using Cfg = FwdCfg<D>;
  constexpr int NT = Cfg::NT, KS = Cfg::KS, VS = Cfg::VS;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (SW128 tiles) as a 32-bit shared address; barriers and tiles are
  // constant offsets from it, so the loops address them without generic-pointer conversions
  const uint32_t sb = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sb - smem_u32(smem_raw));  // generic view of the same base
  const uint32_t q_full = sb + Cfg::SMEM_BAR;  // mbarriers, 8 bytes each
  const uint32_t k_full = q_full + 8 * NT;
  const uint32_t k_empty = k_full + 8 * KS;
  const uint32_t v_full = k_empty + 8 * KS;
  const uint32_t v_empty = v_full + 8 * VS;
  const uint32_t s_full = v_empty + 8 * VS;
  const uint32_t t_full = s_full + 8 * NT;
  const uint32_t t_empty = t_full + 8 * NT;
  const uint32_t p_part = t_empty + 8 * NT;  // [q][t]: P of part q stored (pass 2 in kPParts parts)
  // prologue pseudo-average (kProSum): K'-sum chunk loaded / consumed, G in TMEM / read out
  const uint32_t ks_full = p_part + 8 * kPParts<D> * NT;
  const uint32_t ks_empty = ks_full + 8, g_free = ks_full + 16, g_full = ks_full + 24;  // g_full[t]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + Cfg::SMEM_BAR + 8 * Cfg::NUM_BARS);

  const int warp = static_cast<int>(warp_id());
  const int lane = threadIdx.x & 31;
  // Causal: heads vary fastest so the longest (LPT-first) units of every head
  // start first.  Non-causal: units vary fastest so the CTAs in flight share
  // one head's K'/V in L2 instead of streaming all heads at once.
  const int head_id = CAUSAL ? blockIdx.x : blockIdx.y;
  const int unit = CAUSAL ? blockIdx.y : blockIdx.x;
  const int b = head_id / p.Hkv;
  const int hkv = head_id % p.Hkv;
  TileInfo tl[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) tl[t] = tile_info(p, hkv, unit * NT + t, CAUSAL);
  int nmax = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) nmax = max(nmax, tl[t].nblk);
  const int nch = kProSum ? (nmax + kGChunk - 1) / kGChunk : 0;  // prologue G chunks

  if (threadIdx.x == 0) {
    for (int t = 0; t < NT; ++t) {
      mbar_init(q_full + 8 * (t), 1);
      mbar_init(s_full + 8 * (t), 1);
      for (int q = 0; q < kPParts<D>; ++q) mbar_init(p_part + 8 * (q * NT + t), 4 * Cfg::HALVES);
      mbar_init(t_full + 8 * (t), 1);
      mbar_init(t_empty + 8 * (t), 4 * Cfg::HALVES);
    }
    for (int s = 0; s < KS; ++s) {
      mbar_init(k_full + 8 * (s), 1);
      mbar_init(k_empty + 8 * (s), kSplitIssue ? NT : 1);  // one release per MMA issuer
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(v_full + 8 * (s), 1);
      mbar_init(v_empty + 8 * (s), kSplitIssue ? NT : 1);
    }
    mbar_init(ks_full, 1);
    mbar_init(ks_empty, 1);
    for (int t = 0; t < NT; ++t) mbar_init(g_full + 8 * t, 1);
    mbar_init(g_free, 4 * Cfg::HALVES * NT);  // every softmax warp, every chunk
    fence_barrier_init();
  }
  if (kTcSum) {  // rows 2-15 of the K'-sum boxes read as zero (TMA writes rows 0-1)
    uint4* z = reinterpret_cast<uint4*>(smem + Cfg::SMEM_KS);
    for (int e = threadIdx.x; e < KS * Cfg::NBOX * Cfg::KS_BOX / 16; e += blockDim.x)
      z[e] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (p.s2 < kTile) {
    // Short KV blocks: TMA fills rows [0, s2) of each stage, the rest must read as
    // zero for the whole kernel (zero K' rows give S' = 0, zero V' rows add nothing).
    uint4* z = reinterpret_cast<uint4*>(smem + Cfg::SMEM_K);
    for (int e = threadIdx.x; e < (KS + VS) * Cfg::TILE_BYTES / 16; e += blockDim.x)
      z[e] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Everything above touches only this CTA's shared memory, TMEM and the kernel
  // parameters; the inputs (Q, K', V', max|V|) may come from the previous grid.
  pdl_wait();
#ifdef PASA_TRACE_CTA  // per-CTA lifetime (globaltimer ns) and SM id: p.trace[4 * linear id]
  unsigned long long cta_t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_t0));
#endif
  // A 512-column allocation is the whole TMEM of the SM, so it starts at lane 0, column 0:
  // the base is the constant 0 (no per-thread register, no spill, uniform addressing).
  static_assert(Cfg::TMEM_COLS == 512, "tmem_base = 0 needs the full allocation");
  constexpr uint32_t tmem_base = 0;
  (void)tmem_holder;

  // Register budget: 640 threads x 96 at launch = 61440 per CTA; setmaxnreg
  // moves registers only within the CTA: 128 x 56 + 512 x 104 = 60416.
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 " PASA_STR(PASA_WG0_REGS) ";");
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_kp);
      tma_prefetch(&tm_v);
      if (kTcSum || kProSum) tma_prefetch(&tm_ks);
      auto load_q = [&](int t) {
        if (!tl[t].valid) return;
        mbar_expect_tx(q_full + 8 * (t), Cfg::TILE_BYTES);
        for (int bx = 0; bx < Cfg::NBOX; ++bx)
          // BHSD (c, s, b Hq + h); BSHD (h D + c, s, b) on the {Hq D, S1, B} map
          tma_load_3d(sb + Cfg::SMEM_Q + t * Cfg::TILE_BYTES + bx * Cfg::BOX_BYTES, &tm_q,
                      q_full + 8 * (t), (p.q_bshd ? tl[t].hq * D : 0) + bx * 64, tl[t].i * kTile,
                      p.q_bshd ? b : b * p.Hq + tl[t].hq);
      };
      // Start-up order Q_0, K'(0), Q_1, V'(0): the CTA's first S' waits for the loads
      // ahead of it (per-SM load bandwidth sets the start-up time), so tile 0's S'(0)
      // issues once 2/3 of the first S' operands have landed.  The prologue GEMM
      // (kProSum) reads every Q tile first.
      const bool q_early = kProSum || nmax == 0;
      for (int t = 0; t < NT; ++t)
        if (t == 0 || q_early) load_q(t);
      // Prologue (kProSum): the head's K' block sums, 128 blocks at a time, into the V'
      // stages (free until the first V' load): box (hl, bx) = the hi (hl = 0) or lo rows,
      // columns [64 bx, 64 bx + 64), 128 blocks x 128 B (SW128, K-major like K').
      for (int c = 0; c < nch; ++c) {
        mbar_wait(ks_empty, (c & 1) ^ 1);
        mbar_expect_tx(ks_full, 2 * Cfg::NBOX * 128 * p.ks_rows);  // whole boxes (OOB rows = 0)
        for (int hl = 0; hl < 2; ++hl)
          for (int bx = 0; bx < Cfg::NBOX; ++bx)
            tma_load_4d(sb + Cfg::SMEM_V + (hl * Cfg::NBOX + bx) * Cfg::BOX_BYTES, &tm_ks, ks_full,
                        bx * 64, hl, c * kGChunk, b * p.Hkv + hkv);
      }
      for (int j = 0; j < nmax; ++j) {
        const int ks = j % KS, vs = j % VS;
        mbar_wait(k_empty + 8 * (ks), ((j / KS) & 1) ^ 1);
        mbar_expect_tx(k_full + 8 * (ks), Cfg::NBOX * 128 * (p.s2 + (kTcSum ? 2 : 0)));
        for (int bx = 0; bx < Cfg::NBOX; ++bx) {
          tma_load_3d(sb + Cfg::SMEM_K + ks * Cfg::TILE_BYTES + bx * Cfg::BOX_BYTES, &tm_kp,
                      k_full + 8 * (ks), (p.kv_bshd ? hkv * D : 0) + bx * 64, j * p.s2,
                      p.kv_bshd ? b : b * p.Hkv + hkv);
          if (kTcSum)
            tma_load_3d(sb + Cfg::SMEM_KS + (ks * Cfg::NBOX + bx) * Cfg::KS_BOX, &tm_ks,
                        k_full + 8 * (ks), bx * 64, 2 * j, b * p.Hkv + hkv);
        }
        if (j == 0 && !q_early)
          for (int t = 1; t < NT; ++t) load_q(t);
        if (kProSum && j == 0 && nch > 0) mbar_wait(ks_empty, (nch - 1) & 1);  // V area free
        mbar_wait(v_empty + 8 * (vs), ((j / VS) & 1) ^ 1);
        mbar_expect_tx(v_full + 8 * (vs), Cfg::NBOX * 128 * p.s2);
        for (int bx = 0; bx < Cfg::NBOX; ++bx)
          tma_load_3d(sb + Cfg::SMEM_V + vs * Cfg::TILE_BYTES + bx * Cfg::BOX_BYTES, &tm_v,
                      v_full + 8 * (vs), (p.kv_bshd ? hkv * D : 0) + bx * 64, j * p.s2,
                      p.kv_bshd ? b : b * p.Hkv + hkv);
      }
    }
  } else if (kSplitIssue ? warp <= NT : warp == 1) {
   if constexpr (kSplitIssue) {
    // ------------------------------------------------------------ MMA issuers
    // Warp 1 issues tile 0's MMAs, warp 2 tile 1's (tcgen05.commit tracks the issuing
    // thread's MMAs), each a linear sequence with blocking waits, so neither tile's
    // waits hold up the other's MMAs:
    //   S'(0) [G(0)] | PV(0) parts, S'(1) [G(1)] | PV(1) parts, S'(2) [G(2)] | ...
    // G(j) (tensor-core row sum, kTcSum): Q K'sum_j, M = 128, N = 16, FP32 accumulator,
    // B rows = (hi, lo) of the block's K' column sums -> TMEM columns TM_G + {0, 1}.
    const int t = warp - 1;
    if (elect_one()) {
      constexpr uint32_t kIdS = idesc_f16(128, 128, 0, 0, 0);  // F16 acc, K-major A/B
      constexpr uint32_t kIdPV = idesc_f16(128, D, 0, 0, 1);   // F16 acc, V MN-major
      constexpr uint32_t kIdG = idesc_f16(128, 16, 1, 0, 0);   // F32 acc, K-major A/B, N = 16
      const uint32_t s_tmem = tmem_base + t * Cfg::TMEM_TILE;
      const uint32_t o_tmem = s_tmem + 128;
      const uint32_t qa = sb + Cfg::SMEM_Q + t * Cfg::TILE_BYTES;
      auto issue_s = [&](int ks) {
        const uint32_t ka = sb + Cfg::SMEM_K + ks * Cfg::TILE_BYTES;
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32;
          umma_ss(s_tmem, smem_desc_sw128(qa + off, 16, 1024), smem_desc_sw128(ka + off, 16, 1024),
                  kIdS, s > 0);
        }
        if (kTcSum) {
          const uint32_t ga = sb + Cfg::SMEM_KS + ks * Cfg::NBOX * Cfg::KS_BOX;
#pragma unroll
          for (int s = 0; s < D / 16; ++s) {
            const uint32_t qoff = (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32;
            const uint32_t goff = (s / 4) * Cfg::KS_BOX + (s % 4) * 32;
            umma_ss(s_tmem + Cfg::TM_G, smem_desc_sw128(qa + qoff, 16, 1024),
                    smem_desc_sw128(ga + goff, 16, 1024), kIdG, s > 0);
          }
        }
      };
      // PV in kPParts parts: part q covers the K-steps whose keys pass 2 stored in its
      // part q (half h's pairs -> K-steps 4h + [q, q + 4/kPParts)), issued on p_part[q].
      auto issue_pv = [&](int vs, int part) {
        const uint32_t va = sb + Cfg::SMEM_V + vs * Cfg::TILE_BYTES;
        constexpr int SP = 4 / kPParts<D>;  // K-steps per half per part
#pragma unroll
        for (int k = 0; k < 2 * SP; ++k) {
          const int s = 4 * (k / SP) + part * SP + k % SP;
          umma_ts(o_tmem, s_tmem + s * 8, smem_desc_sw128(va + s * 2048, Cfg::BOX_BYTES, 1024),
                  kIdPV, part > 0 || k > 0);
        }
      };
      const int nb = tl[t].nblk;
      if (nb > 0) {
        mbar_wait(q_full + 8 * t, 0);
        mbar_wait(k_full, 0);
        tc_fence_after();
        issue_s(0);
        tc_commit(s_full + 8 * t);
        tc_commit(k_empty);
      }
      for (int j = 0; j < nb; ++j) {
        const int vs = j % VS;
        PASA_TR(2, j, 4 * t + 0);
        mbar_wait(p_part + 8 * t, j & 1);
        PASA_TR(2, j, 4 * t + 1);
        mbar_wait(v_full + 8 * vs, (j / VS) & 1);
        mbar_wait(t_empty + 8 * t, (j & 1) ^ 1);  // T(j-1) read
        tc_fence_after();
        issue_pv(vs, 0);
        for (int q = 1; q < kPParts<D>; ++q) {
          mbar_wait(p_part + 8 * (q * NT + t), j & 1);
          tc_fence_after();
          issue_pv(vs, q);
        }
        PASA_TR(2, j, 4 * t + 2);
        tc_commit(t_full + 8 * t);
        tc_commit(v_empty + 8 * vs);
        if (j + 1 < nb) {
          const int ks = (j + 1) % KS;
          mbar_wait(k_full + 8 * ks, ((j + 1) / KS) & 1);
          tc_fence_after();
          issue_s(ks);
          tc_commit(s_full + 8 * t);
          tc_commit(k_empty + 8 * ks);
          PASA_TR(2, j, 4 * t + 3);
        }
      }
      // Blocks of the CTA this tile does not need (causal tiles differ in length):
      // release their K'/V stages in the producer's order so it can proceed.
      for (int j = nb; j < nmax; ++j) {
        mbar_wait(k_empty + 8 * (j % KS), ((j / KS) & 1) ^ 1);
        mbar_arrive(k_empty + 8 * (j % KS));
        mbar_wait(v_empty + 8 * (j % VS), ((j / VS) & 1) ^ 1);
        mbar_arrive(v_empty + 8 * (j % VS));
      }
    }
   } else {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t kIdS = idesc_f16(128, 128, 0, 0, 0);  // F16 acc, K-major A/B
      constexpr uint32_t kIdPV = idesc_f16(128, D, 0, 0, 1);   // F16 acc, V MN-major
      // S'(j) and, with the tensor-core row sum, G(j) = Q K'sum_j (M = 128, N = 16, FP32
      // accumulator; B rows = (hi, lo) of the block's K' column sums) -> this tile's S' row
      // sums in TMEM columns TM_G + {0, 1}, committed together on s_full.
      auto issue_s = [&](int t, int ks) {
        const uint32_t d_tmem = tmem_base + t * Cfg::TMEM_TILE;
        const uint32_t qa = sb + Cfg::SMEM_Q + t * Cfg::TILE_BYTES;
        const uint32_t ka = sb + Cfg::SMEM_K + ks * Cfg::TILE_BYTES;
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32;
          umma_ss(d_tmem, smem_desc_sw128(qa + off, 16, 1024), smem_desc_sw128(ka + off, 16, 1024),
                  kIdS, s > 0);
        }
        if (kTcSum) {
          constexpr uint32_t kIdG = idesc_f16(128, 16, 1, 0, 0);
          const uint32_t ga = sb + Cfg::SMEM_KS + ks * Cfg::NBOX * Cfg::KS_BOX;
#pragma unroll
          for (int s = 0; s < D / 16; ++s) {
            const uint32_t qoff = (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32;
            const uint32_t goff = (s / 4) * Cfg::KS_BOX + (s % 4) * 32;
            umma_ss(d_tmem + Cfg::TM_G, smem_desc_sw128(qa + qoff, 16, 1024),
                    smem_desc_sw128(ga + goff, 16, 1024), kIdG, s > 0);
          }
        }
      };
      // PV in kPParts parts: part q covers the K-steps whose keys pass 2 stored in its
      // part q (half h's pairs -> K-steps 4h + [q, q + 4/kPParts)), issued on p_part[q].
      auto issue_pv = [&](int t, int vs, int part) {
        const uint32_t d_tmem = tmem_base + t * Cfg::TMEM_TILE + 128;
        const uint32_t a_tmem = tmem_base + t * Cfg::TMEM_TILE;
        const uint32_t va = sb + Cfg::SMEM_V + vs * Cfg::TILE_BYTES;
        constexpr int SP = 4 / kPParts<D>;  // K-steps per half per part
#pragma unroll
        for (int k = 0; k < 2 * SP; ++k) {
          const int s = 4 * (k / SP) + part * SP + k % SP;
          umma_ts(d_tmem, a_tmem + s * 8, smem_desc_sw128(va + s * 2048, Cfg::BOX_BYTES, 1024),
                  kIdPV, part > 0 || k > 0);
        }
      };
      if (kProSum)
        for (int t = 0; t < NT; ++t)
          if (tl[t].valid) mbar_wait(q_full + 8 * (t), 0);
      // Prologue (kProSum): G_t = [Q_t | Q_t] [hi | lo]^T (K = 2 D) for 128 blocks at a
      // time into tile t's T columns [256 t + 128, 256 t + 128 + nb) (FP32), read out by the
      // softmax warps (g_free); S'(0) is issued after the last chunk's GEMMs, into the S'
      // columns, and runs while the last chunk is read out.
      for (int c = 0; c < nch; ++c) {
        mbar_wait(ks_full, c & 1);
        if (c > 0) mbar_wait(g_free, (c - 1) & 1);
        tc_fence_after();
        for (int t = 0; t < NT; ++t) {
          const int nb = min(kGChunk, tl[t].nblk - c * kGChunk);
          if (nb <= 0) continue;
          const uint32_t idg = idesc_f16(128, 16 * ((nb + 15) / 16), 1, 0, 0);
          const uint32_t qa = sb + Cfg::SMEM_Q + t * Cfg::TILE_BYTES;
#pragma unroll
          for (int s = 0; s < 2 * D / 16; ++s)
            umma_ss(tmem_base + t * Cfg::TMEM_TILE + 128,
                    smem_desc_sw128(qa + ((s % (D / 16)) / 4) * Cfg::BOX_BYTES + (s % 4) * 32, 16, 1024),
                    smem_desc_sw128(sb + Cfg::SMEM_V + (s / 4) * Cfg::BOX_BYTES + (s % 4) * 32, 16, 1024),
                    idg, s > 0);
          tc_commit(g_full + 8 * t);  // tile t's softmax reads out while tile t + 1's GEMM runs
        }
        for (int t = 0; t < NT; ++t)  // a tile without blocks in this chunk: nothing to wait for
          if (min(kGChunk, tl[t].nblk - c * kGChunk) <= 0) mbar_arrive(g_full + 8 * t);
        tc_commit(ks_empty);
      }
      if (nmax > 0) {
        mbar_wait(k_full + 8 * (0), 0);
        for (int t = 0; t < NT; ++t) {
          if (tl[t].nblk == 0) continue;
          mbar_wait(q_full + 8 * (t), 0);  // Q_1 lands after K'(0)
          tc_fence_after();
          issue_s(t, 0);
          tc_commit(s_full + 8 * (t));
        }
        tc_commit(k_empty + 8 * (0));
      }
      for (int j = 0; j < nmax; ++j) {
        const int vs = j % VS;
        mbar_wait(v_full + 8 * (vs), (j / VS) & 1);
        if (j == 0 && nch > 0) {  // PV(0) overwrites the last chunk's G columns
          mbar_wait(g_free, (nch - 1) & 1);
          tc_fence_after();
        }
        bool k_next = false;
        // Serve the tile whose first P part is ready first (no head-of-line blocking
        // when the two tiles' exp passes overlap).
        int first = 0;
        if (PASA_DYN_ORDER && j < tl[0].nblk && j < tl[1].nblk &&
            !mbar_test_wait(p_part + 8 * (0), j & 1) && mbar_test_wait(p_part + 8 * (1), j & 1))
          first = 1;
        for (int tt = 0; tt < NT; ++tt) {
          const int t = tt ^ first;
          if (j >= tl[t].nblk) continue;
          PASA_TR(2, j, 4 * t + 0);
          mbar_wait(p_part + 8 * (t), j & 1);
          PASA_TR(2, j, 4 * t + 1);
          mbar_wait(t_empty + 8 * (t), (j & 1) ^ 1);
          tc_fence_after();
          issue_pv(t, vs, 0);
          for (int q = 1; q < kPParts<D>; ++q) {
            mbar_wait(p_part + 8 * (q * NT + t), j & 1);
            tc_fence_after();
            issue_pv(t, vs, q);
          }
          PASA_TR(2, j, 4 * t + 2);
          tc_commit(t_full + 8 * (t));
          if (j + 1 < tl[t].nblk) {
            const int ks = (j + 1) % KS;
            if (!k_next) {
              mbar_wait(k_full + 8 * (ks), ((j + 1) / KS) & 1);
              tc_fence_after();
              k_next = true;
            }
            issue_s(t, ks);
            tc_commit(s_full + 8 * (t));
            PASA_TR(2, j, 4 * t + 3);
          }
        }
        tc_commit(v_empty + 8 * (vs));
        if (k_next) tc_commit(k_empty + 8 * ((j + 1) % KS));
      }
    }
   }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 " PASA_STR(PASA_SM_REGS) ";");
    // ------------------------------------------------------------ softmax WGs
    // Two threads per row: warps 4-7 / 8-11 hold columns 0-63 / 64-127 of
    // tile 0's rows, warps 12-15 / 16-19 those of tile 1.  Row max and sum are
    // exchanged through shared memory (named barrier per quadrant pair); each
    // thread keeps its own partial l and D/2 output columns.
    const int sw = warp - 4;
    const int t = sw / 8;
    const int h = (sw / 4) & 1;
    const int quad = warp % 4;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const TileInfo ti = tile_info(p, hkv, unit * NT + t, CAUSAL);
    const uint32_t t_s = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + t * Cfg::TMEM_TILE;
    const uint32_t t_t = t_s + 128;
    // exchange slots [parity][t][half][row] of float2, as shared-memory addresses
    const uint32_t xs_mine = sb + Cfg::SMEM_XCH + ((t * Cfg::HALVES + h) * kTile + row) * 8;
    const uint32_t xs_other = xs_mine + (1 - 2 * h) * kTile * 8;
    constexpr uint32_t kXPar = NT * Cfg::HALVES * kTile * 8;  // parity stride
    // plain C++ accesses (not asm volatile): the compiler schedules around them, and the
    // named barrier orders them (+3 % PASA, +10 % FA16 at Qwen 16K vs st/ld.shared asm)
    auto st_xch = [&](uint32_t a, float x, float y) {
      *reinterpret_cast<float2*>(smem + (a - sb)) = make_float2(x, y);
    };
    auto ld_xch = [&](uint32_t a) { return *reinterpret_cast<const float2*>(smem + (a - sb)); };
    const uint32_t xbar = 3 + t * 4 + quad;  // named barrier of this row quadrant's two warps
    float* dslot = reinterpret_cast<float*>(smem + Cfg::SMEM_DIAG) + (threadIdx.x - 128) * 5;
    if (DIAGNOSE) {
      dslot[0] = __int_as_float(0x7f800000);  // +inf
      dslot[1] = __int_as_float(0xff800000);  // -inf
      dslot[2] = dslot[3] = dslot[4] = 0.f;
    }
    // kProSum: this row's S' sums, G[j] at grow[128 j] in this SM's scratch slot (written
    // below from the prologue GEMM, read back one block ahead of use)
    const float* grow = nullptr;
    float gnext = 0.f;
#ifdef PASA_TRACE
    const long long tp0 = clock64();
    long long tp1 = tp0;
#endif
    if (kProSum) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      if (smid >= static_cast<uint32_t>(p.gslots)) asm volatile("trap;");
      float* gw = p.gsum + (static_cast<size_t>(smid * NT + t) * p.nkv) * kTile + row;
      for (int c = 0; c < nch; ++c) {
        mbar_wait(g_full + 8 * t, c & 1);
#ifdef PASA_TRACE
        if (c == 0) tp1 = clock64();
#endif
        tc_fence_after();
        const int nb = min(kGChunk, ti.nblk - c * kGChunk);  // tile-uniform
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          const int jb = 64 * h + 32 * q2;  // this half's 64 blocks, 32 at a time
          if (jb >= nb) break;
          uint32_t g[32];
          tmem_ld_32cols_b32(t_s + 128 + jb, g);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (jb + i < nb) gw[static_cast<size_t>(c * kGChunk + jb + i) * kTile] = __uint_as_float(g[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(g_free);
      }
      named_bar_sync(xbar, 64);  // the row's other half wrote the other blocks' sums
      grow = gw;
      if (ti.nblk > 0) gnext = grow[0];
    }
#ifdef PASA_TRACE  // prologue: kernel start -> G ready -> G stored (CTA x = 0, y < kTraceCtas)
    if (p.trace && blockIdx.x == 0 && blockIdx.y < kTraceCtas && h == 0 && quad == 0 && lane == 0) {
      float* st = reinterpret_cast<float*>(p.trace + kTraceStateOffset) + kStateIters * 8;
      st[(blockIdx.y * NT + t) * 2] = static_cast<float>(tp1 - tp0);
      st[(blockIdx.y * NT + t) * 2 + 1] = static_cast<float>(clock64() - tp1);
    }
#endif
    if (ti.nblk > 0) {
      // O-bounding exponent: V arrives pre-scaled by 2^-c0; the
      // epilogue multiplies by 2^c0.
      const int c0 = MODE == kModePasa ? pasa_inflation(p.S2_bound, p.vmax[b * p.Hkv + hkv]) : 0;
      constexpr int NP = 32;  // pairs per thread
      uint32_t o[D / 4];
#pragma unroll
      for (int i = 0; i < D / 4; ++i) o[i] = 0u;
      uint32_t s[NP];
      float m_run = 0.f, l_run = 0.f, fbar = 0.f;
      float rcp_j = 1.0f;  // 1/(j+1), computed off the critical path

      // both tiles' block counts (identical in every thread of the CTA)
      const int nmin = min(tile_info(p, hkv, unit * NT, CAUSAL).nblk,
                           tile_info(p, hkv, unit * NT + 1, CAUSAL).nblk);
      const bool pingpong = kPingPong<D>;
      for (int j = 0; j < ti.nblk; ++j) {
        const float gcur = gnext;  // kProSum: sum_c S'_c of block j
        if (kProSum && j + 1 < ti.nblk) gnext = grow[static_cast<size_t>(j + 1) * kTile];
        const bool tr = h == 0 && quad == 0 && lane == 0;
        if (tr) PASA_TR(t, j, 0);
        mbar_wait(s_full + 8 * (t), j & 1);
        if (tr) PASA_TR(t, j, 1);
        tc_fence_after();
        tmem_ld_32cols_pack16(t_s + 64 * h, s);
        tmem_ld_32cols_pack16(t_s + 64 * h + 32, s + 16);
        uint32_t g[2] = {0u, 0u};  // tensor-core row sum: this row's S' sum as hi and lo parts
        if (kTcSum) tmem_ld_2cols_b32(t_s + Cfg::TM_G, g);
        tmem_wait_ld();
        if (tr) PASA_TR(t, j, 2);
        // masked columns: causal diagonal block (c > row) or a short KV block (c >= s2)
        // causal: block j (s2 keys) shows row r of the tile its first vis0 + r keys (any
        // S2 - S1 and s2: the tile's last blocks are partial, some fully masked for a row)
        const bool short_blk = p.s2 < kTile;
        const int vis0 = ti.i * kTile + p.qoff - j * (short_blk ? p.s2 : kTile) + 1;
        const bool cdiag = CAUSAL && vis0 < (short_blk ? p.s2 : kTile);
        const bool diag = cdiag || short_blk;
        const int lim = cdiag ? (short_blk ? min(vis0 + row, p.s2) : vis0 + row) : p.s2;
        if (DIAGNOSE) track_store_block<NP>(s, lim, NP * h, diag, dslot);
        constexpr bool kSum = MODE == kModePasa && !kTcSum && !kProSum;
        float mh, sh = 0.f;
        if (diag) row_max_sum<true, NP, kSum>(s, lim, NP * h, mh, sh);
        else row_max_sum<false, NP, kSum>(s, lim, NP * h, mh, sh);
        st_xch(xs_mine + (j & 1) * kXPar, mh, sh);
        named_bar_sync(xbar, 64);
        const float2 other = ld_xch(xs_other + (j & 1) * kXPar);
        const float mloc = fmaxf(mh, other.x);
        const int jc = j + 1;
        float mnew, ep, fnew = 0.f;
        uint32_t cj2, scale2 = 0;
        bool fast2 = true;  // PASA: the exp argument is one HFMA2 (see below)
        if (MODE == kModePasa) {
          // sum_c S'_c (pasa.cpp:131): the two halves' FP32 sums, or G's hi + lo columns
          const float ssum = kTcSum    ? __fadd_rn(__uint_as_float(g[0]), __uint_as_float(g[1]))
                             : kProSum ? gcur
                                       : (h == 0 ? __fadd_rn(sh, other.y) : __fadd_rn(other.y, sh));
          const float sbar = __fmul_rn(ssum, p.inv_s2);
          fnew = (jc == 1) ? sbar : __fadd_rn(fbar, __fmul_rn(__fsub_rn(sbar, fbar), rcp_j));
          const float dmc = __fmul_rn(p.inva, __fsub_rn(sbar, fnew));
          const float dmp = (jc == 1) ? 0.f : __fmul_rn(p.inva, __fsub_rn(fbar, fnew));
          const float cand = __fadd_rn(mloc, dmc);
          const float mprev = __fadd_rn(m_run, dmp);
          mnew = (jc == 1) ? cand : fmaxf(mprev, cand);
          const __half cj = __float2half_rn(__fsub_rn(mnew, dmc));
          ep = (jc == 1) ? 0.f
                         : __half2float(__float2half_rn(ex2_f32(__fmul_rn(2.f, __fsub_rn(mprev, mnew)))));
          // x = fl16(2 S' - 2 c_j) in one HFMA2 while -2 c_j is representable (every
          // row of the warp: |c_j| <= 32752); otherwise 2 fl16(S' - c_j) (below).
          fast2 = __all_sync(0xFFFFFFFFu, __habs(cj) <= __float2half_rn(32752.f));
          cj2 = fast2 ? h2_as_u32(__half2half2(__hmul(cj, __float2half_rn(-2.f))))
                      : h2_as_u32(__half2half2(cj));
          scale2 = h2_as_u32(__float2half2_rn(2.f));
        } else {
          // naive FP16 FA (attention.cpp:92-180): running max of the FP16-stored
          // scores, P = 2^(S*s - m*s) with s = log2(e)/alpha applied after the store
          mnew = (jc == 1) ? mloc : fmaxf(m_run, mloc);
          ep = (jc == 1) ? 0.f
                         : __half2float(__float2half_rn(ex2_f32(__fmul_rn(__fsub_rn(m_run, mnew), p.qk_scale))));
          cj2 = h2_as_u32(__half2half2(__hneg(__float2half_rn(__fmul_rn(mnew, p.qk_scale)))));
          scale2 = h2_as_u32(__half2half2(__float2half_rn(p.qk_scale)));
        }
        if (tr) PASA_TR(t, j, 3);
        // Ping-pong the MUFU-heavy exp pass between the two tiles:
        // turns go T0(0), T1(0), T0(1), T1(1), ... while both tiles have blocks.
        if (pingpong && j < nmin && (t == 1 || j > 0)) named_bar_sync(1 + t, 512);
        if (tr) PASA_TR(t, j, 8);
        // P packed two per column: this half's 32 pairs -> columns [32h, 32h + 32), stored
        // part by part so the PV MMA starts on each part while the exp continues.
        auto mid = [&](int q) {
          constexpr int W = NP / kPParts<D>;
          if (W == 16) {
            tmem_st_16cols_b32(t_s + NP * h + q * W, s + q * W);
          } else if (W == 8) {
            tmem_st_8cols_b32(t_s + NP * h + q * W, s + q * W);
          } else {
            tmem_st_16cols_b32(t_s + NP * h, s);
            tmem_st_16cols_b32(t_s + NP * h + 16, s + 16);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_part + 8 * (q * NT + t));
          if (q == 0 && tr) PASA_TR(t, j, 9);  // first P part released
        };
        if (MODE == kModePasa && !fast2) {
          // rare (|c_j| > 32752 somewhere in the warp): the split form 2 fl16(S' - c_j) as
          // S' <- fl16(S' - c_j) here, then the common pass with c = 0 (fl16(2 d) = 2 d
          // exactly) -- one exp-pass instantiation instead of two (instruction cache)
#pragma unroll
          for (int i = 0; i < NP; ++i) s[i] = h2_as_u32(__hsub2(u32_as_h2(s[i]), u32_as_h2(cj2)));
          cj2 = 0u;
        }
        const float lsum = diag ? row_exp_sum<D, true, NP>(s, lim, NP * h, cj2, scale2, mid)
                                : row_exp_sum<D, false, NP>(s, lim, NP * h, cj2, scale2, mid);
        if (pingpong && ((t == 0 && j < nmin) || (t == 1 && j + 1 < nmin)))
          named_bar_arrive(2 - t, 512);
        PASA_STATE(j, 0, mloc);
        PASA_STATE(j, 1, MODE == kModePasa ? (h == 0 ? __fadd_rn(sh, other.y) : 0.f) : 0.f);
        PASA_STATE(j, 2, fnew);
        PASA_STATE(j, 3, mnew);
        PASA_STATE(j, 4, __half2float(__low2half(u32_as_h2(cj2))));
        PASA_STATE(j, 5, ep);
        PASA_STATE(j, 6, lsum);
        if (tr) PASA_TR(t, j, 7);
        if (tr) PASA_TR(t, j, 4);
        l_run = (jc == 1) ? lsum : __fadd_rn(__fmul_rn(ep, l_run), lsum);
        PASA_STATE(j, 7, l_run);
        m_run = mnew;
        fbar = fnew;
        rcp_j = __frcp_rn(static_cast<float>(jc + 1));
        // T = P V_j -> this half's D/2 output columns
        mbar_wait(t_full + 8 * (t), j & 1);
        if (tr) PASA_TR(t, j, 5);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tmem_ld_32cols_pack16(t_t + (D / 2) * h + c * 32, s + c * 16);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(t_empty + 8 * (t));
        if (tr) PASA_TR(t, j, 6);
        {  // O <- e_prev O + T; block 1 has e_prev = 0 and O = 0 (no branch, no copies)
          const __half2 ep2 = __float2half2_rn(ep);
#pragma unroll
          for (int i = 0; i < D / 4; ++i)
            o[i] = h2_as_u32(__hfma2(ep2, u32_as_h2(o[i]), u32_as_h2(s[i])));
        }
      }
      // Epilogue: global recovering O / l (pasa.cpp:184-194), fp16 store.
      st_xch(xs_mine + (ti.nblk & 1) * kXPar, l_run, 0.f);
      named_bar_sync(xbar, 64);
      const float lo_other = ld_xch(xs_other + (ti.nblk & 1) * kXPar).x;
      const float l_tot = h == 0 ? __fadd_rn(l_run, lo_other) : __fadd_rn(lo_other, l_run);
      const float inv_l = __fmul_rn(__frcp_rn(l_tot), ldexpf(1.0f, c0));  // exact 2^c0
      // O goes out by TMA: each thread writes its D/2 outputs into tile t's Q buffer (dead:
      // the tile's last S' MMA finished before its last T was ready), in the SW128 box
      // layout of the O map (= Q's), then one thread stores the tile -- rows past S1 (a
      // ragged last tile) are clipped by the map.  The threads' 16-byte stores go to smem
      // instead of 512 STGs drained at CTA exit.
      const uint32_t ostage = sb + Cfg::SMEM_Q + t * Cfg::TILE_BYTES;
#pragma unroll
      for (int i = 0; i < D / 4; i += 4) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half a = __float2half_rn(__fmul_rn(lo_f(o[i + k]), inv_l));
          const __half c = __float2half_rn(__fmul_rn(hi_f(o[i + k]), inv_l));
          w[k] = h2_as_u32(__halves2half2(a, c));
        }
        const int col = (D / 2) * h + 2 * i;  // first of these 8 output columns
        const uint32_t a = ostage + (col / 64) * Cfg::BOX_BYTES + row * 128 +
                           ((((col % 64) / 8) ^ (row & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3])
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar_sync(11 + t, 4 * Cfg::HALVES * 32);  // the tile's 256 softmax threads
      if (h == 0 && quad == 0 && lane == 0) {
        for (int bx = 0; bx < Cfg::NBOX; ++bx)
          tma_store_3d(&tm_o, ostage + bx * Cfg::BOX_BYTES, (p.q_bshd ? ti.hq * D : 0) + bx * 64,
                       ti.i * kTile, p.q_bshd ? b : b * p.Hq + ti.hq);
        tma_store_commit_wait_read();  // the buffer must outlive the read before the CTA exits
      }
      if (DIAGNOSE) {  // out_nonfinite / out_total (pasa.cpp:275-286) and the store stats
        const bool row_ok = ti.i * kTile + row < p.S1;  // ragged last query tile
        DiagAccum* g = static_cast<DiagAccum*>(p.diag);
        unsigned nf = 0;
#pragma unroll
        for (int i = 0; i < D / 4; ++i) {
          const float a = __fmul_rn(lo_f(o[i]), inv_l), c = __fmul_rn(hi_f(o[i]), inv_l);
          nf += !isfinite(__half2float(__float2half_rn(a))) + !isfinite(__half2float(__float2half_rn(c)));
        }
        unsigned long long cnt[5] = {row_ok ? nf : 0u, row_ok ? unsigned(D / 2) : 0u,
                                     __float_as_uint(dslot[2]), __float_as_uint(dslot[3]),
                                     __float_as_uint(dslot[4])};
        float mn = __fmul_rn(dslot[0], p.diag_scale), mx = __fmul_rn(dslot[1], p.diag_scale);
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) {
#pragma unroll
          for (int k = 0; k < 5; ++k) cnt[k] += __shfl_xor_sync(0xffffffffu, cnt[k], o2);
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o2));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
        }
        if (lane == 0) {
          unsigned long long* c = &g->out_nonfinite;
#pragma unroll
          for (int k = 0; k < 5; ++k)
            if (cnt[k]) atomicAdd(c + k, cnt[k]);
          if (mn <= mx) {
            atomic_min_f(&g->store_finite_min, mn);
            atomic_max_f(&g->store_finite_max, mx);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
#ifdef PASA_TRACE_CTA
  if (threadIdx.x == 0 && p.trace) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long* e = p.trace + 4 * (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x);
    e[0] = static_cast<long long>(cta_t0);
    e[1] = static_cast<long long>(t1);
    e[2] = smid;
    e[3] = nmax;
  }
#endif
}

// ---------------------------------------------------------------- launcher
template <int D, bool CAUSAL, int MODE>
cudaError_t launch_fwd_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const CUtensorMap& tks, const CUtensorMap& to, const FwdParams& p,
                         cudaStream_t stream) {
  using Cfg = FwdCfg<D>;
  // RunDiagnostics is a separate instantiation so the production kernel's schedule is
  // untouched by the diagnostic code.
  auto kern = p.diag ? pasa_fwd_kernel<D, CAUSAL, MODE, true> : pasa_fwd_kernel<D, CAUSAL, MODE, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = (p.tiles_per_kv + Cfg::NT - 1) / Cfg::NT;
  const dim3 grid = CAUSAL ? dim3(p.B * p.Hkv, units) : dim3(units, p.B * p.Hkv);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, tks, to, p);
}

cudaError_t launch_fwd(int D, bool causal, int mode, const CUtensorMap& tq, const CUtensorMap& tk,
                       const CUtensorMap& tv, const CUtensorMap& tks, const CUtensorMap& to,
                       const FwdParams& p, cudaStream_t stream) {
#define PASA_LAUNCH(DD, CC, MM) \
  if (D == DD && causal == CC && mode == MM) return launch_fwd_t<DD, CC, MM>(tq, tk, tv, tks, to, p, stream);
  PASA_LAUNCH(128, false, kModePasa)
  PASA_LAUNCH(128, true, kModePasa)
  PASA_LAUNCH(64, false, kModePasa)
  PASA_LAUNCH(64, true, kModePasa)
  PASA_LAUNCH(128, false, kModeFa16)
  PASA_LAUNCH(128, true, kModeFa16)
  PASA_LAUNCH(64, false, kModeFa16)
  PASA_LAUNCH(64, true, kModeFa16)
#undef PASA_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace pasa_b200
