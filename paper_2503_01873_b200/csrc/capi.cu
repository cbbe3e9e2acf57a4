// capi.cu -- the C-ABI of libpasa_b200.so (declared in include/pasa_b200.h).
//
// Host side of the drop-in boundary: argument validation with the reference's
// rules (tensor.cpp:19-55, pasa.cpp:200-211), the shifting-matrix scalars
// (pasa.cpp:16-35), TMA descriptors, workspace carving and the two launches
// (key pre-pass, fused forward).  No exceptions cross the ABI.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pasa_b200.h"
#include "pasa_kernels.cuh"

namespace pasa_b200 {
cudaError_t launch_kprep(const KprepParams& p, int B, int Hkv, cudaStream_t stream);
cudaError_t launch_vscale(const VscaleParams& p, cudaStream_t stream);
cudaError_t launch_ksum(const void* kp, void* ks, int BH, int S2, int s2, int D, cudaStream_t stream);
cudaError_t launch_fwd_packed(int D, int mode, const CUtensorMap& tq, const CUtensorMap& tk,
                              const CUtensorMap& tv, const CUtensorMap& to, const PackedParams& p,
                              cudaStream_t stream);
cudaError_t launch_fwd(int D, bool causal, int mode, const CUtensorMap& tq, const CUtensorMap& tk,
                       const CUtensorMap& tv, const CUtensorMap& tks, const CUtensorMap& to,
                       const FwdParams& p, cudaStream_t stream);
cudaError_t launch_generate(const GenParams& p, void* out, cudaStream_t stream);
cudaError_t launch_generate_resonance(const ResonanceParams& p, void* out, cudaStream_t stream);
}  // namespace pasa_b200

using namespace pasa_b200;

// Stream-ordered scratch (the K' block sums of the d = 64 path) comes from a memory pool
// the library owns, one per device, whose freed blocks stay cached (release threshold =
// max): a per-launch allocation is then a pool hit, not a fresh mapping (which cost
// 2.8 ms per launch), and the process's default pool is left untouched.
static cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
  }
  return pools[dev];
}


namespace {

__global__ void nsmid_kernel(int* out) {
  uint32_t n;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
  *out = static_cast<int>(n);
}

// %nsmid of the current device (SM ids are < it; they need not be contiguous), queried once
// per device on a private stream; falls back to twice the SM count.
int device_nsmid() {
  static std::mutex mu;
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 2 * current_sm_count();
  std::lock_guard<std::mutex> lock(mu);
  if (cache[dev] > 0) return cache[dev];
  int n = 0;
  int* d = nullptr;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
      cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(int), st) == cudaSuccess) {
    nsmid_kernel<<<1, 1, 0, st>>>(d);
    if (cudaMemcpyAsync(&n, d, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) n = 0;
    cudaFreeAsync(d, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) n = 0;
  }
  if (st) cudaStreamDestroy(st);
  cudaGetLastError();
  cache[dev] = n > 0 ? n : 2 * current_sm_count();
  return cache[dev];
}

thread_local std::string g_last_error;
long long* g_trace = nullptr;  // PASA_TRACE builds: clock64 timeline buffer

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(PASA_B200_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr double kLog2e = 1.4426950408889634;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- TMA encode
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D view {d, seq, batch*heads} of a BHSD fp16 tensor, box {64, rows, 1}, 128B swizzle.
int make_tmap(CUtensorMap* m, const void* base, int d, int seq, int bh, int rows = kTile) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(PASA_B200_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(seq),
                        static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2,
                           static_cast<cuuint64_t>(d) * 2 * static_cast<cuuint64_t>(seq)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PASA_B200_ECUDA, "cuTensorMapEncodeTiled failed");
  return PASA_B200_OK;
}

// 4-D view {d, 2, nblk, bh} of the K'-sum buffer [bh][nblk][hi, lo][d] (pasa_ksum_kernel):
// box {64, 1, rows, 1} -- the hi (or lo) rows of `rows` consecutive blocks, 128B swizzle.
int make_tmap_ks4(CUtensorMap* m, const void* base, int d, int nblk, int bh, int rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(PASA_B200_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t row = static_cast<cuuint64_t>(d) * 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), 2, static_cast<cuuint64_t>(nblk),
                        static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[3] = {row, 2 * row, 2 * row * static_cast<cuuint64_t>(nblk)};
  cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PASA_B200_ECUDA, "cuTensorMapEncodeTiled (K' sums) failed");
  return PASA_B200_OK;
}

int check_desc(const pasa_b200_desc* d) {
  if (!d) return fail(PASA_B200_EINVAL, "desc is NULL");
  if (d->batch <= 0 || d->heads_q <= 0 || d->seq_q <= 0 || d->head_dim <= 0)
    return fail(PASA_B200_EINVAL, "problem: empty query tensor");  // tensor.cpp:20-22
  if (d->heads_kv <= 0 || d->heads_q % d->heads_kv != 0)
    return fail(PASA_B200_EINVAL, "problem: K heads must divide Q heads");  // tensor.cpp:24-26 (+GQA)
  if (d->seq_kv <= 0) return fail(PASA_B200_EINVAL, "problem: V shape does not match K");
  if (d->s1 <= 0 || d->s2 <= 0 || d->seq_q % d->s1 != 0 || d->seq_kv % d->s2 != 0)
    return fail(PASA_B200_EINVAL,
                "problem: sequence lengths must be nonzero multiples of the block sizes (S1=" +
                    std::to_string(d->seq_q) + ", s1=" + std::to_string(d->s1) +
                    ", S2=" + std::to_string(d->seq_kv) + ", s2=" + std::to_string(d->s2) +
                    "); ragged inputs are rejected, use truncation explicitly");  // tensor.cpp:31-38
  if (d->layout != 0 && d->layout != 1)
    return fail(PASA_B200_EINVAL, "desc: layout must be 0 (BHSD) or 1 (BSHD)");
  if (!(d->beta >= 0.0 && d->beta < 1.0))
    return fail(PASA_B200_EINVAL, "pasa params: beta must lie in [0, 1); beta == 1 has no recovery");
  if (d->alpha != std::sqrt(static_cast<double>(d->head_dim)))
    return fail(PASA_B200_EINVAL, "pasa: params.alpha does not match sqrt(d)");  // pasa.cpp:206-208
  // ---- limits of this build (valid for the reference, unsupported here)
  if (d->head_dim != 64 && d->head_dim != 128)
    return fail(PASA_B200_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (d->s2 > kTile) return fail(PASA_B200_EUNSUPPORTED, "s2 must be <= 128");
  if (d->causal && d->seq_q > d->seq_kv)
    return fail(PASA_B200_EUNSUPPORTED, "causal requires S1 <= S2");
  return PASA_B200_OK;
}

void shift_scalars(int s2, double beta, double alpha, __half* diag, __half* off) {
  const double n = static_cast<double>(s2);
  *diag = __double2half((1.0 - beta / n) / alpha);  // pasa.cpp:26 (RNE)
  *off = __double2half(-beta / (alpha * n));        // pasa.cpp:27
}

size_t kp_bytes(const pasa_b200_desc* d) {
  return static_cast<size_t>(d->batch) * d->heads_kv * d->seq_kv * d->head_dim * 2;
}

}  // namespace

extern "C" {

int pasa_b200_version(void) { return 100; }

const char* pasa_b200_last_error(void) { return g_last_error.c_str(); }

int pasa_b200_shift_entries(int32_t s2, double beta, double alpha, uint16_t* diag_f16,
                            uint16_t* off_f16) {
  if (s2 <= 0) return fail(PASA_B200_EINVAL, "shifting matrix: s2 must be >= 1");
  if (beta < 0.0 || beta > 1.0) return fail(PASA_B200_EINVAL, "shifting matrix: beta must lie in [0, 1]");
  if (!(alpha > 0.0)) return fail(PASA_B200_EINVAL, "shifting matrix: alpha must be positive");
  __half dg, of;
  shift_scalars(s2, beta, alpha, &dg, &of);
  std::memcpy(diag_f16, &dg, 2);
  std::memcpy(off_f16, &of, 2);
  return PASA_B200_OK;
}

int pasa_b200_check(const pasa_b200_desc* desc) {
  g_last_error.clear();
  return check_desc(desc);
}

size_t pasa_b200_workspace_size(const pasa_b200_desc* d) {
  if (!d || d->batch <= 0 || d->heads_kv <= 0 || d->seq_kv <= 0 || d->head_dim <= 0) return 0;
  // K' | V' | max|V| per head
  return 2 * align_up(kp_bytes(d), 256) +
         align_up(static_cast<size_t>(d->batch) * d->heads_kv * 4, 256);
}

static int preprocess_impl(const pasa_b200_desc* d, const void* k, const void* v, void* kp, float* vmax,
                    float lscale, __half dg, __half of, cudaStream_t st, bool rank1 = false) {
  if (d->head_dim != 64 && d->head_dim != 128)
    return fail(PASA_B200_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (d->s2 <= 0 || d->s2 > kTile || d->seq_kv % d->s2 != 0)
    return fail(PASA_B200_EUNSUPPORTED, "s2 must be <= 128 and divide S2");
  KprepParams p{};
  p.s2 = d->s2;
  p.k = static_cast<const uint16_t*>(k);
  p.v = static_cast<const uint16_t*>(v ? v : k);
  p.kp = static_cast<uint16_t*>(kp);
  float* scratch = nullptr;
  if (!vmax) {
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return fail(PASA_B200_ECUDA, "cudaMemPoolCreate failed");
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&scratch),
                                    static_cast<size_t>(d->batch) * d->heads_kv * 4, pool, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync");
  }
  p.vmax = vmax ? vmax : scratch;
  p.S2 = d->seq_kv;
  p.D = d->head_dim;
  p.diag = __half2float(dg);
  p.off = __half2float(of);
  p.lscale = lscale;
  p.rank1 = rank1;  // the fused path: rank-1 form for any block size
  p.Hkv = d->heads_kv;
  const Strides3 is = layout_strides(d->layout, d->heads_kv, d->seq_kv, d->head_dim);
  p.in_bs = is.bs;
  p.in_hs = is.hs;
  p.in_ss = is.ss;
  if (d->layout != 0 && !(rank1 && v && (d->head_dim == 64 || d->head_dim == 128)))
    return fail(PASA_B200_EUNSUPPORTED, "preprocess_keys: the reference-form pre-pass reads BHSD only");
  cudaError_t e = cudaMemsetAsync(p.vmax, 0, static_cast<size_t>(d->batch) * d->heads_kv * 4, st);
  if (e == cudaSuccess) e = launch_kprep(p, d->batch, d->heads_kv, st);
  if (scratch) cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "pasa_kprep launch");
  return PASA_B200_OK;
}

int pasa_b200_preprocess_keys(const pasa_b200_desc* d, const void* k, const void* v, void* kp,
                              float* vmax, float lscale, void* stream) {
  g_last_error.clear();
  if (!d || !k || !kp) return fail(PASA_B200_EINVAL, "preprocess_keys: NULL argument");
  if (!(d->beta >= 0.0 && d->beta <= 1.0) || !(d->alpha > 0.0))
    return fail(PASA_B200_EINVAL, "shifting matrix: invalid beta/alpha");
  __half dg, of;
  shift_scalars(d->s2, d->beta, d->alpha, &dg, &of);
  return preprocess_impl(d, k, v, kp, vmax, lscale, dg, of, static_cast<cudaStream_t>(stream));
}

int pasa_b200_preprocess_keys_host(const pasa_b200_desc* d, const uint16_t* k, uint16_t* kp,
                                   double m_diag, double m_off) {
  g_last_error.clear();
  if (!d || !k || !kp) return fail(PASA_B200_EINVAL, "preprocess_keys: NULL argument");
  const __half dg = __double2half(m_diag), of = __double2half(m_off);
  if (static_cast<double>(__half2float(dg)) != m_diag || static_cast<double>(__half2float(of)) != m_off)
    return fail(PASA_B200_EINVAL, "preprocess_keys: shifting-matrix entries must be FP16 values");
  const size_t nk = kp_bytes(d);
  uint8_t* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 2 * align_up(nk, 256));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  uint8_t* dk = buf;
  uint8_t* dkp = buf + align_up(nk, 256);
  e = cudaMemcpy(dk, k, nk, cudaMemcpyHostToDevice);
  int rc = PASA_B200_OK;
  if (e != cudaSuccess) rc = cuda_fail(e, "H2D copy");
  if (rc == PASA_B200_OK) rc = preprocess_impl(d, dk, nullptr, dkp, nullptr, 1.0f, dg, of, nullptr);
  if (rc == PASA_B200_OK && (e = cudaMemcpy(kp, dkp, nk, cudaMemcpyDeviceToHost)) != cudaSuccess)
    rc = cuda_fail(e, "D2H copy / kernel");
  cudaFree(buf);
  return rc;
}

int pasa_b200_preprocess(const pasa_b200_desc* d, const void* k, const void* v, void* kp,
                         void* vp, float* vmax, void* stream) {
  g_last_error.clear();
  if (!d || !k || !v || !kp || !vp || !vmax) return fail(PASA_B200_EINVAL, "preprocess: NULL argument");
  if (!(d->beta > 0.0 && d->beta < 1.0) || !(d->alpha > 0.0))
    return fail(PASA_B200_EINVAL, "preprocess: beta must lie in (0, 1), alpha > 0");
  __half dg, of;
  shift_scalars(d->s2, d->beta, d->alpha, &dg, &of);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // K' carries log2(e)/2: the kernel's exp argument is 2 fl16(S' - c_j)
  int rc = preprocess_impl(d, k, v, kp, vmax, static_cast<float>(0.5 * kLog2e), dg, of, st,
                           /*rank1=*/true);
  if (rc) return rc;
  VscaleParams vs{};
  vs.v = static_cast<const uint16_t*>(v);
  vs.vp = static_cast<uint16_t*>(vp);
  vs.vmax = vmax;
  vs.per_head = static_cast<long long>(d->seq_kv) * d->head_dim;
  vs.total = vs.per_head * d->batch * d->heads_kv;
  vs.S2 = d->seq_kv;
  vs.D = d->head_dim;
  vs.Hkv = d->heads_kv;
  const Strides3 vst = layout_strides(d->layout, d->heads_kv, d->seq_kv, d->head_dim);
  vs.in_bs = vst.bs;
  vs.in_hs = vst.hs;
  vs.in_ss = vst.ss;
  cudaError_t e = launch_vscale(vs, st);
  if (e != cudaSuccess) return cuda_fail(e, "pasa_vscale launch");
  return PASA_B200_OK;
}

constexpr long long kMaxGridY = 65535;

// Short sequences (one KV block each, N <= 64) run on the packed kernel (pasa_fwd_packed.cu).
static bool packed_shape(const pasa_b200_desc* d, const pasa_b200_diag* diag, int s2_bound) {
  return !diag && !d->causal && d->heads_q == d->heads_kv && d->layout == 0 && d->seq_q == d->seq_kv &&
         d->seq_kv == d->s2 && d->s2 <= 64 && (s2_bound <= 0 || s2_bound == d->seq_kv);
}

// self_prep (PASA, packed shapes): keys / v are the raw K, V and the packed kernel runs the
// pre-pass per tile in shared memory (no K', V' round trip through HBM).
// [tile_lo, tile_hi): the 128-row query tiles computed (of every (b, h)); -1 = all.  Every
// tile is computed exactly as in the whole problem (same S1, S2, causal offset, K', V', c0),
// so query-row shards are bit-identical to the unsharded output.
static int launch_forward(const pasa_b200_desc* d, int mode, const void* q, const void* keys,
                          const void* v, const float* vmax, void* o, void* stream,
                          pasa_b200_diag* diag = nullptr, int s2_bound = 0, bool self_prep = false,
                          int tile_lo = 0, int tile_hi = -1) {
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(keys) |
       reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(o)) & 15)
    return fail(PASA_B200_EINVAL, "attention_fwd: tensors must be 16-byte aligned");
  const int nq_all = (d->seq_q + kTile - 1) / kTile;
  if (tile_hi < 0) tile_hi = nq_all;
  if (tile_hi <= tile_lo) return PASA_B200_OK;  // an empty query range
  int rc;
  // The fused kernel's grid has B Hkv kv heads in one dimension (y when non-causal) and the
  // query units in the other; beyond the 65535 limit of y the batch is cut into launches.
  {
    const long long units = (static_cast<long long>(d->heads_q / d->heads_kv) * (tile_hi - tile_lo) + 1) / 2;
    const bool packed = packed_shape(d, diag, 0);
    const long long ydim = d->causal ? units : static_cast<long long>(d->batch) * d->heads_kv;
    if (!packed && ydim > kMaxGridY && d->batch > 1) {
      const int per_b = d->causal ? 0 : static_cast<int>(kMaxGridY / d->heads_kv);
      if (per_b < 1) return fail(PASA_B200_EUNSUPPORTED, "attention_fwd: grid too large");
      const size_t qb = static_cast<size_t>(d->heads_q) * d->seq_q * d->head_dim * 2;
      const size_t kb = static_cast<size_t>(d->heads_kv) * d->seq_kv * d->head_dim * 2;
      for (int b0 = 0; b0 < d->batch; b0 += per_b) {
        pasa_b200_desc cd = *d;
        cd.batch = b0 + per_b <= d->batch ? per_b : d->batch - b0;
        rc = launch_forward(&cd, mode, static_cast<const uint8_t*>(q) + qb * b0,
                            static_cast<const uint8_t*>(keys) + kb * b0,
                            static_cast<const uint8_t*>(v) + kb * b0,
                            vmax ? vmax + static_cast<size_t>(b0) * d->heads_kv : nullptr,
                            static_cast<uint8_t*>(o) + qb * b0, stream, diag, s2_bound, false, tile_lo,
                            tile_hi);
        if (rc) return rc;
      }
      return PASA_B200_OK;
    }
    if (!packed && ydim > kMaxGridY)
      return fail(PASA_B200_EUNSUPPORTED, "attention_fwd: grid too large");
  }
  CUtensorMap tq, tk, tv;
  // Short sequences (one KV block each, N <= 64): packed P = 128 / N per tensor-core tile
  if (packed_shape(d, diag, s2_bound)) {
    const int bh = d->batch * d->heads_q, rows = bh * d->seq_q, n = d->seq_q;
    if ((rc = make_tmap(&tq, q, d->head_dim, rows, 1, n))) return rc;
    if ((rc = make_tmap(&tk, keys, d->head_dim, rows, 1, n))) return rc;
    if ((rc = make_tmap(&tv, v, d->head_dim, rows, 1, n))) return rc;
    CUtensorMap tom;  // O: stored by TMA from the staged tile, one box of N rows per sequence
    if ((rc = make_tmap(&tom, o, d->head_dim, rows, 1, n))) return rc;
    PackedParams pp{};
    pp.BH = bh;
    pp.N = n;
    pp.W = 16 * ((n + 15) / 16);
    pp.P = kTile / pp.W;
    pp.qk_scale = static_cast<float>(kLog2e / d->alpha);
    pp.vmax = vmax;
    pp.trace = g_trace;
    if (self_prep && mode == kModePasa) {
      __half dg, of;
      shift_scalars(d->s2, d->beta, d->alpha, &dg, &of);
      pp.self_prep = 1;
      pp.dm = __half2float(dg) - __half2float(of);  // exact: both are FP16 values
      pp.off = __half2float(of);
      pp.lscale = static_cast<float>(0.5 * kLog2e);  // the fused path's K' carries log2(e)/2
    }
    cudaError_t e = launch_fwd_packed(d->head_dim, mode, tq, tk, tv, tom, pp, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "pasa_fwd_packed launch");
    return PASA_B200_OK;
  }
  // BHSD: a {d, S, B H} map, box coordinates (c, s, b H + h); BSHD: the rows of a batch
  // hold every head's d values, so a {H d, S, B} map with coordinates (h d + c, s, b).
  // K and V are the caller's in FA16 mode, the BHSD workspace (K', V') in PASA mode.
  const bool kv_bshd = mode == kModeFa16 && d->layout == 1;
  CUtensorMap to;  // O: Q's shape and layout (the epilogue's TMA store)
  if (d->layout == 1) {
    if ((rc = make_tmap(&tq, q, d->heads_q * d->head_dim, d->seq_q, d->batch))) return rc;
    if ((rc = make_tmap(&to, o, d->heads_q * d->head_dim, d->seq_q, d->batch))) return rc;
  } else {
    if ((rc = make_tmap(&tq, q, d->head_dim, d->seq_q, d->batch * d->heads_q))) return rc;
    if ((rc = make_tmap(&to, o, d->head_dim, d->seq_q, d->batch * d->heads_q))) return rc;
  }
  if (kv_bshd) {
    if ((rc = make_tmap(&tk, keys, d->heads_kv * d->head_dim, d->seq_kv, d->batch, d->s2))) return rc;
    if ((rc = make_tmap(&tv, v, d->heads_kv * d->head_dim, d->seq_kv, d->batch, d->s2))) return rc;
  } else {
    if ((rc = make_tmap(&tk, keys, d->head_dim, d->seq_kv, d->batch * d->heads_kv, d->s2))) return rc;
    if ((rc = make_tmap(&tv, v, d->head_dim, d->seq_kv, d->batch * d->heads_kv, d->s2))) return rc;
  }
  FwdParams p{};
  p.B = d->batch;
  p.Hq = d->heads_q;
  p.Hkv = d->heads_kv;
  p.S1 = d->seq_q;
  p.S2 = d->seq_kv;
  p.S2_bound = s2_bound > 0 ? s2_bound : d->seq_kv;
  p.q_bshd = d->layout == 1;
  p.kv_bshd = kv_bshd;
  p.nq = (d->seq_q + kTile - 1) / kTile;
  p.nkv = d->seq_kv / d->s2;
  p.qoff = d->causal ? d->seq_kv - d->seq_q : 0;
  p.s2 = d->s2;
  p.inv_s2 = static_cast<float>(1.0 / d->s2);
  p.group = d->heads_q / d->heads_kv;
  p.tile_hi = tile_hi;
  p.tiles_per_kv = p.group * (tile_hi - tile_lo);
  p.inva = static_cast<float>(d->beta / (1.0 - d->beta));  // pasa.cpp:85
  p.qk_scale = static_cast<float>(kLog2e / d->alpha);
  p.vmax = vmax;
  p.trace = g_trace;
  p.diag = diag;
  p.diag_scale = mode == kModePasa ? static_cast<float>(2.0 / kLog2e) : 1.0f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // PASA at D = 64: the S' row sums come from the tensor core (pseudo-average GEMM
  // against the block sums of K', pasa_tc_rowsum); the sums are a stream-ordered scratch
  // of B Hkv (S2 / s2) 2 D halves (1.6 % of K' at s2 = 128) from the library's pool.
  //
  // PASA at D = 128: the same K' block sums feed the fused kernel's prologue GEMM (256-row
  // boxes, 128 blocks per chunk); its per-row results go to an L2-resident scratch of one
  // slot per SM id (%nsmid x 2 tiles x blocks x 128 rows FP32), also from the pool.
  CUtensorMap tks = tk;
  void* ks = nullptr;
  void* gs = nullptr;
  cudaError_t e = cudaSuccess;
  if (mode == kModePasa && (pasa_tc_rowsum(d->head_dim) || pasa_prologue_rowsum(d->head_dim))) {
    const int bh = d->batch * d->heads_kv, nblk = d->seq_kv / d->s2;
    const bool pro = pasa_prologue_rowsum(d->head_dim);
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return fail(PASA_B200_ECUDA, "cudaMemPoolCreate failed");
    e = cudaMallocFromPoolAsync(&ks, static_cast<size_t>(bh) * nblk * 2 * d->head_dim * 2, pool, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync");
    p.ks_rows = pro ? (nblk < 128 ? nblk : 128) : 2;
    if ((rc = pro ? make_tmap_ks4(&tks, ks, d->head_dim, nblk, bh, p.ks_rows)
                  : make_tmap(&tks, ks, d->head_dim, 2 * nblk, bh, p.ks_rows))) {
      cudaFreeAsync(ks, st);
      return rc;
    }
    if (pro) {
      p.gslots = device_nsmid();
      e = cudaMallocFromPoolAsync(&gs, static_cast<size_t>(p.gslots) * 2 * nblk * kTile * 4, pool, st);
      if (e != cudaSuccess) {
        cudaFreeAsync(ks, st);
        return cuda_fail(e, "cudaMallocFromPoolAsync");
      }
      p.gsum = static_cast<float*>(gs);
    }
    e = launch_ksum(keys, ks, bh, d->seq_kv, d->s2, d->head_dim, st);
  }
  if (e == cudaSuccess) e = launch_fwd(d->head_dim, d->causal != 0, mode, tq, tk, tv, tks, to, p, st);
  if (ks) cudaFreeAsync(ks, st);
  if (gs) cudaFreeAsync(gs, st);
  if (e != cudaSuccess) return cuda_fail(e, "pasa_fwd launch");
  return PASA_B200_OK;
}

int pasa_b200_attention_fwd_prepped(const pasa_b200_desc* d, const void* q, const void* kp,
                                    const void* vp, const float* vmax, void* o, void* stream) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !kp || !vp || !o || !vmax)
    return fail(PASA_B200_EINVAL, "attention_fwd: NULL tensor");
  if (d->beta == 0.0)
    return fail(PASA_B200_EINVAL, "attention_fwd_prepped: beta == 0 has no key pre-pass");
  return launch_forward(d, kModePasa, q, kp, vp, vmax, o, stream);
}

int pasa_b200_flash_fp16_fwd(const pasa_b200_desc* d, const void* q, const void* k, const void* v,
                             void* o, void* stream) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !k || !v || !o) return fail(PASA_B200_EINVAL, "flash_fp16_fwd: NULL tensor");
  return launch_forward(d, kModeFa16, q, k, v, nullptr, o, stream);
}

int pasa_b200_attention_fwd(const pasa_b200_desc* d, const void* q, const void* k, const void* v,
                            void* o, void* workspace, size_t workspace_bytes,
                            pasa_b200_diag* diag, void* stream) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !k || !v || !o || !workspace)
    return fail(PASA_B200_EINVAL, "attention_fwd: NULL tensor or workspace");
  if (workspace_bytes < pasa_b200_workspace_size(d))
    return fail(PASA_B200_EINVAL, "attention_fwd: workspace too small");
  // beta == 0 degrades to the blocked FP16 attention (pasa.cpp:212-221)
  if (d->beta == 0.0) return launch_forward(d, kModeFa16, q, k, v, nullptr, o, stream, diag);
  // short sequences: one packed kernel with the pre-pass fused (bit-identical to the path below)
  if (packed_shape(d, diag, 0))
    return launch_forward(d, kModePasa, q, k, v, nullptr, o, stream, nullptr, 0, /*self_prep=*/true);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* kp = ws;
  void* vp = ws + align_up(kp_bytes(d), 256);
  float* vmax = reinterpret_cast<float*>(ws + 2 * align_up(kp_bytes(d), 256));
  rc = pasa_b200_preprocess(d, k, v, kp, vp, vmax, stream);
  if (rc) return rc;
  if (!diag) return pasa_b200_attention_fwd_prepped(d, q, kp, vp, vmax, o, stream);
  return launch_forward(d, kModePasa, q, kp, vp, vmax, o, stream, diag);
}

int pasa_b200_attention_fwd_tiles(const pasa_b200_desc* d, const void* q, const void* k, const void* v,
                                  void* o, void* workspace, size_t workspace_bytes, int32_t tile0,
                                  int32_t ntiles, void* stream) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !k || !v || !o || !workspace)
    return fail(PASA_B200_EINVAL, "attention_fwd_tiles: NULL tensor or workspace");
  if (workspace_bytes < pasa_b200_workspace_size(d))
    return fail(PASA_B200_EINVAL, "attention_fwd_tiles: workspace too small");
  const int nq = (d->seq_q + kTile - 1) / kTile;
  if (tile0 < 0 || ntiles < 0 || tile0 > nq || ntiles > nq - tile0)
    return fail(PASA_B200_EINVAL, "attention_fwd_tiles: tile range outside [0, ceil(seq_q / 128))");
  if (ntiles == 0) return PASA_B200_OK;
  if (d->beta == 0.0) return launch_forward(d, kModeFa16, q, k, v, nullptr, o, stream, nullptr, 0, false, tile0,
                                            tile0 + ntiles);
  if (packed_shape(d, nullptr, 0))  // one query tile per sequence: the range is the whole problem
    return launch_forward(d, kModePasa, q, k, v, nullptr, o, stream, nullptr, 0, /*self_prep=*/true);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* kp = ws;
  void* vp = ws + align_up(kp_bytes(d), 256);
  float* vmax = reinterpret_cast<float*>(ws + 2 * align_up(kp_bytes(d), 256));
  rc = pasa_b200_preprocess(d, k, v, kp, vp, vmax, stream);  // every key: K', V', c0 as unsharded
  if (rc) return rc;
  return launch_forward(d, kModePasa, q, kp, vp, vmax, o, stream, nullptr, 0, false, tile0, tile0 + ntiles);
}

__global__ void diag_reset_kernel(pasa_b200_diag* g) {
  *g = pasa_b200_diag{0ull, 0ull, 0ull, 0ull, 0ull, __int_as_float(0x7f800000),
                      __int_as_float(0xff800000)};
}

int pasa_b200_diag_reset(pasa_b200_diag* diag, void* stream) {
  g_last_error.clear();
  if (!diag) return fail(PASA_B200_EINVAL, "diag_reset: NULL");
  diag_reset_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(diag);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "diag_reset");
}

static int attention_host_impl(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                               const uint16_t* v, uint16_t* o, pasa_b200_diag* hdiag);

int pasa_b200_attention_host(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                             const uint16_t* v, uint16_t* o) {
  return attention_host_impl(d, q, k, v, o, nullptr);
}

int pasa_b200_attention_host_diag(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                                  const uint16_t* v, uint16_t* o, pasa_b200_diag* diag) {
  if (!diag) {
    g_last_error.clear();
    return fail(PASA_B200_EINVAL, "attention_host_diag: NULL diag");
  }
  return attention_host_impl(d, q, k, v, o, diag);
}

// The host entry point's device buffers, streams and events, cached per host thread (and
// re-created when the thread switches device).  release() frees them: the multi-device
// entry point's worker threads call it before they exit.
struct HostCache {
  static constexpr int kComp = 4, kRing = 64;
  int dev = -1;
  uint8_t* buf = nullptr;
  size_t bytes = 0;
  cudaStream_t st[3 + kComp] = {};
  cudaEvent_t ev[3][kRing] = {};  // kv copied / piece copied in / piece computed
  cudaEvent_t prep[kRing] = {}, comp_done[kComp] = {};
  void release() {
    if (buf) cudaFree(buf);
    buf = nullptr;
    bytes = 0;
    for (auto& x : st)
      if (x) cudaStreamDestroy(x), x = nullptr;
    for (auto& row : ev)
      for (auto& x : row)
        if (x) cudaEventDestroy(x), x = nullptr;
    for (auto& x : prep)
      if (x) cudaEventDestroy(x), x = nullptr;
    for (auto& x : comp_done)
      if (x) cudaEventDestroy(x), x = nullptr;
    dev = -1;
  }
};
static thread_local HostCache g_host_cache;

// One piece of a query-tile split (more devices than (b, kv head) units): units [u0, u1),
// query tiles [t0, t0 + nt) of each, on the current device.  Q rows of those tiles and the
// units' K, V go in, pasa_b200_attention_fwd_tiles computes them exactly as the whole problem
// does, the O rows come back.  Not pipelined: a split piece is a small share.
struct TilePiece {
  int u0, u1, t0, nt;
};

static int host_tile_piece(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                           uint16_t* o, const TilePiece& pc) {
  const int group = d->heads_q / d->heads_kv, nu = pc.u1 - pc.u0;
  pasa_b200_desc sd = *d;  // the piece's units as one batch of nu kv heads (BHSD)
  sd.batch = 1;
  sd.heads_kv = nu;
  sd.heads_q = nu * group;
  const size_t head = static_cast<size_t>(d->seq_q) * d->head_dim * 2;  // bytes per q head
  const size_t kunit = static_cast<size_t>(d->seq_kv) * d->head_dim * 2;
  const int r0 = pc.t0 * kTile, r1 = std::min(d->seq_q, (pc.t0 + pc.nt) * kTile);
  const size_t rows_b = static_cast<size_t>(r1 - r0) * d->head_dim * 2, off_b = static_cast<size_t>(r0) * d->head_dim * 2;
  const size_t qb = head * nu * group, kb = kunit * nu, wsb = pasa_b200_workspace_size(&sd);
  cudaStream_t st = nullptr;
  void *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr, *ws = nullptr;
  int rc = PASA_B200_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&dq, qb);
  if (e == cudaSuccess) e = cudaMalloc(&dout, qb);
  if (e == cudaSuccess) e = cudaMalloc(&dk, kb);
  if (e == cudaSuccess) e = cudaMalloc(&dv, kb);
  if (e == cudaSuccess) e = cudaMalloc(&ws, wsb);
  const uint8_t* qh = reinterpret_cast<const uint8_t*>(q) + head * group * pc.u0;
  uint8_t* oh = reinterpret_cast<uint8_t*>(o) + head * group * pc.u0;
  if (e == cudaSuccess)  // the tiles' rows of every q head of the piece (pitch: one head)
    e = cudaMemcpy2DAsync(static_cast<uint8_t*>(dq) + off_b, head, qh + off_b, head, rows_b, nu * group,
                          cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dk, reinterpret_cast<const uint8_t*>(k) + kunit * pc.u0, kb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dv, reinterpret_cast<const uint8_t*>(v) + kunit * pc.u0, kb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "attention_host_multi: piece setup");
  if (rc == PASA_B200_OK) rc = pasa_b200_attention_fwd_tiles(&sd, dq, dk, dv, dout, ws, wsb, pc.t0, pc.nt, st);
  if (rc == PASA_B200_OK) {
    e = cudaMemcpy2DAsync(oh + off_b, head, static_cast<uint8_t*>(dout) + off_b, head, rows_b, nu * group,
                          cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "attention_host_multi: piece copy-out");
  }
  if (st) cudaStreamSynchronize(st);
  for (void* b : {dq, dk, dv, dout, ws})
    if (b) cudaFree(b);
  if (st) cudaStreamDestroy(st);
  return rc;
}

// partition_work of multi.py: the unit-major (unit, tile) items cut into n runs of equal
// key-block cost (an item goes to the run holding its cost midpoint); a run is at most three
// pieces (a unit's tail, whole units, a unit's head).
static std::vector<std::vector<TilePiece>> tile_partition(const pasa_b200_desc* d, int n) {
  const int nq = (d->seq_q + kTile - 1) / kTile, nkv = d->seq_kv / d->s2, qoff = d->seq_kv - d->seq_q;
  const int units = d->batch * d->heads_kv;
  std::vector<long long> cost(nq), prefix(nq + 1, 0);
  for (int i = 0; i < nq; ++i) {
    cost[i] = d->causal ? std::min((std::min(d->seq_q, kTile * (i + 1)) - 1 + qoff) / d->s2 + 1, nkv) : nkv;
    prefix[i + 1] = prefix[i] + cost[i];
  }
  const long long per_unit = prefix[nq], total = per_unit * units;
  auto owner = [&](int u, int i) {
    const long long mid2 = 2 * (u * per_unit + prefix[i]) + cost[i];
    return total ? static_cast<int>(std::min<long long>(n - 1, mid2 * n / (2 * total))) : 0;
  };
  std::vector<std::vector<TilePiece>> runs(n);
  for (int u = 0; u < units; ++u)
    for (int lo = 0; lo < nq;) {
      const int r = owner(u, lo);
      int hi = lo;
      while (hi < nq && owner(u, hi) == r) ++hi;
      auto& pcs = runs[r];
      if (!pcs.empty() && lo == 0 && hi == nq && pcs.back().t0 == 0 && pcs.back().nt == nq && pcs.back().u1 == u)
        pcs.back().u1 = u + 1;
      else
        pcs.push_back({u, u + 1, lo, hi - lo});
      lo = hi;
    }
  return runs;
}

int pasa_b200_attention_host_multi(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                                   const uint16_t* v, uint16_t* o, const int32_t* devices,
                                   int32_t n_devices) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !k || !v || !o || !devices || n_devices <= 0)
    return fail(PASA_B200_EINVAL, "attention_host_multi: NULL buffer or empty device list");
  if (d->layout != 0)
    return fail(PASA_B200_EUNSUPPORTED, "attention_host_multi: BHSD only (units must be contiguous)");
  // The (batch, kv head) units, contiguous in BHSD, are split evenly across the devices
  // (no exchange -- each device computes its units' whole output); one host
  // thread per device runs the pipelined host entry point on its share.  With more devices
  // than units, query tiles are split too (tile_partition; bit-identical, like multi.py).
  const int units = d->batch * d->heads_kv, group = d->heads_q / d->heads_kv;
  if (n_devices > units && !packed_shape(d, nullptr, 0) && (d->seq_q + kTile - 1) / kTile > 1) {
    const auto runs = tile_partition(d, n_devices);
    std::vector<int> rcs(n_devices, PASA_B200_OK);
    std::vector<std::string> errs(n_devices);
    std::vector<std::thread> pool;
    for (int r = 0; r < n_devices; ++r) {
      if (runs[r].empty()) continue;
      pool.emplace_back([&, r] {
        if (cudaSetDevice(devices[r]) != cudaSuccess) {
          rcs[r] = PASA_B200_ENODEV;
          errs[r] = "attention_host_multi: cudaSetDevice failed";
          return;
        }
        for (const TilePiece& pc : runs[r])
          if ((rcs[r] = host_tile_piece(d, q, k, v, o, pc)) != PASA_B200_OK) {
            errs[r] = g_last_error;
            break;
          }
      });
    }
    for (auto& th : pool) th.join();
    for (int r = 0; r < n_devices; ++r)
      if (rcs[r]) {
        g_last_error = errs[r];
        return rcs[r];
      }
    return PASA_B200_OK;
  }
  const int n = n_devices < units ? n_devices : units;
  const size_t q_unit = static_cast<size_t>(group) * d->seq_q * d->head_dim;  // halves
  const size_t k_unit = static_cast<size_t>(d->seq_kv) * d->head_dim;
  std::vector<int> rcs(n, PASA_B200_OK);
  std::vector<std::string> errs(n);
  std::vector<std::thread> pool;
  for (int r = 0; r < n; ++r) {
    const int u0 = static_cast<int>(static_cast<long long>(units) * r / n);
    const int u1 = static_cast<int>(static_cast<long long>(units) * (r + 1) / n);
    pool.emplace_back([&, r, u0, u1] {
      cudaError_t e = cudaSetDevice(devices[r]);
      if (e != cudaSuccess) {
        rcs[r] = PASA_B200_ENODEV;
        errs[r] = "attention_host_multi: cudaSetDevice failed";
        return;
      }
      pasa_b200_desc sd = *d;  // the share as one batch of (u1 - u0) kv heads (BHSD)
      sd.batch = 1;
      sd.heads_kv = u1 - u0;
      sd.heads_q = (u1 - u0) * group;
      rcs[r] = attention_host_impl(&sd, q + q_unit * u0, k + k_unit * u0, v + k_unit * u0,
                                   o + q_unit * u0, nullptr);
      if (rcs[r]) errs[r] = g_last_error;
      cudaDeviceSynchronize();  // nothing of this share may still use the buffers
      g_host_cache.release();   // the worker thread ends: free its cached buffers
    });
  }
  for (auto& th : pool) th.join();
  for (int r = 0; r < n; ++r)
    if (rcs[r]) {
      g_last_error = errs[r];
      return rcs[r];
    }
  return PASA_B200_OK;
}

static int attention_host_run(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                              const uint16_t* v, uint16_t* o, pasa_b200_diag* hdiag,
                              pasa_b200_diag** ddiag_out);

// A failed call returns only after everything it enqueued has finished: no copy may still
// read the caller's buffers (or write the cached device buffers) once it has returned.
static int attention_host_impl(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                               const uint16_t* v, uint16_t* o, pasa_b200_diag* hdiag) {
  pasa_b200_diag* ddiag = nullptr;
  const int rc = attention_host_run(d, q, k, v, o, hdiag, &ddiag);
  if (rc != PASA_B200_OK) {
    const std::string err = g_last_error;
    for (auto st : g_host_cache.st)
      if (st) cudaStreamSynchronize(st);
    if (ddiag) cudaFree(ddiag);
    g_last_error = err;
  }
  return rc;
}

static int attention_host_run(const pasa_b200_desc* d, const uint16_t* q, const uint16_t* k,
                              const uint16_t* v, uint16_t* o, pasa_b200_diag* hdiag,
                              pasa_b200_diag** ddiag_out) {
  g_last_error.clear();
  int rc = check_desc(d);
  if (rc) return rc;
  if (!q || !k || !v || !o) return fail(PASA_B200_EINVAL, "attention_host: NULL buffer");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(PASA_B200_ENODEV, "no CUDA device");
  // The problem is cut into ~kTargetPieces pieces of query heads -- a few query heads of
  // one (batch, kv head) unit, or a run of whole units -- that are copied in, computed and
  // copied out in a pipeline: one H2D stream (K/V of a unit before its first piece, then the
  // piece's Q), one pre-pass stream (K', V' per unit), kComp compute streams (so the small
  // kernels of consecutive pieces share the SMs) and one D2H stream (PCIe is full duplex).
  // Small pieces keep the pipeline's fill (the first piece's H2D) and drain (the last
  // piece's kernel and D2H) short; the whole call is then bound by the H2D copy
  // (tools/pcie_probe.py).  Device buffers, streams and events are cached per thread and device.
  constexpr int kTargetPieces = 32, kComp = HostCache::kComp, kRing = HostCache::kRing;
  HostCache& cache = g_host_cache;
  const int group = d->heads_q / d->heads_kv;
  const int units = d->batch * d->heads_kv;
  const size_t q_head = static_cast<size_t>(d->seq_q) * d->head_dim * 2;
  const size_t q_unit = q_head * group;
  const size_t k_unit = static_cast<size_t>(d->seq_kv) * d->head_dim * 2;
  const size_t nq = q_unit * units, nk = k_unit * units;
  const bool pasa = d->beta != 0.0;
  // piece size in query heads; below a unit's group the unit is split, above it whole units
  const int total = units * group;
  const int ph = (total + kTargetPieces - 1) / kTargetPieces;
  int hper = group, uper = 1;
  if (ph < group) {
    const int parts = (group + ph - 1) / ph;
    hper = (group + parts - 1) / parts;
  } else {
    uper = ph / group;
  }
  const size_t total_bytes = 2 * align_up(nq, 256) + 4 * align_up(nk, 256) +
                             align_up(static_cast<size_t>(units) * 4, 256) + 256;
  cudaError_t e = cudaSuccess;
  if (cache.dev != dev || cache.bytes < total_bytes) {
    if (cache.buf) cudaFree(cache.buf);
    if (cache.dev != dev) {
      for (auto& st : cache.st)
        if (st) cudaStreamDestroy(st), st = nullptr;
      for (auto& row : cache.ev)
        for (auto& x : row)
          if (x) cudaEventDestroy(x), x = nullptr;
      for (auto& x : cache.prep)
        if (x) cudaEventDestroy(x), x = nullptr;
      for (auto& x : cache.comp_done)
        if (x) cudaEventDestroy(x), x = nullptr;
    }
    cache.buf = nullptr;
    cache.bytes = 0;
    if ((e = cudaMalloc(&cache.buf, total_bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    cache.bytes = total_bytes;
    cache.dev = dev;
  }
  for (auto& st : cache.st)
    if (!st && (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  auto mk = [&](cudaEvent_t& x) {
    return x ? cudaSuccess : cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  };
  for (auto& row : cache.ev)
    for (auto& x : row)
      if ((e = mk(x)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  for (auto& x : cache.prep)
    if ((e = mk(x)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  for (auto& x : cache.comp_done)
    if ((e = mk(x)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  uint8_t* dq = cache.buf;
  uint8_t* dk = dq + align_up(nq, 256);
  uint8_t* dv = dk + align_up(nk, 256);
  uint8_t* dkp = dv + align_up(nk, 256);  // K', V', max|V| of every unit (pre-pass output)
  uint8_t* dvp = dkp + align_up(nk, 256);
  uint8_t* dout = dvp + align_up(nk, 256);
  float* dvmax = reinterpret_cast<float*>(dout + align_up(nq, 256));
  pasa_b200_diag* ddiag = nullptr;
  cudaStream_t s_in = cache.st[0], s_prep = cache.st[1], s_out = cache.st[2];
  const cudaStream_t* s_comp = cache.st + 3;
  if (hdiag) {
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return fail(PASA_B200_ECUDA, "cudaMemPoolCreate failed");
    if ((e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ddiag), sizeof(pasa_b200_diag), pool,
                                     s_prep)))
      return cuda_fail(e, "cudaMallocFromPoolAsync");
    *ddiag_out = ddiag;  // freed on s_out on success, by the caller on failure
    if ((rc = pasa_b200_diag_reset(ddiag, s_prep))) return rc;
    if ((e = cudaEventRecord(cache.prep[0], s_prep)) != cudaSuccess) return cuda_fail(e, "event");
    for (int c = 0; c < kComp; ++c)
      if ((e = cudaStreamWaitEvent(s_comp[c], cache.prep[0], 0)) != cudaSuccess) return cuda_fail(e, "event");
  }
  const uint8_t* hq = reinterpret_cast<const uint8_t*>(q);
  const uint8_t* hk = reinterpret_cast<const uint8_t*>(k);
  const uint8_t* hv = reinterpret_cast<const uint8_t*>(v);
  uint8_t* ho = reinterpret_cast<uint8_t*>(o);
  if (d->layout == 1) {
    // BSHD: a unit's rows are not contiguous, so no pieces -- one copy-in, compute, copy-out
    cudaEvent_t ev_in = cache.ev[1][0], ev_done = cache.ev[2][0];
    const cudaStream_t sc = s_comp[0];
    e = cudaMemcpyAsync(dq, hq, nq, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dk, hk, nk, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dv, hv, nk, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in, s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev_in, 0);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    if (pasa) {
      if ((rc = pasa_b200_preprocess(d, dk, dv, dkp, dvp, dvmax, sc))) return rc;
      rc = launch_forward(d, kModePasa, dq, dkp, dvp, dvmax, dout, sc, ddiag);
    } else {
      rc = launch_forward(d, kModeFa16, dq, dk, dv, nullptr, dout, sc, ddiag);
    }
    if (rc) return rc;
    e = cudaEventRecord(ev_done, sc);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, ev_done, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ho, dout, nq, cudaMemcpyDeviceToHost, s_out);
    if (e == cudaSuccess && hdiag)
      e = cudaMemcpyAsync(hdiag, ddiag, sizeof(pasa_b200_diag), cudaMemcpyDeviceToHost, s_out);
    if (e == cudaSuccess && hdiag && (e = cudaFreeAsync(ddiag, s_out)) == cudaSuccess)
      *ddiag_out = nullptr;
    if (e == cudaSuccess) e = cudaStreamSynchronize(s_out);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy / kernel");
    return PASA_B200_OK;
  }
  int piece = 0, kvc = 0;
  cudaEvent_t last_dep = nullptr;  // the last unit's K/V (FA16) or pre-pass (PASA) event
  // PASA_B200_HOST_TRACE=1 (diagnostic): per-piece H2D / compute / D2H completion times
  static const bool trace = getenv("PASA_B200_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  std::vector<double> thost;  // host time (ms after the first mark) when each piece was enqueued
  const auto h0 = std::chrono::steady_clock::now();
  auto tmark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, st);
    tev.push_back(x);
    if (st == s_out)
      thost.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
  };
  tmark(s_in);
  // one piece: query rows [r0, r0 + nr) of heads [g0, g0 + nh) of units [u0, u0 + nu) on
  // keys [0, skv) (row pieces of a causal head stay bit-identical to the whole head; V's O
  // bound keeps the full key count).  Pieces are whole heads today: cutting the last
  // unit's causal heads by rows (cheap early rows last) did not shorten the drain (a
  // late-row piece keeps a 128-block CTA chain), and cutting every head doubled the copy
  // chunks, whose per-copy DMA overhead cost more (PASA_B200_HOST_TRACE timelines,
  // tools/pcie_probe.py).
  auto run_piece = [&](int u0, int nu, int g0, int nh, int r0, int nr, int skv,
                       cudaEvent_t dep) -> int {
    const size_t ok = k_unit * u0;
    const size_t row_bytes = static_cast<size_t>(d->head_dim) * 2;
    // contiguous: whole heads, or rows of one head
    const size_t oq = q_unit * u0 + q_head * g0 + row_bytes * r0;
    const size_t bq = nr < d->seq_q ? row_bytes * nr : (nu == 1 ? q_head * nh : q_unit * nu);
    cudaEvent_t ev_in = cache.ev[1][piece % kRing], ev_done = cache.ev[2][piece % kRing];
    const cudaStream_t sc = s_comp[piece % kComp];
    ++piece;
    cudaError_t e2 = cudaMemcpyAsync(dq + oq, hq + oq, bq, cudaMemcpyHostToDevice, s_in);
    if (e2 == cudaSuccess) e2 = cudaEventRecord(ev_in, s_in);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(sc, ev_in, 0);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(sc, dep, 0);
    if (e2 != cudaSuccess) return cuda_fail(e2, "H2D copy");
    tmark(s_in);
    pasa_b200_desc pd = *d;
    pd.batch = 1;
    pd.heads_kv = nu;
    pd.heads_q = nu == 1 ? nh : nu * group;
    pd.seq_q = nr;
    pd.seq_kv = skv;
    int rc2 = pasa ? launch_forward(&pd, kModePasa, dq + oq, dkp + ok, dvp + ok, dvmax + u0, dout + oq,
                                    sc, ddiag, d->seq_kv)
                   : launch_forward(&pd, kModeFa16, dq + oq, dk + ok, dv + ok, nullptr, dout + oq, sc,
                                    ddiag, d->seq_kv);
    if (rc2) return rc2;
    tmark(sc);
    e2 = cudaEventRecord(ev_done, sc);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(s_out, ev_done, 0);
    if (e2 == cudaSuccess) e2 = cudaMemcpyAsync(ho + oq, dout + oq, bq, cudaMemcpyDeviceToHost, s_out);
    if (e2 != cudaSuccess) return cuda_fail(e2, "D2H copy");
    tmark(s_out);
    return PASA_B200_OK;
  };
  for (int u0 = 0; u0 < units; u0 += uper) {
    const int nu = u0 + uper <= units ? uper : units - u0;
    const size_t ok = k_unit * u0, bk = k_unit * nu;
    // K and V of the piece's units, then (PASA) their pre-pass on its own stream
    cudaEvent_t ev_kv = cache.ev[0][kvc % kRing], ev_prep = cache.prep[kvc % kRing];
    ++kvc;
    e = cudaMemcpyAsync(dk + ok, hk + ok, bk, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dv + ok, hv + ok, bk, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaEventRecord(ev_kv, s_in);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    if (pasa) {
      pasa_b200_desc ud = *d;
      ud.batch = 1;
      ud.heads_kv = nu;
      ud.heads_q = nu * group;
      if ((e = cudaStreamWaitEvent(s_prep, ev_kv, 0)) != cudaSuccess) return cuda_fail(e, "event");
      if ((rc = pasa_b200_preprocess(&ud, dk + ok, dv + ok, dkp + ok, dvp + ok, dvmax + u0, s_prep)))
        return rc;
      if ((e = cudaEventRecord(ev_prep, s_prep)) != cudaSuccess) return cuda_fail(e, "event");
    }
    last_dep = pasa ? ev_prep : ev_kv;
    for (int g0 = 0; g0 < group; g0 += hper) {
      const int nh = g0 + hper <= group ? hper : group - g0;
      if ((rc = run_piece(u0, nu, g0, nh, 0, d->seq_q, d->seq_kv, last_dep))) return rc;
      if (nu > 1) break;  // whole units: one piece covers all their query heads
    }
  }
  if (hdiag) {
    for (int c = 0; c < kComp; ++c) {
      e = cudaEventRecord(cache.comp_done[c], s_comp[c]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, cache.comp_done[c], 0);
      if (e != cudaSuccess) return cuda_fail(e, "event");
    }
    e = cudaMemcpyAsync(hdiag, ddiag, sizeof(pasa_b200_diag), cudaMemcpyDeviceToHost, s_out);
    if (e == cudaSuccess && (e = cudaFreeAsync(ddiag, s_out)) == cudaSuccess) *ddiag_out = nullptr;
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  }
  // every compute stream's last kernel precedes a D2H on s_out, so s_out completes last
  if ((e = cudaStreamSynchronize(s_out)) != cudaSuccess) return cuda_fail(e, "D2H copy / kernel");
  if (trace) {  // piece: H2D done, compute done, D2H done (ms after the call's first copy)
    for (size_t i = 1; i + 2 < tev.size(); i += 3) {
      float a = 0, b = 0, c = 0;
      cudaEventElapsedTime(&a, tev[0], tev[i]);
      cudaEventElapsedTime(&b, tev[0], tev[i + 1]);
      cudaEventElapsedTime(&c, tev[0], tev[i + 2]);
      fprintf(stderr, "piece %2zu  in %.3f  comp %.3f  out %.3f  enqueued %.3f\n", i / 3, a, b, c,
              thost[i / 3]);
    }
    for (auto x : tev) cudaEventDestroy(x);
  }
  return PASA_B200_OK;
}

#if defined(PASA_TRACE) || defined(PASA_TRACE_CTA)
// Profiling builds only (libpasa_b200_trace.so): device buffer of
// kTraceCtas * 3 * 32 * 8 int64 that the fused kernel fills with clock64().
__attribute__((visibility("default"))) int pasa_b200_debug_set_trace(void* device_buf) {
  g_trace = static_cast<long long*>(device_buf);
  return PASA_B200_OK;
}
#endif

}  // extern "C"

int pasa_b200_generate(int32_t kind, double x0, double am, double p, uint64_t seed,
                       uint64_t tensor_id, uint64_t start, uint64_t n, void* out, void* stream) {
  g_last_error.clear();
  if (kind != 0 && kind != 1) return fail(PASA_B200_EINVAL, "generate: kind must be 0 or 1");
  if (kind == 1 && !(p > 0.0 && p < 1.0))
    return fail(PASA_B200_EINVAL, "generate: p must lie in (0, 1)");  // bench.cpp:59-61
  if (n && !out) return fail(PASA_B200_EINVAL, "generate: NULL output");
  GenParams gp{kind, x0, am, p, seed, tensor_id, start, n};
  const cudaError_t e = launch_generate(gp, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "generate");
}

int pasa_b200_generate_resonance(uint64_t seed, int32_t tensor_id, int32_t batch, int32_t heads,
                                 int32_t seq, int32_t head_dim, double qa, double ka, void* out,
                                 void* stream) {
  g_last_error.clear();
  if (tensor_id < 0 || tensor_id > 2)
    return fail(PASA_B200_EINVAL, "generate_resonance: tensor_id must be 0, 1 or 2");
  if (batch < 0 || heads < 0 || seq < 0 || head_dim <= 0)
    return fail(PASA_B200_EINVAL, "generate_resonance: negative or zero extent");
  if (!out && batch && heads && seq) return fail(PASA_B200_EINVAL, "generate_resonance: NULL output");
  ResonanceParams rp{seed, tensor_id, batch, heads, seq, head_dim, qa, ka};
  const cudaError_t e = launch_generate_resonance(rp, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "generate_resonance");
}
