/*
 * pasa_b200.h -- C-ABI of the B200-native PASA forward (libpasa_b200.so).
 *
 * Plain C types only: device or host pointers, sizes, a status code.  Every
 * entry point replaces one piece of the reference C++ operator API in
 * /root/reference/proj (citations are include/pasa/<file>:<line> or
 * src/<file>:<line>); INTEGRATION.md shows the bindings a maintainer adds.
 *
 * Layouts (reference tensor.hpp:13-29): Q is (B, Hq, S1, d), K and V are
 * (B, Hkv, S2, d), O is (B, Hq, S1, d); dense row-major BHSD, IEEE binary16
 * (the reference carries FP16-exact values in doubles, tensor.hpp:19-20).
 * Hq == Hkv reproduces the reference; Hq % Hkv == 0 adds grouped-query heads.
 *
 * Status codes: 0 success, otherwise one of PASA_B200_E* (negative).  The
 * reference throws std::invalid_argument for the same conditions
 * (pasa.cpp:200-211, tensor.cpp:19-55); pasa_b200_last_error() returns the
 * message of the last failure on the calling thread.  NaN/Inf in the OUTPUT
 * are results, not errors.
 */
#ifndef PASA_B200_H_
#define PASA_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PASA_B200_API __attribute__((visibility("default")))
#else
#define PASA_B200_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PASA_B200_OK 0
#define PASA_B200_EINVAL -1      /* shape / parameter violation (invalid_argument) */
#define PASA_B200_EUNSUPPORTED -2 /* valid for the reference, not for this build   */
#define PASA_B200_ECUDA -3       /* CUDA runtime error                            */
#define PASA_B200_ENODEV -4      /* no sm_100 device                              */

/* Problem + parameters: AttentionProblem (tensor.hpp:41-51) + PasaParams
 * (pasa.hpp:57-64) + the causal extension.  The shifting matrix M is not
 * passed: it is fully determined by (s2, beta, alpha) at FP16
 * (pasa.cpp:97-108, built by bench.cpp:196 with Prec::FP16). */
typedef struct pasa_b200_desc {
  int32_t batch;     /* B                                                      */
  int32_t heads_q;   /* Hq                                                     */
  int32_t heads_kv;  /* Hkv; must divide Hq (reference requires equality)      */
  int32_t seq_q;     /* S1, multiple of s1                                     */
  int32_t seq_kv;    /* S2, multiple of s2                                     */
  int32_t head_dim;  /* d in {64, 128}                                         */
  int32_t s1;        /* query block; numerically irrelevant (any divisor of S1) */
  int32_t s2;        /* KV block = shifting-matrix size, <= 128 (128 is fastest)*/
  int32_t causal;    /* 0: reference semantics; 1: causal, bottom-right aligned: query
                        row r sees keys <= r + S2 - S1 (S1 <= S2, any s2 and offset) */
  int32_t layout;    /* Q, K, V, O memory order: 0 = BHSD (the reference's Tensor4D,
                        tensor.hpp:27-29), 1 = BSHD ((B, S, H, d) row-major, as most model
                        code stores activations); the workspace (K', V') is always BHSD.
                        BSHD: fused path and host entry point; the reference-parity
                        pasa_b200_preprocess_keys* stay BHSD */
  double beta;       /* shift fraction in [0, 1) (pasa.cpp:98-101); 0 = FP16 FA */
  double alpha;      /* static scale, must equal sqrt(d) (pasa.cpp:206-208)     */
} pasa_b200_desc;

/* RunDiagnostics (attention.hpp:30-48) accumulated on the device: the scores the
 * tensor core stored (S' in PASA mode, S in the FP16 FA mode; masked entries
 * excluded) -- finite min/max in the reference's units (S'/alpha-scaled, i.e. the
 * kernel's log2(e)/2-scaled store divided back) and inf/NaN counts -- and the
 * output counters.  A DEVICE pointer, reset with pasa_b200_diag_reset; pass NULL
 * to skip (no cost).  Accumulates (merge semantics) across calls. */
typedef struct pasa_b200_diag {
  unsigned long long out_nonfinite;
  unsigned long long out_total;
  unsigned long long store_pos_inf;
  unsigned long long store_neg_inf;
  unsigned long long store_nan;
  float store_finite_min; /* +inf when nothing finite was stored */
  float store_finite_max; /* -inf when nothing finite was stored */
} pasa_b200_diag;

/* Library version (major*10000 + minor*100 + patch). */
PASA_B200_API int pasa_b200_version(void);

/* Message of the last failing call on this thread ("" if none). */
PASA_B200_API const char* pasa_b200_last_error(void);

/* The two distinct entries of the shifting matrix M, as binary16 bit
 * patterns: diag = fl16((1 - beta/s2)/alpha), off = fl16(-beta/(alpha*s2)).
 * Replaces build_shifting_matrix (pasa.hpp:27-28, pasa.cpp:16-35) /
 * PasaParams::make (pasa.cpp:97-108) with prec = FP16. */
PASA_B200_API int pasa_b200_shift_entries(int32_t s2, double beta, double alpha, uint16_t* diag_f16,
                            uint16_t* off_f16);

/* Validate a descriptor exactly like make_problem (tensor.cpp:19-55) and
 * pasa_attention (pasa.cpp:200-211); 0 if the fused path accepts it. */
PASA_B200_API int pasa_b200_check(const pasa_b200_desc* desc);

/* Bytes of device workspace pasa_b200_attention_fwd needs (K' and the
 * scaled V' for every KV head and block, plus per-head statistics). */
PASA_B200_API size_t pasa_b200_workspace_size(const pasa_b200_desc* desc);

/* Key pre-pass K'_j = K_j^T M for every (b, kv head, j) (pasa.cpp:53-56, the
 * loop at :231-240), device pointers, stream-ordered.  Output layout is
 * K-major: kp[(b, h, j*s2 + c), t] = K'_j[t][c].  lscale = 1 gives the
 * reference's bits exactly (FP32 sequential accumulate, one FP16 rounding);
 * the fused path uses lscale = log2(e)/2.  vmax (nullable, B*Hkv floats) gets
 * max|V| per head when v is non-NULL. */
PASA_B200_API int pasa_b200_preprocess_keys(const pasa_b200_desc* desc, const void* k, const void* v,
                              void* kp, float* vmax, float lscale, void* stream);

/* The key pre-pass from HOST buffers with the shifting matrix given by its
 * two entries (as PasaParams::m holds them; they must be FP16 values): the
 * drop-in for preprocess_keys (pasa.hpp:34-36) called per block by a CPU
 * caller (the reference's range_report, bench.cpp:136).  lscale = 1, so the
 * result carries the reference's bits.  Synchronous. */
PASA_B200_API int pasa_b200_preprocess_keys_host(const pasa_b200_desc* desc, const uint16_t* k,
                                                 uint16_t* kp, double m_diag, double m_off);

/* The PASA forward, device pointers, stream-ordered, asynchronous.
 * Replaces pasa::pasa_attention (pasa.hpp:95-99, pasa.cpp:196-293) for the
 * PASA_FP16 policy; beta == 0 runs pasa_b200_flash_fp16_fwd like the reference
 * (pasa.cpp:212-221).  workspace must hold pasa_b200_workspace_size() bytes.
 * stream is a cudaStream_t (NULL = legacy default stream). */
PASA_B200_API int pasa_b200_attention_fwd(const pasa_b200_desc* desc, const void* q, const void* k,
                            const void* v, void* o, void* workspace, size_t workspace_bytes,
                            pasa_b200_diag* diag, void* stream);

/* Query-row shard of pasa_b200_attention_fwd: computes the rows of query tiles
 * [tile0, tile0 + ntiles) (128 rows each; the last tile may be ragged) of every (b, h) and
 * leaves the other rows of o untouched.  The key pre-pass runs over every key, and each tile
 * is computed exactly as in the whole problem (same S1, S2, causal offset, K', V', c0), so
 * the union of shards is bit-identical to one pasa_b200_attention_fwd call.  This is what
 * balances a problem with fewer (b, kv head) units than GPUs (split q-tiles).
 * Replaces: the (b, h, i) loop of pasa_attention restricted to a range of i
 * (pasa.cpp:243-287). */
PASA_B200_API int pasa_b200_attention_fwd_tiles(const pasa_b200_desc* d, const void* q, const void* k,
                                                const void* v, void* o, void* workspace,
                                                size_t workspace_bytes, int32_t tile0, int32_t ntiles,
                                                void* stream);

/* The full pre-pass of the fused kernel, device pointers, stream-ordered:
 * kp = K'^T blocks with lscale = log2(e)/2 (as pasa_b200_preprocess_keys),
 * vmax = max|V| per (b, kv head), and vp = V * 2^-c0 per head with
 * c0 = max(0, ceil(log2(S2 * vmax / 2^14))) -- the exact power-of-two scale
 * that keeps the FP16 O accumulator bounded. */
PASA_B200_API int pasa_b200_preprocess(const pasa_b200_desc* desc, const void* k, const void* v,
                                       void* kp, void* vp, float* vmax, void* stream);

/* The fused forward on pre-processed keys and values (kp, vp, vmax from
 * pasa_b200_preprocess).  Lets a caller keep K'/V' resident and reuse them
 * across calls (same keys, many query batches). */
PASA_B200_API int pasa_b200_attention_fwd_prepped(const pasa_b200_desc* desc, const void* q,
                                                  const void* kp, const void* vp, const float* vmax,
                                                  void* o, void* stream);

/* The naive FP16 FlashAttention on the same pipeline: flash_attention with
 * the FA_PARTIAL_FP16 policy (attention.cpp:92-180): raw K, FP16 score store,
 * the 1/alpha scale applied AFTER the store (so |QK^T| > 65504 overflows to
 * inf and the output to NaN, :134-136), FP16 running max, no shift.  desc->beta
 * is ignored; pasa_b200_attention_fwd routes beta == 0 here (pasa.cpp:212-221).
 * The baseline PASA is measured against. */
PASA_B200_API int pasa_b200_flash_fp16_fwd(const pasa_b200_desc* desc, const void* q,
                                           const void* k, const void* v, void* o, void* stream);

/* Reset a device pasa_b200_diag (counters 0, min +inf, max -inf), stream-ordered. */
PASA_B200_API int pasa_b200_diag_reset(pasa_b200_diag* diag, void* stream);

/* pasa_b200_attention_fwd from HOST buffers (binary16 bit patterns): copies
 * Q, K, V in, runs, copies O back and synchronizes.  The drop-in for a CPU
 * caller of pasa_attention (the reference's `sweep`, bench.cpp:224).  Pipelined
 * over ~32 pieces of query heads (a few heads of one (batch, kv head) unit, or a
 * run of whole units): one H2D stream, a pre-pass stream, four compute streams and
 * one D2H stream, so copy-in, compute and copy-out of different pieces overlap and
 * the call is bound by the H2D copy.  Device buffers are cached per thread and
 * device; pinned host buffers copy at DMA speed (and overlap), pageable ones
 * through the driver's staging path.  With PASA_B200_HOST_TRACE set in the
 * environment the call prints each piece's H2D / compute / D2H completion times
 * to stderr (diagnostic). */
PASA_B200_API int pasa_b200_attention_host(const pasa_b200_desc* desc, const uint16_t* q, const uint16_t* k,
                             const uint16_t* v, uint16_t* o);

/* pasa_b200_attention_host that also fills a HOST pasa_b200_diag (overwritten):
 * the drop-in for pasa_attention(..., RunDiagnostics* diag) (pasa.cpp:244-291). */
PASA_B200_API int pasa_b200_attention_host_diag(const pasa_b200_desc* desc, const uint16_t* q,
                                                const uint16_t* k, const uint16_t* v, uint16_t* o,
                                                pasa_b200_diag* diag);

/* pasa_b200_attention_host over several GPUs of one process: the
 * (batch, kv head) units are split evenly over `devices` (n_devices entries; a device
 * may repeat), one host thread per device runs the pipelined host path on its share;
 * no exchange between devices.  The output is bit-identical to the single-device call.
 * BHSD only.  Blocks until every share is back in `o`. */
PASA_B200_API int pasa_b200_attention_host_multi(const pasa_b200_desc* desc, const uint16_t* q,
                                                 const uint16_t* k, const uint16_t* v, uint16_t* o,
                                                 const int32_t* devices, int32_t n_devices);

/* Device-side input generator: elements [start,
 * start + n) of tensor `tensor_id` (0 = Q, 1 = K, 2 = V) of the reference's
 * generate() (bench.cpp:28-72, rng.hpp:14-40) as binary16 into device memory:
 * kind 0 = uniform x0 - am + 2 am u, kind 1 = hybrid x0 + N(0,1) plus a
 * Bernoulli(p)-gated am * N(0,1) outlier.  Uniform is bit-identical to the
 * reference; hybrid agrees except within an ulp of an FP16 rounding boundary
 * (device log/cos).  Errors: p outside (0, 1) for hybrid -> EINVAL with the
 * reference's message.  Stream-ordered. */
PASA_B200_API int pasa_b200_generate(int32_t kind, double x0, double am, double p, uint64_t seed,
                                     uint64_t tensor_id, uint64_t start, uint64_t n, void* out,
                                     void* stream);

/* Resonance inputs (the SVD d = 64 case): BHSD tensor
 * `tensor_id` with Q = qa cos(2 pi 3c/d + 0.3h) + U(-1,1),
 * K = -ka (1 + 0.1 sin(2 pi s/512)) cos(...) + U(-1,1), V = U(-1,1).  Matches
 * the oracle's orc_generate_resonance.  Stream-ordered. */
PASA_B200_API int pasa_b200_generate_resonance(uint64_t seed, int32_t tensor_id, int32_t batch,
                                               int32_t heads, int32_t seq, int32_t head_dim,
                                               double qa, double ka, void* out, void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* PASA_B200_H_ */
