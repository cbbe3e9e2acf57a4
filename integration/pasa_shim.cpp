// integration/pasa_shim.cpp -- link-time drop-in for the reference's pasa.o.
//
// Compiled against the REFERENCE's own headers (include/pasa/pasa.hpp), it
// defines the symbols other reference objects bind to -- build_shifting_matrix,
// shifting_matrix_inverse, PasaParams::make, preprocess_keys and pasa_attention
// (pasa.hpp:27-99) -- on top of libpasa_b200.so's C-ABI.  The per-block CPU primitives
// (recover_global_mean, correction_terms, OnlineState) are not provided: the B200 build
// runs that recursion on the device inside pasa_attention.  Linking the reference's bench.o (whose
// `sweep` calls PasaParams::make, pasa_attention and preprocess_keys,
// bench.cpp:136, :196, :224) against this file instead of pasa.o runs the
// reference's own harness on the B200 kernel.  INTEGRATION.md shows the recipe.
//
// Semantics follow the reference: same validation and exception types
// (pasa.cpp:200-211), inputs are FP16-exact doubles (tensor.hpp:19-20), output
// is tagged with the policy's vector precision (pasa.cpp:242).  Only the
// PASA_FP16 policy is offloaded; pasa_attention with any other policy throws (no CPU
// fallback); preprocess_keys under a non-PASA policy is the reference's FP64 range
// diagnostic and keeps the reference's own gemm.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pasa/matrix.hpp"
#include "pasa/pasa.hpp"
#include "pasa_b200.h"

namespace {

[[noreturn]] void rethrow_status(int rc) {
  const std::string msg = pasa_b200_last_error();
  if (rc == PASA_B200_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("pasa_b200: " + msg);
}

std::vector<uint16_t> to_half_bits(const pasa::Tensor4D& t) {
  std::vector<uint16_t> out(t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    const _Float16 h = static_cast<_Float16>(t.data[i]);
    std::memcpy(&out[i], &h, 2);
  }
  return out;
}

double half_bits_to_double(uint16_t b) {
  _Float16 h;
  std::memcpy(&h, &b, 2);
  return static_cast<double>(h);
}

bool is_pasa_fp16(const pasa::PrecisionPolicy& p) {
  return p.gemm_accum == pasa::Prec::FP32 && p.gemm_store == pasa::Prec::FP16 &&
         p.vector_prec == pasa::Prec::FP16;
}

}  // namespace

namespace pasa {

// Theorem 2.1's closed-form inverse of (I - lambda J): I + lambda / (1 - lambda s) J, FP64
// (pasa.cpp:37-51); singular exactly when lambda s == 1 (beta == 1).
Matrix2D shifting_matrix_inverse(size_t s, double lambda) {
  const double denom = 1.0 - lambda * static_cast<double>(s);
  if (denom == 0.0) throw SingularMatrixError("shifting matrix is singular: lambda * s == 1 (beta == 1)");
  const double off = lambda / denom;
  Matrix2D m(s, s, Prec::FP64);
  for (size_t r = 0; r < s; ++r) {
    double* row = m.row(r);
    for (size_t c = 0; c < s; ++c) row[c] = r == c ? 1.0 + off : off;
  }
  return m;
}

Matrix2D build_shifting_matrix(size_t s2, double beta, double alpha, Prec prec) {
  if (s2 == 0) throw std::invalid_argument("shifting matrix: s2 must be >= 1");
  if (beta < 0.0 || beta > 1.0)
    throw std::invalid_argument("shifting matrix: beta must lie in [0, 1]");
  if (!(alpha > 0.0)) throw std::invalid_argument("shifting matrix: alpha must be positive");
  double diag, off;
  if (prec == Prec::FP16) {
    uint16_t d16, o16;
    const int rc = pasa_b200_shift_entries(static_cast<int32_t>(s2), beta, alpha, &d16, &o16);
    if (rc) rethrow_status(rc);
    diag = half_bits_to_double(d16);
    off = half_bits_to_double(o16);
  } else {
    const double n = static_cast<double>(s2);
    diag = round_to(prec, (1.0 - beta / n) / alpha);
    off = round_to(prec, -beta / (alpha * n));
  }
  Matrix2D m(s2, s2, prec);
  for (size_t r = 0; r < s2; ++r)
    for (size_t c = 0; c < s2; ++c) m.at(r, c) = (r == c) ? diag : off;
  return m;
}

PasaParams PasaParams::make(size_t s2, double beta, double alpha, Prec prec) {
  if (beta < 0.0 || beta >= 1.0)
    throw std::invalid_argument("pasa params: beta must lie in [0, 1); beta == 1 has no recovery");
  PasaParams p;
  p.beta = beta;
  p.alpha = alpha;
  p.s2 = s2;
  p.m = build_shifting_matrix(s2, beta, alpha, prec);
  return p;
}

// K^T * M on the device (bit-exact with the reference's FP32 sequential GEMM).
//
// Other policies are the reference's own diagnostics, not the offloaded path: range_report
// (bench.cpp:136, run by sweep() when SweepOptions::diagnose is set) asks for the FP64 K'
// ranges with the GoldenFp64 policy.  Those go to the reference's gemm (matrix.o, in the
// link set) exactly as pasa.cpp:53-56 does, so the drop-in keeps every pasa.o feature.
Matrix2D preprocess_keys(const Matrix2D& k_block, const Matrix2D& m,
                         const PrecisionPolicy& policy) {
  if (!is_pasa_fp16(policy)) return gemm(transpose(k_block), m, false, policy);
  const size_t s2 = k_block.rows, d = k_block.cols;
  if (m.rows != s2 || m.cols != s2) throw std::invalid_argument("gemm: inner dimensions disagree");
  // Recover (beta, alpha) from the two distinct entries: diag - off = 1/alpha.
  const double alpha = 1.0 / (m.at(0, 0) - (s2 > 1 ? m.at(0, 1) : 0.0));
  const double beta = -(s2 > 1 ? m.at(0, 1) : 0.0) * alpha * static_cast<double>(s2);
  Tensor4D kt(1, 1, s2, d, Prec::FP16);
  std::memcpy(kt.data.data(), k_block.data.data(), s2 * d * sizeof(double));
  std::vector<uint16_t> kh = to_half_bits(kt), kp(s2 * d);
  pasa_b200_desc desc{1, 1, 1, static_cast<int32_t>(s2), static_cast<int32_t>(s2),
                      static_cast<int32_t>(d), static_cast<int32_t>(s2),
                      static_cast<int32_t>(s2), 0, 0, beta, alpha};
  // The device entry point takes device buffers: stage through the host API
  // of the pre-pass via a tiny device round trip.
  int rc = pasa_b200_preprocess_keys_host(&desc, kh.data(), kp.data(), m.at(0, 0),
                                          s2 > 1 ? m.at(0, 1) : 0.0);
  if (rc) rethrow_status(rc);
  Matrix2D out(d, s2, policy.gemm_store);
  for (size_t c = 0; c < s2; ++c)
    for (size_t t = 0; t < d; ++t) out.at(t, c) = half_bits_to_double(kp[c * d + t]);
  return out;
}

Tensor4D pasa_attention(const AttentionProblem& problem, const PasaParams& params,
                        const PrecisionPolicy& policy, const AttnOptions& opts,
                        RunDiagnostics* diag) {
  // opts.threads is a CPU-loop knob; opts.diagnose's FP64 side channel is not offloaded
  if (params.s2 != problem.s2) throw std::invalid_argument("pasa: params.s2 does not match the problem");
  if (params.m.rows != params.s2 || params.m.cols != params.s2)
    throw std::invalid_argument("pasa: shifting matrix has the wrong shape");
  if (params.alpha != problem.alpha)
    throw std::invalid_argument("pasa: params.alpha does not match sqrt(d)");
  if (params.beta == 1.0) throw std::invalid_argument("pasa: beta == 1 has no recovery");
  if (!is_pasa_fp16(policy))  // PASA_FP16 and, for beta == 0, FA_PARTIAL_FP16 share these precisions
    throw std::invalid_argument("pasa_b200 offloads the PASA_FP16 policy only");
  // beta == 0 degrades to the blocked FP16 attention (pasa.cpp:212-221); the device runs it
  // as the FA16 mode of the same kernel, which implements the -inf initial max only.
  if (params.beta == 0.0 && opts.m0 != M0Mode::NegInf)
    throw std::invalid_argument("pasa_b200: beta == 0 offloads the m0 = -inf flash_attention only");
  const Tensor4D& q = problem.q;
  pasa_b200_desc desc{static_cast<int32_t>(q.batch), static_cast<int32_t>(q.heads),
                      static_cast<int32_t>(problem.k.heads), static_cast<int32_t>(q.seq),
                      static_cast<int32_t>(problem.k.seq), static_cast<int32_t>(q.dim),
                      static_cast<int32_t>(problem.s1), static_cast<int32_t>(problem.s2), 0, 0,
                      params.beta, problem.alpha};
  std::vector<uint16_t> qh = to_half_bits(q), kh = to_half_bits(problem.k),
                        vh = to_half_bits(problem.v), oh(q.size());
  pasa_b200_diag dd{};
  const int rc = diag ? pasa_b200_attention_host_diag(&desc, qh.data(), kh.data(), vh.data(),
                                                      oh.data(), &dd)
                      : pasa_b200_attention_host(&desc, qh.data(), kh.data(), vh.data(), oh.data());
  if (rc) rethrow_status(rc);
  Tensor4D out(q.batch, q.heads, q.seq, q.dim, policy.vector_prec);
  for (size_t i = 0; i < out.size(); ++i) out.data[i] = half_bits_to_double(oh[i]);
  if (diag) {  // the device's RunDiagnostics (store statistics + output counters)
    RunDiagnostics d;
    d.store_finite_min = dd.store_finite_min;
    d.store_finite_max = dd.store_finite_max;
    d.store_pos_inf = dd.store_pos_inf;
    d.store_neg_inf = dd.store_neg_inf;
    d.store_nan = dd.store_nan;
    d.out_total = dd.out_total;
    d.out_nonfinite = dd.out_nonfinite;
    diag->merge(d);
  }
  return out;
}

}  // namespace pasa
