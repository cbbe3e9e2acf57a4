// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A thin extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// tests and bench.py's reference arm drive the reference's own public API
// (pasa::pasa_attention, pasa::flash_attention, pasa::golden_attention,
// pasa::generate, ...) through ctypes.  No reference source is copied here;
// this file only includes the reference headers at build time.
//
// Every function returns 0 on success and -1 when the reference threw; the
// message is then available from ref_last_error().

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pasa/attention.hpp"
#include "pasa/bench.hpp"
#include "pasa/beta_solver.hpp"
#include "pasa/pasa.hpp"
#include "pasa/tensor.hpp"

namespace {

thread_local std::string g_err;

pasa::Tensor4D to_tensor(const double* src, size_t b, size_t h, size_t s,
                         size_t d) {
  pasa::Tensor4D t(b, h, s, d, pasa::Prec::FP16);
  std::memcpy(t.data.data(), src, t.size() * sizeof(double));
  return t;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

pasa::PolicyId policy_from(int id) { return static_cast<pasa::PolicyId>(id); }

// RunDiagnostics -> {store_finite_min, store_finite_max, store_pos_inf,
// store_neg_inf, store_nan, out_nonfinite, out_total} (nullable destination).
void put_diag(const pasa::RunDiagnostics& d, double* out7) {
  if (!out7) return;
  out7[0] = d.store_finite_min;
  out7[1] = d.store_finite_max;
  out7[2] = static_cast<double>(d.store_pos_inf);
  out7[3] = static_cast<double>(d.store_neg_inf);
  out7[4] = static_cast<double>(d.store_nan);
  out7[5] = static_cast<double>(d.out_nonfinite);
  out7[6] = static_cast<double>(d.out_total);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// PolicyId values: 0 GOLDEN_FP64, 1 FA_FP32, 2 FA_PARTIAL_FP16, 3 FA_FULL_FP16,
// 4 PASA_FP16 (precision.hpp:41-47).
int ref_pasa_attention(size_t B, size_t H, size_t S1, size_t S2, size_t d,
                       size_t s1, size_t s2, const double* q, const double* k,
                       const double* v, double beta, int m_prec, int policy,
                       int threads, double* out, double* diag7) {
  return guarded([&] {
    auto prob = pasa::make_problem(to_tensor(q, B, H, S1, d),
                                   to_tensor(k, B, H, S2, d),
                                   to_tensor(v, B, H, S2, d), s1, s2);
    auto params = pasa::PasaParams::make(s2, beta, prob.alpha,
                                         static_cast<pasa::Prec>(m_prec));
    pasa::AttnOptions opts;
    opts.threads = threads;
    pasa::RunDiagnostics diag;
    auto o = pasa::pasa_attention(prob, params, pasa::policy_for(policy_from(policy)), opts,
                                  diag7 ? &diag : nullptr);
    std::memcpy(out, o.data.data(), o.size() * sizeof(double));
    put_diag(diag, diag7);
  });
}

int ref_flash_attention(size_t B, size_t H, size_t S1, size_t S2, size_t d,
                        size_t s1, size_t s2, const double* q, const double* k,
                        const double* v, int policy, int m0_zero, int threads,
                        double* out, double* diag7) {
  return guarded([&] {
    auto prob = pasa::make_problem(to_tensor(q, B, H, S1, d),
                                   to_tensor(k, B, H, S2, d),
                                   to_tensor(v, B, H, S2, d), s1, s2);
    pasa::AttnOptions opts;
    opts.threads = threads;
    opts.m0 = m0_zero ? pasa::M0Mode::Zero : pasa::M0Mode::NegInf;
    pasa::RunDiagnostics diag;
    auto o = pasa::flash_attention(prob, pasa::policy_for(policy_from(policy)), opts,
                                   diag7 ? &diag : nullptr);
    std::memcpy(out, o.data.data(), o.size() * sizeof(double));
    put_diag(diag, diag7);
  });
}

int ref_golden(size_t B, size_t H, size_t S1, size_t S2, size_t d, size_t s1,
               size_t s2, const double* q, const double* k, const double* v,
               int threads, double* out) {
  return guarded([&] {
    auto prob = pasa::make_problem(to_tensor(q, B, H, S1, d),
                                   to_tensor(k, B, H, S2, d),
                                   to_tensor(v, B, H, S2, d), s1, s2);
    auto o = pasa::golden_attention(prob, threads);
    std::memcpy(out, o.data.data(), o.size() * sizeof(double));
  });
}

// kind 0 uniform, 1 hybrid (bench.hpp:24).  Writes Q, K, V (B,H,S,d).
int ref_generate(int kind, double x0, double am, double p, uint64_t seed,
                 size_t B, size_t H, size_t S, size_t d, double* q, double* k,
                 double* v) {
  return guarded([&] {
    pasa::DistributionSpec spec;
    spec.kind = kind ? pasa::DistKind::Hybrid : pasa::DistKind::Uniform;
    spec.x0 = x0;
    spec.am = am;
    spec.p = p;
    spec.seed = seed;
    spec.batch = B;
    spec.heads = H;
    spec.seq = S;
    spec.dim = d;
    auto g = pasa::generate(spec);
    std::memcpy(q, g.q.data.data(), g.q.size() * sizeof(double));
    std::memcpy(k, g.k.data.data(), g.k.size() * sizeof(double));
    std::memcpy(v, g.v.data.data(), g.v.size() * sizeof(double));
  });
}

double ref_rmse(size_t n, const double* x, const double* g) {
  double r = 0.0;
  int rc = guarded([&] {
    pasa::Tensor4D a(1, 1, 1, n, pasa::Prec::FP64), b(1, 1, 1, n, pasa::Prec::FP64);
    std::memcpy(a.data.data(), x, n * sizeof(double));
    std::memcpy(b.data.data(), g, n * sizeof(double));
    r = pasa::rmse(a, b);
  });
  return rc ? -1.0 : r;
}

double ref_nan_stats(size_t n, const double* x) {
  pasa::Tensor4D a(1, 1, 1, n, pasa::Prec::FP64);
  std::memcpy(a.data.data(), x, n * sizeof(double));
  return pasa::nan_stats(a);
}

// The two distinct shifting-matrix entries as built by PasaParams::make.
int ref_shift_entries(size_t s2, double beta, double alpha, int prec,
                      double* diag, double* off) {
  return guarded([&] {
    auto m = pasa::build_shifting_matrix(s2, beta, alpha,
                                         static_cast<pasa::Prec>(prec));
    *diag = m.at(0, 0);
    *off = s2 > 1 ? m.at(0, 1) : 0.0;
  });
}

// K'_j = K_j^T * M for one s2 x d block, output d x s2 (reference layout).
int ref_preprocess_keys(size_t s2, size_t d, const double* kblock, double beta,
                        double alpha, int policy, double* out) {
  return guarded([&] {
    pasa::Matrix2D kb(s2, d, pasa::Prec::FP16);
    std::memcpy(kb.data.data(), kblock, s2 * d * sizeof(double));
    auto m = pasa::build_shifting_matrix(s2, beta, alpha, pasa::Prec::FP16);
    auto kp = pasa::preprocess_keys(kb, m, pasa::policy_for(policy_from(policy)));
    std::memcpy(out, kp.data.data(), kp.data.size() * sizeof(double));
  });
}

int ref_optimal_beta(double beta0, size_t n, double tol, double* beta_star,
                     size_t* iters, double* rel_err) {
  return guarded([&] {
    auto s = pasa::optimal_beta(beta0, n, tol);
    *beta_star = s.beta_star;
    *iters = s.iterations;
    *rel_err = s.report.rel_err;
  });
}

int ref_invariance(double beta, size_t n, double* out5) {
  return guarded([&] {
    auto r = pasa::invariance_parameter(beta, n);
    out5[0] = r.a;
    out5[1] = r.b;
    out5[2] = r.inva_ideal;
    out5[3] = r.inva_actual;
    out5[4] = r.rel_err;
  });
}

// The reference's report text (bench.cpp:249-316) for n rows given field by
// field: nums[i*14 + ...] = {x0, am, p, beta, rmse, nan_pct, s_min_before,
// s_max_before, s_min_after, s_max_after, wall_s, -, -, -}, ints[i*6 + ...] =
// {seed, B, N, S, d, has_ranges}; json = 0 -> report_csv, 1 -> report_json_rows.
// Returns the byte count written (truncated to cap - 1), or -1.
long ref_report(int n, const char* const* policy, const char* const* kind,
                const char* const* error, const double* nums, const long long* ints,
                int json, char* out, size_t cap) {
  std::string text;
  const int rc = guarded([&] {
    std::vector<pasa::RunReport> rows(n);
    for (int i = 0; i < n; ++i) {
      pasa::RunReport& r = rows[i];
      const double* f = nums + 14 * i;
      const long long* z = ints + 6 * i;
      r.policy = policy[i];
      r.kind = kind[i];
      r.error = error[i];
      r.x0 = f[0]; r.am = f[1]; r.p = f[2]; r.beta = f[3]; r.rmse = f[4]; r.nan_pct = f[5];
      r.s_min_before = f[6]; r.s_max_before = f[7]; r.s_min_after = f[8]; r.s_max_after = f[9];
      r.wall_s = f[10];
      r.seed = static_cast<uint64_t>(z[0]);
      r.batch = z[1]; r.heads = z[2]; r.seq = z[3]; r.dim = z[4];
      r.has_ranges = z[5] != 0;
    }
    text = json ? pasa::report_json_rows(rows) : pasa::report_csv(rows);
  });
  if (rc) return -1;
  const size_t m = text.size() < cap ? text.size() : cap - 1;
  std::memcpy(out, text.data(), m);
  out[m] = 0;
  return static_cast<long>(m);
}

}  // extern "C"
