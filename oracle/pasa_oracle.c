/*
 * oracle/pasa_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement of the reference PASA path (arXiv 2503.01873, reference at
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU baseline -- never as the thing measured or shipped.
 *
 * Two families of entry points live here:
 *
 *  (1) Reference restatements (orc_ref_*, orc_golden, orc_flash_ref, the
 *      generators, rmse, nan_pct).  These follow the reference's rounding
 *      points one for one and are pinned BIT-EXACTLY against the reference
 *      itself (compiled out-of-tree into oracle/_ref by oracle/Makefile) in
 *      tests/test_oracle_vs_ref.py.  Citations are proj/src/<file>:<line>.
 *
 *  (2) The kernel-numerics model (orc_model_*): the same algorithm with the
 *      numerics the B200 kernel documents in DESIGN.md section 4 (FP32 row
 *      statistics, incremental global mean, bounded O, log2 domain, causal and
 *      GQA extensions).  It is the tight oracle for the CUDA path; the
 *      restatement (1) is the loose "same inputs as the reference" oracle.
 *
 * Binary16 rounding uses the compiler's IEEE conversion to _Float16 (RNE,
 * overflow to inf at |x| >= 65520), which is the correctly rounded operation
 * the reference emulates in half.hpp:28-46.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Precision helpers (reference precision.hpp:20-32, half.hpp:28-46)         */
/* ------------------------------------------------------------------------ */

enum { P64 = 0, P32 = 1, P16 = 2, PR1 = 3 /* rank-1 pre-pass, accumulation mode only */ };

static inline double fl16(double x) { return (double)(_Float16)x; }
static inline double fl32(double x) { return (double)(float)x; }
static inline double rnd(int p, double x) {
  return p == P16 ? fl16(x) : (p == P32 ? fl32(x) : x);
}
/* exp in extended precision, one rounding at p (precision.hpp:30-32). */
static inline double exp_p(int p, double x) {
  return rnd(p, (double)expl((long double)x));
}
/* NaN-poisoning max (attention.cpp:86-91). */
static inline double nanmax2(double a, double b) {
  if (isnan(a) || isnan(b)) return NAN;
  return a > b ? a : b;
}

ORC_API double orc_f16_round(double x) { return fl16(x); }

ORC_API void orc_f16_round_array(const double* x, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] = fl16(x[i]);
}

static int resolve_threads(int requested) {
  if (requested > 0) return requested;
  const char* env = getenv("PASA_THREADS");
  if (env && atoi(env) > 0) return atoi(env);
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Shifting matrix and beta solver                                          */
/* ------------------------------------------------------------------------ */

/* The two distinct entries of M = I/alpha - beta*J/(alpha*s2), each rounded
 * once at `prec` (pasa.cpp:16-35, the diag/off expressions at :26-27). */
ORC_API int orc_shift_entries(size_t s2, double beta, double alpha, int prec,
                              double* diag, double* off) {
  if (s2 == 0 || beta < 0.0 || beta > 1.0 || !(alpha > 0.0)) return -1;
  const double n = (double)s2;
  *diag = rnd(prec, (1.0 - beta / n) / alpha);
  *off = rnd(prec, -beta / (alpha * n));
  return 0;
}

/* Invariance of the rounded shift (beta_solver.cpp:11-30). Out array:
 * {a, b, inva_ideal, inva_actual, rel_err}. */
ORC_API int orc_invariance(double beta, size_t n, double* out5) {
  if (!(beta > 0.0) || !(beta < 1.0) || n == 0) return -1;
  const double nd = (double)n;
  const double b = fl16(beta / nd);
  const double a = fl16(1.0 - beta / nd) + b;
  const double den = a - b * nd;
  if (den == 0.0) return -2;
  const double actual = b * nd / (a * den) + (1.0 - a) / a;
  const double ideal = beta / (1.0 - beta);
  out5[0] = a;
  out5[1] = b;
  out5[2] = ideal;
  out5[3] = actual;
  out5[4] = fabs(ideal - actual) / fabs(ideal);
  return 0;
}

/* Fixed point beta <- f/(1+f) (beta_solver.cpp:32-52). */
ORC_API int orc_optimal_beta(double beta0, size_t n, double tol,
                             double* beta_star, int* iters) {
  if (!(tol > 0.0)) return -1;
  double beta = beta0, rep[5];
  for (int it = 1; it <= 10000; ++it) {
    if (orc_invariance(beta, n, rep) != 0) return -2;
    const double f = rep[3];
    const double next = f / (1.0 + f);
    const double err = fabs(next - beta) / fabs(beta);
    beta = next;
    if (err <= tol) {
      *beta_star = beta;
      *iters = it;
      return 0;
    }
  }
  return -3;
}

/* ------------------------------------------------------------------------ */
/* Synthetic inputs (reference bench.cpp:28-72 over rng.hpp:14-41)           */
/* ------------------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline double draw_u01(uint64_t seed, uint64_t stream, uint64_t ctr) {
  const uint64_t h = mix64(mix64(mix64(seed) ^ stream) ^ ctr);
  return (double)(h >> 11) * 0x1.0p-53;
}
static inline double draw_normal(uint64_t seed, uint64_t stream, uint64_t i) {
  const double u1 = 1.0 - draw_u01(seed, stream, 2 * i);
  const double u2 = draw_u01(seed, stream, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* kind 0 = uniform(x0 +- am), 1 = hybrid normal + Bernoulli-gated outlier.
 * Fills n elements of tensor `tensor_id` (0=Q,1=K,2=V) starting at flat
 * index `start`, rounded to binary16 (bench.cpp:28-48). */
ORC_API int orc_generate(int kind, double x0, double am, double p,
                         uint64_t seed, uint64_t tensor_id, uint64_t start,
                         size_t n, double* out) {
  if (kind == 1 && !(p > 0.0 && p < 1.0)) return -1;
#pragma omp parallel for schedule(static)
  for (long long ii = 0; ii < (long long)n; ++ii) {
    const uint64_t idx = start + (uint64_t)ii;
    double v;
    if (kind == 0) {
      const double u = draw_u01(seed, tensor_id, idx);
      v = x0 - am + 2.0 * am * u;
    } else {
      const uint64_t base = tensor_id * 4;
      const double core = x0 + draw_normal(seed, base, idx);
      const int gate = draw_u01(seed, base + 2, idx) < p;
      v = gate ? core + am * draw_normal(seed, base + 1, idx) : core;
    }
    out[ii] = fl16(v);
  }
  return 0;
}

/* Resonance inputs: Q and
 * K share a head-dim cosine with a 180-degree lag, so Q.K^T is large and
 * negative.  BHSD layout, tensor_id as above. */
ORC_API void orc_generate_resonance(uint64_t seed, int tensor_id, size_t B,
                                    size_t H, size_t S, size_t d, double qa,
                                    double ka, double* out) {
  const double twopi = 2.0 * 3.14159265358979323846;
#pragma omp parallel for schedule(static)
  for (long long ii = 0; ii < (long long)(B * H * S * d); ++ii) {
    const size_t c = (size_t)ii % d;
    const size_t s = ((size_t)ii / d) % S;
    const size_t h = ((size_t)ii / (d * S)) % H;
    const double noise = 2.0 * draw_u01(seed, (uint64_t)tensor_id, ii) - 1.0;
    const double wave = cos(twopi * 3.0 * (double)c / (double)d + 0.3 * (double)h);
    double v;
    if (tensor_id == 0) {
      v = qa * wave + noise;
    } else if (tensor_id == 1) {
      v = -ka * (1.0 + 0.1 * sin(twopi * (double)s / 512.0)) * wave + noise;
    } else {
      v = noise;
    }
    out[ii] = fl16(v);
  }
}

/* ------------------------------------------------------------------------ */
/* Metrics (bench.cpp:74-100)                                                */
/* ------------------------------------------------------------------------ */

/* ||x - g|| / ||g|| with compensated sums; NaN if x is non-finite anywhere;
 * returns -1 when ||g|| == 0 (the reference throws ZeroNormError). */
ORC_API double orc_rmse(const double* x, const double* g, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return NAN;
  double s1 = 0, c1 = 0, s2 = 0, c2 = 0;
  for (size_t i = 0; i < n; ++i) {
    const double d = x[i] - g[i];
    double y = d * d - c1, t = s1 + y;
    c1 = (t - s1) - y;
    s1 = t;
    y = g[i] * g[i] - c2;
    t = s2 + y;
    c2 = (t - s2) - y;
    s2 = t;
  }
  if (s2 == 0.0) return -1.0;
  return sqrt(s1) / sqrt(s2);
}

ORC_API double orc_nan_pct(const double* x, size_t n) {
  if (n == 0) return 0.0;
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += !isfinite(x[i]);
  return 100.0 * (double)bad / (double)n;
}

/* ------------------------------------------------------------------------ */
/* Shared shapes                                                             */
/* ------------------------------------------------------------------------ */

/* Problem description shared by every attention entry point.  Q is
 * (B, Hq, S1, d), K and V are (B, Hkv, S2, d), all dense row-major BHSD
 * (tensor.hpp:27-29).  Hq must be a multiple of Hkv (GQA extension; the
 * reference requires Hq == Hkv, tensor.cpp:24-26).  q_offset is the absolute
 * position of Q row 0 (for sampled-query-block oracles under causal masks). */
typedef struct {
  size_t B, Hq, Hkv, S1, S2, d, s1, s2;
  int causal;
  size_t q_offset;
} orc_shape;

static inline const double* row_ptr(const double* t, size_t H, size_t S,
                                    size_t d, size_t b, size_t h, size_t s) {
  return t + ((b * H + h) * S + s) * d;
}

/* ------------------------------------------------------------------------ */
/* Golden FP64 attention (attention.cpp:66-90) + causal/GQA extension        */
/* ------------------------------------------------------------------------ */

ORC_API int orc_golden(const orc_shape* sh, const double* q, const double* k,
                       const double* v, double* o, int threads) {
  if (sh->Hq % sh->Hkv) return -1;
  const double alpha = sqrt((double)sh->d);
  const size_t grp = sh->Hq / sh->Hkv;
  const int nt = resolve_threads(threads);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long x = 0; x < (long long)(sh->B * sh->Hq * sh->S1); ++x) {
    const size_t r = (size_t)x % sh->S1;
    const size_t h = ((size_t)x / sh->S1) % sh->Hq;
    const size_t b = (size_t)x / (sh->S1 * sh->Hq);
    const size_t hk = h / grp;
    const double* qr = row_ptr(q, sh->Hq, sh->S1, sh->d, b, h, r);
    size_t ncols = sh->S2;
    if (sh->causal) {
      const size_t pos = sh->q_offset + r;
      ncols = pos + 1 < sh->S2 ? pos + 1 : sh->S2;
    }
    double* s = (double*)malloc(sizeof(double) * (ncols ? ncols : 1));
    double mx = -INFINITY;
    for (size_t c = 0; c < ncols; ++c) {
      const double* kr = row_ptr(k, sh->Hkv, sh->S2, sh->d, b, hk, c);
      double acc = 0.0;
      for (size_t t = 0; t < sh->d; ++t) acc = acc + qr[t] * kr[t];
      s[c] = acc / alpha;
      if (isnan(s[c])) mx = NAN;
      else if (!isnan(mx) && s[c] > mx) mx = s[c];
    }
    double l = 0.0;
    for (size_t c = 0; c < ncols; ++c) {
      s[c] = (double)expl((long double)(s[c] - mx));
      l = l + s[c];
    }
    double* orow = o + ((b * sh->Hq + h) * sh->S1 + r) * sh->d;
    for (size_t n = 0; n < sh->d; ++n) orow[n] = 0.0;
    for (size_t c = 0; c < ncols; ++c) {
      const double pc = s[c] / l;
      const double* vr = row_ptr(v, sh->Hkv, sh->S2, sh->d, b, hk, c);
      for (size_t n = 0; n < sh->d; ++n) orow[n] = orow[n] + pc * vr[n];
    }
    free(s);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Policy GEMM element (matrix.cpp:26-74): sequential ascending inner index, */
/* every product and add rounded at `acc`, one rounding at `store`.          */
/* ------------------------------------------------------------------------ */

static inline double dot_policy(const double* a, size_t astride,
                                const double* b, size_t bstride, size_t n,
                                int acc, int store) {
  double s = 0.0;
  if (acc == P32) {
    for (size_t t = 0; t < n; ++t) s = fl32(s + fl32(a[t * astride] * b[t * bstride]));
  } else if (acc == P16) {
    for (size_t t = 0; t < n; ++t) s = fl16(s + fl16(a[t * astride] * b[t * bstride]));
  } else {
    for (size_t t = 0; t < n; ++t) s = s + a[t * astride] * b[t * bstride];
  }
  return rnd(store, s);
}

/* ------------------------------------------------------------------------ */
/* Blocked FA under a policy (attention.cpp:92-180), GQA extension.           */
/* policy = {accum, store, vec}; m0_zero selects the conformance m0 = 0.      */
/* ------------------------------------------------------------------------ */

ORC_API int orc_flash_ref(const orc_shape* sh, const double* q,
                          const double* k, const double* v, double* o,
                          int p_acc, int p_store, int p_vec, int m0_zero,
                          int threads) {
  if (sh->Hq % sh->Hkv || sh->causal) return -1;
  if (sh->S1 % sh->s1 || sh->S2 % sh->s2) return -2;
  const size_t s1 = sh->s1, s2 = sh->s2, d = sh->d;
  const size_t nq = sh->S1 / s1, nkv = sh->S2 / s2, grp = sh->Hq / sh->Hkv;
  const double alpha = sqrt((double)d);
  const int nt = resolve_threads(threads);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long x = 0; x < (long long)(sh->B * sh->Hq * nq); ++x) {
    const size_t i = (size_t)x % nq;
    const size_t h = ((size_t)x / nq) % sh->Hq;
    const size_t b = (size_t)x / (nq * sh->Hq);
    const size_t hk = h / grp;
    double* m = malloc(sizeof(double) * s1);
    double* l = calloc(s1, sizeof(double));
    double* oacc = calloc(s1 * d, sizeof(double));
    double* S = malloc(sizeof(double) * s1 * s2);
    double* T = malloc(sizeof(double) * s1 * d);
    for (size_t r = 0; r < s1; ++r) m[r] = m0_zero ? 0.0 : -INFINITY;
    for (size_t j = 0; j < nkv; ++j) {
      for (size_t r = 0; r < s1; ++r) {
        const double* qr = row_ptr(q, sh->Hq, sh->S1, d, b, h, i * s1 + r);
        for (size_t c = 0; c < s2; ++c) {
          const double* kr = row_ptr(k, sh->Hkv, sh->S2, d, b, hk, j * s2 + c);
          const double sv = dot_policy(qr, 1, kr, 1, d, p_acc, p_store);
          S[r * s2 + c] = rnd(p_vec, sv / alpha); /* scale after store :134-136 */
        }
      }
      for (size_t r = 0; r < s1; ++r) {
        double* sr = S + r * s2;
        double mloc = -INFINITY;
        for (size_t c = 0; c < s2; ++c) {
          if (isnan(sr[c])) { mloc = NAN; break; }
          if (sr[c] > mloc) mloc = sr[c];
        }
        const double mnew = nanmax2(m[r], mloc);
        double lloc = 0.0;
        for (size_t c = 0; c < s2; ++c) {
          sr[c] = exp_p(p_vec, rnd(p_vec, sr[c] - mnew));
          lloc = rnd(p_vec, lloc + sr[c]);
        }
        const double fac = exp_p(p_vec, rnd(p_vec, m[r] - mnew));
        l[r] = rnd(p_vec, rnd(p_vec, fac * l[r]) + lloc);
        for (size_t n = 0; n < d; ++n) {
          const double* vcol = row_ptr(v, sh->Hkv, sh->S2, d, b, hk, j * s2) + n;
          T[r * d + n] = dot_policy(sr, 1, vcol, d, s2, p_acc, p_store);
          oacc[r * d + n] = rnd(p_vec, rnd(p_vec, fac * oacc[r * d + n]) + T[r * d + n]);
        }
        m[r] = mnew;
      }
    }
    for (size_t r = 0; r < s1; ++r) {
      double* orow = o + ((b * sh->Hq + h) * sh->S1 + i * s1 + r) * d;
      for (size_t n = 0; n < d; ++n) orow[n] = rnd(p_vec, oacc[r * d + n] / l[r]);
    }
    free(m); free(l); free(oacc); free(S); free(T);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Key pre-pass K'_j = K_j^T * M (pasa.cpp:53-56 via matrix.cpp:26-74).       */
/* Output layout is the kernel's: kp[c*d + t] = K'_j[t][c] (s2 x d, K-major). */
/* `lscale` != 1 multiplies the FP32 chain once before the store rounding     */
/* (the log2-domain variant the B200 kernel uses; 1.0 reproduces the ref).    */
/* ------------------------------------------------------------------------ */

static void prepass_block(const double* kb, size_t s2, size_t d, double diag,
                          double off, int p_acc, int p_store, double lscale,
                          double* kp) {
  if (p_acc == PR1) {
    /* The fused path's rank-1 pre-pass (pasa_kprep_rank1_kernel): M = (diag-off) I
     * + off J, so K'[t][c] = fl16(fl32(fma(diag - off, K[c][t], fl32(off * colsum[t])))
     * * lscale) with colsum the FP32 sum over p ascending. */
    const double dm = (double)((float)diag - (float)off);
    for (size_t t = 0; t < d; ++t) {
      float cs = 0.f;
      for (size_t p = 0; p < s2; ++p) cs = cs + (float)kb[p * d + t];
      const double os = fl32(off * (double)cs);
      for (size_t c = 0; c < s2; ++c) {
        double a = fl32(fma(dm, kb[c * d + t], os));
        a = fl32(a * (double)(float)lscale);
        kp[c * d + t] = rnd(p_store, a);
      }
    }
    return;
  }
  for (size_t t = 0; t < d; ++t) {
    for (size_t c = 0; c < s2; ++c) {
      double acc = 0.0;
      for (size_t p = 0; p < s2; ++p) {
        const double mpc = (p == c) ? diag : off;
        const double prod = kb[p * d + t] * mpc;
        if (p_acc == P32) acc = fl32(acc + fl32(prod));
        else if (p_acc == P16) acc = fl16(acc + fl16(prod));
        else acc = acc + prod;
      }
      if (lscale != 1.0) acc = fl32(acc * (double)(float)lscale); /* FP32 multiply */
      kp[c * d + t] = rnd(p_store, acc);
    }
  }
}

ORC_API int orc_preprocess_keys(const double* k, size_t B, size_t Hkv,
                                size_t S2, size_t d, size_t s2, double diag,
                                double off, int p_acc, int p_store,
                                double lscale, double* kp, int threads) {
  if (S2 % s2) return -1;
  const size_t nkv = S2 / s2;
  const int nt = resolve_threads(threads);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long x = 0; x < (long long)(B * Hkv * nkv); ++x) {
    const size_t off_rows = (size_t)x * s2; /* (b, h, j) blocks are contiguous */
    prepass_block(k + off_rows * d, s2, d, diag, off, p_acc, p_store, lscale,
                  kp + off_rows * d);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Reference PASA restatement (pasa.cpp:196-293; absorb :117-182; finalize    */
/* :184-194), general policy so the FP64-equivalence KAT can run.             */
/* diag/off are the shift entries as rounded by PasaParams::make.             */
/* ------------------------------------------------------------------------ */

ORC_API int orc_pasa_ref(const orc_shape* sh, const double* q, const double* k,
                         const double* v, double* o, double beta, double diag,
                         double off, int p_acc, int p_store, int p_vec,
                         int threads) {
  if (sh->Hq % sh->Hkv || sh->causal) return -1;
  if (sh->S1 % sh->s1 || sh->S2 % sh->s2) return -2;
  if (!(beta > 0.0 && beta < 1.0)) return -3; /* beta==0 routes to FA (:212) */
  const size_t s1 = sh->s1, s2 = sh->s2, d = sh->d;
  const size_t nq = sh->S1 / s1, nkv = sh->S2 / s2, grp = sh->Hq / sh->Hkv;
  const double inva = beta / (1.0 - beta); /* pasa.cpp:85 */
  const int nt = resolve_threads(threads);
  double* kp = malloc(sizeof(double) * sh->B * sh->Hkv * sh->S2 * d);
  orc_preprocess_keys(k, sh->B, sh->Hkv, sh->S2, d, s2, diag, off, p_acc,
                      p_store, 1.0, kp, nt);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long x = 0; x < (long long)(sh->B * sh->Hq * nq); ++x) {
    const size_t i = (size_t)x % nq;
    const size_t h = ((size_t)x / nq) % sh->Hq;
    const size_t b = (size_t)x / (nq * sh->Hq);
    const size_t hk = h / grp;
    double* m = calloc(s1, sizeof(double));
    double* l = calloc(s1, sizeof(double));
    double* fbar = calloc(s1, sizeof(double));
    double* oacc = calloc(s1 * d, sizeof(double));
    double* S = malloc(sizeof(double) * s2);
    for (size_t j = 1; j <= nkv; ++j) {
      const double* kpj = kp + ((b * sh->Hkv + hk) * sh->S2 + (j - 1) * s2) * d;
      const double* vj = row_ptr(v, sh->Hkv, sh->S2, d, b, hk, (j - 1) * s2);
      for (size_t r = 0; r < s1; ++r) {
        const double* qr = row_ptr(q, sh->Hq, sh->S1, d, b, h, i * s1 + r);
        /* S' = q_i K'_j at policy (pasa.cpp:256). */
        for (size_t c = 0; c < s2; ++c)
          S[c] = dot_policy(qr, 1, kpj + c * d, 1, d, p_acc, p_store);
        /* absorb (pasa.cpp:128-131): m', P, l', rowmean. */
        double mloc = -INFINITY;
        for (size_t c = 0; c < s2; ++c) {
          if (isnan(S[c])) { mloc = NAN; break; }
          if (S[c] > mloc) mloc = S[c];
        }
        double ssum = 0.0;
        for (size_t c = 0; c < s2; ++c) ssum = rnd(p_vec, ssum + S[c]);
        const double sbar = rnd(p_vec, ssum / (double)s2);
        double lloc = 0.0;
        for (size_t c = 0; c < s2; ++c) {
          S[c] = exp_p(p_vec, rnd(p_vec, S[c] - mloc)); /* S now holds P */
          lloc = rnd(p_vec, lloc + S[c]);
        }
        /* recover_global_mean (pasa.cpp:58-75). */
        double fnew;
        if (j == 1) fnew = sbar;
        else {
          const double t = rnd(p_vec, rnd(p_vec, (double)(j - 1) * fbar[r]) + sbar);
          fnew = rnd(p_vec, t / (double)j);
        }
        /* correction_terms (pasa.cpp:77-95); j==1 uses F_prev = F_new. */
        const double fprev = (j == 1) ? fnew : fbar[r];
        const double dmp = rnd(p_vec, inva * rnd(p_vec, fprev - fnew));
        const double dmc = rnd(p_vec, inva * rnd(p_vec, sbar - fnew));
        /* corrected max (pasa.cpp:139-148). */
        const double cand_cur = rnd(p_vec, mloc + dmc);
        const double mnew = (j == 1) ? cand_cur
                                     : nanmax2(rnd(p_vec, m[r] + dmp), cand_cur);
        /* exp corrections (pasa.cpp:150-160). */
        const double ecur = exp_p(p_vec, rnd(p_vec, rnd(p_vec, mloc - mnew) + dmc));
        double eprev = 0.0;
        if (j > 1) eprev = exp_p(p_vec, rnd(p_vec, rnd(p_vec, m[r] - mnew) + dmp));
        /* l (pasa.cpp:162-166). */
        const double lcur = rnd(p_vec, ecur * lloc);
        l[r] = (j == 1) ? lcur : rnd(p_vec, rnd(p_vec, eprev * l[r]) + lcur);
        /* O (pasa.cpp:168-178): T = P V_j at policy, then combine. */
        double* orow = oacc + r * d;
        for (size_t n = 0; n < d; ++n) {
          const double tn = dot_policy(S, 1, vj + n, d, s2, p_acc, p_store);
          const double cur = rnd(p_vec, ecur * tn);
          orow[n] = (j == 1) ? cur : rnd(p_vec, cur + rnd(p_vec, eprev * orow[n]));
        }
        m[r] = mnew;
        fbar[r] = fnew;
      }
    }
    /* finalize (pasa.cpp:184-194). */
    for (size_t r = 0; r < s1; ++r) {
      double* dst = o + ((b * sh->Hq + h) * sh->S1 + i * s1 + r) * d;
      for (size_t n = 0; n < d; ++n) dst[n] = rnd(p_vec, oacc[r * d + n] / l[r]);
    }
    free(m); free(l); free(fbar); free(oacc); free(S);
  }
  free(kp);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Kernel-numerics model.                              */
/*                                                                           */
/* Same recurrence as orc_pasa_ref with these documented deviations, each    */
/* exact in real arithmetic:                                                 */
/*  - every score lives in the L domain (lscale = log2 e: 2^x replaces e^x), */
/*  - row statistics (sum of S', mean, F, corrections, running max, l) are   */
/*    FP32; the S' row sum runs as eight chains (kernel order) or, at d <=  */
/*    112, is the tensor core's q . (sum of the block's K' columns) (the    */
/*    pseudo-average GEMM); the P row sum runs as eight chains               */
/*  - F_j = F_{j-1} + (Sbar - F_{j-1}) * fl32(1/j) (no (j-1)*F product),     */
/*  - e_cur is folded into P: P = 2^(fl16(S' - c_j)) with c_j = fl16(m_j -   */
/*    dm_cur), so O <- fl16(e_p * O + T); V enters as V' = fl16(V 2^-c0) with */
/*    c0 >= 0 the per-head bound exponent (O < 2^14) and the epilogue scales  */
/*    by 2^c0,                                                               */
/*  - causal: the block mean uses all s2 columns, masked entries get P = 0,  */
/*    fully masked blocks are skipped and j counts consumed blocks.          */
/* tc_mode: 0 = GEMMs accumulate sequentially in FP32 then round once to    */
/* FP16; 1 = FP16 accumulation with one rounding per 16-long chunk (tensor-  */
/* core F16 accumulator model).                                              */
/* ------------------------------------------------------------------------ */

static inline double tc_dot(const double* a, size_t as, const double* b,
                            size_t bs, size_t n, int tc_mode) {
  if (tc_mode == 0) {
    double s = 0.0;
    for (size_t t = 0; t < n; ++t) s = fl32(s + a[t * as] * b[t * bs]);
    return fl16(s);
  }
  double s = 0.0;
  for (size_t t0 = 0; t0 < n; t0 += 16) {
    double chunk = 0.0;
    for (size_t t = t0; t < t0 + 16 && t < n; ++t) chunk += a[t * as] * b[t * bs];
    s = fl16(s + chunk);
  }
  return s;
}

typedef struct {
  double beta, diag, off, lscale;
  int tc_mode;
  double c0;     /* inflation in L units; < 0 selects the kernel's automatic rule */
  double xscale; /* exact power of two applied after the store: the exp argument is
                    xscale*fl16(S' - c_j) (the kernel: lscale = log2(e)/2,
                    xscale = 2, so the FP16 S' store holds 1/ln 2 / 2 = 0.72 x the
                    reference's scores and overflows later than the reference) */
  int rowsum;    /* the pseudo-average's row sum: 1 = tensor core, q . hi and q . lo (the
                    K' block sums split into FP16 hi + lo) in two FP32 accumulators, then
                    added (the kernel at d = 64, per block); 2 = one FP32 accumulator over
                    [q | q] . [hi | lo] (d = 128, the prologue GEMM); 0 = the CUDA-core
                    FP32 chains over the stored FP16 scores (PASA_PRO_SUM=0 builds) */
} orc_model_params;

/* The kernel's O-bounding exponent (pasa_kernels.cuh: pasa_inflation): the
 * smallest integer c0 >= 0 with S2 * vmax <= 2^14 * 2^c0, in FP32 exactly as
 * the device computes it.  V is scaled by 2^-c0 before PV; the epilogue
 * multiplies by 2^c0.  (lscale is accepted for API compatibility.) */
ORC_API double orc_model_inflation(double vmax, size_t S2, double lscale) {
  (void)lscale;
  const float need = (float)S2 * (float)vmax * (1.0f / 16384.0f);
  if (!(need > 1.0f) || !(need < 3.0e38f)) return 0.0; /* non-finite V: c0 = 0 */
  int e = ilogbf(need); /* floor(log2 need), exact */
  return (double)(ldexpf(1.0f, e) == need ? e : e + 1);
}

ORC_API int orc_model_pasa(const orc_shape* sh, const double* q,
                           const double* k, const double* v, double* o,
                           const orc_model_params* mp, int threads) {
  if (sh->Hq % sh->Hkv) return -1;
  if (sh->S1 % sh->s1 || sh->S2 % sh->s2) return -2;
  if (sh->causal && sh->S1 + sh->q_offset > sh->S2) return -4;
  const size_t s1 = sh->s1, s2 = sh->s2, d = sh->d;
  const size_t nq = sh->S1 / s1, nkv = sh->S2 / s2, grp = sh->Hq / sh->Hkv;
  const float inva = (float)(mp->beta / (1.0 - mp->beta));
  const double L = mp->lscale;
  const int log2dom = (L != 1.0);
  const double xs = mp->xscale > 0.0 ? mp->xscale : 1.0;
  const int nt = resolve_threads(threads);
  double* kp = malloc(sizeof(double) * sh->B * sh->Hkv * sh->S2 * d);
  /* the kernel's pre-pass: the rank-1 form (any block size) */
  orc_preprocess_keys(k, sh->B, sh->Hkv, sh->S2, d, s2, mp->diag, mp->off,
                      L != 1.0 ? PR1 : P32, P16, L, kp, nt);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long x = 0; x < (long long)(sh->B * sh->Hq * nq); ++x) {
    const size_t i = (size_t)x % nq;
    const size_t h = ((size_t)x / nq) % sh->Hq;
    const size_t b = (size_t)x / (nq * sh->Hq);
    const size_t hk = h / grp;
    /* O-bound exponent for this kv head and the scaled V' = fl16(V 2^-c0) */
    const double* vh = row_ptr(v, sh->Hkv, sh->S2, d, b, hk, 0);
    double c0 = mp->c0;
    if (c0 < 0.0) {
      double vmax = 0.0;
      for (size_t e = 0; e < sh->S2 * d; ++e) vmax = fmax(vmax, fabs(vh[e]));
      c0 = orc_model_inflation(vmax, sh->S2, L);
    }
    double* vsc = malloc(sizeof(double) * sh->S2 * d);
    for (size_t e = 0; e < sh->S2 * d; ++e) vsc[e] = fl16(vh[e] * ldexp(1.0, -(int)c0));
    float* m = calloc(s1, sizeof(float));
    float* l = calloc(2 * s1, sizeof(float)); /* per half-row partial l */
    float* fbar = calloc(s1, sizeof(float));
    double* oacc = calloc(s1 * d, sizeof(double));
    double* S = malloc(sizeof(double) * s2);
    const int tcsum = mp->rowsum != 0;
    double* ksh = malloc(sizeof(double) * d); /* K' block sums, hi / lo parts */
    double* ksl = malloc(sizeof(double) * d);
    size_t jc = 0; /* consumed blocks */
    for (size_t j = 0; j < nkv; ++j) {
      const size_t row0 = sh->q_offset + i * s1;
      if (sh->causal && j * s2 > row0 + s1 - 1) break; /* fully masked */
      ++jc;
      const double* kpj = kp + ((b * sh->Hkv + hk) * sh->S2 + j * s2) * d;
      const double* vj = vsc + j * s2 * d;
      /* the K'-sum kernel: per head-dim index t, four FP32 chains over the keys
       * (c % 4), ((a0 + a1) + (a2 + a3)), split hi = fl16(sum), lo = fl16(sum - hi) */
      for (size_t t = 0; tcsum && t < d; ++t) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        size_t c = 0;
        for (; c + 4 <= s2; c += 4)
          for (int u = 0; u < 4; ++u) acc[u] += (float)kpj[(c + u) * d + t];
        for (; c < s2; ++c) acc[0] += (float)kpj[c * d + t];
        const float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        ksh[t] = fl16((double)sum);
        ksl[t] = fl16((double)(sum - (float)ksh[t]));
      }
      for (size_t r = 0; r < s1; ++r) {
        const double* qr = row_ptr(q, sh->Hq, sh->S1, d, b, h, i * s1 + r);
        const size_t pos = row0 + r;
        for (size_t c = 0; c < s2; ++c) S[c] = tc_dot(qr, 1, kpj + c * d, 1, d, mp->tc_mode);
        /* Pseudo-average.  From the tensor core (rowsum = 1; per block at d = 64, from
         * the prologue GEMM at d = 128): sum_c S'_c = q . ksum_j with the
         * block's K' column sums split as (hi, lo) FP16 (the K'-sum kernel), each
         * product exact, accumulated to FP32 (modelled as FP64 then one rounding),
         * columns hi and lo added in FP32. */
        float ssum;
        if (tcsum) {
          double ghi = 0.0, glo = 0.0;
          for (size_t t = 0; t < d; ++t) {
            ghi += qr[t] * ksh[t];
            glo += qr[t] * ksl[t];
          }
          ssum = mp->rowsum == 2 ? (float)(ghi + glo) /* one FP32 accumulator over K = 2 d */
                                 : (float)ghi + (float)glo;
        } else {
          /* rowsum = 0 (CUDA cores): two threads per row (tile columns [0, 64)
           * and [64, 128)); in each half eight FP32 chains: column c -> chain
           * 2*((c/2)%4) + c%2 (the kernel's pair-register order), combined
           * ((t0+t1)+(t2+t3)), t_r = a_2r + a_2r+1; the row total is half0 + half1. */
          float sacc[2][8] = {{0.f}};
          for (size_t c = 0; c < s2; ++c) {
            const int ch = 2 * (int)((c / 2) % 4) + (int)(c % 2);
            sacc[c >= 64][ch] = sacc[c >= 64][ch] + (float)S[c];
          }
          float shalf[2];
          for (int hh = 0; hh < 2; ++hh)
            shalf[hh] = ((sacc[hh][0] + sacc[hh][1]) + (sacc[hh][2] + sacc[hh][3])) +
                        ((sacc[hh][4] + sacc[hh][5]) + (sacc[hh][6] + sacc[hh][7]));
          ssum = shalf[0] + shalf[1];
        }
        double mloc = -INFINITY;
        for (size_t c = 0; c < s2; ++c) {
          const int masked = sh->causal && (j * s2 + c > pos);
          if (!masked && S[c] > mloc) mloc = S[c];
        }
        const float sbar = ssum * (float)(1.0 / (double)s2);
        const float rcp = 1.0f / (float)jc; /* the kernel multiplies by 1/j */
        float fnew = (jc == 1) ? sbar : fbar[r] + (sbar - fbar[r]) * rcp;
        const float dmc = inva * (sbar - fnew);
        const float dmp = (jc == 1) ? 0.f : inva * (fbar[r] - fnew);
        const float cand = (float)mloc + dmc;
        float mnew = (jc == 1) ? cand : fmaxf(m[r] + dmp, cand);
        const float cjf = mnew - dmc;
        const double cj = fl16((double)cjf);
        double ep = 0.0;
        if (jc > 1) {
          const float earg = ((m[r] + dmp) - mnew) * (float)xs;
          ep = fl16(log2dom ? exp2((double)earg) : exp((double)earg));
        }
        float lacc[2][8] = {{0.f}}; /* same chains, per half row */
        for (size_t c = 0; c < s2; ++c) {
          const int masked = sh->causal && (j * s2 + c > pos);
          /* the kernel's one-HFMA2 form fl16(xs S' - xs c_j) while xs c_j fits FP16,
           * else xs fl16(S' - c_j) (both exact scalings of the same rounding
           * except in the subnormal range) */
          const double a = (fabs(xs * cj) <= 65504.0) ? fl16(xs * S[c] - xs * cj)
                                                      : xs * fl16(S[c] - cj);
          S[c] = masked ? 0.0 : fl16(log2dom ? exp2(a) : exp(a));
          const int ch = 2 * (int)((c / 2) % 4) + (int)(c % 2);
          lacc[c >= 64][ch] = lacc[c >= 64][ch] + (float)S[c];
        }
        for (int hh = 0; hh < 2; ++hh) { /* each half keeps its own partial l */
          const float lloc = ((lacc[hh][0] + lacc[hh][1]) + (lacc[hh][2] + lacc[hh][3])) +
                             ((lacc[hh][4] + lacc[hh][5]) + (lacc[hh][6] + lacc[hh][7]));
          l[2 * r + hh] = (jc == 1) ? lloc : (float)ep * l[2 * r + hh] + lloc;
        }
        double* orow = oacc + r * d;
        for (size_t n = 0; n < d; ++n) {
          const double tn = tc_dot(S, 1, vj + n, d, s2, mp->tc_mode);
          orow[n] = (jc == 1) ? tn : fl16(ep * orow[n] + tn);
        }
        m[r] = mnew;
        fbar[r] = fnew;
      }
    }
    for (size_t r = 0; r < s1; ++r) {
      double* dst = o + ((b * sh->Hq + h) * sh->S1 + i * s1 + r) * d;
      const float invl = (1.0f / (l[2 * r] + l[2 * r + 1])) * ldexpf(1.0f, (int)c0);
      for (size_t n = 0; n < d; ++n) dst[n] = fl16((float)oacc[r * d + n] * invl);
    }
    free(m); free(l); free(fbar); free(oacc); free(S); free(vsc); free(ksh); free(ksl);
  }
  free(kp);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Model of the kernel's FA16 mode (the naive FP16 FlashAttention, beta = 0, */
/* attention.cpp:92-180 with FA_PARTIAL_FP16): raw K, FP16 score store (F16  */
/* accumulator), scale applied after the store by one HFMA2                  */
/* x = fl16(S * fl16(s) - fl16(m * s)) with s = fl32(log2 e / alpha), FP32   */
/* running max of the stored scores, P = fl16(2^x), FP32 half-row l, FP16 O  */
/* via fl16(e_p * O + T).  Overflow of the store propagates to NaN exactly   */
/* like the reference.                                                       */
/* ------------------------------------------------------------------------ */
ORC_API int orc_model_fa16(const orc_shape* sh, const double* q, const double* k,
                           const double* v, double* o, int tc_mode, int threads) {
  if (sh->Hq % sh->Hkv) return -1;
  if (sh->S1 % sh->s1 || sh->S2 % sh->s2) return -2;
  if (sh->causal && sh->S1 + sh->q_offset > sh->S2) return -4;
  const size_t s1 = sh->s1, s2 = sh->s2, d = sh->d;
  const size_t nq = sh->S1 / s1, nkv = sh->S2 / s2, grp = sh->Hq / sh->Hkv;
  const float scale_f = (float)(1.4426950408889634 / sqrt((double)d));
  const double scale_h = fl16((double)scale_f);
  const int nt = resolve_threads(threads);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long x = 0; x < (long long)(sh->B * sh->Hq * nq); ++x) {
    const size_t i = (size_t)x % nq;
    const size_t h = ((size_t)x / nq) % sh->Hq;
    const size_t b = (size_t)x / (nq * sh->Hq);
    const size_t hk = h / grp;
    float* m = calloc(s1, sizeof(float));
    float* l = calloc(2 * s1, sizeof(float));
    double* oacc = calloc(s1 * d, sizeof(double));
    double* S = malloc(sizeof(double) * s2);
    size_t jc = 0;
    for (size_t j = 0; j < nkv; ++j) {
      const size_t row0 = sh->q_offset + i * s1;
      if (sh->causal && j * s2 > row0 + s1 - 1) break;
      ++jc;
      const double* kj = row_ptr(k, sh->Hkv, sh->S2, d, b, hk, j * s2);
      const double* vj = row_ptr(v, sh->Hkv, sh->S2, d, b, hk, j * s2);
      for (size_t r = 0; r < s1; ++r) {
        const double* qr = row_ptr(q, sh->Hq, sh->S1, d, b, h, i * s1 + r);
        const size_t pos = row0 + r;
        double mloc = -INFINITY;
        for (size_t c = 0; c < s2; ++c) {
          S[c] = tc_dot(qr, 1, kj + c * d, 1, d, tc_mode);
          const int masked = sh->causal && (j * s2 + c > pos);
          if (!masked && S[c] > mloc) mloc = S[c];
        }
        const float mnew = (jc == 1) ? (float)mloc : fmaxf(m[r], (float)mloc);
        double ep = 0.0;
        if (jc > 1) ep = fl16(exp2((double)((m[r] - mnew) * scale_f)));
        const double ms = fl16((double)(mnew * scale_f));
        float lacc[2][8] = {{0.f}};
        for (size_t c = 0; c < s2; ++c) {
          const int masked = sh->causal && (j * s2 + c > pos);
          const double a = fl16(S[c] * scale_h - ms);
          S[c] = masked ? 0.0 : fl16(exp2(a));
          const int ch = 2 * (int)((c / 2) % 4) + (int)(c % 2);
          lacc[c >= 64][ch] = lacc[c >= 64][ch] + (float)S[c];
        }
        for (int hh = 0; hh < 2; ++hh) {
          const float lloc = ((lacc[hh][0] + lacc[hh][1]) + (lacc[hh][2] + lacc[hh][3])) +
                             ((lacc[hh][4] + lacc[hh][5]) + (lacc[hh][6] + lacc[hh][7]));
          l[2 * r + hh] = (jc == 1) ? lloc : (float)ep * l[2 * r + hh] + lloc;
        }
        double* orow = oacc + r * d;
        for (size_t n = 0; n < d; ++n) {
          const double tn = tc_dot(S, 1, vj + n, d, s2, tc_mode);
          orow[n] = (jc == 1) ? tn : fl16(ep * orow[n] + tn);
        }
        m[r] = mnew;
      }
    }
    for (size_t r = 0; r < s1; ++r) {
      double* dst = o + ((b * sh->Hq + h) * sh->S1 + i * s1 + r) * d;
      const float invl = 1.0f / (l[2 * r] + l[2 * r + 1]);
      for (size_t n = 0; n < d; ++n) dst[n] = fl16((float)oacc[r * d + n] * invl);
    }
    free(m); free(l); free(oacc); free(S);
  }
  return 0;
}
