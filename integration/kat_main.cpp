// integration/kat_main.cpp -- host known-answer checks of the drop-in's closed-form pieces,
// linked like ref_sweep_b200 (pasa_shim.o in place of the reference's pasa.o); no GPU needed.
//   * Theorem 2.1 (SPEC KAT): shifting_matrix_inverse(s, lambda) inverts I - lambda J, and
//     throws SingularMatrixError exactly at lambda s == 1 (pasa.cpp:37-51);
//   * build_shifting_matrix at FP16: the two distinct entries of pasa.cpp:26-27 at d = 128
//     (diag 0.0877075195, off -6.79969788e-4).
#include <cmath>
#include <cstdio>

#include "pasa/pasa.hpp"

int main() {
  using namespace pasa;
  int bad = 0;
  for (double beta : {0.5, 0.9375, 0.984497}) {
    const size_t s = 128;
    const double lam = beta / static_cast<double>(s);
    const Matrix2D inv = shifting_matrix_inverse(s, lam);
    double worst = 0.0;  // (I - lam J) inv - I
    for (size_t r = 0; r < s; ++r)
      for (size_t c = 0; c < s; ++c) {
        double col_sum = 0.0;
        for (size_t k = 0; k < s; ++k) col_sum += inv.row(k)[c];
        const double v = inv.row(r)[c] - lam * col_sum - (r == c ? 1.0 : 0.0);
        worst = std::fmax(worst, std::fabs(v));
      }
    std::printf("inverse beta=%g: max |(I - lambda J) M^-1 - I| = %.3g\n", beta, worst);
    bad += !(worst < 1e-12);
  }
  try {
    shifting_matrix_inverse(128, 1.0 / 128.0);
    std::printf("singular: no exception\n");
    ++bad;
  } catch (const SingularMatrixError&) {
    std::printf("singular: SingularMatrixError\n");
  }
  const Matrix2D m = build_shifting_matrix(128, 0.984497, std::sqrt(128.0), Prec::FP16);
  std::printf("M(FP16) d=128: diag %.10g off %.9g\n", m.row(0)[0], m.row(0)[1]);
  bad += !(std::fabs(m.row(0)[0] - 0.0877075195) < 1e-10 && std::fabs(m.row(0)[1] + 6.79969788e-4) < 1e-12);
  std::printf(bad ? "KAT FAIL\n" : "KAT OK\n");
  return bad ? 1 : 0;
}
