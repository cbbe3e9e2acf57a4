// integration/sweep_main.cpp -- drives the REFERENCE's own harness
// (pasa::sweep, bench.cpp:170-247) with pasa.o replaced by pasa_shim.o, so
// every PASA_FP16 cell runs on the B200 while FA_PARTIAL_FP16 stays on the
// reference CPU path.  Prints the reference's CSV report (bench.hpp:105-107).
// Usage: ref_sweep_b200 [heads] [seq] [diagnose 0|1]  (diagnose: the reference's FP64 range
// report, whose K' pre-pass under GoldenFp64 stays on the reference's gemm)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pasa/bench.hpp"

int main(int argc, char** argv) {
  const size_t heads = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 4;
  const size_t seq = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 1280;
  std::vector<pasa::DistributionSpec> specs;
  // Appendix E cells at (1, heads, seq, 128).
  const struct { pasa::DistKind k; double x0, am; } cells[] = {
      {pasa::DistKind::Uniform, 30, 0.5}, {pasa::DistKind::Uniform, 20, 15},
      {pasa::DistKind::Uniform, 20, 20},  {pasa::DistKind::Hybrid, 30, 10},
      {pasa::DistKind::Hybrid, 20, 50},   {pasa::DistKind::Hybrid, 20, 100}};
  for (const auto& c : cells) {
    pasa::DistributionSpec s;
    s.kind = c.k;
    s.x0 = c.x0;
    s.am = c.am;
    s.seed = 0;
    s.batch = 1;
    s.heads = heads;
    s.seq = seq;
    s.dim = 128;
    specs.push_back(s);
  }
  pasa::SweepOptions opts;
  opts.diagnose = argc > 3 && std::strtoul(argv[3], nullptr, 10) != 0;
  opts.policies = {pasa::PolicyId::PasaFp16, pasa::PolicyId::FaPartialFp16};
  const auto rows = pasa::sweep(specs, opts);
  std::fputs(pasa::report_csv(rows).c_str(), stdout);
  for (const auto& r : rows)
    if (!r.error.empty()) {
      std::fprintf(stderr, "cell error: %s\n", r.error.c_str());
      return 1;
    }
  return 0;
}
