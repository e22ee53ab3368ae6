// Adapter check — TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/).
//
// Compiles the reference GOFMM headers (unmodified, against oracle/eigen_shim) together with the
// header-only C++ adapter include/gofmm_b200_gfmm.hpp and the product library, then runs the
// reference's own compress() and evaluate() next to the adapter's GPU evaluate on the same
// HMatrix: the drop-in a maintainer would add, exercised for real.
// Exit code 0 iff: stored-block and matrix-free GPU results match evaluate() to 1e-12 (relative
// 2-norm), the flop counters are equal, and a wrong-sized W throws std::invalid_argument.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gfmm/gfmm.hpp"
#include "gofmm_b200_gfmm.hpp"

using namespace gfmm;

static double rel2(const Matrix& a, const Matrix& b) {
  double num = 0.0, den = 0.0;
  for (long j = 0; j < long(a.cols()); ++j)
    for (long i = 0; i < long(a.rows()); ++i) {
      const double d = a(i, j) - b(i, j);
      num += d * d;
      den += b(i, j) * b(i, j);
    }
  return std::sqrt(num / den);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 2048;
  const int r = argc > 2 ? std::atoi(argv[2]) : 16;
  PointCloud pc = PointCloud::random_gaussian(n, 3, 11);
  GaussianKernelOracle K(pc, 1.0);
  RunConfig cfg;
  cfg.m = 128;
  cfg.s = 64;
  cfg.tau = 1e-7;
  cfg.kappa = 16;
  cfg.budget = 0.05;
  cfg.seed = 3;
  HMatrix h = compress(K, &pc, cfg);
  Rng rng(7, 0x1);
  Matrix w(n, r);
  for (int c = 0; c < r; ++c)
    for (int i = 0; i < n; ++i) w(i, c) = rng.gauss();
  const Potentials ref = evaluate(h, w);

  B200Evaluator stored(h);
  const Potentials g1 = evaluate_b200(stored, w);
  B200Evaluator mfree(h, &pc, 1.0);
  const Potentials g2 = mfree.evaluate(w);
  const double e1 = rel2(g1.u, ref.u), e2 = rel2(g2.u, ref.u);
  bool threw = false;
  try {
    stored.evaluate(Matrix(n + 1, 2));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  const bool ok = e1 <= 1e-12 && e2 <= 1e-12 && g1.flops == ref.flops && g2.flops == ref.flops && threw;
  std::printf("adapter n=%d r=%d stored_rel=%.3e matrixfree_rel=%.3e flops_ref=%lld flops_gpu=%lld invalid_arg=%d ok=%d\n",
              n, r, e1, e2, static_cast<long long>(ref.flops), static_cast<long long>(g1.flops), threw ? 1 : 0,
              ok ? 1 : 0);
  return ok ? 0 : 1;
}
