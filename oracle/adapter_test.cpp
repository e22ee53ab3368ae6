// Adapter check — TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/).
//
// Compiles the reference GOFMM headers (unmodified, against oracle/eigen_shim) together with the
// header-only C++ adapter include/gofmm_b200_gfmm.hpp and the product library, then runs the
// reference's own compress(), evaluate() and error_eps2() next to the adapter on the same HMatrix:
// the drop-in a maintainer would add, exercised for real.
// Exit code 0 iff:
//   * evaluate_b200(h, w, opts) (cached per-HMatrix evaluator, stored blocks), the explicit
//     stored evaluator and the matrix-free evaluators (Gaussian, Laplace, Exponential) match
//     evaluate() to 1e-12 (relative 2-norm) with equal flop counters;
//   * error_eps2_b200 reproduces error_eps2 (same sampled rows, eps2 to 1e-10 relative);
//   * 4 host threads calling evaluate_b200 on ONE HMatrix concurrently get results
//     bitwise equal to the same calls made serially;
//   * a wrong-sized W throws std::invalid_argument.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

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

static bool bitwise_equal(const Matrix& a, const Matrix& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() &&
         std::memcmp(a.data(), b.data(), sizeof(double) * size_t(a.rows()) * size_t(a.cols())) == 0;
}

static Matrix rhs(int n, int r, std::uint64_t seed) {
  Rng rng(seed, 0x1);
  Matrix w(n, r);
  for (int c = 0; c < r; ++c)
    for (int i = 0; i < n; ++i) w(i, c) = rng.gauss();
  return w;
}

// Matérn-1/2 through the reference plugin point (EntryOracle, oracle.hpp:34-66), as in
// oracle/ref_harness.cpp: BASELINE config 4's kernel, absent from the reference.
class ExpOracle final : public EntryOracle {
 public:
  ExpOracle(PointCloud p, double h) : p_(std::move(p)), h_(h) {}
  int size() const override { return p_.size(); }
  void eval_block(std::span<const int> I, std::span<const int> J, Matrix& out) const override {
    out.resize(I.size(), J.size());
    const double inv = 1.0 / h_;
    for (size_t c = 0; c < J.size(); ++c) {
      auto xj = p_.coords.col(J[c]);
      for (size_t r = 0; r < I.size(); ++r) out(r, c) = std::exp(-(p_.coords.col(I[r]) - xj).norm() * inv);
    }
  }
  Vector eval_diag(std::span<const int> I) const override { return Vector::Ones(I.size()); }

 private:
  PointCloud p_;
  double h_;
};

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 2048;
  const int r = argc > 2 ? std::atoi(argv[2]) : 16;
  PointCloud pc = PointCloud::random_gaussian(n, 3, 11);
  RunConfig cfg;
  cfg.m = 128;
  cfg.s = 64;
  cfg.tau = 1e-7;
  cfg.kappa = 16;
  cfg.budget = 0.05;
  cfg.seed = 3;
  bool ok = true;
  auto check = [&](const char* what, bool cond) {
    std::printf("  %-44s %s\n", what, cond ? "ok" : "FAIL");
    ok = ok && cond;
  };

  // --- Gaussian: cached evaluate_b200(h, ...), explicit stored and matrix-free evaluators
  GaussianKernelOracle K(pc, 1.0);
  HMatrix h = compress(K, &pc, cfg);
  const Matrix w = rhs(n, r, 7);
  const Potentials ref = evaluate(h, w);
  const Potentials c1 = evaluate_b200(h, w);  // builds the cached evaluator
  const Potentials c2 = evaluate_b200(h, w, EvalOptions{});  // reuses it
  B200Evaluator stored(h);
  const Potentials g1 = evaluate_b200(stored, w);
  B200Evaluator mfree(h, &pc, 1.0);
  const Potentials g2 = mfree.evaluate(w);
  std::printf("gaussian n=%d r=%d cached=%.3e stored=%.3e matrixfree=%.3e flops_ref=%lld flops_gpu=%lld\n", n, r,
              rel2(c1.u, ref.u), rel2(g1.u, ref.u), rel2(g2.u, ref.u), (long long)ref.flops, (long long)c1.flops);
  check("evaluate_b200(h, w) == evaluate(h, w)", rel2(c1.u, ref.u) <= 1e-12 && c1.flops == ref.flops);
  check("cached evaluator reused bitwise", bitwise_equal(c1.u, c2.u));
  check("stored evaluator", rel2(g1.u, ref.u) <= 1e-12 && g1.flops == ref.flops);
  check("matrix-free gaussian", rel2(g2.u, ref.u) <= 1e-12 && g2.flops == ref.flops);

  // --- the distributed evaluator's data plane on a single rank (no communicator needed): the
  // subtree-split stages + the in-library exchange path, every row owned
  {
    auto d1 = B200Evaluator::distributed(h, &pc, GOFMM_KERNEL_GAUSSIAN, 1.0, 0.0, 0, 1);
    const auto rows = d1->own_rows();
    const Potentials pd = d1->evaluate_dist(w);
    std::printf("distributed(1 rank) rows=[%lld,%lld) rel=%.3e flops=%lld\n", (long long)rows.first,
                (long long)rows.second, rel2(pd.u, ref.u), (long long)pd.flops);
    check("distributed evaluator, 1 rank", rows.first == 0 && rows.second == n && rel2(pd.u, ref.u) <= 1e-12 &&
                                               pd.flops == ref.flops);
  }

  // --- error_eps2 routed to the GPU
  const ErrorReport e_ref = error_eps2(h, K, 2, 100, 42);
  const ErrorReport e_gpu = error_eps2_b200(h, K, 2, 100, 42);
  std::printf("eps2 ref=%.9g gpu=%.9g\n", e_ref.eps2, e_gpu.eps2);
  check("error_eps2_b200 sampled rows", e_ref.sample_rows == e_gpu.sample_rows);
  check("error_eps2_b200 eps2", std::abs(e_gpu.eps2 - e_ref.eps2) <= 1e-10 * e_ref.eps2 &&
                                     e_gpu.eval_flops == e_ref.eval_flops);

  // --- concurrent evaluate on one HMatrix with different w, bitwise == serial
  {
    const int T = 4;
    std::vector<Matrix> ws, serial(T), conc(T);
    for (int t = 0; t < T; ++t) ws.push_back(rhs(n, 3 + t, 100 + t));
    for (int t = 0; t < T; ++t) serial[t] = evaluate_b200(h, ws[t]).u;
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (int rep = 0; rep < 3; ++rep) conc[t] = evaluate_b200(h, ws[t]).u;
      });
    for (auto& x : th) x.join();
    bool same = true;
    for (int t = 0; t < T; ++t) same = same && bitwise_equal(serial[t], conc[t]);
    check("4 threads concurrently, bitwise == serial", same);
  }
  b200_release(h);

  // --- Laplace (from the oracle object) and Exponential matrix-free
  {
    LaplaceKernelOracle L(pc, 0.05);
    HMatrix hl = compress(L, &pc, cfg);
    const Potentials rl = evaluate(hl, w);
    auto gl = B200Evaluator::matrix_free(hl, L);
    const Potentials pl = gl->evaluate(w);
    std::printf("laplace rel=%.3e\n", rel2(pl.u, rl.u));
    check("matrix-free laplace", rel2(pl.u, rl.u) <= 1e-12 && pl.flops == rl.flops);
  }
  {
    ExpOracle E(pc, 1.0);
    HMatrix he = compress(E, &pc, cfg);
    const Potentials re = evaluate(he, w);
    B200Evaluator ge(he, &pc, GOFMM_KERNEL_EXPONENTIAL, 1.0);
    const Potentials pe = ge.evaluate(w);
    std::printf("exponential rel=%.3e\n", rel2(pe.u, re.u));
    check("matrix-free exponential", rel2(pe.u, re.u) <= 1e-12 && pe.flops == re.flops);
  }

  bool threw = false;
  try {
    evaluate_b200(h, Matrix(n + 1, 2));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  check("wrong-sized W -> std::invalid_argument", threw);
  std::printf("adapter ok=%d\n", ok ? 1 : 0);
  return ok ? 0 : 1;
}
