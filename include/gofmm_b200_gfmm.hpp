// gofmm_b200_gfmm.hpp — header-only C++ adapter for the reference GOFMM API.
//
// Include AFTER the reference headers ("gfmm/gfmm.hpp"). It flattens a gfmm::HMatrix
// (compress.hpp:65-79) into gofmm_tree_desc once, and offers gfmm::evaluate()'s exact contract
// (evaluate.hpp:287-317: W in original order, Potentials.u in permuted order, the reference flop
// counter, std::invalid_argument on bad W) on the B200 through the C-ABI of gofmm_b200.h:
//
//   gfmm::Potentials p = gfmm::evaluate_b200(h, w, opts);   // evaluate(h, w, opts)'s exact signature
//   gfmm::ErrorReport e = gfmm::error_eps2_b200(h, oracle, r, rows, seed, opts);  // error_eps2's
//
// evaluate_b200(h, ...) keeps one device-resident evaluator per HMatrix (stored blocks, any
// EntryOracle), created on first use and reused by every later call on the same HMatrix — from
// any thread: SPEC.md:429 concurrent calls are serialised on the device handle (gofmm_b200.h).
// error_eps2's body (evaluate.hpp:348) is the one place the reference calls evaluate(); routing
// it to the GPU means calling error_eps2_b200 instead, which draws the same rows and W from the
// same Rng stream (incl. the up-to-3 redraws) and evaluates them with evaluate_b200.
//
// Explicit evaluators: B200Evaluator gpu(h) (stored blocks), or matrix-free — near / far blocks
// regenerated from the coordinates on the device — for the reference kernel oracles:
//   B200Evaluator(h, &points, bandwidth)                           Gaussian   oracle.hpp:141-163
//   B200Evaluator(h, &points, GOFMM_KERNEL_LAPLACE, delta)          Laplace    oracle.hpp:165-195
//   B200Evaluator(h, &points, GOFMM_KERNEL_POLYNOMIAL, c, degree)   Polynomial oracle.hpp:197-219
//   B200Evaluator(h, &points, GOFMM_KERNEL_EXPONENTIAL, h)          Matern-1/2 (BASELINE config 4)
//   B200Evaluator::matrix_free(h, laplace_oracle)                   from the oracle object itself
// Multi-GPU (one process per GPU): B200Evaluator::distributed(h, &points, kernel, p0, p1, rank,
// nranks) + init_comm(id) + evaluate_dist(w) — this rank's rows of u (gofmm_dist_evaluate_host).
#ifndef GOFMM_B200_GFMM_HPP
#define GOFMM_B200_GFMM_HPP

#include <chrono>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "gofmm_b200.h"

namespace gfmm {

class B200Evaluator {
 public:
  /// Stored blocks exactly as HMatrix holds them (leaf_diag, near_field[t].k, far_field[t].k).
  explicit B200Evaluator(const HMatrix& h, int device = 0) { build(h, nullptr, -1, 0.0, 0.0, device); }
  /// Gaussian kernel tree evaluated matrix-free from the point coordinates (oracle.hpp:148-159).
  B200Evaluator(const HMatrix& h, const PointCloud* points, double bandwidth, int device = 0) {
    build(h, points, GOFMM_KERNEL_GAUSSIAN, bandwidth, 0.0, device);
  }
  /// Any GOFMM_KERNEL_* evaluated matrix-free (kparam p0, p1 as in gofmm_tree_desc::kparam).
  B200Evaluator(const HMatrix& h, const PointCloud* points, int kernel, double p0, double p1 = 0.0,
                int device = 0) {
    if (!points) throw std::invalid_argument("matrix-free evaluation needs the point cloud");
    build(h, points, kernel, p0, p1, device);
  }
  /// One rank of the subtree-split evaluation over nranks GPUs (north_star (4)),
  /// matrix-free from the point coordinates. Every rank builds it from the same HMatrix; rank 0 gets
  /// a unique id from nccl_unique_id(), the caller broadcasts it (e.g. MPI_Bcast) and every rank
  /// calls init_comm(id) — then evaluate_dist(w) on every rank, once per evaluation.
  static std::unique_ptr<B200Evaluator> distributed(const HMatrix& h, const PointCloud* points, int kernel, double p0,
                                                    double p1, int rank, int nranks, int device = 0) {
    if (!points) throw std::invalid_argument("distributed evaluation needs the point cloud");
    std::unique_ptr<B200Evaluator> ev(new B200Evaluator());
    ev->build(h, points, kernel, p0, p1, device, rank, nranks);
    return ev;
  }
  static std::vector<unsigned char> nccl_unique_id() {
    std::vector<unsigned char> id(GOFMM_NCCL_UNIQUE_ID_BYTES);
    if (gofmm_nccl_unique_id(id.data()) != GOFMM_OK)
      throw std::runtime_error(std::string("gofmm_nccl_unique_id: ") + gofmm_last_error());
    return id;
  }
  /// Collective over the nranks processes (ncclCommInitRank); not needed for a single rank.
  void init_comm(const void* unique_id) {
    if (gofmm_dist_init_comm(h_, unique_id) != GOFMM_OK)
      throw std::runtime_error(std::string("gofmm_dist_init_comm: ") + gofmm_last_error());
  }
  /// This rank's permuted rows [first, second) of u.
  std::pair<int64_t, int64_t> own_rows() const {
    gofmm_dist_info info{};
    if (gofmm_dist_get_info(h_, &info) != GOFMM_OK) throw std::runtime_error(gofmm_last_error());
    return {info.own_row_begin, info.own_row_end};
  }
  /// evaluate() of this rank's share: W (full, original order) in, u_perm with this rank's rows
  /// [own_rows()) filled (zeros elsewhere); flops = this rank's reference-counted share.
  Potentials evaluate_dist(const Matrix& w) const {
    if (w.rows() != n_) throw std::invalid_argument("evaluate: w has wrong row count");
    if (w.cols() < 1) throw std::invalid_argument("evaluate: w needs at least one column");
    Potentials p;
    p.u = Matrix::Zero(w.rows(), w.cols());
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = gofmm_dist_evaluate_host(h_, w.data(), w.rows(), static_cast<int32_t>(w.cols()), p.u.data(),
                                            p.u.rows(), nullptr);
    if (rc == GOFMM_ERR_INVALID) throw std::invalid_argument(gofmm_last_error());
    if (rc != GOFMM_OK) throw std::runtime_error(std::string("gofmm_dist_evaluate_host: ") + gofmm_last_error());
    gofmm_dist_info info{};
    gofmm_dist_get_info(h_, &info);
    p.flops = info.flops_per_rhs * w.cols();
    p.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return p;
  }
  /// Matrix-free from the reference oracle object (its points and parameter).
  static std::unique_ptr<B200Evaluator> matrix_free(const HMatrix& h, const LaplaceKernelOracle& k, int device = 0) {
    return std::make_unique<B200Evaluator>(h, &k.points(), GOFMM_KERNEL_LAPLACE, k.regularization(), 0.0, device);
  }
  B200Evaluator(const B200Evaluator&) = delete;
  B200Evaluator& operator=(const B200Evaluator&) = delete;
  ~B200Evaluator() {
    if (h_) gofmm_destroy(h_);
  }

  int size() const { return n_; }

  /// evaluate.hpp:287-317 on the GPU: u = K~ w, u in permuted order.
  Potentials evaluate(const Matrix& w) const {
    if (w.rows() != n_) throw std::invalid_argument("evaluate: w has wrong row count");
    if (w.cols() < 1) throw std::invalid_argument("evaluate: w needs at least one column");
    Potentials p;
    p.u = Matrix(w.rows(), w.cols());
    gofmm_eval_stats st{};
    const int rc = gofmm_evaluate(h_, w.data(), w.rows(), static_cast<int32_t>(w.cols()), p.u.data(), p.u.rows(),
                                  &st);
    if (rc == GOFMM_ERR_INVALID) throw std::invalid_argument(gofmm_last_error());
    if (rc != GOFMM_OK) throw std::runtime_error(std::string("gofmm_evaluate: ") + gofmm_last_error());
    p.flops = st.flops;
    p.seconds = st.seconds;
    return p;
  }

 private:
  B200Evaluator() = default;
  void build(const HMatrix& h, const PointCloud* pts, int kernel, double p0, double p1, int device, int rank = 0,
             int nranks = 0) {
    const MetricTree& t = h.tree;
    n_ = h.n;
    const int nn = static_cast<int>(t.nodes.size());
    for (const TreeNode& nd : t.nodes) {
      parent_.push_back(nd.parent);
      left_.push_back(nd.left);
      right_.push_back(nd.right);
      level_.push_back(nd.level);
      start_.push_back(nd.start);
      end_.push_back(nd.end);
    }
    iperm_.assign(t.iperm.begin(), t.iperm.end());
    skel_off_.push_back(0);
    proj_off_.push_back(0);
    for (int i = 0; i < nn; ++i) {
      const Skeleton& sk = h.skeletons[i];
      rank_.push_back(sk.valid() ? sk.rank() : -1);
      if (sk.valid()) {
        skel_.insert(skel_.end(), sk.skel.begin(), sk.skel.end());
        proj_.insert(proj_.end(), sk.proj.data(), sk.proj.data() + sk.proj.rows() * sk.proj.cols());
      }
      skel_off_.push_back(static_cast<int64_t>(skel_.size()));
      proj_off_.push_back(static_cast<int64_t>(proj_.size()));
    }
    diag_off_.push_back(0);
    for (int i = 0; i < nn; ++i) {
      const Matrix& d = h.leaf_diag[i];
      diag_.insert(diag_.end(), d.data(), d.data() + d.rows() * d.cols());
      diag_off_.push_back(static_cast<int64_t>(diag_.size()));
    }
    near_off_.push_back(0);
    for (const auto& b : h.near_field) {
      na_.push_back(b.a);
      nb_.push_back(b.b);
      near_.insert(near_.end(), b.k.data(), b.k.data() + b.k.rows() * b.k.cols());
      near_off_.push_back(static_cast<int64_t>(near_.size()));
    }
    far_off_.push_back(0);
    for (const auto& b : h.far_field) {
      fa_.push_back(b.a);
      fb_.push_back(b.b);
      far_.insert(far_.end(), b.k.data(), b.k.data() + b.k.rows() * b.k.cols());
      far_off_.push_back(static_cast<int64_t>(far_.size()));
    }
    gofmm_tree_desc d{};
    d.n = h.n;
    d.num_nodes = nn;
    d.parent = parent_.data();
    d.left = left_.data();
    d.right = right_.data();
    d.level = level_.data();
    d.start = start_.data();
    d.end = end_.data();
    d.iperm = iperm_.data();
    d.rank = rank_.data();
    d.skel_offset = skel_off_.data();
    d.skel_idx = skel_.empty() ? nullptr : skel_.data();
    d.proj_offset = proj_off_.data();
    d.proj = proj_.empty() ? nullptr : proj_.data();
    d.num_near = static_cast<int64_t>(na_.size());
    d.near_a = na_.data();
    d.near_b = nb_.data();
    d.num_far = static_cast<int64_t>(fa_.size());
    d.far_a = fa_.data();
    d.far_b = fb_.data();
    if (pts) {
      if (pts->size() != h.n) throw std::invalid_argument("point cloud size differs from the HMatrix");
      d.source = GOFMM_SOURCE_KERNEL;
      d.kernel = kernel;
      d.dim = pts->dim();
      d.coords = pts->coords.data();
      d.kparam[0] = p0;
      d.kparam[1] = p1;
    } else {
      d.source = GOFMM_SOURCE_STORED;
      d.diag_offset = diag_off_.data();
      d.diag_blocks = diag_.empty() ? nullptr : diag_.data();
      d.near_offset = near_off_.data();
      d.near_blocks = near_.empty() ? nullptr : near_.data();
      d.far_offset = far_off_.data();
      d.far_blocks = far_.empty() ? nullptr : far_.data();
    }
    gofmm_options o{};
    o.device = device;
    const int rc = nranks > 0 ? gofmm_create_dist(&d, &o, rank, nranks, &h_) : gofmm_create(&d, &o, &h_);
    if (rc == GOFMM_ERR_INVALID) throw std::invalid_argument(gofmm_last_error());
    if (rc != GOFMM_OK) throw std::runtime_error(std::string("gofmm_create: ") + gofmm_last_error());
  }

  gofmm_handle* h_ = nullptr;
  int n_ = 0;
  std::vector<int32_t> parent_, left_, right_, level_, start_, end_, iperm_, rank_, skel_, na_, nb_, fa_, fb_;
  std::vector<int64_t> skel_off_, proj_off_, diag_off_, near_off_, far_off_;
  std::vector<double> proj_, diag_, near_, far_;
};

/// evaluate()'s signature (evaluate.hpp:287) routed to the GPU; opts.mode / opts.threads do not
/// change results in the reference (evaluate.hpp:118) and are not needed here.
inline Potentials evaluate_b200(const B200Evaluator& gpu, const Matrix& w, const EvalOptions& = {}) {
  return gpu.evaluate(w);
}

namespace b200_detail {
// One device-resident evaluator per HMatrix. The key is the HMatrix's address plus a fingerprint
// of what it owns (sizes and the addresses of its block storage), so a different HMatrix that
// reuses a freed address is rebuilt rather than served a stale tree.
struct CacheKey {
  const HMatrix* h;
  int n;
  size_t nodes, near, far;
  const double* diag0;
  const double* proj0;
  bool operator<(const CacheKey& o) const {
    return std::tie(h, n, nodes, near, far, diag0, proj0) < std::tie(o.h, o.n, o.nodes, o.near, o.far, o.diag0, o.proj0);
  }
};
inline CacheKey key_of(const HMatrix& h) {
  const double* d0 = nullptr;
  for (const Matrix& m : h.leaf_diag)
    if (m.size()) {
      d0 = m.data();
      break;
    }
  const double* p0 = nullptr;
  for (const Skeleton& sk : h.skeletons)
    if (sk.valid() && sk.proj.size()) {
      p0 = sk.proj.data();
      break;
    }
  return {&h, h.n, h.tree.nodes.size(), h.near_field.size(), h.far_field.size(), d0, p0};
}
inline std::mutex& cache_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<CacheKey, std::shared_ptr<B200Evaluator>>& cache() {
  static std::map<CacheKey, std::shared_ptr<B200Evaluator>> c;
  return c;
}
inline std::shared_ptr<B200Evaluator> evaluator_for(const HMatrix& h) {
  const CacheKey k = key_of(h);
  std::lock_guard<std::mutex> g(cache_mutex());
  auto& c = cache();
  auto it = c.find(k);
  if (it != c.end()) return it->second;
  for (auto i = c.begin(); i != c.end();)  // same address, different contents: stale
    i = (i->first.h == &h) ? c.erase(i) : std::next(i);
  auto ev = std::make_shared<B200Evaluator>(h);
  c.emplace(k, ev);
  return ev;
}
}  // namespace b200_detail

/// Drop the cached device copy of `h` (call before destroying an HMatrix to free HBM early).
inline void b200_release(const HMatrix& h) {
  std::lock_guard<std::mutex> g(b200_detail::cache_mutex());
  auto& c = b200_detail::cache();
  for (auto i = c.begin(); i != c.end();) i = (i->first.h == &h) ? c.erase(i) : std::next(i);
}

/// evaluate(h, w, opts) (evaluate.hpp:287-317) on the B200, same signature and contract.
inline Potentials evaluate_b200(const HMatrix& h, const Matrix& w, const EvalOptions& opts = {}) {
  if (w.rows() != h.n) throw std::invalid_argument("evaluate: w has wrong row count");
  if (w.cols() < 1) throw std::invalid_argument("evaluate: w needs at least one column");
  return evaluate_b200(*b200_detail::evaluator_for(h), w, opts);
}

/// error_eps2(h, oracle, r, sample_rows, seed, opts) (evaluate.hpp:330-373) with its evaluate()
/// routed to the B200: the same sampled rows and W (the reference Rng stream, restated in the
/// C-ABI: gofmm_rng_eps2_draw_attempt), up to three draws while the sampled rows of K w vanish,
/// exact rows from the caller's oracle on the host, the same report fields.
inline ErrorReport error_eps2_b200(const HMatrix& h, const EntryOracle& oracle, int r, int sample_rows,
                                   std::uint64_t seed, const EvalOptions& opts = {}) {
  if (sample_rows < 1) throw std::invalid_argument("sample_rows must be >= 1");
  if (r < 1) throw std::invalid_argument("r must be >= 1");
  const int n = h.n;
  const int k = std::min(sample_rows, n);
  ErrorReport rep;
  rep.sample_rows.resize(k);
  IndexList all(n);
  std::iota(all.begin(), all.end(), 0);
  for (int attempt = 0; attempt < 3; ++attempt) {
    Matrix w(n, r);
    if (gofmm_rng_eps2_draw_attempt(seed, n, r, sample_rows, attempt, rep.sample_rows.data(), w.data(), n) !=
        GOFMM_OK)
      throw std::runtime_error(std::string("gofmm_rng_eps2_draw_attempt: ") + gofmm_last_error());
    const Potentials pot = evaluate_b200(h, w, opts);
    const Matrix u = unpermute(h.tree, pot.u);
    rep.eval_flops = pot.flops;
    rep.eval_seconds = pot.seconds;
    const Matrix exact = oracle.block(rep.sample_rows, all) * w;
    double num = 0.0, den = 0.0;
    std::vector<double> rel;
    rel.reserve(k);
    for (int t = 0; t < k; ++t) {
      const double dn = (u.row(rep.sample_rows[t]) - exact.row(t)).norm();
      const double de = exact.row(t).norm();
      num += dn * dn;
      den += de * de;
      rel.push_back(de > 0 ? dn / de : 0.0);
    }
    if (den == 0.0) continue;
    rep.eps2 = std::sqrt(num / den);
    rep.per_entry.assign(rel.begin(), rel.begin() + std::min<size_t>(10, rel.size()));
    rep.mean_sample = std::accumulate(rel.begin(), rel.end(), 0.0) / double(rel.size());
    return rep;
  }
  throw numeric_error("error_eps2: sampled rows of Kw vanished repeatedly");
}

}  // namespace gfmm

#endif  // GOFMM_B200_GFMM_HPP
