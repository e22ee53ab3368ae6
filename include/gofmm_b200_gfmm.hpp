// gofmm_b200_gfmm.hpp — header-only C++ adapter for the reference GOFMM API.
//
// Include AFTER the reference headers ("gfmm/gfmm.hpp"). It flattens a gfmm::HMatrix
// (compress.hpp:65-79) into gofmm_tree_desc once, and offers gfmm::evaluate()'s exact contract
// (evaluate.hpp:287-317: W in original order, Potentials.u in permuted order, the reference flop
// counter, std::invalid_argument on bad W) on the B200 through the C-ABI of gofmm_b200.h:
//
//   gfmm::B200Evaluator gpu(h);                 // stored blocks, any EntryOracle
//   gfmm::Potentials p = gpu.evaluate(w);       // == gfmm::evaluate(h, w) to 1e-12 (fp64)
//   gfmm::Potentials q = gfmm::evaluate_b200(gpu, w, opts);  // evaluate()-shaped free function
//
// A Gaussian kernel tree can instead be evaluated matrix-free (near/far blocks regenerated from
// the coordinates on the device) with B200Evaluator(h, &points, bandwidth).
#ifndef GOFMM_B200_GFMM_HPP
#define GOFMM_B200_GFMM_HPP

#include <stdexcept>
#include <string>
#include <vector>

#include "gofmm_b200.h"

namespace gfmm {

class B200Evaluator {
 public:
  /// Stored blocks exactly as HMatrix holds them (leaf_diag, near_field[t].k, far_field[t].k).
  explicit B200Evaluator(const HMatrix& h, int device = 0) { build(h, nullptr, 0.0, device); }
  /// Gaussian kernel tree evaluated matrix-free from the point coordinates (oracle.hpp:148-159).
  B200Evaluator(const HMatrix& h, const PointCloud* points, double bandwidth, int device = 0) {
    build(h, points, bandwidth, device);
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
  void build(const HMatrix& h, const PointCloud* pts, double bandwidth, int device) {
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
      d.source = GOFMM_SOURCE_KERNEL;
      d.kernel = GOFMM_KERNEL_GAUSSIAN;
      d.dim = pts->dim();
      d.coords = pts->coords.data();
      d.kparam[0] = bandwidth;
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
    const int rc = gofmm_create(&d, &o, &h_);
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

}  // namespace gfmm

#endif  // GOFMM_B200_GFMM_HPP
