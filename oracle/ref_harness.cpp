// Oracle harness — TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference GOFMM headers UNMODIFIED from /root/reference/proj/include (against the
// Eigen-subset shim in oracle/eigen_shim, see oracle/Makefile) and exposes them through a small
// C API so the Python tests and bench.py's reference/cpu_baseline legs can drive the reference's
// own code path:
//   compress()      compress.hpp:331-434   (produces the HMatrix the hot path consumes)
//   evaluate()      evaluate.hpp:287-317   (THE reference hot path, timed as the CPU baseline)
//   error_eps2()    evaluate.hpp:330-373
//   unpermute       evaluate.hpp:21-25
// plus export/import of the compressed structure so the GPU product and this oracle consume the
// SAME tree. Nothing in the product links or loads this library (paper_1707_00164_b200/ never
// imports oracle/); only tests/, __graft_entry__.smoke() and bench.py's reference legs do.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <vector>
#include <exception>
#include <memory>
#include <string>

#include "gfmm/gfmm.hpp"

using namespace gfmm;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// Map the reference's exception types to the CLI exit codes (gfmm_cli.cpp:289-305).
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(2, e.what());
  } catch (const io_error& e) {
    return fail(3, e.what());
  } catch (const numeric_error& e) {
    return fail(4, e.what());
  } catch (const std::exception& e) {
    return fail(1, e.what());
  }
}

/// Matérn-1/2 ("Exponential") kernel K_ij = exp(-|x_i - x_j| / h). Not present in the
/// reference (SURVEY.md §0 finding 6; BASELINE config 4); added through the reference's own
/// plugin point, EntryOracle (oracle.hpp:34-66), written like GaussianKernelOracle
/// (oracle.hpp:148-159): distance from the difference vector, then exp.
class ExponentialKernelOracle final : public EntryOracle {
 public:
  ExponentialKernelOracle(PointCloud points, double bandwidth)
      : points_(std::move(points)), h_(bandwidth) {
    points_.validate();
    if (!(bandwidth > 0)) throw std::invalid_argument("exponential bandwidth must be positive");
  }
  int size() const override { return points_.size(); }
  void eval_block(std::span<const int> I, std::span<const int> J, Matrix& out) const override {
    out.resize(I.size(), J.size());
    const double inv = 1.0 / h_;
    for (size_t c = 0; c < J.size(); ++c) {
      auto xj = points_.coords.col(J[c]);
      for (size_t r = 0; r < I.size(); ++r) {
        double d = (points_.coords.col(I[r]) - xj).norm();
        out(r, c) = std::exp(-d * inv);
      }
    }
  }
  Vector eval_diag(std::span<const int> I) const override { return Vector::Ones(I.size()); }

 private:
  PointCloud points_;
  double h_;
};

/// Serves one given block: rows are sample indices [0, rows), columns are candidates
/// [rows, rows + cols). Lets skeletonize_node (compress.hpp:149-187) run unmodified on a block
/// supplied by the test (the GPU batch gets the very same block).
class GivenBlockOracle final : public EntryOracle {
 public:
  GivenBlockOracle(const double* b, int rows, int cols) : b_(b), rows_(rows), cols_(cols) {}
  int size() const override { return rows_ + cols_; }
  void eval_block(std::span<const int> I, std::span<const int> J, Matrix& out) const override {
    out.resize(I.size(), J.size());
    for (size_t c = 0; c < J.size(); ++c)
      for (size_t r = 0; r < I.size(); ++r) out(r, c) = b_[size_t(J[c] - rows_) * rows_ + I[r]];
  }

 private:
  const double* b_;
  int rows_, cols_;
};

}  // namespace

extern "C" {

struct gfmm_ref_config {
  int32_t m, s;
  double tau;
  int32_t kappa;
  double budget;
  int32_t kind;  // 0 geom, 1 kernel, 2 angle (DistanceKind, metric.hpp:8)
  uint64_t seed;
  int32_t r;
  int32_t ann_iterations;
  int32_t threads;
};

// kernel ids shared with include/gofmm_b200.h
enum { REF_GAUSSIAN = 0, REF_LAPLACE = 1, REF_POLYNOMIAL = 2, REF_COSINE = 3, REF_EXPONENTIAL = 4 };

struct gfmm_ref {
  std::unique_ptr<EntryOracle> oracle;
  PointCloud pc;
  bool has_points = false;
  HMatrix h;
};

struct gfmm_ref_sizes {
  int32_t n, num_nodes, depth, num_leaves, dim, has_points;
  int64_t skel_total, proj_total, num_near, num_far, diag_total, near_total, far_total;
};

const char* gfmm_ref_last_error() { return g_err.c_str(); }

void gfmm_ref_free(gfmm_ref* p) { delete p; }

// PointCloud::random_gaussian (oracle.hpp:18-25), d x n column-major.
void gfmm_ref_points_gaussian(int32_t n, int32_t d, uint64_t seed, double* out) {
  PointCloud pc = PointCloud::random_gaussian(n, d, seed);
  std::memcpy(out, pc.coords.data(), sizeof(double) * size_t(n) * size_t(d));
}

// Column-major standard-normal fill from Rng(seed, stream), c outer / i inner — the order of
// random_rhs (test_evaluate.cpp:15-21, stream 0) and error_eps2's W (evaluate.hpp:344-346).
void gfmm_ref_rng_gauss(int64_t n, int32_t r, uint64_t seed, uint64_t stream, double* out) {
  Rng rng(seed, stream);
  for (int32_t c = 0; c < r; ++c)
    for (int64_t i = 0; i < n; ++i) out[i + c * n] = rng.gauss();
}

uint64_t gfmm_ref_splitmix64(uint64_t x) { return splitmix64(x); }

static RunConfig to_cfg(const gfmm_ref_config* c) {
  RunConfig cfg;
  cfg.m = c->m;
  cfg.s = c->s;
  cfg.tau = c->tau;
  cfg.kappa = c->kappa;
  cfg.budget = c->budget;
  cfg.kind = static_cast<DistanceKind>(c->kind);
  cfg.seed = c->seed;
  cfg.r = c->r;
  cfg.ann_iterations = c->ann_iterations;
  cfg.threads = c->threads;
  return cfg;
}

static std::unique_ptr<EntryOracle> make_kernel(int32_t kernel, const PointCloud& pc, double p0, double p1) {
  switch (kernel) {
    case REF_GAUSSIAN: return gaussian_kernel_oracle(pc, p0);
    case REF_LAPLACE: return laplace_kernel_oracle(pc, p0 < 0 ? default_laplace_floor(pc) : p0);
    case REF_POLYNOMIAL: return polynomial_kernel_oracle(pc, p0, static_cast<int>(p1));
    case REF_COSINE: return cosine_kernel_oracle(pc, p0);
    case REF_EXPONENTIAL: return std::make_unique<ExponentialKernelOracle>(pc, p0);
  }
  throw std::invalid_argument("unknown kernel id");
}

// Laplace default floor (oracle.hpp:276-288) so callers can pass the resolved value to the GPU.
double gfmm_ref_default_laplace_floor(const double* coords, int32_t d, int32_t n, uint64_t seed) {
  PointCloud pc;
  pc.coords.resize(d, n);
  std::memcpy(pc.coords.data(), coords, sizeof(double) * size_t(d) * size_t(n));
  return default_laplace_floor(pc, seed);
}

int gfmm_ref_compress_kernel(int32_t kernel, const double* coords, int32_t d, int32_t n, double p0,
                             double p1, const gfmm_ref_config* cfg, gfmm_ref** out) {
  return guarded([&] {
    auto ref = std::make_unique<gfmm_ref>();
    ref->pc.coords.resize(d, n);
    std::memcpy(ref->pc.coords.data(), coords, sizeof(double) * size_t(d) * size_t(n));
    ref->has_points = true;
    ref->oracle = make_kernel(kernel, ref->pc, p0, p1);
    ref->h = compress(*ref->oracle, &ref->pc, to_cfg(cfg));
    *out = ref.release();
  });
}

int gfmm_ref_compress_dense(const double* K, int32_t n, const gfmm_ref_config* cfg, gfmm_ref** out) {
  return guarded([&] {
    auto ref = std::make_unique<gfmm_ref>();
    Matrix k(n, n);
    std::memcpy(k.data(), K, sizeof(double) * size_t(n) * size_t(n));
    ref->oracle = std::make_unique<DenseOracle>(std::move(k));
    ref->h = compress(*ref->oracle, nullptr, to_cfg(cfg));
    *out = ref.release();
  });
}

// random_spd_oracle (oracle.hpp:321-333) — the exact-representation fixtures of
// test_evaluate.cpp:38-51,155-171 and acceptance criterion 1.
int gfmm_ref_compress_randspd(int32_t n, uint64_t seed, const gfmm_ref_config* cfg, gfmm_ref** out) {
  return guarded([&] {
    auto ref = std::make_unique<gfmm_ref>();
    ref->oracle = random_spd_oracle(n, seed);
    ref->h = compress(*ref->oracle, nullptr, to_cfg(cfg));
    *out = ref.release();
  });
}

// Dense K from the source oracle (desk scale) for independent dense checks.
int gfmm_ref_dense(const gfmm_ref* ref, double* K) {
  return guarded([&] {
    int n = ref->oracle->size();
    if (n > kDeskScaleCap) throw io_error("dense: N exceeds desk-scale cap");
    IndexList all(n);
    for (int i = 0; i < n; ++i) all[i] = i;
    Matrix k = ref->oracle->block(all, all);
    std::memcpy(K, k.data(), sizeof(double) * size_t(n) * size_t(n));
  });
}

// Rows of K (original indices) times W: the "exact" side of error_eps2 (evaluate.hpp:353).
int gfmm_ref_exact_rows(const gfmm_ref* ref, const int32_t* rows, int32_t nrows, const double* w,
                        int32_t r, double* out) {
  return guarded([&] {
    int n = ref->oracle->size();
    IndexList rl(rows, rows + nrows), all(n);
    for (int i = 0; i < n; ++i) all[i] = i;
    Matrix wm(n, r);
    std::memcpy(wm.data(), w, sizeof(double) * size_t(n) * size_t(r));
    Matrix ex = ref->oracle->block(rl, all) * wm;
    std::memcpy(out, ex.data(), sizeof(double) * size_t(nrows) * size_t(r));
  });
}

int gfmm_ref_get_sizes(const gfmm_ref* ref, gfmm_ref_sizes* s) {
  return guarded([&] {
    const HMatrix& h = ref->h;
    std::memset(s, 0, sizeof(*s));
    s->n = h.n;
    s->num_nodes = static_cast<int32_t>(h.tree.nodes.size());
    s->depth = h.tree.depth;
    s->num_leaves = static_cast<int32_t>(h.tree.leaf_ids.size());
    s->dim = ref->has_points ? ref->pc.dim() : 0;
    s->has_points = ref->has_points;
    for (const Skeleton& sk : h.skeletons) {
      if (!sk.valid()) continue;
      s->skel_total += sk.rank();
      s->proj_total += sk.proj.size();
    }
    s->num_near = static_cast<int64_t>(h.near_field.size());
    s->num_far = static_cast<int64_t>(h.far_field.size());
    for (const Matrix& m : h.leaf_diag) s->diag_total += m.size();
    for (const auto& b : h.near_field) s->near_total += b.k.size();
    for (const auto& b : h.far_field) s->far_total += b.k.size();
  });
}

struct gfmm_ref_export_args {
  int32_t *parent, *left, *right, *level, *start, *end;  // [num_nodes]
  int32_t* iperm;                                         // [n]
  int32_t* rank;                                          // [num_nodes], -1 = invalid skeleton
  int32_t* ncand;                                         // [num_nodes] proj columns
  int64_t* skel_off;                                      // [num_nodes+1]
  int32_t* skel_idx;                                      // [skel_total]
  int64_t* proj_off;                                      // [num_nodes+1]
  double* proj;                                           // [proj_total]
  int32_t *near_a, *near_b, *far_a, *far_b;
  int64_t* diag_off;  // [num_nodes+1]
  double* diag;       // [diag_total]
  int64_t* near_off;  // [num_near+1]
  double* near_blk;
  int64_t* far_off;  // [num_far+1]
  double* far_blk;
  double* coords;  // d x n, original order
};

int gfmm_ref_export(const gfmm_ref* ref, const gfmm_ref_export_args* a) {
  return guarded([&] {
    const HMatrix& h = ref->h;
    const MetricTree& t = h.tree;
    int nn = static_cast<int>(t.nodes.size());
    for (int i = 0; i < nn; ++i) {
      const TreeNode& nd = t.nodes[i];
      if (a->parent) a->parent[i] = nd.parent;
      if (a->left) a->left[i] = nd.left;
      if (a->right) a->right[i] = nd.right;
      if (a->level) a->level[i] = nd.level;
      if (a->start) a->start[i] = nd.start;
      if (a->end) a->end[i] = nd.end;
    }
    if (a->iperm) std::memcpy(a->iperm, t.iperm.data(), sizeof(int32_t) * t.iperm.size());
    int64_t so = 0, po = 0;
    for (int i = 0; i < nn; ++i) {
      const Skeleton& sk = h.skeletons[i];
      if (a->rank) a->rank[i] = sk.valid() ? sk.rank() : -1;
      if (a->ncand) a->ncand[i] = sk.valid() ? static_cast<int32_t>(sk.proj.cols()) : 0;
      if (a->skel_off) a->skel_off[i] = so;
      if (a->proj_off) a->proj_off[i] = po;
      if (sk.valid()) {
        if (a->skel_idx) std::memcpy(a->skel_idx + so, sk.skel.data(), sizeof(int32_t) * sk.skel.size());
        if (a->proj) std::memcpy(a->proj + po, sk.proj.data(), sizeof(double) * sk.proj.size());
        so += sk.rank();
        po += sk.proj.size();
      }
    }
    if (a->skel_off) a->skel_off[nn] = so;
    if (a->proj_off) a->proj_off[nn] = po;
    int64_t off = 0;
    for (int i = 0; i < nn; ++i) {
      if (a->diag_off) a->diag_off[i] = off;
      if (a->diag && h.leaf_diag[i].size())
        std::memcpy(a->diag + off, h.leaf_diag[i].data(), sizeof(double) * h.leaf_diag[i].size());
      off += h.leaf_diag[i].size();
    }
    if (a->diag_off) a->diag_off[nn] = off;
    off = 0;
    for (size_t t2 = 0; t2 < h.near_field.size(); ++t2) {
      const auto& b = h.near_field[t2];
      if (a->near_a) a->near_a[t2] = b.a;
      if (a->near_b) a->near_b[t2] = b.b;
      if (a->near_off) a->near_off[t2] = off;
      if (a->near_blk) std::memcpy(a->near_blk + off, b.k.data(), sizeof(double) * b.k.size());
      off += b.k.size();
    }
    if (a->near_off) a->near_off[h.near_field.size()] = off;
    off = 0;
    for (size_t t2 = 0; t2 < h.far_field.size(); ++t2) {
      const auto& b = h.far_field[t2];
      if (a->far_a) a->far_a[t2] = b.a;
      if (a->far_b) a->far_b[t2] = b.b;
      if (a->far_off) a->far_off[t2] = off;
      if (a->far_blk) std::memcpy(a->far_blk + off, b.k.data(), sizeof(double) * b.k.size());
      off += b.k.size();
    }
    if (a->far_off) a->far_off[h.far_field.size()] = off;
    if (a->coords && ref->has_points)
      std::memcpy(a->coords, ref->pc.coords.data(), sizeof(double) * ref->pc.coords.size());
  });
}

// Build a reference HMatrix from an externally produced compressed structure (e.g. the
// synthetic c3-shaped trees bench.py generates, which the reference compress would take hours
// to produce at N=2^20). Blocks D / S / far are materialised through the reference's own
// oracle.block() exactly as compress() does (compress.hpp:365-420).
struct gfmm_ref_import_args {
  int32_t n, num_nodes, kernel, dim;
  double p0, p1;
  const double* coords;  // d x n original order
  const int32_t *parent, *left, *right, *level, *start, *end, *iperm;
  const int32_t* rank;  // -1 invalid
  const int64_t* skel_off;
  const int32_t* skel_idx;
  const int64_t* proj_off;
  const double* proj;
  int64_t num_near;
  const int32_t *near_a, *near_b;
  int64_t num_far;
  const int32_t *far_a, *far_b;
  int32_t threads;
};

int gfmm_ref_import(const gfmm_ref_import_args* a, gfmm_ref** out) {
  return guarded([&] {
    auto ref = std::make_unique<gfmm_ref>();
    ref->pc.coords.resize(a->dim, a->n);
    std::memcpy(ref->pc.coords.data(), a->coords, sizeof(double) * size_t(a->dim) * size_t(a->n));
    ref->has_points = true;
    ref->oracle = make_kernel(a->kernel, ref->pc, a->p0, a->p1);
    HMatrix& h = ref->h;
    h.n = a->n;
    MetricTree& t = h.tree;
    t.nodes.resize(a->num_nodes);
    t.iperm.assign(a->iperm, a->iperm + a->n);
    t.perm.resize(a->n);
    for (int i = 0; i < a->n; ++i) t.perm[t.iperm[i]] = i;
    t.depth = 0;
    for (int i = 0; i < a->num_nodes; ++i) {
      TreeNode& nd = t.nodes[i];
      nd.id = i;
      nd.parent = a->parent[i];
      nd.left = a->left[i];
      nd.right = a->right[i];
      nd.level = a->level[i];
      nd.start = a->start[i];
      nd.end = a->end[i];
      t.depth = std::max(t.depth, nd.level);
      if (nd.is_leaf()) t.leaf_ids.push_back(i);
    }
    std::sort(t.leaf_ids.begin(), t.leaf_ids.end(),
              [&](int x, int y) { return t.nodes[x].start < t.nodes[y].start; });
    h.skeletons.resize(a->num_nodes);
    for (int i = 0; i < a->num_nodes; ++i) {
      if (a->rank[i] < 0) continue;
      Skeleton& sk = h.skeletons[i];
      sk.node_id = i;
      sk.skel.assign(a->skel_idx + a->skel_off[i], a->skel_idx + a->skel_off[i + 1]);
      int64_t np = a->proj_off[i + 1] - a->proj_off[i];
      int k = a->rank[i];
      int c = k ? static_cast<int>(np / k) : 0;
      sk.proj.resize(k, c);
      std::memcpy(sk.proj.data(), a->proj + a->proj_off[i], sizeof(double) * size_t(np));
    }
    int threads = std::max(1, a->threads);
    h.leaf_diag.resize(a->num_nodes);
    int nl = static_cast<int>(t.leaf_ids.size());
    parallel_for(0, nl, threads, [&](int li) {
      int id = t.leaf_ids[li];
      IndexList ids = t.node_indices(id);
      h.leaf_diag[id] = ref->oracle->block(ids, ids);
    });
    h.near_field.resize(a->num_near);
    parallel_for(0, static_cast<int>(a->num_near), threads, [&](int q) {
      int x = a->near_a[q], y = a->near_b[q];
      h.near_field[q] = {x, y, ref->oracle->block(t.node_indices(x), t.node_indices(y))};
    });
    h.far_field.resize(a->num_far);
    parallel_for(0, static_cast<int>(a->num_far), threads, [&](int q) {
      int x = a->far_a[q], y = a->far_b[q];
      h.far_field[q] = {x, y, ref->oracle->block(h.skeletons[x].skel, h.skeletons[y].skel)};
    });
    *out = ref.release();
  });
}

// evaluate() (evaluate.hpp:287-317): w is n x r original order, u_perm receives the permuted
// potentials. mode: 0 LevelByLevel, 1 TaskDag.
// nrows is w's row count: a mismatch reaches evaluate() and throws there (evaluate.hpp:288).
int gfmm_ref_evaluate(const gfmm_ref* ref, const double* w, int32_t nrows, int32_t r, double* u_perm,
                      int32_t mode, int32_t threads, int64_t* flops, double* seconds) {
  return guarded([&] {
    const HMatrix& h = ref->h;
    Matrix wm(nrows, r);
    if (nrows && r > 0) std::memcpy(wm.data(), w, sizeof(double) * size_t(nrows) * size_t(r));
    EvalOptions o;
    o.mode = mode == 0 ? TraversalMode::LevelByLevel : TraversalMode::TaskDag;
    o.threads = threads;
    Potentials p = evaluate(h, wm, o);
    std::memcpy(u_perm, p.u.data(), sizeof(double) * size_t(p.u.size()));
    if (flops) *flops = p.flops;
    if (seconds) *seconds = p.seconds;
  });
}

// unpermute (evaluate.hpp:21-25)
int gfmm_ref_unpermute(const gfmm_ref* ref, const double* u_perm, int32_t r, double* u) {
  return guarded([&] {
    const HMatrix& h = ref->h;
    Matrix up(h.n, r);
    std::memcpy(up.data(), u_perm, sizeof(double) * size_t(h.n) * size_t(r));
    Matrix o = unpermute(h.tree, up);
    std::memcpy(u, o.data(), sizeof(double) * size_t(o.size()));
  });
}

// error_eps2 (evaluate.hpp:330-373). first10 has room for 10, rows_out for min(sample_rows, n).
int gfmm_ref_error_eps2(const gfmm_ref* ref, int32_t r, int32_t sample_rows, uint64_t seed, int32_t mode,
                        int32_t threads, double* eps2, double* first10, int32_t* nfirst, double* mean,
                        int64_t* flops, double* seconds, int32_t* rows_out) {
  return guarded([&] {
    EvalOptions o;
    o.mode = mode == 0 ? TraversalMode::LevelByLevel : TraversalMode::TaskDag;
    o.threads = threads;
    ErrorReport rep = error_eps2(ref->h, *ref->oracle, r, sample_rows, seed, o);
    *eps2 = rep.eps2;
    *nfirst = static_cast<int32_t>(rep.per_entry.size());
    for (size_t i = 0; i < rep.per_entry.size(); ++i) first10[i] = rep.per_entry[i];
    *mean = rep.mean_sample;
    *flops = rep.eval_flops;
    *seconds = rep.eval_seconds;
    if (rows_out)
      for (size_t i = 0; i < rep.sample_rows.size(); ++i) rows_out[i] = rep.sample_rows[i];
  });
}

// Rng::sample_without_replacement then the column-major gauss W, in error_eps2's consumption
// order (evaluate.hpp:336-346), for attempt 0. Lets the GPU side reproduce eps2 exactly.
int gfmm_ref_eps2_draw(int32_t n, int32_t r, int32_t sample_rows, uint64_t seed, int32_t* rows_out,
                       double* w_out) {
  return guarded([&] {
    Rng rng(seed, 0xe952);
    IndexList rows = rng.sample_without_replacement(n, std::min(sample_rows, n));
    for (size_t i = 0; i < rows.size(); ++i) rows_out[i] = rows[i];
    for (int32_t c = 0; c < r; ++c)
      for (int32_t i = 0; i < n; ++i) w_out[i + size_t(c) * n] = rng.gauss();
  });
}

int gfmm_ref_compress_stats(const gfmm_ref* ref, int64_t* entries, int64_t* cflops, int64_t* near_entries,
                            int32_t* max_skel, double* mean_skel, double* cseconds) {
  return guarded([&] {
    const CompressStats& s = ref->h.stats;
    *entries = s.entries_evaluated;
    *cflops = s.compress_flops;
    *near_entries = s.near_field_entries;
    *max_skel = s.max_skeleton;
    *mean_skel = s.mean_skeleton;
    *cseconds = s.compress_seconds;
  });
}

/// The reference skeletonize_node (compress.hpp:149-187) over a batch of given blocks (node t:
/// column-major rows[t] x cols[t] at blocks + off[t]), parallel over nodes like compress() does
/// (parallel_for, common.hpp:109-126). Outputs as gofmm_skeletonize_batch: rank, achieved_tol,
/// skel (pivot index per skeleton entry, slot of cols[t] ints), proj (slot of
/// min(s, rows, cols) * cols doubles, rank x cols column-major). seconds = wall time of the loop.
int gfmm_ref_skeletonize_batch(int32_t nnodes, const int32_t* rows, const int32_t* cols, const int64_t* off,
                               const double* blocks, int32_t s, double tau, int32_t threads, int32_t* rank_out,
                               double* achieved_out, int32_t* skel_out, double* proj_out, double* seconds) {
  return guarded([&] {
    std::vector<int64_t> soff(nnodes + 1, 0), poff(nnodes + 1, 0);
    for (int t = 0; t < nnodes; ++t) {
      soff[t + 1] = soff[t] + cols[t];
      poff[t + 1] = poff[t] + int64_t(std::min({s, rows[t], cols[t]})) * cols[t];
    }
    auto t0 = std::chrono::steady_clock::now();
    parallel_for(0, nnodes, std::max(1, threads), [&](int t) {
      GivenBlockOracle o(blocks + off[t], rows[t], cols[t]);
      IndexList sample(rows[t]), cand(cols[t]);
      for (int i = 0; i < rows[t]; ++i) sample[i] = i;
      for (int j = 0; j < cols[t]; ++j) cand[j] = rows[t] + j;
      Skeleton sk = skeletonize_node(t, cand, sample, o, s, tau);
      rank_out[t] = sk.rank();
      achieved_out[t] = sk.achieved_tol;
      for (int l = 0; l < sk.rank(); ++l) skel_out[soff[t] + l] = sk.skel[l] - rows[t];
      for (int64_t e = 0; e < int64_t(sk.rank()) * cols[t]; ++e) proj_out[poff[t] + e] = sk.proj.data()[e];
    });
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- ANN (neighbors.hpp:88-106): the random tree's leaves and one reference ann_iteration on a
// given table, for the GPU leaf all-pairs + merge parity (tests/test_ann_gpu.py).
// kind: 0 = GeometricL2, 1 = KernelL2 over a Gaussian oracle of bandwidth h (metric.hpp).
struct AnnCtx {
  PointCloud pc;
  std::unique_ptr<EntryOracle> oracle;
  std::unique_ptr<Metric> metric;
  AnnCtx(const double* coords, int32_t d, int32_t n, int32_t kind, double h) {
    pc.coords.resize(d, n);
    std::memcpy(pc.coords.data(), coords, sizeof(double) * size_t(d) * size_t(n));
    oracle = std::make_unique<GaussianKernelOracle>(pc, h);
    metric = std::make_unique<Metric>(kind == 0 ? DistanceKind::GeometricL2 : DistanceKind::KernelL2, *oracle,
                                      &pc);
  }
};

int gfmm_ref_ann_leaves(const double* coords, int32_t d, int32_t n, int32_t kind, double h, int32_t m,
                        uint64_t seed, int32_t* leaf_off, int32_t* leaf_idx, int32_t* nleaves) {
  return guarded([&] {
    AnnCtx c(coords, d, n, kind, h);
    MetricTree tree = build_random_tree(*c.metric, m, seed);
    int pos = 0;
    leaf_off[0] = 0;
    for (size_t l = 0; l < tree.leaf_ids.size(); ++l) {
      IndexList idx = tree.node_indices(tree.leaf_ids[l]);
      for (int i : idx) leaf_idx[pos++] = i;
      leaf_off[l + 1] = pos;
    }
    *nleaves = int32_t(tree.leaf_ids.size());
  });
}

int gfmm_ref_ann_iteration(const double* coords, int32_t d, int32_t n, int32_t kind, double h, int32_t kappa,
                           int32_t m, uint64_t seed, int32_t threads, int32_t* tj, double* td, int32_t* tlen,
                           double* seconds) {
  return guarded([&] {
    AnnCtx c(coords, d, n, kind, h);
    NeighborTable table = NeighborTable::empty(n, kappa);
    for (int i = 0; i < n; ++i)
      for (int t = 0; t < tlen[i]; ++t)
        table.lists[i].emplace_back(tj[size_t(i) * kappa + t], td[size_t(i) * kappa + t]);
    auto t0 = std::chrono::steady_clock::now();
    ann_iteration(table, *c.metric, m, seed, std::max(1, threads));
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int i = 0; i < n; ++i) {
      tlen[i] = int32_t(table.lists[i].size());
      for (int t = 0; t < tlen[i]; ++t) {
        tj[size_t(i) * kappa + t] = table.lists[i][t].first;
        td[size_t(i) * kappa + t] = table.lists[i][t].second;
      }
    }
  });
}

}  // extern "C"
