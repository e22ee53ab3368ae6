// gofmm_compress.cu — the compress phase that produces the evaluator's input.
//
// Restates gfmm::compress (compress.hpp:331-434) and the pieces it calls — kernel oracles
// (oracle.hpp:141-219, plus the Matérn-1/2 kernel of BASELINE config 4), Metric (metric.hpp:20-150),
// the metric / random ball trees (tree.hpp:126-246), ann_search (neighbors.hpp:88-183),
// select_near_field (compress.hpp:85-144), StructureWalker (compress.hpp:196-324), sample_columns
// (compress.hpp:191-229) and skeletonize_node (compress.hpp:149-187) — as a host pipeline around
// three device stages:
//   * ANN leaf passes: gofmm_ann_leaf_merge (csrc/gofmm_ann.cu), one launch per iteration;
//   * sampled blocks K(sample_cols, candidates) of a whole tree level generated in HBM
//     (sampled_block_kernel below, entries as the oracle builds them);
//   * the level's batched column-pivoted QR / interpolative decomposition (csrc/gofmm_skel.cu,
//     bit-identical to the reference on the same block).
// D / near / far blocks are not stored: the evaluator regenerates them inside its GEMMs
// (matrix-free), and the entries they would cost are counted like the reference's CountingOracle.
//
// Two entry modes (gofmm_compress_config.entries):
//   GOFMM_ENTRIES_HOST   — every kernel entry that steers a discrete decision (tree pivots, ANN
//                          lists, sampled blocks) is computed on the host with the reference's
//                          formulas and reduction order (Eigen 3.4 SSE2 redux, glibc exp/pow), so
//                          the tree, neighbour lists, skeletons and proj are bit-identical to the
//                          reference compress (tests/test_compress_gpu.py); CPQR still runs on the GPU.
//   GOFMM_ENTRIES_DEVICE — ANN leaf passes and sampled blocks on the GPU (libdevice exp/pow, a few
//                          ulps from glibc): the same algorithm, orders of magnitude faster at 1M
//                          points; decisions can differ from the reference at exact near-ties.
// The metric tree is built on the host in both modes (O(N log N) entries).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/gofmm_b200.h"
#include "gofmm_kernels.cuh"
#include "gofmm_rng.h"
#include "gofmm_skel_internal.h"

namespace gofmm {
namespace cmp {

using IndexList = std::vector<int>;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
thread_local std::string g_err;

// ---------------------------------------------------------------- reductions (Eigen 3.4, SSE2)
// redux over a unit-stride expression: 2-wide packets, two packet accumulators (Eigen
// redux_impl<LinearVectorizedTraversal>), element i = get(i); strided (row) views reduce in order.
template <class F>
inline double redux_packet(int64_t n, F get) {
  const int64_t aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  if (aligned) {
    double a0 = get(0), a1 = get(1);
    if (aligned > 2) {
      double b0 = get(2), b1 = get(3);
      for (int64_t i = 4; i < aligned2; i += 4) {
        a0 = a0 + get(i);
        a1 = a1 + get(i + 1);
        b0 = b0 + get(i + 2);
        b1 = b1 + get(i + 3);
      }
      a0 = a0 + b0;
      a1 = a1 + b1;
      if (aligned > aligned2) {
        a0 = a0 + get(aligned2);
        a1 = a1 + get(aligned2 + 1);
      }
    }
    double res = a0 + a1;
    for (int64_t i = aligned; i < n; ++i) res = res + get(i);
    return res;
  }
  double res = get(0);
  for (int64_t i = 1; i < n; ++i) res = res + get(i);
  return res;
}
template <class F>
inline double redux_seq(int64_t n, F get) {
  double res = get(0);
  for (int64_t i = 1; i < n; ++i) res = res + get(i);
  return res;
}

// Static partition (common.hpp:109-126): chunk t takes indices begin + t, begin + t + threads, ...
template <class F>
void parallel_for(int begin, int end, int threads, F&& body) {
  const int n = end - begin;
  if (n <= 0) return;
  threads = std::max(1, std::min(threads, n));
  if (threads == 1) {
    for (int i = begin; i < end; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(threads);
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int i = begin + t; i < end; i += threads) body(i);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// ---------------------------------------------------------------- kernel oracle (oracle.hpp)
struct Oracle {
  int kernel = GOFMM_KERNEL_GAUSSIAN, d = 0, n = 0;
  const double* x = nullptr;  // d x n column-major (point-major)
  double p0 = 0, p1 = 0;      // as gofmm_tree_desc::kparam
  mutable std::atomic<int64_t> count{0};  // CountingOracle (oracle.hpp:68-90)

  const double* col(int i) const { return x + int64_t(i) * d; }
  // K_ij exactly as the reference generator computes it (not counted)
  double raw(int i, int j) const {
    const double *a = col(i), *b = col(j);
    switch (kernel) {
      case GOFMM_KERNEL_GAUSSIAN: {  // oracle.hpp:148-159
        const double inv = 1.0 / (2.0 * p0 * p0);
        const double d2 = redux_packet(d, [&](int64_t q) {
          const double e = a[q] - b[q];
          return e * e;
        });
        return std::exp(-d2 * inv);
      }
      case GOFMM_KERNEL_EXPONENTIAL: {  // Matérn-1/2 through EntryOracle (oracle/ref_harness.cpp)
        const double inv = 1.0 / p0;
        const double dd = std::sqrt(redux_packet(d, [&](int64_t q) {
          const double e = a[q] - b[q];
          return e * e;
        }));
        return std::exp(-dd * inv);
      }
      case GOFMM_KERNEL_LAPLACE: {  // oracle.hpp:178-192
        const double p = double(d - 2);
        const double dd = std::sqrt(redux_packet(d, [&](int64_t q) {
          const double e = a[q] - b[q];
          return e * e;
        }));
        const double rr = std::max(dd, p0);
        if (rr <= 0.0) throw Error(GOFMM_ERR_NUMERIC, "laplace kernel: zero distance with delta=0");
        return std::pow(rr, -p);
      }
      case GOFMM_KERNEL_POLYNOMIAL: {  // oracle.hpp:208-218
        const double ip = redux_packet(d, [&](int64_t q) { return a[q] * b[q]; });
        return std::pow(ip + p0, int(p1));
      }
    }
    throw Error(GOFMM_ERR_INVALID, "unsupported kernel id");
  }
  // block(I, J) column-major |I| x |J| (counted)
  void block(const int* I, int ni, const int* J, int nj, double* out) const {
    count.fetch_add(int64_t(ni) * nj, std::memory_order_relaxed);
    for (int c = 0; c < nj; ++c)
      for (int r = 0; r < ni; ++r) out[r + int64_t(c) * ni] = raw(I[r], J[c]);
  }
  double entry(int i, int j) const {
    count.fetch_add(1, std::memory_order_relaxed);
    return raw(i, j);
  }
  // eval_diag over all indices (counted n): unit diagonal for Gaussian / Matérn overrides,
  // the generic entry-by-entry default otherwise (oracle.hpp:44-53,161-163)
  std::vector<double> diag() const {
    count.fetch_add(n, std::memory_order_relaxed);
    std::vector<double> dg(n, 1.0);
    if (kernel == GOFMM_KERNEL_LAPLACE || kernel == GOFMM_KERNEL_POLYNOMIAL)
      for (int i = 0; i < n; ++i) dg[i] = raw(i, i);
    return dg;
  }
};

// ---------------------------------------------------------------- metric (metric.hpp)
struct Metric {
  int kind;  // GOFMM_DIST_*
  const Oracle* o;
  std::vector<double> dg;

  Metric(int k, const Oracle& oracle) : kind(k), o(&oracle) { dg = oracle.diag(); }
  int size() const { return o->n; }

  double geom(int i, int j) const {
    const double *a = o->col(i), *b = o->col(j);
    return std::sqrt(redux_packet(o->d, [&](int64_t q) {
      const double e = a[q] - b[q];
      return e * e;
    }));
  }
  double from_entry(int i, int j, double kij) const {
    if (kind == GOFMM_DIST_KERNEL) return std::sqrt(std::max(0.0, dg[i] + dg[j] - 2.0 * kij));
    const double dd = 1.0 - (kij * kij) / (dg[i] * dg[j]);
    return std::clamp(dd, 0.0, 1.0);
  }
  double operator()(int i, int j) const {
    if (i == j) return 0.0;
    if (kind == GOFMM_DIST_GEOMETRIC) return geom(i, j);
    return from_entry(i, j, o->entry(i, j));
  }
  void distances_from(int i, const int* J, int nj, double* out) const {
    if (kind == GOFMM_DIST_GEOMETRIC) {
      for (int t = 0; t < nj; ++t) out[t] = geom(i, J[t]);
      return;
    }
    std::vector<double> row(nj);
    o->block(&i, 1, J, nj, row.data());
    for (int t = 0; t < nj; ++t) out[t] = (J[t] == i) ? 0.0 : from_entry(i, J[t], row[t]);
  }
  // |I| x |I| distances, column-major
  void pairwise(const int* I, int ni, double* out) const {
    if (kind == GOFMM_DIST_GEOMETRIC) {
      for (int b = 0; b < ni; ++b)
        for (int a = 0; a < ni; ++a) out[a + int64_t(b) * ni] = geom(I[a], I[b]);
      return;
    }
    o->block(I, ni, I, ni, out);
    for (int b = 0; b < ni; ++b)
      for (int a = 0; a < ni; ++a) {
        double& v = out[a + int64_t(b) * ni];
        v = (I[a] == I[b]) ? 0.0 : from_entry(I[a], I[b], v);
      }
  }
  struct Centroid {
    IndexList sample;
    double self = 0.0;
    std::vector<double> mean;
  };
  // throws Error(GOFMM_ERR_NUMERIC + 100) for a degenerate angle centroid
  Centroid centroid(const IndexList& sample) const {
    Centroid c;
    c.sample = sample;
    const int ns = int(sample.size());
    if (kind == GOFMM_DIST_GEOMETRIC) {
      c.mean.assign(o->d, 0.0);
      for (int s : sample)
        for (int q = 0; q < o->d; ++q) c.mean[q] = c.mean[q] + o->col(s)[q];
      for (int q = 0; q < o->d; ++q) c.mean[q] = c.mean[q] / double(ns);
      return c;
    }
    std::vector<double> g(size_t(ns) * ns);
    o->block(sample.data(), ns, sample.data(), ns, g.data());
    const double nc = double(ns);
    if (kind == GOFMM_DIST_ANGLE) {
      for (int b = 0; b < ns; ++b)
        for (int a = 0; a < ns; ++a) g[a + size_t(b) * ns] /= std::sqrt(dg[sample[a]] * dg[sample[b]]);
      c.self = redux_packet(int64_t(ns) * ns, [&](int64_t i) { return g[i]; }) / (nc * nc);
      if (c.self <= 1e-14) throw Error(GOFMM_ERR_NUMERIC + 100, "angle centroid has (near-)zero norm");
      return c;
    }
    c.self = redux_packet(int64_t(ns) * ns, [&](int64_t i) { return g[i]; }) / (nc * nc);
    return c;
  }
  void distances_to_centroid(const int* I, int ni, const Centroid& c, double* out) const {
    if (kind == GOFMM_DIST_GEOMETRIC) {
      for (int t = 0; t < ni; ++t) {
        const double* a = o->col(I[t]);
        out[t] = std::sqrt(redux_packet(o->d, [&](int64_t q) {
          const double e = a[q] - c.mean[q];
          return e * e;
        }));
      }
      return;
    }
    const int ns = int(c.sample.size());
    std::vector<double> cross(size_t(ni) * ns);
    o->block(I, ni, c.sample.data(), ns, cross.data());
    const double nc = double(ns);
    for (int t = 0; t < ni; ++t) {
      if (kind == GOFMM_DIST_KERNEL) {
        const double si = redux_seq(ns, [&](int64_t s) { return cross[t + size_t(s) * ni]; });
        const double d2 = dg[I[t]] - 2.0 * si / nc + c.self;
        out[t] = std::sqrt(std::max(0.0, d2));
      } else {
        double si = 0.0;
        for (int s = 0; s < ns; ++s) si += cross[t + size_t(s) * ni] / std::sqrt(dg[I[t]] * dg[c.sample[s]]);
        const double dd = 1.0 - (si * si) / (nc * nc * c.self);
        out[t] = std::clamp(dd, 0.0, 1.0);
      }
    }
  }
};

// ---------------------------------------------------------------- trees (tree.hpp)
struct Node {
  int id = -1, parent = -1, left = -1, right = -1, level = 0, start = 0, end = 0;
  uint64_t path = 1;
  bool leaf() const { return left < 0; }
  int count() const { return end - start; }
};
struct Tree {
  std::vector<Node> nodes;
  IndexList perm, iperm;
  std::vector<int> leaf_ids;
  int depth = 0;
};
struct Split {
  IndexList left, right;
};

constexpr int kCentroidSample = 32;  // tree.hpp:11

Split even_split(const int* idx, int n) {
  Split r;
  const int lsize = n - n / 2;
  r.left.assign(idx, idx + lsize);
  r.right.assign(idx + lsize, idx + n);
  return r;
}

// tree.hpp:58-101: left = the ceil(n/2) smallest (score, position) pairs, both sides in position order
Split split_by_pivots(const int* idx, int n, const Metric& m, int p, int q) {
  std::vector<double> dp(n), dq(n), s(n);
  m.distances_from(p, idx, n, dp.data());
  m.distances_from(q, idx, n, dq.data());
  for (int i = 0; i < n; ++i) s[i] = dp[i] - dq[i];
  bool seen = false, all_tie = true;
  double first = 0.0;
  for (int i = 0; i < n; ++i) {
    if (idx[i] == p || idx[i] == q) continue;
    if (!seen) {
      first = s[i];
      seen = true;
    } else if (s[i] != first) {
      all_tie = false;
      break;
    }
  }
  if (seen && all_tie) return even_split(idx, n);
  std::vector<std::pair<double, int>> order(n);
  for (int i = 0; i < n; ++i) order[i] = {s[i], i};
  const int lsize = n - n / 2;
  std::nth_element(order.begin(), order.begin() + lsize, order.end());
  IndexList lpos(lsize), rpos(n - lsize);
  for (int i = 0; i < lsize; ++i) lpos[i] = order[i].second;
  for (int i = lsize; i < n; ++i) rpos[i - lsize] = order[i].second;
  std::sort(lpos.begin(), lpos.end());
  std::sort(rpos.begin(), rpos.end());
  Split r;
  r.left.reserve(lsize);
  r.right.reserve(n - lsize);
  for (int t : lpos) r.left.push_back(idx[t]);
  for (int t : rpos) r.right.push_back(idx[t]);
  return r;
}

int argmax_index(const int* idx, const double* d, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (d[i] > d[best] || (d[i] == d[best] && idx[i] < idx[best])) best = i;
  return best;
}

// tree.hpp:126-152
Split metric_split(const int* idx, int n, const Metric& m, RefRng& rng) {
  std::vector<double> dc(n);
  bool have = false;
  for (int attempt = 0; attempt < 4 && !have; ++attempt) {
    IndexList pos = rng.sample_without_replacement(n, std::min(kCentroidSample, n));
    IndexList sample(pos.size());
    for (size_t t = 0; t < pos.size(); ++t) sample[t] = idx[pos[t]];
    try {
      Metric::Centroid c = m.centroid(sample);
      m.distances_to_centroid(idx, n, c, dc.data());
      have = true;
    } catch (const Error& e) {
      if (e.code != GOFMM_ERR_NUMERIC + 100) throw;  // degenerate_centroid: fresh sample
    }
  }
  if (!have) return even_split(idx, n);
  const int p = idx[argmax_index(idx, dc.data(), n)];
  std::vector<double> dp(n);
  m.distances_from(p, idx, n, dp.data());
  if (*std::max_element(dp.begin(), dp.end()) == 0.0) return even_split(idx, n);
  const int q = idx[argmax_index(idx, dp.data(), n)];
  return split_by_pivots(idx, n, m, p, q);
}

// tree.hpp:156-167
Split randomized_split(const int* idx, int n, const Metric& m, RefRng& rng) {
  for (int attempt = 0; attempt < 8; ++attempt) {
    const int a = rng.uniform(n);
    int b = rng.uniform(n - 1);
    if (b >= a) ++b;
    const int p = idx[a], q = idx[b];
    if (m(p, q) > 0.0) return split_by_pivots(idx, n, m, p, q);
  }
  return even_split(idx, n);
}

// tree.hpp:171-239 — BFS order, node ids in queue order. The nodes of one BFS level are split
// concurrently (each split only reads its own range and its own path-keyed Rng), then their
// children are appended in the queue's order.
Tree build_tree(const Metric& m, int leaf, uint64_t seed, bool random_pivots, int threads) {
  const int n = m.size();
  Tree t;
  t.iperm.resize(n);
  std::iota(t.iperm.begin(), t.iperm.end(), 0);
  Node root;
  root.id = 0;
  root.start = 0;
  root.end = n;
  t.nodes.push_back(root);
  std::vector<int> frontier{0};
  while (!frontier.empty()) {
    std::vector<int> todo;
    for (int id : frontier)
      if (t.nodes[id].count() > leaf) todo.push_back(id);
    std::vector<Split> res(todo.size());
    parallel_for(0, int(todo.size()), threads, [&](int k) {
      const Node& nd = t.nodes[todo[k]];
      RefRng rng(seed, splitmix64(nd.path));
      const int* idx = t.iperm.data() + nd.start;
      res[k] = random_pivots ? randomized_split(idx, nd.count(), m, rng) : metric_split(idx, nd.count(), m, rng);
    });
    std::vector<int> next;
    for (size_t k = 0; k < todo.size(); ++k) {
      const int id = todo[k];
      Node nd = t.nodes[id];
      std::copy(res[k].left.begin(), res[k].left.end(), t.iperm.begin() + nd.start);
      std::copy(res[k].right.begin(), res[k].right.end(), t.iperm.begin() + nd.start + res[k].left.size());
      const int mid = nd.start + int(res[k].left.size());
      Node lc, rc;
      lc.parent = rc.parent = id;
      lc.level = rc.level = nd.level + 1;
      lc.start = nd.start;
      lc.end = mid;
      rc.start = mid;
      rc.end = nd.end;
      lc.path = nd.path * 2;
      rc.path = nd.path * 2 + 1;
      lc.id = int(t.nodes.size());
      rc.id = lc.id + 1;
      t.nodes[id].left = lc.id;
      t.nodes[id].right = rc.id;
      t.nodes.push_back(lc);
      t.nodes.push_back(rc);
      next.push_back(lc.id);
      next.push_back(rc.id);
    }
    frontier = std::move(next);
  }
  t.perm.resize(n);
  for (int i = 0; i < n; ++i) t.perm[t.iperm[i]] = i;
  for (const Node& nd : t.nodes) {
    t.depth = std::max(t.depth, nd.level);
    if (nd.leaf()) t.leaf_ids.push_back(nd.id);
  }
  std::sort(t.leaf_ids.begin(), t.leaf_ids.end(), [&](int a, int b) { return t.nodes[a].start < t.nodes[b].start; });
  return t;
}

// ---------------------------------------------------------------- neighbours (neighbors.hpp)
using Nbr = std::pair<int, double>;
struct Table {
  int k = 0;
  std::vector<std::vector<Nbr>> lists;
};
inline bool nbr_less(const Nbr& a, const Nbr& b) {
  if (a.second != b.second) return a.second < b.second;
  return a.first < b.first;
}
// neighbors.hpp:35-63
void merge_candidates(std::vector<Nbr>& list, std::vector<Nbr>& cand, int k) {
  std::sort(cand.begin(), cand.end(), nbr_less);
  std::vector<Nbr> merged;
  merged.reserve(std::min<size_t>(k, list.size() + cand.size()));
  size_t a = 0, b = 0;
  int last = -1;
  while (int(merged.size()) < k && (a < list.size() || b < cand.size())) {
    const Nbr* next;
    if (b >= cand.size() || (a < list.size() && nbr_less(list[a], cand[b])))
      next = &list[a++];
    else
      next = &cand[b++];
    if (next->first == last) continue;
    bool dup = false;
    for (auto it = merged.rbegin(); it != merged.rend() && it->second == next->second; ++it)
      if (it->first == next->first) {
        dup = true;
        break;
      }
    if (dup) continue;
    merged.push_back(*next);
    last = next->first;
  }
  list = std::move(merged);
}

struct Config {
  gofmm_compress_config c;
  bool device_entries() const { return c.entries == GOFMM_ENTRIES_DEVICE; }
};

// one ann_iteration (neighbors.hpp:88-106): host leaf pass, or the GPU one (geometric / kernel L2
// over a Gaussian: gofmm_ann_leaf_merge, which merges exactly as merge_candidates does)
void ann_iteration(Table& tab, const Metric& m, const Config& cfg, uint64_t seed, double* kernel_ms) {
  Tree tr = build_tree(m, cfg.c.m, seed, true, cfg.c.threads);
  const int nl = int(tr.leaf_ids.size());
  const Oracle& o = *m.o;
  const bool gpu = cfg.device_entries() && tab.k >= 1 && tab.k <= 32 &&
                   (m.kind == GOFMM_DIST_GEOMETRIC ||
                    (m.kind == GOFMM_DIST_KERNEL && o.kernel == GOFMM_KERNEL_GAUSSIAN)) &&
                   o.d <= 16 && cfg.c.m <= 1024;
  if (gpu) {
    const int n = o.n, k = tab.k;
    std::vector<int32_t> off(nl + 1, 0), idx(n), tj(size_t(n) * k), tl(n);
    std::vector<double> td(size_t(n) * k);
    for (int li = 0; li < nl; ++li) {
      const Node& nd = tr.nodes[tr.leaf_ids[li]];
      off[li + 1] = off[li] + nd.count();
      std::copy(tr.iperm.begin() + nd.start, tr.iperm.begin() + nd.end, idx.begin() + off[li]);
    }
    for (int i = 0; i < n; ++i) {
      tl[i] = int(tab.lists[i].size());
      for (int t = 0; t < tl[i]; ++t) {
        tj[size_t(i) * k + t] = tab.lists[i][t].first;
        td[size_t(i) * k + t] = tab.lists[i][t].second;
      }
    }
    double ms = 0.0;
    const int rc = gofmm_ann_leaf_merge(n, o.d, o.x, m.kind == GOFMM_DIST_GEOMETRIC ? 0 : 1, o.p0, k, nl, off.data(),
                                        idx.data(), cfg.c.device, tj.data(), td.data(), tl.data(), &ms);
    if (rc != GOFMM_OK) throw Error(rc, std::string("ANN leaf pass: ") + gofmm_ann_last_error());
    if (kernel_ms) *kernel_ms += ms;
    // CountingOracle: pairwise(leaf) evaluates the whole ln x ln block (kernel kinds)
    if (m.kind != GOFMM_DIST_GEOMETRIC)
      for (int li = 0; li < nl; ++li) o.count.fetch_add(int64_t(off[li + 1] - off[li]) * (off[li + 1] - off[li]));
    for (int i = 0; i < n; ++i) {
      tab.lists[i].resize(tl[i]);
      for (int t = 0; t < tl[i]; ++t) tab.lists[i][t] = {tj[size_t(i) * k + t], td[size_t(i) * k + t]};
    }
    return;
  }
  parallel_for(0, nl, cfg.c.threads, [&](int li) {
    const Node& nd = tr.nodes[tr.leaf_ids[li]];
    const int ln = nd.count();
    const int* leaf = tr.iperm.data() + nd.start;
    std::vector<double> d(size_t(ln) * ln);
    m.pairwise(leaf, ln, d.data());
    std::vector<Nbr> cand;
    for (int a = 0; a < ln; ++a) {
      cand.clear();
      cand.reserve(ln - 1);
      for (int b = 0; b < ln; ++b)
        if (b != a) cand.emplace_back(leaf[b], d[a + size_t(b) * ln]);
      merge_candidates(tab.lists[leaf[a]], cand, tab.k);
    }
  });
}

// neighbors.hpp:114-183 (recall against brute force on min(10, N) probes)
Table ann_search(const Metric& m, const Config& cfg, uint64_t seed, std::vector<double>& recall, double* kernel_ms) {
  const int n = m.size();
  Table tab;
  tab.k = std::min(cfg.c.kappa, n - 1);
  tab.lists.resize(n);
  const int recall_sample = 10;
  RefRng rng(seed, 0x7ec411);
  IndexList probe = rng.sample_without_replacement(n, std::min(recall_sample, n));
  std::vector<IndexList> exact(probe.size());
  IndexList all(n);
  std::iota(all.begin(), all.end(), 0);
  parallel_for(0, int(probe.size()), cfg.c.threads, [&](int t) {
    const int i = probe[t];
    std::vector<double> d(n);
    m.distances_from(i, all.data(), n, d.data());
    std::vector<Nbr> cand;
    cand.reserve(n - 1);
    for (int j = 0; j < n; ++j)
      if (j != i) cand.emplace_back(j, d[j]);
    std::partial_sort(cand.begin(), cand.begin() + tab.k, cand.end(), nbr_less);
    IndexList ids;
    for (int q = 0; q < tab.k; ++q) ids.push_back(cand[q].first);
    std::sort(ids.begin(), ids.end());
    exact[t] = std::move(ids);
  });
  for (int it = 0; it < cfg.c.ann_iterations; ++it) {
    ann_iteration(tab, m, cfg, splitmix64(seed) + uint64_t(it), kernel_ms);
    int64_t hit = 0, total = 0;
    for (size_t t = 0; t < probe.size(); ++t) {
      for (const Nbr& e : tab.lists[probe[t]])
        if (std::binary_search(exact[t].begin(), exact[t].end(), e.first)) ++hit;
      total += int64_t(exact[t].size());
    }
    recall.push_back(total ? double(hit) / double(total) : 1.0);
  }
  return tab;
}

// ---------------------------------------------------------------- interaction structure
// compress.hpp:85-144: greedy admission of leaf pairs by shared-neighbour count under budget*N^2
std::vector<std::pair<int, int>> select_near_field(const Tree& t, const Table& tab, double budget) {
  const int nl = int(t.leaf_ids.size()), n = int(t.perm.size());
  std::vector<std::pair<int, int>> out;
  if (nl < 2 || budget <= 0.0) return out;
  std::vector<int> leaf_of(n);
  for (int li = 0; li < nl; ++li) {
    const Node& nd = t.nodes[t.leaf_ids[li]];
    for (int q = nd.start; q < nd.end; ++q) leaf_of[t.iperm[q]] = li;
  }
  auto cnt = [&](int li) { return int64_t(t.nodes[t.leaf_ids[li]].count()); };
  const double cap = budget * double(n) * double(n);
  // total over all pairs: 2 * sum_{a<b} c_a c_b
  int64_t total_all = 0, pre = 0;
  for (int a = 0; a < nl; ++a) {
    total_all += 2 * cnt(a) * pre;
    pre += cnt(a);
  }
  auto emit = [&](int a, int b) {
    const int ia = t.leaf_ids[a], ib = t.leaf_ids[b];
    out.emplace_back(std::min(ia, ib), std::max(ia, ib));
  };
  if (double(total_all) <= cap) {
    for (int a = 0; a < nl; ++a)
      for (int b = a + 1; b < nl; ++b) emit(a, b);
    return out;
  }
  // score of every leaf-ordinal pair (a < b): count of (i, j in list(i)) with leaves {a, b}
  std::vector<uint64_t> keys;
  keys.reserve(size_t(n) * tab.k);
  for (int i = 0; i < n; ++i)
    for (const Nbr& e : tab.lists[i]) {
      const int a = leaf_of[i], b = leaf_of[e.first];
      if (a == b) continue;
      keys.push_back((uint64_t(std::min(a, b)) << 32) | uint64_t(std::max(a, b)));
    }
  std::sort(keys.begin(), keys.end());
  std::vector<std::pair<int64_t, uint64_t>> ranked;  // (score, pair key)
  for (size_t i = 0; i < keys.size();) {
    size_t j = i;
    while (j < keys.size() && keys[j] == keys[i]) ++j;
    ranked.push_back({int64_t(j - i), keys[i]});
    i = j;
  }
  std::stable_sort(ranked.begin(), ranked.end(), [](const auto& x, const auto& y) {
    if (x.first != y.first) return x.first > y.first;
    return x.second < y.second;  // pair ascending (a, then b)
  });
  int64_t used = 0;
  for (const auto& [sc, key] : ranked) {
    const int a = int(key >> 32), b = int(key & 0xffffffffu);
    const int64_t cost = 2 * cnt(a) * cnt(b);
    if (double(used + cost) > cap) continue;
    used += cost;
    emit(a, b);
  }
  std::sort(out.begin(), out.end());
  return out;
}

// compress.hpp:196-324 with crossed() from sorted per-leaf partner lists: (a, b) is crossed iff
// some admitted pair joins a leaf under a with a leaf under b (every admitted pair is visited
// through the smaller of the two leaf-ordinal ranges, each row by binary search)
struct Structure {
  std::vector<std::pair<int, int>> near, far;
};
Structure walk_structure(const Tree& t, const std::vector<std::pair<int, int>>& admitted) {
  const int nn = int(t.nodes.size()), nl = int(t.leaf_ids.size());
  std::vector<int> ord(nn, -1), lo(nn), hi(nn);
  for (int li = 0; li < nl; ++li) ord[t.leaf_ids[li]] = li;
  for (int i = nn - 1; i >= 0; --i) {  // children have larger ids (BFS)
    const Node& nd = t.nodes[i];
    if (nd.leaf()) {
      lo[i] = ord[i];
      hi[i] = ord[i] + 1;
    } else {
      lo[i] = lo[nd.left];
      hi[i] = hi[nd.right];
    }
  }
  std::vector<std::vector<int>> partners(nl);
  for (auto [a, b] : admitted) {
    const int x = ord[a], y = ord[b];
    partners[x].push_back(y);
    partners[y].push_back(x);
  }
  for (auto& p : partners) std::sort(p.begin(), p.end());
  std::vector<int> has(nl + 1, 0);  // prefix count of leaves with any partner
  for (int x = 0; x < nl; ++x) has[x + 1] = has[x] + (partners[x].empty() ? 0 : 1);
  auto crossed = [&](int a, int b) {
    int r0 = lo[a], r1 = hi[a], c0 = lo[b], c1 = hi[b];
    if (r1 - r0 > c1 - c0) {
      std::swap(r0, c0);
      std::swap(r1, c1);
    }
    if (has[r1] == has[r0] || has[c1] == has[c0]) return false;
    for (int x = r0; x < r1; ++x) {
      const auto& p = partners[x];
      if (p.empty()) continue;
      auto it = std::lower_bound(p.begin(), p.end(), c0);
      if (it != p.end() && *it < c1) return true;
    }
    return false;
  };
  Structure s;
  std::vector<std::pair<int, int>> stack;
  for (int i = 0; i < nn; ++i)
    if (!t.nodes[i].leaf()) stack.push_back({t.nodes[i].left, t.nodes[i].right});
  while (!stack.empty()) {
    auto [a, b] = stack.back();
    stack.pop_back();
    if (!crossed(a, b)) {
      s.far.emplace_back(std::min(a, b), std::max(a, b));
      continue;
    }
    const Node &na = t.nodes[a], &nb = t.nodes[b];
    if (na.leaf() && nb.leaf()) {
      s.near.emplace_back(std::min(a, b), std::max(a, b));
    } else if (na.leaf()) {
      stack.push_back({a, nb.left});
      stack.push_back({a, nb.right});
    } else if (nb.leaf()) {
      stack.push_back({na.left, b});
      stack.push_back({na.right, b});
    } else {
      stack.push_back({na.left, nb.left});
      stack.push_back({na.left, nb.right});
      stack.push_back({na.right, nb.left});
      stack.push_back({na.right, nb.right});
    }
  }
  std::sort(s.near.begin(), s.near.end());
  std::sort(s.far.begin(), s.far.end());
  return s;
}

// compress.hpp:191-229
IndexList sample_columns(const Tree& t, int id, const Table& tab, int n_samples, RefRng& rng) {
  const Node& nd = t.nodes[id];
  const int n = int(t.perm.size());
  const int outside = n - nd.count();
  if (outside == 0) return {};
  n_samples = std::min(n_samples, outside);
  auto in_node = [&](int o) {
    const int p = t.perm[o];
    return p >= nd.start && p < nd.end;
  };
  IndexList cols;
  std::unordered_set<int> seen;
  cols.reserve(n_samples);
  for (int q = nd.start; q < nd.end && int(cols.size()) < n_samples; ++q) {
    const int i = t.iperm[q];
    for (const Nbr& e : tab.lists[i]) {
      if (int(cols.size()) >= n_samples) break;
      if (in_node(e.first) || seen.count(e.first)) continue;
      seen.insert(e.first);
      cols.push_back(e.first);
    }
  }
  int attempts = 0;
  while (int(cols.size()) < n_samples && attempts < 100 * n_samples) {
    ++attempts;
    const int o = rng.uniform(n);
    if (in_node(o) || seen.count(o)) continue;
    seen.insert(o);
    cols.push_back(o);
  }
  if (int(cols.size()) < n_samples)
    for (int o = 0; o < n && int(cols.size()) < n_samples; ++o)
      if (!in_node(o) && !seen.count(o)) cols.push_back(o);
  return cols;
}

// ---------------------------------------------------------------- device sampled blocks
struct BlockDesc {
  int64_t out_off;           // column-major rows x cols block in the output blob
  int64_t row_off, col_off;  // into the concatenated sample / candidate index lists
  int32_t rows, cols;
};

// K(x[rows], x[cols]) of every node of a level, column-major, entries as the reference oracle
// computes them (kernel_entry: difference vector, Eigen reduction order, libdevice exp / pow).
// grid.x = node, grid.y = 32-column slab; one thread per row, the slab's column points in smem.
template <int KIND>
__global__ void __launch_bounds__(256) sampled_block_kernel(const BlockDesc* __restrict__ descs,
                                                            const int32_t* __restrict__ rows_idx,
                                                            const int32_t* __restrict__ cols_idx,
                                                            const double* __restrict__ x, KernelParams kp,
                                                            double* __restrict__ out) {
  const BlockDesc b = descs[blockIdx.x];
  const int c0 = blockIdx.y * 32;
  if (c0 >= b.cols) return;
  const int nc = min(32, b.cols - c0);
  const int dim = kp.dim;
  __shared__ double sx[32 * kMaxDimRt];
  for (int i = threadIdx.x; i < nc * dim; i += blockDim.x) {
    const int c = i / dim, q = i - c * dim;
    sx[c * kMaxDimRt + q] = x[int64_t(cols_idx[b.col_off + c0 + c]) * dim + q];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < b.rows; r += blockDim.x) {
    double xr[kMaxDimRt];
    const double* src = x + int64_t(rows_idx[b.row_off + r]) * dim;
    for (int q = 0; q < dim; ++q) xr[q] = src[q];
    double* o = out + b.out_off + r;
    for (int c = 0; c < nc; ++c) o[int64_t(c0 + c) * b.rows] = kernel_entry<KIND, 0>(xr, sx + c * kMaxDimRt, kp);
  }
}

struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevMem() {
    if (p) cudaFree(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, std::max<size_t>(b, 8));
    if (e != cudaSuccess) throw Error(GOFMM_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    bytes = b;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

#define CMP_CUDA(x)                                                                                    \
  do {                                                                                                 \
    const cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw Error(GOFMM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------- the result
struct Skel {
  IndexList skel;
  std::vector<double> proj;  // rank x cols column-major
  bool valid = false;
};

}  // namespace cmp
}  // namespace gofmm

struct gofmm_compressed {
  int32_t n = 0, dim = 0, kernel = 0;
  double kparam[4] = {0, 0, 0, 0};
  std::vector<double> coords;
  std::vector<int32_t> parent, left, right, level, start, end, iperm, rank, skel_idx, near_a, near_b, far_a, far_b;
  std::vector<int64_t> skel_off, proj_off;
  std::vector<double> proj;
  gofmm_compress_stats stats{};
};

namespace gofmm {
namespace cmp {

// compress.hpp:331-434
void compress(gofmm_compressed* R, const Oracle& o, const Config& cfg) {
  using clock = std::chrono::steady_clock;
  auto since = [](clock::time_point t0) { return std::chrono::duration<double>(clock::now() - t0).count(); };
  const auto t_total = clock::now();
  const gofmm_compress_config& c = cfg.c;
  gofmm_compress_stats& st = R->stats;
  Metric metric(c.distance, o);
  const int n = o.n;

  // neighbour search first, then the partitioning tree
  Table table;
  table.k = std::min(c.kappa, n - 1);
  table.lists.resize(n);
  std::vector<double> recall;
  const auto t_ann = clock::now();
  double ann_ms = 0.0;
  if (c.kappa > 0 && n > 1) table = ann_search(metric, cfg, splitmix64(c.seed ^ 0xa221), recall, &ann_ms);
  st.ann_seconds = since(t_ann);
  st.ann_kernel_ms = ann_ms;
  st.ann_iterations_done = int32_t(recall.size());
  for (size_t i = 0; i < recall.size() && i < 64; ++i) st.ann_recall[i] = recall[i];

  const auto t_tree = clock::now();
  Tree tree = build_tree(metric, c.m, c.seed, false, c.threads);
  st.tree_seconds = since(t_tree);

  const auto admitted = select_near_field(tree, table, c.budget);
  Structure structure = walk_structure(tree, admitted);

  // D and S blocks: evaluated matrix-free later; counted as the reference's CountingOracle does
  for (int id : tree.leaf_ids) o.count.fetch_add(int64_t(tree.nodes[id].count()) * tree.nodes[id].count());
  int64_t near_entries = 0;
  for (auto [a, b] : structure.near) {
    const int64_t e = int64_t(tree.nodes[a].count()) * tree.nodes[b].count();
    o.count.fetch_add(e);
    near_entries += 2 * e;
  }
  st.near_field_entries = near_entries;

  // skeletons, bottom-up by level; one GPU batch per level
  const int nn = int(tree.nodes.size());
  std::vector<Skel> sk(nn);
  std::vector<int64_t> node_flops(nn, 0);
  const int n_samples_target = std::min(n, 2 * c.s + 32);
  const auto t_skel = clock::now();
  double skel_ms = 0.0;
  DevMem d_blocks, d_desc, d_ri, d_ci, d_x;
  if (cfg.device_entries()) {
    d_x.ensure(size_t(o.n) * o.d * sizeof(double));
    CMP_CUDA(cudaMemcpy(d_x.p, o.x, size_t(o.n) * o.d * sizeof(double), cudaMemcpyHostToDevice));
  }
  for (int lev = tree.depth; lev >= 1; --lev) {
    std::vector<int> lnodes;
    for (const Node& nd : tree.nodes)
      if (nd.level == lev) lnodes.push_back(nd.id);
    const int L = int(lnodes.size());
    std::vector<IndexList> cand(L), cols(L);
    parallel_for(0, L, c.threads, [&](int t) {
      const int id = lnodes[t];
      const Node& nd = tree.nodes[id];
      if (nd.leaf()) {
        cand[t].assign(tree.iperm.begin() + nd.start, tree.iperm.begin() + nd.end);
      } else {
        const IndexList &ls = sk[nd.left].skel, &rs = sk[nd.right].skel;
        cand[t].reserve(ls.size() + rs.size());
        cand[t].insert(cand[t].end(), ls.begin(), ls.end());
        cand[t].insert(cand[t].end(), rs.begin(), rs.end());
      }
      RefRng rng(c.seed ^ 0x51e7, splitmix64(nd.path));
      cols[t] = sample_columns(tree, id, table, n_samples_target, rng);
    });
    // the level's blocks K(cols, cand), column-major, concatenated
    std::vector<gofmm_skel::NodeDesc> nd;
    std::vector<int> which;  // level slot of each batch entry
    int64_t off = 0;
    for (int t = 0; t < L; ++t) {
      if (cols[t].empty() || cand[t].empty()) continue;  // non-compressible (caller handles)
      nd.push_back({off, 0, 0, 0, int32_t(cols[t].size()), int32_t(cand[t].size())});
      which.push_back(t);
      off += int64_t(cols[t].size()) * int64_t(cand[t].size());
    }
    if (nd.empty()) continue;
    d_blocks.ensure(size_t(off) * sizeof(double));
    for (size_t q = 0; q < nd.size(); ++q) o.count.fetch_add(int64_t(nd[q].rows) * nd[q].cols);
    if (cfg.device_entries()) {
      std::vector<BlockDesc> bd;
      std::vector<int32_t> ri, ci;
      int maxc = 0;
      for (size_t q = 0; q < nd.size(); ++q) {
        const int t = which[q];
        bd.push_back({nd[q].in_off, int64_t(ri.size()), int64_t(ci.size()), nd[q].rows, nd[q].cols});
        ri.insert(ri.end(), cols[t].begin(), cols[t].end());
        ci.insert(ci.end(), cand[t].begin(), cand[t].end());
        maxc = std::max(maxc, nd[q].cols);
      }
      d_desc.ensure(bd.size() * sizeof(BlockDesc));
      d_ri.ensure(ri.size() * 4);
      d_ci.ensure(ci.size() * 4);
      CMP_CUDA(cudaMemcpy(d_desc.p, bd.data(), bd.size() * sizeof(BlockDesc), cudaMemcpyHostToDevice));
      CMP_CUDA(cudaMemcpy(d_ri.p, ri.data(), ri.size() * 4, cudaMemcpyHostToDevice));
      CMP_CUDA(cudaMemcpy(d_ci.p, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice));
      KernelParams kp{};
      kp.dim = o.d;
      if (o.kernel == GOFMM_KERNEL_GAUSSIAN) kp.p0 = 1.0 / (2.0 * o.p0 * o.p0);
      if (o.kernel == GOFMM_KERNEL_EXPONENTIAL) kp.p0 = 1.0 / o.p0;
      if (o.kernel == GOFMM_KERNEL_LAPLACE) {
        kp.p0 = o.p0;
        kp.p1 = double(o.d - 2);
      }
      if (o.kernel == GOFMM_KERNEL_POLYNOMIAL) {
        kp.p0 = o.p0;
        kp.p1 = double(int(o.p1));
      }
      dim3 grid(unsigned(bd.size()), unsigned((maxc + 31) / 32));
      const BlockDesc* dd = d_desc.as<BlockDesc>();
      const int32_t *dri = d_ri.as<int32_t>(), *dci = d_ci.as<int32_t>();
      const double* dx = d_x.as<double>();
      double* db = d_blocks.as<double>();
      switch (o.kernel) {
        case GOFMM_KERNEL_GAUSSIAN: sampled_block_kernel<kGaussian><<<grid, 256>>>(dd, dri, dci, dx, kp, db); break;
        case GOFMM_KERNEL_EXPONENTIAL:
          sampled_block_kernel<kExponential><<<grid, 256>>>(dd, dri, dci, dx, kp, db);
          break;
        case GOFMM_KERNEL_LAPLACE: sampled_block_kernel<kLaplace><<<grid, 256>>>(dd, dri, dci, dx, kp, db); break;
        default: sampled_block_kernel<kPolynomial><<<grid, 256>>>(dd, dri, dci, dx, kp, db); break;
      }
      CMP_CUDA(cudaGetLastError());
    } else {
      std::vector<double> hb(static_cast<size_t>(off));
      parallel_for(0, int(nd.size()), c.threads, [&](int q) {
        const int t = which[q];
        for (int cc = 0; cc < nd[q].cols; ++cc)
          for (int r = 0; r < nd[q].rows; ++r)
            hb[size_t(nd[q].in_off) + r + size_t(cc) * nd[q].rows] = o.raw(cols[t][r], cand[t][cc]);
      });
      CMP_CUDA(cudaMemcpy(d_blocks.p, hb.data(), size_t(off) * sizeof(double), cudaMemcpyHostToDevice));
    }
    const int B = int(nd.size());
    std::vector<int32_t> rank(B);
    std::vector<double> ach(B), lead(B);
    int64_t pe = 0, pj = 0;
    for (const auto& q : nd) {
      pe += q.cols;
      pj += int64_t(std::min({c.s, q.rows, q.cols})) * q.cols;
    }
    std::vector<int32_t> perm(size_t(std::max<int64_t>(pe, 1)));
    std::vector<double> proj(size_t(std::max<int64_t>(pj, 1)));
    float ms = 0.f;
    std::string err;
    const int rc = gofmm_skel::skel_device(nd, d_blocks.as<double>(), c.s, c.tau, rank.data(), ach.data(), lead.data(),
                                           perm.data(), proj.data(), &ms, &err);
    if (rc != GOFMM_OK) throw Error(rc, err);
    skel_ms += ms;
    for (int q = 0; q < B; ++q) {
      const int t = which[q], id = lnodes[t];
      const int rows = nd[q].rows, cc = nd[q].cols, k = rank[q];
      Skel& s = sk[id];
      s.valid = true;
      s.skel.resize(k);
      const int32_t* pm = perm.data() + nd[q].perm_off;
      for (int l = 0; l < k; ++l) s.skel[l] = cand[t][pm[l]];
      s.proj.assign(proj.begin() + nd[q].proj_off, proj.begin() + nd[q].proj_off + int64_t(k) * cc);
      int64_t f = 4LL * rows * cc * std::min(rows, cc);
      if (cc > k && lead[q] > 0.0) f += 1LL * k * k * (cc - k);
      node_flops[id] = f;
    }
  }
  st.skeleton_seconds = since(t_skel);
  st.skel_kernel_ms = skel_ms;
  for (int64_t f : node_flops) st.compress_flops += f;

  // UV coupling blocks K(skel a, skel b): counted, regenerated by the evaluator
  for (auto [a, b] : structure.far) o.count.fetch_add(int64_t(sk[a].skel.size()) * sk[b].skel.size());

  // flattened HMatrix (gofmm_tree_desc layout)
  R->parent.resize(nn);
  R->left.resize(nn);
  R->right.resize(nn);
  R->level.resize(nn);
  R->start.resize(nn);
  R->end.resize(nn);
  R->rank.resize(nn);
  R->skel_off.assign(nn + 1, 0);
  R->proj_off.assign(nn + 1, 0);
  int64_t rank_sum = 0;
  int nsk = 0;
  for (int i = 0; i < nn; ++i) {
    const Node& nd = tree.nodes[i];
    R->parent[i] = nd.parent;
    R->left[i] = nd.left;
    R->right[i] = nd.right;
    R->level[i] = nd.level;
    R->start[i] = nd.start;
    R->end[i] = nd.end;
    R->rank[i] = sk[i].valid ? int32_t(sk[i].skel.size()) : -1;
    if (sk[i].valid) {
      R->skel_idx.insert(R->skel_idx.end(), sk[i].skel.begin(), sk[i].skel.end());
      R->proj.insert(R->proj.end(), sk[i].proj.begin(), sk[i].proj.end());
      rank_sum += int64_t(sk[i].skel.size());
      st.max_skeleton = std::max<int32_t>(st.max_skeleton, int32_t(sk[i].skel.size()));
      ++nsk;
    }
    R->skel_off[i + 1] = int64_t(R->skel_idx.size());
    R->proj_off[i + 1] = int64_t(R->proj.size());
  }
  st.mean_skeleton = nsk ? double(rank_sum) / nsk : 0.0;
  R->iperm.assign(tree.iperm.begin(), tree.iperm.end());
  for (auto [a, b] : structure.near) {
    R->near_a.push_back(a);
    R->near_b.push_back(b);
  }
  for (auto [a, b] : structure.far) {
    R->far_a.push_back(a);
    R->far_b.push_back(b);
  }
  st.entries_evaluated = o.count.load();
  st.depth = tree.depth;
  st.num_nodes = nn;
  st.num_leaves = int32_t(tree.leaf_ids.size());
  st.num_near = int64_t(structure.near.size());
  st.num_far = int64_t(structure.far.size());
  st.compress_seconds = since(t_total);
}

}  // namespace cmp
}  // namespace gofmm

extern "C" {

const char* gofmm_compress_last_error(void) { return gofmm::cmp::g_err.c_str(); }

void gofmm_compress_default_config(gofmm_compress_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  // RunConfig defaults (compress.hpp:12-34)
  c->m = 256;
  c->s = 256;
  c->tau = 1e-5;
  c->kappa = 32;
  c->budget = 0.03;
  c->distance = GOFMM_DIST_KERNEL;
  c->seed = 0;
  c->ann_iterations = 10;
  c->threads = int32_t(std::max(1u, std::thread::hardware_concurrency()));
  c->entries = GOFMM_ENTRIES_DEVICE;
  c->device = 0;
}

int gofmm_compress(int32_t kernel, const double* kparam, int32_t dim, int32_t n, const double* coords,
                   const gofmm_compress_config* config, gofmm_compressed** out) {
  using namespace gofmm::cmp;
  try {
    if (!out || !coords || !kparam || !config) throw Error(GOFMM_ERR_INVALID, "compress: null argument");
    *out = nullptr;
    const gofmm_compress_config& c = *config;
    // RunConfig::validate (compress.hpp:24-33)
    if (c.m < 1) throw Error(GOFMM_ERR_INVALID, "m must be >= 1");
    if (c.s < 1 || c.s > c.m) throw Error(GOFMM_ERR_INVALID, "s must satisfy 1 <= s <= m");
    if (!(c.tau > 0)) throw Error(GOFMM_ERR_INVALID, "tau must be positive");
    if (c.kappa < 0) throw Error(GOFMM_ERR_INVALID, "kappa must be >= 0");
    if (c.budget < 0 || c.budget > 1) throw Error(GOFMM_ERR_INVALID, "budget must be in [0, 1]");
    if (c.ann_iterations < 1) throw Error(GOFMM_ERR_INVALID, "ann iterations must be >= 1");
    if (c.threads < 1) throw Error(GOFMM_ERR_INVALID, "threads must be >= 1");
    if (n < 1 || dim < 1 || dim > gofmm::kMaxDimRt) throw Error(GOFMM_ERR_INVALID, "compress: need n >= 1, 1 <= d <= 16");
    if (c.distance != GOFMM_DIST_GEOMETRIC && c.distance != GOFMM_DIST_KERNEL && c.distance != GOFMM_DIST_ANGLE)
      throw Error(GOFMM_ERR_INVALID, "compress: unknown distance kind");
    if (c.entries != GOFMM_ENTRIES_HOST && c.entries != GOFMM_ENTRIES_DEVICE)
      throw Error(GOFMM_ERR_INVALID, "compress: entries must be GOFMM_ENTRIES_HOST or _DEVICE");
    if (kernel == GOFMM_KERNEL_GAUSSIAN && !(kparam[0] > 0))
      throw Error(GOFMM_ERR_INVALID, "gaussian bandwidth must be positive");
    if (kernel == GOFMM_KERNEL_EXPONENTIAL && !(kparam[0] > 0))
      throw Error(GOFMM_ERR_INVALID, "exponential bandwidth must be positive");
    if (kernel == GOFMM_KERNEL_LAPLACE && kparam[0] < 0) throw Error(GOFMM_ERR_INVALID, "laplace regularization must be >= 0");
    if (kernel == GOFMM_KERNEL_POLYNOMIAL && kparam[1] < 1) throw Error(GOFMM_ERR_INVALID, "polynomial degree must be >= 1");
    if (kernel != GOFMM_KERNEL_GAUSSIAN && kernel != GOFMM_KERNEL_EXPONENTIAL && kernel != GOFMM_KERNEL_LAPLACE &&
        kernel != GOFMM_KERNEL_POLYNOMIAL)
      throw Error(GOFMM_ERR_INVALID, "unsupported kernel id");
    for (int64_t i = 0; i < int64_t(n) * dim; ++i)
      if (!std::isfinite(coords[i])) throw Error(GOFMM_ERR_INVALID, "point cloud has non-finite coordinates");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(GOFMM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    CMP_CUDA(cudaSetDevice(c.device));
    auto R = std::make_unique<gofmm_compressed>();
    R->n = n;
    R->dim = dim;
    R->kernel = kernel;
    R->kparam[0] = kparam[0];
    R->kparam[1] = kparam[1];
    R->coords.assign(coords, coords + int64_t(n) * dim);
    Oracle o;
    o.kernel = kernel;
    o.d = dim;
    o.n = n;
    o.x = R->coords.data();
    o.p0 = kparam[0];
    o.p1 = kparam[1];
    Config cfg{c};
    compress(R.get(), o, cfg);
    *out = R.release();
    g_err.clear();
    return GOFMM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code == GOFMM_ERR_NUMERIC + 100 ? GOFMM_ERR_NUMERIC : e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return GOFMM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GOFMM_ERR_INVALID;
  }
}

int gofmm_compressed_desc(const gofmm_compressed* R, gofmm_tree_desc* d) {
  if (!R || !d) return GOFMM_ERR_INVALID;
  std::memset(d, 0, sizeof(*d));
  d->n = R->n;
  d->num_nodes = int32_t(R->parent.size());
  d->parent = R->parent.data();
  d->left = R->left.data();
  d->right = R->right.data();
  d->level = R->level.data();
  d->start = R->start.data();
  d->end = R->end.data();
  d->iperm = R->iperm.data();
  d->rank = R->rank.data();
  d->skel_offset = R->skel_off.data();
  d->skel_idx = R->skel_idx.data();
  d->proj_offset = R->proj_off.data();
  d->proj = R->proj.data();
  d->num_near = int64_t(R->near_a.size());
  d->near_a = R->near_a.data();
  d->near_b = R->near_b.data();
  d->num_far = int64_t(R->far_a.size());
  d->far_a = R->far_a.data();
  d->far_b = R->far_b.data();
  d->source = GOFMM_SOURCE_KERNEL;
  d->kernel = R->kernel;
  d->dim = R->dim;
  d->coords = R->coords.data();
  for (int i = 0; i < 4; ++i) d->kparam[i] = R->kparam[i];
  return GOFMM_OK;
}

int gofmm_compressed_stats(const gofmm_compressed* R, gofmm_compress_stats* s) {
  if (!R || !s) return GOFMM_ERR_INVALID;
  *s = R->stats;
  return GOFMM_OK;
}

int gofmm_compressed_free(gofmm_compressed* R) {
  delete R;
  return GOFMM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- point sources (CLI inputs)
extern "C" {

// PointCloud::random_gaussian (oracle.hpp:18-25): Rng(seed, 0x9f), point j outer, dimension i inner.
int gofmm_points_gaussian(int32_t n, int32_t d, uint64_t seed, double* out) {
  if (n < 1 || d < 1 || !out) {
    gofmm::cmp::g_err = "points: need n >= 1, d >= 1 and an output buffer";
    return GOFMM_ERR_INVALID;
  }
  gofmm::RefRng rng(seed, 0x9f);
  for (int64_t j = 0; j < n; ++j)
    for (int i = 0; i < d; ++i) out[j * d + i] = rng.gauss();
  return GOFMM_OK;
}

// Rng(seed, stream).gauss() column-major into w (n x r, ld ldw): the bench RHS of the CLI,
// Rng(cfg.seed, 0xbe7c) (gfmm_cli.cpp:195-198), and the tests' Rng(seed, 0) RHS.
int gofmm_rng_gauss_stream(uint64_t seed, uint64_t stream, int32_t n, int32_t r, double* w, int64_t ldw) {
  if (n < 1 || r < 1 || !w || ldw < n) {
    gofmm::cmp::g_err = "rng: bad arguments";
    return GOFMM_ERR_INVALID;
  }
  gofmm::RefRng rng(seed, stream);
  for (int64_t c = 0; c < r; ++c)
    for (int64_t i = 0; i < n; ++i) w[i + c * ldw] = rng.gauss();
  return GOFMM_OK;
}

// default_laplace_floor (oracle.hpp:274-288): 1e-3 x the median pairwise distance of a 100-point
// sample drawn from Rng(seed, 0x1ap1) (the hex-float literal is 52.0 -> stream 52); distances as the
// reference computes them ((xa - xb).norm(): Eigen's packet reduction of the squares, then sqrt).
int gofmm_default_laplace_floor(int32_t d, int32_t n, const double* coords, uint64_t seed, double* out) {
  using gofmm::cmp::redux_packet;
  if (n < 1 || d < 1 || !coords || !out) {
    gofmm::cmp::g_err = "laplace floor: bad arguments";
    return GOFMM_ERR_INVALID;
  }
  gofmm::RefRng rng(seed, 52);
  const std::vector<int> sample = rng.sample_without_replacement(n, std::min(n, 100));
  std::vector<double> dists;
  for (size_t a = 0; a < sample.size(); ++a)
    for (size_t b = a + 1; b < sample.size(); ++b) {
      const double* xa = coords + int64_t(sample[a]) * d;
      const double* xb = coords + int64_t(sample[b]) * d;
      dists.push_back(std::sqrt(redux_packet(d, [&](int64_t q) {
        const double e = xa[q] - xb[q];
        return e * e;
      })));
    }
  if (dists.empty()) {
    *out = 1e-3;
    return GOFMM_OK;
  }
  auto mid = dists.begin() + dists.size() / 2;
  std::nth_element(dists.begin(), mid, dists.end());
  *out = 1e-3 * *mid;
  return GOFMM_OK;
}

}  // extern "C"
