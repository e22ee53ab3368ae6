// gofmm_capi.cu — host side of the B200-native GOFMM evaluation phase behind include/gofmm_b200.h.
//
// Replaces the reference executor (evaluate.hpp:52-120 traversal_schedule, :222-281
// execute_levels / execute_dag, common.hpp:109-126 parallel_for) with a plan built ONCE at
// gofmm_create over a device-resident flattened tree, executed as level-synchronous launches
// on one stream:
//     permute W (K5)  ->  N2S levels depth..1  ->  DOWNWARD levels 1..depth  ->  OUTPUT
// Each launch is the grouped multi-term FP64 DMMA GEMM of gofmm_kernels.cuh.
//
// HBM layout (all FP64):
//   point space    : leaves left-to-right, leaf a at rows [pst_a, pst_a + pad16(n_a)); W_perm and
//                    the permuted coordinates live here (padding rows are zero)
//   skeleton space : nodes in BFS id order (== level order), node a at rows
//                    [soff_a, soff_a + pad16(k_a)); what (N2S output) and c (downward) live here.
//                    Siblings are adjacent, so [what_l; what_r] is one contiguous row range.
//   W_perm / what / c are stored in 16-ROW PANELS: panel p holds rows [16p, 16p+16) of all r_ws
//                    columns contiguously (element (i, j) at (i/16)*16*r_ws + 16*j + i%16), so a
//                    TMA box of 16 rows x BN columns is one contiguous 128*BN-byte run — a plain
//                    column-major N x r layout would make every box touch BN 2 MB pages.
//   proj_a         : k_a x ncand_pad column-major, ld = pad2(k_a); interior proj gets zero
//                    columns so [child l; child r] candidates line up with skeleton space.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gofmm_b200.h"
#include "gofmm_kernels.cuh"
#include "gofmm_kernels_f32.cuh"
#include "gofmm_rng.h"
#include "nccl_dyn.h"

namespace gofmm {
namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GOFMM_CUDA(x)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw Error(GOFMM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
  } while (0)

inline int64_t pad2(int64_t x) { return (x + 1) & ~int64_t(1); }
// point / skeleton space rows are padded to 16 so every node starts a 16-row panel (one TMA box)
inline int64_t pad16(int64_t x) { return (x + 15) & ~int64_t(15); }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b, bool zero = true) {
    release();
    if (b == 0) return;
    GOFMM_CUDA(cudaMalloc(&p, b));
    bytes = b;
    if (zero) GOFMM_CUDA(cudaMemset(p, 0, b));
  }
  template <class T>
  void upload(const std::vector<T>& v) {
    alloc(v.size() * sizeof(T), false);
    if (!v.empty()) GOFMM_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ---------------------------------------------------------------- kernel configurations
// S: stored-operand GEMMs (N2S / downward / output without generation): 128x128 CTA tile,
//    8 consumer warps of 32x64.
// G: generated-operand GEMMs (matrix-free L2L and S2S), r <= 256: 64x256 CTA tile, 16 consumer
//    warps of 16x64. Every A entry is generated once per CTA and amortised over BN columns.
// GW: the same for r > 256: 32x512 CTA tile (two 256-column TMA boxes per stage), 16 warps of
//    32x32, 3 stages. Same accumulator registers per warp as G, but each generated entry feeds
//    512 columns instead of 256: entry generation (FP64 ops on the pipe the DMMAs use) halves per
//    flop (c3: 75.1% -> 81.3% of the FP64 peak); the 32x32 warp tile needs 8 fragment loads per
//    16 DMMAs instead of 10 (-> 82.5%; the same change slows G down).
constexpr int kStagesS = 5, kStagesG = 5, kBM_S = 128, kBN_S = 128, kBM_G = 64, kBN_G = 256;
constexpr int kStagesGW = 3, kBM_GW = 32, kBN_GW = 512;
// GN64 / GN128: the same 64-row tiles for r <= 64 / r <= 128 (config 1: r = 64), so no CTA
// multiplies zero columns and each k-stage is 4x / 2x shorter along the serial term chain.
#define CFG_S kBM_S, kBN_S, 4, 4, kStagesS
#define CFG_G kBM_G, kBN_G, 4, 4, kStagesG
#define CFG_GW kBM_GW, kBN_GW, 1, 16, kStagesGW
#define CFG_GN64 kBM_G, 64, 4, 4, kStagesG
#define CFG_GN128 kBM_G, 128, 4, 4, kStagesG
// GN64W: 32-row tiles for r <= 64 — twice the CTAs and half the stage of GN64 for the
// latency-bound upper levels (config 1: 16-64 groups per level, chains of up to 80 stages)
#define CFG_GN64W kBM_GW, 64, 2, 8, kStagesG
// GM: generated operands, 128 < r <= 256 in 32-row tiles (GW's warp tile shape at half the width)
#define CFG_GM kBM_GW, kBN_G, 1, 16, kStagesG
// SN64: stored operands for r <= 64 (64x64 tiles: twice the CTAs of S, no idle columns)
#define CFG_SN64 kBM_G, 64, 4, 4, kStagesS
constexpr int kBM[3] = {kBM_S, kBM_G, kBM_GW};  // tile-row classes of the FP64 tile lists
// per-CTA fixed cost in the launch-config model, in tile-area x k-stage units (one 128x128 stage)
constexpr double kCtaOverheadArea = double(kBM_S) * kBN_S / 0.8;
constexpr int kThreadsG = kProducerThreads + kConsumerThreads;  // every FP64 config: producer WG + 16 consumer warps

using KernelFn = void (*)(BMaps, const Tile*, const Group*, const Term*, int32_t, KernelParams, double*, int64_t,
                          int32_t, int32_t);

struct GenKernel {
  KernelFn fn, fn_wide, fn_n64, fn_n128, fn_n64w, fn_m;
  size_t smem, smem_wide, smem_n64, smem_n128, smem_n64w, smem_m;
};

template <int KIND, int DIM>
GenKernel gen_kernel() {
  return {&grouped_gemm_f64<CFG_G, KIND, DIM>,           &grouped_gemm_f64<CFG_GW, KIND, DIM>,
          &grouped_gemm_f64<CFG_GN64, KIND, DIM>,        &grouped_gemm_f64<CFG_GN128, KIND, DIM>,
          &grouped_gemm_f64<CFG_GN64W, KIND, DIM>,       &grouped_gemm_f64<CFG_GM, KIND, DIM>,
          gemm_smem_bytes<CFG_G, KIND, DIM>(),           gemm_smem_bytes<CFG_GW, KIND, DIM>(),
          gemm_smem_bytes<CFG_GN64, KIND, DIM>(),        gemm_smem_bytes<CFG_GN128, KIND, DIM>(),
          gemm_smem_bytes<CFG_GN64W, KIND, DIM>(),       gemm_smem_bytes<CFG_GM, KIND, DIM>()};
}

// wide generated tiles (32 x 512) once the chunk has more than 256 columns
inline bool use_wide(int32_t r) { return r > kBN_G; }

GenKernel pick_gen_kernel(int kind, int dim) {
#define GOFMM_DIMS(K)                        \
  switch (dim) {                             \
    case 1: return gen_kernel<K, 1>();       \
    case 2: return gen_kernel<K, 2>();       \
    case 3: return gen_kernel<K, 3>();       \
    case 4: return gen_kernel<K, 4>();       \
    case 6: return gen_kernel<K, 6>();       \
    case 8: return gen_kernel<K, 8>();       \
    default: return gen_kernel<K, 0>();      \
  }
  switch (kind) {
    case kGaussian: GOFMM_DIMS(kGaussian)
    case kLaplace: GOFMM_DIMS(kLaplace)
    case kPolynomial: GOFMM_DIMS(kPolynomial)
    case kExponential: GOFMM_DIMS(kExponential)
  }
#undef GOFMM_DIMS
  throw Error(GOFMM_ERR_INVALID, "unsupported kernel id " + std::to_string(kind));
}

// TMA descriptor encoding through the runtime's driver entry point (no libcuda link needed)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    GOFMM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(GOFMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// B operand view of a panel-layout FP64 buffer (rows x r used columns, r_ws allocated): a 3D
// tensor {16 rows-in-panel, r columns, rows/16 panels}; boxes of 16 x bn x 1, 128-byte swizzle
// (conflict-free fragment loads); columns >= r read as zero.
void encode_bmap(CUtensorMap* map, const double* ptr, int64_t rows, int32_t r, int32_t r_ws, int bn) {
  cuuint64_t dims[3] = {16, cuuint64_t(r), cuuint64_t(rows / 16)};
  cuuint64_t strides[2] = {16 * sizeof(double), cuuint64_t(r_ws) * 16 * sizeof(double)};
  cuuint32_t box[3] = {16, cuuint32_t(bn), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult rc = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw Error(GOFMM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(rc)));
}

// A operand of one stored-A term for TMA (kernels: kABoxRow / kABoxCol): exact extents M x K, so
// every box column / row beyond the block reads as zero (partial m-tiles, the last k-stage).
//   row-major A[m][k] = a[k + m*lda]: dims {K, M}, box {16, kABoxRow}, 128B swizzle
//   column-major A[m][k] = a[m + k*lda]: dims {M, K}, box {kABoxCol, 16}, 64B swizzle
void encode_amap(CUtensorMap* map, const double* a, int64_t lda, int M, int K, bool row_major) {
  cuuint64_t dims[2] = {cuuint64_t(row_major ? K : M), cuuint64_t(row_major ? M : K)};
  cuuint64_t strides[1] = {cuuint64_t(lda) * sizeof(double)};
  cuuint32_t box[2] = {row_major ? 16u : cuuint32_t(kABoxCol), row_major ? cuuint32_t(kABoxRow) : 16u};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a), dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     row_major ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw Error(GOFMM_ERR_CUDA, "cuTensorMapEncodeTiled (A) failed: " + std::to_string(int(rc)));
}

// FP32 stored A (K-major hi / lo copies, A[m][k] = a[k + m*lda]): dims {K, M}, box {16, 128}
// (one UMMA K-major SWIZZLE_64B tile, the layout the A producers write for generated terms).
void encode_amap32(CUtensorMap* map, const float* a, int64_t lda, int M, int K) {
  cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(M)};
  cuuint64_t strides[1] = {cuuint64_t(lda) * sizeof(float)};
  cuuint32_t box[2] = {16u, 128u};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw Error(GOFMM_ERR_CUDA, "cuTensorMapEncodeTiled (A32) failed: " + std::to_string(int(rc)));
}

template <int KIND, int DIM>
void launch_generate(const double* xr, int rows, const double* xc, int cols, double* out, int64_t ld,
                     const KernelParams& kp, cudaStream_t st) {
  dim3 grid((rows + 127) / 128, cols);
  generate_block<KIND, DIM><<<grid, 128, 0, st>>>(xr, rows, xc, cols, out, ld, kp);
}

void generate_dispatch(int kind, int dim, const double* xr, int rows, const double* xc, int cols, double* out,
                       int64_t ld, const KernelParams& kp, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
#define GOFMM_GEN(K)                                                      \
  switch (dim) {                                                          \
    case 3: launch_generate<K, 3>(xr, rows, xc, cols, out, ld, kp, st); return; \
    case 8: launch_generate<K, 8>(xr, rows, xc, cols, out, ld, kp, st); return; \
    default: launch_generate<K, 0>(xr, rows, xc, cols, out, ld, kp, st); return; \
  }
  switch (kind) {
    case kGaussian: GOFMM_GEN(kGaussian)
    case kLaplace: GOFMM_GEN(kLaplace)
    case kPolynomial: GOFMM_GEN(kPolynomial)
    case kExponential: GOFMM_GEN(kExponential)
  }
#undef GOFMM_GEN
  throw Error(GOFMM_ERR_INVALID, "unsupported kernel id " + std::to_string(kind));
}

// ---------------------------------------------------------------- plan
// SM count the split of long downward term chains is sized for (B200: 148). A constant, so the
// summation order of the result does not depend on the device (see build()).
constexpr int kSplitRefSms = 148;

enum class Buf { Wp, What, C, Out };  // B operand / output bases (resolved per workspace)

struct HostTerm {
  int kind;         // 0 stored A, 1 generated
  bool row_major;   // stored A is accessed transposed
  int64_t a_off;    // offset (doubles) into the A blob (blob id below)
  int a_blob;       // 0 proj, 1 diag, 2 near, 3 far
  int64_t lda;
  Buf b_buf;
  int64_t b_row;    // row offset within the B buffer
  int K;
  int64_t xr_off, xc_off;  // generated: point offsets (in points) into coordinate blob
  int x_blob;              // 0 point space (Xp), 1 skeleton space (Xs)
};

struct HostGroup {
  int64_t c_row;
  int M;
  std::vector<HostTerm> terms;
  int flags = 0;  // kGroupLoadC: continue the chain a previous launch left in C
};

struct Launch {
  // FP64 tile lists of this launch's groups, one per tile-row class: kBM[c] rows per tile
  int tfirst[3] = {0, 0, 0}, tn[3] = {0, 0, 0};
  // k-stages (16-deep) of the tiles' term chains: sum over each tile list, and the longest chain
  int64_t chain_sum[3] = {0, 0, 0};
  int64_t chain_max = 0;
  bool gen = false;  // G config (generated operands present)
  Buf out;
  int phase;  // 0 upward, 1 downward, 2 output
  int level;  // tree level (output launch: -1)
  int64_t flops_per_rhs = 0;  // reference-counted flops of this launch per RHS column
  // distributed evaluation: 1 = before the all-gather (own-subtree N2S), 2 = after it, 3 = the
  // own leaves' D + near output terms, which need no exchanged data and run during the all-gather
  int stage = 2;
  int first_group = 0, ngroups = 0;      // groups [first_group, first_group + ngroups)
  int reduce_first = 0, reduce_n = 0;    // split-chain reductions after this launch (chain_reduce)
  int first_tile32 = 0, ntiles32 = 0;    // FP32 plan: 128-row tiles of the same groups
  int64_t chain_sum32 = 0, chain_max32 = 0;  // k-stages over / longest chain of its FP32 tiles
  // output launch of a host-buffer evaluation: split into row-contiguous parts so the D2H of a
  // part's u rows overlaps the next part's kernel. parts[p] = first tile of part p in each tile
  // list and the u_perm rows it completes; parts.back() is the end sentinel. Empty = no split.
  struct Part {
    int tile[3], tile32;
    int64_t row;
  };
  std::vector<Part> parts;
};

constexpr int kOutParts = 8;
static_assert(kOutParts <= 8, "per-part D2H timing events (gofmm_handle::dpev)");

// the part boundaries of an output launch: groups split into kOutParts runs of leaves; valid only
// if consecutive runs cover consecutive u_perm rows (leaves in left-to-right order)
template <class GroupVec, class TileVec>
void split_output_parts(Launch& L, const GroupVec& groups, const TileVec& tiles) {
  L.parts.clear();
  if (L.ngroups < kOutParts) return;
  int64_t expect = -1;
  std::vector<Launch::Part> parts;
  for (int p = 0; p <= kOutParts; ++p) {
    const int gb = L.first_group + int(int64_t(L.ngroups) * p / kOutParts);
    Launch::Part q{};
    auto first_of = [&](int t0, int nt) {
      int t = t0;
      while (t < t0 + nt && tiles[t].group < gb) ++t;
      return t;
    };
    for (int c = 0; c < 3; ++c) q.tile[c] = first_of(L.tfirst[c], L.tn[c]);
    q.tile32 = 0;
    q.row = (p < kOutParts) ? groups[gb].c_row : expect;
    if (p < kOutParts) {
      const int ge = L.first_group + int(int64_t(L.ngroups) * (p + 1) / kOutParts);
      int64_t row = groups[gb].c_row;
      if (expect >= 0 && row != expect) return;  // not row-contiguous: no split
      for (int g = gb; g < ge; ++g) {
        if (groups[g].c_row != row) return;
        row += std::max(groups[g].M, 0);
      }
      expect = row;
    }
    parts.push_back(q);
  }
  L.parts = std::move(parts);
}

// Longest-first order of a launch's tiles (ranges [b, e) of a tile list): the block scheduler
// hands out CTAs roughly in index order, so the long term chains (up to 460 k-stages at c2's leaf
// level vs a mean of 200) start first instead of forming the launch's tail. Ranges are the
// output parts (each part must stay row-contiguous) or the whole list.
template <class GroupVec>
void order_longest_first(std::vector<Tile>& tiles, int b, int e, const GroupVec& groups) {
  std::vector<std::pair<int64_t, Tile>> v;
  v.reserve(size_t(std::max(e - b, 0)));
  for (int i = b; i < e; ++i) {
    int64_t w = 0;
    for (const auto& term : groups[tiles[i].group].terms) w += (term.K + 15) / 16;
    v.push_back({w, tiles[i]});
  }
  std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  for (int i = b; i < e; ++i) tiles[i] = v[size_t(i - b)].second;
}

// ---------------------------------------------------------------- subtree-split distribution
// north_star (4): for P = 2^l GPUs the tree is split into subtrees at level s = l + up to
// kSplitExtra, and rank g owns a contiguous, work-balanced run of them (make_dist_plan); nodes
// above level s ("top") are evaluated redundantly by every rank. One all-gather per evaluation
// exchanges, from every rank, the skeleton weights (what) other ranks need (all level-s nodes
// for the top N2S, plus far-field
// partners across subtrees) and the W rows of leaves that are near-field partners across
// subtrees. Everything below is pure host logic over the flattened tree.
struct Seg {
  int32_t buf;   // 0 = what (skeleton space), 1 = W_perm (point space)
  int64_t row;   // first row (16-aligned)
  int64_t rows;  // multiple of 16
};

struct DistPlan {
  int nranks = 1, split = 0;
  std::vector<int32_t> owner;              // -1 = top (replicated)
  std::vector<std::vector<Seg>> exports;   // per rank, in send-buffer order
  std::vector<int64_t> send_rows;          // per rank
  int64_t max_send_rows = 0;
};

inline int64_t pad16_(int64_t x) { return (x + 15) & ~int64_t(15); }

// levels below log2(P) the subtree split may go for load balance (more, smaller subtrees per rank;
// everything above the split is replicated on every rank)
constexpr int kSplitExtra = 3;

DistPlan make_dist_plan(int nranks, int nn, const int32_t* left, const int32_t* right, const int32_t* level,
                        const int32_t* start, const int32_t* end, const int32_t* rank, int64_t n_near,
                        const int32_t* near_a, const int32_t* near_b, int64_t n_far, const int32_t* far_a,
                        const int32_t* far_b) {
  DistPlan P;
  P.nranks = nranks;
  if (nranks < 1 || (nranks & (nranks - 1)))
    throw Error(GOFMM_ERR_INVALID, "the number of ranks must be a power of two");
  int l = 0;
  while ((1 << l) < nranks) ++l;
  // every node above the split must be interior (no leaf above level l)
  int min_leaf_level = 1 << 30;
  for (int i = 0; i < nn; ++i)
    if (left[i] < 0) min_leaf_level = std::min(min_leaf_level, int(level[i]));
  if (min_leaf_level < l) throw Error(GOFMM_ERR_INVALID, "tree too shallow for " + std::to_string(nranks) + " ranks");
  // Load balance: the split goes up to kSplitExtra levels deeper than log2(P) (tree permitting),
  // and each rank owns a CONTIGUOUS run of those subtrees (left to right, so its rows stay one
  // range) chosen to minimise the largest per-rank work. The work of a subtree is the reference
  // flop counter of the tasks whose output it owns (evaluate.hpp:154-214, per RHS column).
  const int extra = nranks > 1 ? std::min(kSplitExtra, min_leaf_level - l) : 0;
  const int ls = l + extra;
  P.split = ls;
  std::vector<int> at_split;
  for (int i = 0; i < nn; ++i)
    if (level[i] == ls) at_split.push_back(i);
  std::sort(at_split.begin(), at_split.end(), [&](int x, int y) { return start[x] < start[y]; });
  if (int(at_split.size()) != (1 << ls)) throw Error(GOFMM_ERR_INVALID, "split level is not a complete tree level");
  std::vector<double> work(nn, 0.0);
  {
    std::vector<int32_t> par(nn, -1);
    for (int i = 0; i < nn; ++i)
      if (left[i] >= 0) par[left[i]] = par[right[i]] = i;
    auto npts = [&](int i) { return double(end[i] - start[i]); };
    for (int i = 0; i < nn; ++i) {
      const double k = rank[i] >= 0 ? double(rank[i]) : 0.0;
      if (left[i] < 0) {
        work[i] += 2.0 * npts(i) * npts(i) + 2.0 * k * npts(i) + 2.0 * k * npts(i);  // D, leaf S2N, N2S
      } else if (rank[i] >= 0) {
        const double c = double(std::max(rank[left[i]], 0) + std::max(rank[right[i]], 0));
        work[i] += 2.0 * k * c;  // N2S
      }
      if (par[i] >= 0 && rank[par[i]] >= 0 && rank[i] >= 0) work[i] += 2.0 * rank[par[i]] * k;  // S2N
    }
    for (int64_t t = 0; t < n_far; ++t) {
      const double f = 2.0 * std::max(rank[far_a[t]], 0) * std::max(rank[far_b[t]], 0);
      work[far_a[t]] += f;
      work[far_b[t]] += f;
    }
    for (int64_t t = 0; t < n_near; ++t) {
      const double f = 2.0 * npts(near_a[t]) * npts(near_b[t]);
      work[near_a[t]] += f;
      work[near_b[t]] += f;
    }
    for (int i = nn - 1; i >= 0; --i)  // BFS ids: children after parents
      if (left[i] >= 0 && level[i] >= ls) work[i] += work[left[i]] + work[right[i]];
  }
  // optimal contiguous partition of the S subtrees into nranks runs (min over max run work)
  const int S = int(at_split.size());
  std::vector<double> pre(S + 1, 0.0);
  for (int t = 0; t < S; ++t) pre[t + 1] = pre[t] + work[at_split[t]];
  std::vector<std::vector<double>> best(nranks + 1, std::vector<double>(S + 1, 1e300));
  std::vector<std::vector<int>> cut(nranks + 1, std::vector<int>(S + 1, 0));
  best[0][0] = 0.0;
  for (int g = 1; g <= nranks; ++g)
    for (int e = g; e <= S; ++e)
      for (int b = g - 1; b < e; ++b) {
        const double v = std::max(best[g - 1][b], pre[e] - pre[b]);
        if (v < best[g][e]) {
          best[g][e] = v;
          cut[g][e] = b;
        }
      }
  P.owner.assign(nn, -1);
  for (int g = nranks, e = S; g >= 1; --g) {
    const int b = cut[g][e];
    for (int t = b; t < e; ++t) P.owner[at_split[t]] = g - 1;
    e = b;
  }
  for (int i = 0; i < nn; ++i)  // BFS order: parents first
    if (level[i] >= ls && left[i] >= 0) P.owner[left[i]] = P.owner[right[i]] = P.owner[i];
  for (int i = 0; i < nn; ++i)
    if (level[i] > ls && P.owner[i] < 0) {
      // children were assigned from their parent above; a node deeper than l with no owner
      // would mean an inconsistent tree
      throw Error(GOFMM_ERR_INVALID, "node below the split without an owning subtree");
    }
  // W is replicated (every rank receives the full N x r input), so the W rows of cross-subtree
  // near-field partners are permuted locally in stage 1 and never exchanged; only skeleton weights
  // (what) travel.
  std::vector<char> need_what(nn, 0);
  if (nranks > 1) {
    for (int i : at_split) need_what[i] = 1;  // every rank's top N2S needs all level-l what
    auto request = [&](int requester_node, int target) {
      const int ro = P.owner[requester_node], to = P.owner[target];
      if (to < 0) return;                 // top what is recomputed by everyone
      if (ro < 0 || ro != to) need_what[target] = 1;  // top requesters run on every rank
    };
    for (int64_t t = 0; t < n_far; ++t) {
      request(far_a[t], far_b[t]);
      request(far_b[t], far_a[t]);
    }
  }
  // skeleton space offsets (same formula as build())
  std::vector<int64_t> soff(nn, -1);
  int64_t off = 0;
  for (int i = 0; i < nn; ++i)
    if (rank[i] >= 0) {
      soff[i] = off;
      off += pad16_(rank[i]);
    }
  P.exports.assign(nranks, {});
  P.send_rows.assign(nranks, 0);
  for (int i = 0; i < nn; ++i)
    if (need_what[i] && P.owner[i] >= 0) {
      if (rank[i] < 0) throw Error(GOFMM_ERR_INVALID, "exported node has no skeleton");
      P.exports[P.owner[i]].push_back({0, soff[i], pad16_(rank[i])});
    }
  for (int g = 0; g < nranks; ++g) {
    for (const Seg& sg : P.exports[g]) P.send_rows[g] += sg.rows;
    P.max_send_rows = std::max(P.max_send_rows, P.send_rows[g]);
  }
  return P;
}

}  // namespace
}  // namespace gofmm

struct gofmm_handle {
  // SPEC.md:429 allows concurrent evaluate() calls on one HMatrix. Every entry point that touches
  // the plan, workspace or timing state holds `mu` (host side), and every enqueue waits on
  // `ws_free` before its first launch and records it after its last, so evaluations issued on
  // different streams (or threads) never overlap on the shared device workspace.
  mutable std::mutex mu;
  cudaEvent_t ws_free = nullptr;
  int device = 0;
  int num_sms = 148;  // launch-config costing (queried at create)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  // host-buffer evaluation pipeline (evaluate_host): H2D / D2H copy streams and, per staging
  // buffer b, events in_ready / comp_done / out_free and copy-timing pairs
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  // CUDA graph of a whole single-chunk evaluation (all level launches in one graph),
  // captured on cap_stream and replayed on the caller's stream while the key matches
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::tuple<const void*, int64_t, const void*, int64_t, int32_t, int32_t, int32_t> gkey{};
  bool graphs = true;  // GOFMM_NO_GRAPH=1 disables replay
  // programmatic dependent launch between level launches (GOFMM_NO_PDL=1 disables); never in timed
  // (event-instrumented) enqueues: an event between two launches breaks the programmatic edge, and
  // the host pipeline measured slower and jittery with it (N = 2^16: 37-47 vs 34 ms per call)
  bool pdl = true;
  cudaEvent_t pev[2][4] = {};
  cudaEvent_t tev[2][4] = {};
  cudaEvent_t dpev[8][2] = {};  // per-part D2H timing of a split output launch (<= kOutParts)
  cudaEvent_t hpev[8] = {};     // column pieces of a single-chunk upload landed (H2D / N2S overlap)
  cudaEvent_t upev[2] = {};     // upward phase of a piece-pipelined evaluation (timing)
  gofmm::DevBuf d_win2[2], d_uout2[2];
  std::vector<cudaEvent_t> lev;  // per-launch start/stop events (timed evaluations only)
  std::vector<float> launch_ms;  // durations of the last timed evaluation (summed over chunks)
  float phase_ms[4] = {0, 0, 0, 0};
  int32_t max_chunk = 0;         // options.max_rhs_chunk (0 = size from free HBM)
  int32_t n = 0, num_nodes = 0, depth = 0, dim = 0, kernel = -1, source = 0;
  gofmm::KernelParams kp{};
  int near_mode = GOFMM_BLOCKS_MATRIX_FREE, far_mode = GOFMM_BLOCKS_MATRIX_FREE;

  // host copies of the structure
  std::vector<int32_t> parent, left, right, level, start, end, iperm, rank;
  std::vector<int32_t> leaf_ids;
  std::vector<int64_t> pst, soff;  // point / skeleton space offsets per node (-1 if none)
  int64_t ld_wp = 0, ld_s = 0;
  std::vector<int32_t> near_a, near_b, far_a, far_b;

  // device tree
  gofmm::DevBuf d_proj, d_diag, d_near, d_far, d_xp, d_xs, d_prow, d_iperm;
  gofmm::DevBuf d_amaps;  // TMA descriptors of the stored-A terms (upload_plan)
  gofmm::DevBuf d_perm32;  // FP32 two-pass permutation: row-major copy of W (large W only)
  int32_t perm2 = -1;      // GOFMM_PERM2=1 / 0 forces the two-pass FP32 permutation on / off
  bool perm2_on = false;   // the current chunk uses it (prepare32)
  std::vector<int64_t> proj_off, diag_off, near_off, far_off;  // device blob offsets (doubles)

  // plan
  std::vector<gofmm::HostGroup> groups;
  std::vector<gofmm::Launch> launches;
  std::vector<gofmm::Tile> tiles;
  gofmm::DevBuf d_tiles, d_groups, d_terms;
  std::vector<gofmm::ChainReduce> reduces;  // split term chains (FP64 downward levels)
  std::vector<int64_t> reduce_src;
  gofmm::DevBuf d_reduces, d_reduce_src;
  int64_t scratch_rows = 0;  // skeleton-space rows appended after the nodes for split segments
  bool plan_uploaded = false;
  int32_t plan_r = 0;  // workspace r the device term pointers were built for

  // workspace
  gofmm::DevBuf d_wp, d_what, d_c, d_win, d_uout;
  int32_t ws_r = 0;

  // distribution (nranks == 1: single-GPU evaluation)
  int32_t drank = 0, nranks = 1;
  gofmm::DistPlan dist;
  int64_t own_pst_begin = 0, own_pst_end = 0;  // own leaves' rows in point space
  int64_t own_begin = 0, own_end = 0;          // own permuted rows [start, end)
  int64_t full_flops_per_rhs = 0;              // the whole (undistributed) evaluation
  gofmm::DevBuf d_segs;                        // pack / unpack segment table
  // in-library data plane (gofmm_dist_evaluate): the NCCL communicator over the nranks GPUs
  // (owned when created from a unique id), a high-priority stream for the all-gather, the send /
  // receive slots, and the events that order stage 1 -> all-gather -> stage 4
  gofmm::nccl::comm_t comm = nullptr;
  bool own_comm = false;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_gath = nullptr, dtev[4] = {};
  gofmm::DevBuf d_send, d_recv;
  std::vector<double> coords_host;             // d x n original order (kernel sources; exact rows)
  gofmm::DevBuf d_ex_groups, d_ex_terms, d_ex_tiles, d_ex_x, d_ex_part;  // exact-rows scratch
  int32_t n_pack = 0, n_unpack = 0;

  // FP32 (3xTF32 tcgen05) plan, precision == GOFMM_PRECISION_F32: stored A operands as K-major
  // hi / lo copies (d_a32h / d_a32l, offsets per term), FP32 coordinates, 128-row tiles, and a
  // workspace of hi / lo panel buffers [0] = hi, [1] = lo
  int32_t precision = GOFMM_PRECISION_F64;
  gofmm::DevBuf d_a32h, d_a32l, d_xp32, d_xs32, d_xpn32, d_xsn32, d_terms32, d_tiles32;
  std::vector<int64_t> term_a32_off, term_a32_ld;  // per plan term (flattened group order), -1 if generated
  gofmm::DevBuf d_wp32[2], d_what32[2], d_c32[2], d_win32, d_uout32;
  int32_t ws32_r = 0;
  bool plan32_uploaded = false;
  gofmm::f32::KernelParams kp32{};
  // FP32 kernels and B maps per N tile (index 0/1/2 = 64/128/256 columns); each launch picks its own
  gofmm::f32::GemmKernel k32_s[3], k32_g[3];
  gofmm::f32::BMaps maps32[3]{};
  int32_t maps32_rv[3] = {0, 0, 0};

  gofmm::KernelFn kfn_sw = nullptr, kfn_sg = nullptr, kfn_sn64w = nullptr;
  size_t smem_sw = 0, smem_sg = 0, smem_sn64w = 0;
  gofmm::KernelFn kfn_s = nullptr, kfn_sn64 = nullptr, kfn_g = nullptr, kfn_gw = nullptr, kfn_gn64 = nullptr,
                  kfn_gn128 = nullptr, kfn_gn64w = nullptr, kfn_gm = nullptr;
  size_t smem_s = 0, smem_sn64 = 0, smem_g = 0, smem_gw = 0, smem_gn64 = 0, smem_gn128 = 0, smem_gn64w = 0,
         smem_gm = 0;
  double gm_eff = 0.74;  // GM candidate efficiency in the launch-config model (GOFMM_GM_EFF; 0 = off)
  gofmm::BMaps maps_s{}, maps_g{}, maps_n64{};  // B boxes of 128 / 256 / 64 columns
  int32_t maps_r = 0;  // r the tensor maps were encoded for
  int64_t flops_per_rhs = 0;
  int64_t phase_flops_per_rhs[3] = {0, 0, 0};  // upward, downward, output
};

namespace gofmm {
namespace {

void validate(const gofmm_tree_desc* d) {
  if (!d) throw Error(GOFMM_ERR_INVALID, "null descriptor");
  if (d->n < 1) throw Error(GOFMM_ERR_INVALID, "n must be >= 1");
  if (d->num_nodes < 1) throw Error(GOFMM_ERR_INVALID, "num_nodes must be >= 1");
  if (!d->parent || !d->left || !d->right || !d->level || !d->start || !d->end || !d->iperm || !d->rank)
    throw Error(GOFMM_ERR_INVALID, "missing node arrays");
  const int nn = d->num_nodes;
  for (int i = 0; i < nn; ++i) {
    if (d->start[i] < 0 || d->end[i] > d->n || d->start[i] > d->end[i])
      throw Error(GOFMM_ERR_INVALID, "node range out of bounds");
    if (d->left[i] >= 0) {
      if (d->left[i] >= nn || d->right[i] != d->left[i] + 1 || d->right[i] >= nn)
        throw Error(GOFMM_ERR_INVALID, "children must be consecutive ids (tree.hpp:213-217)");
      if (d->left[i] <= i) throw Error(GOFMM_ERR_INVALID, "nodes must be in BFS order");
    }
    if (i > 0 && (d->level[i] < d->level[i - 1]))
      throw Error(GOFMM_ERR_INVALID, "nodes must be in level (BFS) order");
  }
  if (d->parent[0] != -1 || d->start[0] != 0 || d->end[0] != d->n)
    throw Error(GOFMM_ERR_INVALID, "node 0 must be the root covering [0, n)");
  if (d->num_near < 0 || d->num_far < 0) throw Error(GOFMM_ERR_INVALID, "negative list size");
  if (d->source != GOFMM_SOURCE_STORED && d->source != GOFMM_SOURCE_KERNEL)
    throw Error(GOFMM_ERR_INVALID, "unknown entry source");
  if (d->source == GOFMM_SOURCE_KERNEL && (!d->coords || d->dim < 1 || d->dim > kMaxDimRt))
    throw Error(GOFMM_ERR_INVALID, "kernel source needs coords and 1 <= dim <= 16");
  if (d->source == GOFMM_SOURCE_STORED && (!d->diag_offset || !d->diag_blocks))
    throw Error(GOFMM_ERR_INVALID, "stored source needs leaf_diag blocks");
}


// ---------------------------------------------------------------- FP32 plan (3xTF32 tcgen05)
// The FP64 device tree built above is converted once: every stored-A operand a plan term reads
// becomes a K-major FP32 hi / lo copy (split_to_kmajor; proj twice — transposed for N2S, as is
// for S2N — and both orientations of stored near / far blocks), coordinates become FP32, and the
// same groups are re-tiled into 128-row tiles (UMMA M = 128). The FP64 blobs are released.
int f32_bn(int32_t r) { return r > 128 ? 256 : r > 64 ? 128 : 64; }

void build_f32(gofmm_handle* H) {
  const double* blobs[4] = {H->d_proj.as<double>(), H->d_diag.as<double>(), H->d_near.as<double>(),
                            H->d_far.as<double>()};
  struct Key {
    int blob;
    int64_t off;
    int rm, M, K;
    bool operator<(const Key& o) const {
      return std::tie(blob, off, rm, M, K) < std::tie(o.blob, o.off, o.rm, o.M, o.K);
    }
  };
  std::map<Key, std::pair<int64_t, int64_t>> seen;
  std::vector<f32::SplitJob> jobs;
  int64_t total = 0;
  H->term_a32_off.clear();
  H->term_a32_ld.clear();
  for (const HostGroup& g : H->groups)
    for (const HostTerm& t : g.terms) {
      if (t.kind != 0) {
        H->term_a32_off.push_back(-1);
        H->term_a32_ld.push_back(0);
        continue;
      }
      const Key key{t.a_blob, t.a_off, t.row_major ? 1 : 0, g.M, t.K};
      auto it = seen.find(key);
      if (it == seen.end()) {
        const int64_t ldd = (int64_t(t.K) + 3) & ~int64_t(3);  // 16-byte rows for cp.async
        f32::SplitJob J{};
        J.src = blobs[t.a_blob] + t.a_off;
        J.lds = t.lda;
        J.dst = total;
        J.rows = g.M;
        J.cols = t.K;
        J.ldd = int32_t(ldd);
        J.trans = t.row_major ? 0 : 1;
        jobs.push_back(J);
        it = seen.emplace(key, std::make_pair(total, ldd)).first;
        total += int64_t(g.M) * ldd;
      }
      H->term_a32_off.push_back(it->second.first);
      H->term_a32_ld.push_back(it->second.second);
    }
  H->d_a32h.alloc(size_t(std::max<int64_t>(total, 4)) * sizeof(float), false);
  H->d_a32l.alloc(size_t(std::max<int64_t>(total, 4)) * sizeof(float), false);
  if (!jobs.empty()) {
    DevBuf d_jobs;
    d_jobs.upload(jobs);
    GOFMM_CUDA(f32::launch_split(d_jobs.as<f32::SplitJob>(), int(jobs.size()), H->d_a32h.as<float>(),
                                 H->d_a32l.as<float>(), H->stream));
    GOFMM_CUDA(cudaStreamSynchronize(H->stream));
  }
  if (H->source == GOFMM_SOURCE_KERNEL) {
    // skeleton-space coordinates exist for the node rows only (split-chain scratch rows extend
    // ld_s after d_xs was sized and carry no points)
    const int64_t xs_rows = int64_t(H->d_xs.bytes / sizeof(double)) / std::max(H->dim, 1);
    const int64_t nxp = int64_t(H->ld_wp) * H->dim, nxs = xs_rows * H->dim;
    H->d_xp32.alloc(size_t(nxp) * sizeof(float), false);
    H->d_xs32.alloc(size_t(std::max<int64_t>(nxs, 1)) * sizeof(float), false);
    GOFMM_CUDA(f32::launch_to_f32(H->d_xp.as<double>(), nxp, H->d_xp32.as<float>(), H->stream));
    if (H->d_xs.p) GOFMM_CUDA(f32::launch_to_f32(H->d_xs.as<double>(), nxs, H->d_xs32.as<float>(), H->stream));
    if (H->kernel == kGaussian) {
      // norm expansion operands: -log2(e)/(2h^2) |x|^2, from the FP64 coordinates
      const double sc = -H->kp.p0 * 1.4426950408889634;
      H->d_xpn32.alloc(size_t(std::max<int64_t>(H->ld_wp, 16)) * sizeof(float));
      H->d_xsn32.alloc(size_t(std::max<int64_t>(H->ld_s, 16)) * sizeof(float));
      GOFMM_CUDA(f32::launch_scaled_norms(H->d_xp.as<double>(), H->ld_wp, H->dim, sc, H->d_xpn32.as<float>(), H->stream));
      if (H->d_xs.p)
        GOFMM_CUDA(f32::launch_scaled_norms(H->d_xs.as<double>(), xs_rows, H->dim, sc, H->d_xsn32.as<float>(), H->stream));
    }
    GOFMM_CUDA(cudaStreamSynchronize(H->stream));
  }
  // kernel parameters: exp(x) = 2^(x log2 e) is folded into the scale (ex2.approx in the kernel)
  constexpr double kLog2e = 1.4426950408889634;
  H->kp32 = {};
  H->kp32.dim = H->dim;
  if (H->kernel == kGaussian || H->kernel == kExponential) {
    H->kp32.p0 = float(H->kp.p0 * kLog2e);
  } else {
    H->kp32.p0 = float(H->kp.p0);
    H->kp32.p1 = float(H->kp.p1);
  }
  // 128-row tiles of the same groups
  std::vector<Tile> tiles32;
  for (Launch& L : H->launches) {
    L.first_tile32 = int(tiles32.size());
    for (int gi = L.first_group; gi < L.first_group + L.ngroups; ++gi)
      for (int m0 = 0; m0 < std::max(H->groups[gi].M, 0); m0 += f32::kBM) tiles32.push_back({gi, m0});
    L.ntiles32 = int(tiles32.size()) - L.first_tile32;
    L.chain_sum32 = L.chain_max32 = 0;
    for (int i = L.first_tile32; i < L.first_tile32 + L.ntiles32; ++i) {
      int64_t w = 0;
      for (const HostTerm& t : H->groups[tiles32[i].group].terms) w += (t.K + 15) / 16;
      L.chain_sum32 += w;
      L.chain_max32 = std::max(L.chain_max32, w);
    }
    for (size_t p = 0; p < L.parts.size(); ++p) {
      const int gb = (p + 1 < L.parts.size()) ? L.first_group + int(int64_t(L.ngroups) * p / kOutParts)
                                               : L.first_group + L.ngroups;
      int t = L.first_tile32;
      while (t < L.first_tile32 + L.ntiles32 && tiles32[t].group < gb) ++t;
      L.parts[p].tile32 = t;
    }
    if (L.parts.empty()) {
      order_longest_first(tiles32, L.first_tile32, L.first_tile32 + L.ntiles32, H->groups);
    } else {
      for (size_t p = 0; p + 1 < L.parts.size(); ++p)
        order_longest_first(tiles32, L.parts[p].tile32, L.parts[p + 1].tile32, H->groups);
    }
  }
  H->d_tiles32.upload(tiles32);
  // groups and FP32 terms do not depend on the workspace (B operands go through tensor maps)
  std::vector<Group> gs;
  std::vector<f32::Term> ts;
  const float* xb[2] = {H->d_xp32.as<float>(), H->d_xs32.as<float>()};
  const float* xn[2] = {H->d_xpn32.as<float>(), H->d_xsn32.as<float>()};
  const int bid[4] = {kBufWp, kBufWhat, kBufC, kBufC};
  size_t ti = 0;
  // two TMA views (hi, lo) per stored-A term (64-byte aligned 128-byte descriptors in global memory)
  size_t n_amaps = 0;
  for (const HostGroup& hg : H->groups)
    for (const HostTerm& ht : hg.terms)
      if (ht.kind == 0 && ht.K > 0 && hg.M > 0) n_amaps += 2;
  std::vector<CUtensorMap> amaps;
  amaps.reserve(n_amaps);
  H->d_amaps.alloc(std::max<size_t>(n_amaps, 1) * sizeof(CUtensorMap), false);
  const CUtensorMap* amap_base = H->d_amaps.as<CUtensorMap>();
  for (const HostGroup& hg : H->groups) {
    Group g{};
    g.crow = hg.c_row;
    g.M = hg.M;
    g.flags = hg.flags;
    g.tbeg = int(ts.size());
    for (const HostTerm& ht : hg.terms) {
      f32::Term t{};
      t.bbuf = bid[int(ht.b_buf)];
      t.b_row = ht.b_row;
      t.K = ht.K;
      if (ht.kind == 1) {
        t.flags = kTermGen;
        t.xr = xb[ht.x_blob] + ht.xr_off * H->dim;
        t.xc = xb[ht.x_blob] + ht.xc_off * H->dim;
        if (xn[ht.x_blob]) {
          t.xrn = xn[ht.x_blob] + ht.xr_off;
          t.xcn = xn[ht.x_blob] + ht.xc_off;
        }
      } else {
        t.a_hi = H->d_a32h.as<float>() + H->term_a32_off[ti];
        t.a_lo = H->d_a32l.as<float>() + H->term_a32_off[ti];
        t.lda = H->term_a32_ld[ti];
        if (ht.K > 0 && hg.M > 0) {
          t.amap = amap_base + amaps.size();
          amaps.emplace_back();
          encode_amap32(&amaps.back(), t.a_hi, t.lda, hg.M, ht.K);
          amaps.emplace_back();
          encode_amap32(&amaps.back(), t.a_lo, t.lda, hg.M, ht.K);
        }
      }
      ts.push_back(t);
      ++ti;
    }
    g.tend = int(ts.size());
    gs.push_back(g);
  }
  if (!amaps.empty())
    GOFMM_CUDA(cudaMemcpy(H->d_amaps.p, amaps.data(), amaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  H->d_groups.upload(gs);
  H->d_terms32.upload(ts.empty() ? std::vector<f32::Term>(1) : ts);
  // the FP64 operand blobs are not read by an FP32 handle
  H->d_proj.release();
  H->d_diag.release();
  H->d_near.release();
  H->d_far.release();
}

void build(gofmm_handle* H, const gofmm_tree_desc* d, const gofmm_options* o) {
  const int nn = d->num_nodes;
  H->n = d->n;
  H->num_nodes = nn;
  H->source = d->source;
  H->kernel = d->source == GOFMM_SOURCE_KERNEL ? d->kernel : -1;
  H->dim = d->source == GOFMM_SOURCE_KERNEL ? d->dim : 0;
  if (o) {
    H->near_mode = o->near_mode;
    H->far_mode = o->far_mode;
    H->max_chunk = o->max_rhs_chunk;
    H->precision = o->precision;
  }
  if (const char* e = std::getenv("GOFMM_NO_GRAPH")) H->graphs = !(e[0] == '1');
  if (const char* e = std::getenv("GOFMM_NO_PDL")) H->pdl = !(e[0] == '1');
  if (const char* e = std::getenv("GOFMM_PERM2")) H->perm2 = (e[0] == '1') ? 1 : 0;
  if (const char* e = std::getenv("GOFMM_GM_EFF")) H->gm_eff = std::atof(e);
  auto cp = [&](std::vector<int32_t>& v, const int32_t* p, int64_t k) { v.assign(p, p + k); };
  cp(H->parent, d->parent, nn);
  cp(H->left, d->left, nn);
  cp(H->right, d->right, nn);
  cp(H->level, d->level, nn);
  cp(H->start, d->start, nn);
  cp(H->end, d->end, nn);
  cp(H->iperm, d->iperm, d->n);
  cp(H->rank, d->rank, nn);
  cp(H->near_a, d->near_a, d->num_near);
  cp(H->near_b, d->near_b, d->num_near);
  cp(H->far_a, d->far_a, d->num_far);
  cp(H->far_b, d->far_b, d->num_far);
  H->depth = 0;
  for (int i = 0; i < nn; ++i) H->depth = std::max(H->depth, H->level[i]);

  // kernel parameters exactly as the reference oracles precompute them
  if (H->kernel == kGaussian) {
    double h = d->kparam[0];
    if (!(h > 0)) throw Error(GOFMM_ERR_INVALID, "gaussian bandwidth must be positive");
    H->kp.p0 = 1.0 / (2.0 * h * h);  // oracle.hpp:151
  } else if (H->kernel == kExponential) {
    if (!(d->kparam[0] > 0)) throw Error(GOFMM_ERR_INVALID, "exponential bandwidth must be positive");
    H->kp.p0 = 1.0 / d->kparam[0];
  } else if (H->kernel == kLaplace) {
    if (d->kparam[0] < 0) throw Error(GOFMM_ERR_INVALID, "laplace regularization must be >= 0");
    H->kp.p0 = d->kparam[0];
    H->kp.p1 = double(d->dim - 2);  // oracle.hpp:181
  } else if (H->kernel == kPolynomial) {
    H->kp.p0 = d->kparam[0];
    H->kp.p1 = double(static_cast<int>(d->kparam[1]));
  } else if (d->source == GOFMM_SOURCE_KERNEL) {
    throw Error(GOFMM_ERR_INVALID, "unsupported kernel id");
  }
  H->kp.dim = H->dim;

  // skeleton validity & consistency
  std::vector<int32_t> ncand(nn, 0);
  for (int i = 0; i < nn; ++i) {
    const int k = H->rank[i];
    if (k < 0) continue;
    int64_t np = d->proj_offset[i + 1] - d->proj_offset[i];
    const bool leaf = H->left[i] < 0;
    int64_t c = leaf ? (H->end[i] - H->start[i]) : 0;
    if (!leaf) {
      if (H->rank[H->left[i]] < 0 || H->rank[H->right[i]] < 0)
        throw Error(GOFMM_ERR_INVALID, "interior skeleton needs valid child skeletons");
      c = H->rank[H->left[i]] + H->rank[H->right[i]];
    }
    if (np != int64_t(k) * c) throw Error(GOFMM_ERR_INVALID, "proj size mismatch at node " + std::to_string(i));
    if (d->skel_offset[i + 1] - d->skel_offset[i] != k)
      throw Error(GOFMM_ERR_INVALID, "skeleton index count mismatch at node " + std::to_string(i));
    ncand[i] = static_cast<int32_t>(c);
  }

  // leaves left-to-right (tree.hpp:232-233) and point space
  for (int i = 0; i < nn; ++i)
    if (H->left[i] < 0) H->leaf_ids.push_back(i);
  std::sort(H->leaf_ids.begin(), H->leaf_ids.end(), [&](int a, int b) { return H->start[a] < H->start[b]; });
  H->pst.assign(nn, -1);
  int64_t off = 0;
  for (int id : H->leaf_ids) {
    H->pst[id] = off;
    off += pad16(H->end[id] - H->start[id]);
  }
  H->ld_wp = std::max<int64_t>(pad16(off), 16);
  // skeleton space (BFS id order)
  H->soff.assign(nn, -1);
  off = 0;
  for (int i = 0; i < nn; ++i) {
    if (H->rank[i] < 0) continue;
    H->soff[i] = off;
    off += pad16(H->rank[i]);
  }
  H->ld_s = std::max<int64_t>(pad16(off), 16);

  // subtree split (single GPU: nranks == 1, everything owned by rank 0)
  H->dist = make_dist_plan(H->nranks, nn, d->left, d->right, d->level, d->start, d->end, d->rank, d->num_near,
                           d->near_a, d->near_b, d->num_far, d->far_a, d->far_b);
  if (H->drank < 0 || H->drank >= H->nranks) throw Error(GOFMM_ERR_INVALID, "rank out of range");
  {
    H->own_pst_begin = H->ld_wp;
    H->own_pst_end = 0;
    H->own_begin = d->n;
    H->own_end = 0;
    for (int id : H->leaf_ids)
      if (H->dist.owner[id] == H->drank) {
        H->own_pst_begin = std::min(H->own_pst_begin, H->pst[id]);
        H->own_pst_end = std::max(H->own_pst_end, H->pst[id] + pad16(H->end[id] - H->start[id]));
        H->own_begin = std::min<int64_t>(H->own_begin, H->start[id]);
        H->own_end = std::max<int64_t>(H->own_end, H->end[id]);
      }
  }
  auto active = [&](int i) { return H->dist.owner[i] == H->drank || H->dist.owner[i] < 0; };

  // row map for the permutation kernel, and iperm
  std::vector<int32_t> prow(H->ld_wp, -1);
  for (int id : H->leaf_ids)
    for (int t = H->start[id]; t < H->end[id]; ++t) prow[H->pst[id] + (t - H->start[id])] = H->iperm[t];
  H->d_prow.upload(prow);
  H->d_iperm.upload(H->iperm);

  // padded proj blob. When no node needs padding (even ranks, children ranks multiples of 16 —
  // the saturated large trees) the caller's layout already is the device layout: one H2D copy,
  // no host-side duplicate of a ~13-26 GB array.
  bool proj_identity = true;
  for (int i = 0; i < nn && proj_identity; ++i) {
    const int k = H->rank[i];
    if (k < 0) continue;
    if (k % 2) proj_identity = false;
    if (H->left[i] >= 0 && (H->rank[H->left[i]] % 16 || H->rank[H->right[i]] % 16)) proj_identity = false;
    if (d->proj_offset[i] % 2) proj_identity = false;
  }
  if (proj_identity) {
    H->proj_off.assign(nn, -1);
    for (int i = 0; i < nn; ++i)
      if (H->rank[i] >= 0) H->proj_off[i] = d->proj_offset[i];
    const int64_t total = std::max<int64_t>(d->proj_offset[nn], 2);
    H->d_proj.alloc(size_t(total) * sizeof(double), false);
    if (d->proj_offset[nn] > 0)
      GOFMM_CUDA(cudaMemcpy(H->d_proj.p, d->proj, size_t(d->proj_offset[nn]) * sizeof(double), cudaMemcpyHostToDevice));
  } else {
    std::vector<double> blob;
    H->proj_off.assign(nn, -1);
    for (int i = 0; i < nn; ++i) {
      const int k = H->rank[i];
      if (k < 0) continue;
      const int64_t ld = pad2(k);
      const double* src = d->proj + d->proj_offset[i];
      H->proj_off[i] = static_cast<int64_t>(blob.size());
      if (H->left[i] < 0) {
        const int c = ncand[i];
        blob.resize(blob.size() + ld * c, 0.0);
        double* dst = blob.data() + H->proj_off[i];
        for (int j = 0; j < c; ++j)
          for (int r = 0; r < k; ++r) dst[r + j * ld] = src[r + int64_t(j) * k];
      } else {
        const int kl = H->rank[H->left[i]], kr = H->rank[H->right[i]];
        const int64_t cpad = pad16(kl) + pad16(kr);
        blob.resize(blob.size() + ld * cpad, 0.0);
        double* dst = blob.data() + H->proj_off[i];
        for (int j = 0; j < kl + kr; ++j) {
          const int64_t jj = (j < kl) ? j : pad16(kl) + (j - kl);
          for (int r = 0; r < k; ++r) dst[r + jj * ld] = src[r + int64_t(j) * k];
        }
      }
      while (blob.size() % 2) blob.push_back(0.0);
    }
    H->d_proj.upload(blob);
  }

  // coordinates: permuted point space and skeleton space, point-major
  if (d->source == GOFMM_SOURCE_KERNEL) {
    const int D = d->dim;
    H->coords_host.assign(d->coords, d->coords + int64_t(D) * d->n);
    std::vector<double> xp(size_t(H->ld_wp) * D, 0.0);
    for (int id : H->leaf_ids)
      for (int t = H->start[id]; t < H->end[id]; ++t) {
        const int64_t row = H->pst[id] + (t - H->start[id]);
        const double* src = d->coords + int64_t(H->iperm[t]) * D;
        for (int q = 0; q < D; ++q) xp[row * D + q] = src[q];
      }
    H->d_xp.upload(xp);
    std::vector<double> xs(size_t(H->ld_s) * D, 0.0);
    for (int i = 0; i < nn; ++i) {
      if (H->rank[i] < 0) continue;
      for (int l = 0; l < H->rank[i]; ++l) {
        const int64_t orig = d->skel_idx[d->skel_offset[i] + l];
        if (orig < 0 || orig >= d->n) throw Error(GOFMM_ERR_INVALID, "skeleton index out of range");
        for (int q = 0; q < D; ++q) xs[(H->soff[i] + l) * D + q] = d->coords[orig * D + q];
      }
    }
    H->d_xs.upload(xs);
  }

  // stored / materialised blocks: D (leaf_diag), near, far — column-major, ld = pad2(rows)
  const bool stored = d->source == GOFMM_SOURCE_STORED;
  const bool mat_near = !stored && H->near_mode == GOFMM_BLOCKS_MATERIALIZE;
  const bool mat_far = !stored && H->far_mode == GOFMM_BLOCKS_MATERIALIZE;
  auto nrows = [&](int id) { return H->end[id] - H->start[id]; };
  auto pack_blocks = [&](int64_t count, auto rows_of, auto cols_of, const int64_t* src_off, const double* src,
                         std::vector<int64_t>& offs, DevBuf& dev, bool from_host) {
    offs.assign(count, -1);
    int64_t total = 0;
    for (int64_t t = 0; t < count; ++t) {
      int r = rows_of(t), c = cols_of(t);
      if (r <= 0 || c <= 0) continue;
      offs[t] = total;
      total += pad2(r) * c;
    }
    if (!from_host) {
      dev.alloc(std::max<int64_t>(total, 2) * sizeof(double));
      return;
    }
    std::vector<double> blob(std::max<int64_t>(total, 2), 0.0);
    for (int64_t t = 0; t < count; ++t) {
      if (offs[t] < 0) continue;
      int r = rows_of(t), c = cols_of(t);
      if (src_off[t + 1] - src_off[t] != int64_t(r) * c)
        throw Error(GOFMM_ERR_INVALID, "stored block size mismatch");
      const double* s = src + src_off[t];
      double* dd = blob.data() + offs[t];
      const int64_t ld = pad2(r);
      for (int j = 0; j < c; ++j)
        for (int i = 0; i < r; ++i) dd[i + j * ld] = s[i + int64_t(j) * r];
    }
    dev.upload(blob);
  };
  if (stored || mat_near) {
    pack_blocks(
        nn, [&](int64_t t) { return H->left[t] < 0 ? nrows(int(t)) : 0; },
        [&](int64_t t) { return H->left[t] < 0 ? nrows(int(t)) : 0; }, d->diag_offset, d->diag_blocks, H->diag_off,
        H->d_diag, stored);
    if (stored && d->num_near && (!d->near_offset || !d->near_blocks))
      throw Error(GOFMM_ERR_INVALID, "stored source needs near blocks");
    pack_blocks(
        d->num_near, [&](int64_t t) { return nrows(H->near_a[t]); }, [&](int64_t t) { return nrows(H->near_b[t]); },
        d->near_offset, d->near_blocks, H->near_off, H->d_near, stored);
  }
  if (stored || mat_far) {
    if (stored && d->num_far && (!d->far_offset || !d->far_blocks))
      throw Error(GOFMM_ERR_INVALID, "stored source needs far blocks");
    pack_blocks(
        d->num_far, [&](int64_t t) { return H->rank[H->far_a[t]]; }, [&](int64_t t) { return H->rank[H->far_b[t]]; },
        d->far_offset, d->far_blocks, H->far_off, H->d_far, stored);
  }
  // device-side materialisation from coordinates
  if (mat_near) {
    const double* xp = H->d_xp.as<double>();
    for (int id : H->leaf_ids)
      generate_dispatch(H->kernel, H->dim, xp + H->pst[id] * H->dim, nrows(id), xp + H->pst[id] * H->dim, nrows(id),
                        H->d_diag.as<double>() + H->diag_off[id], pad2(nrows(id)), H->kp, H->stream);
    for (size_t t = 0; t < H->near_a.size(); ++t) {
      int a = H->near_a[t], b = H->near_b[t];
      generate_dispatch(H->kernel, H->dim, xp + H->pst[a] * H->dim, nrows(a), xp + H->pst[b] * H->dim, nrows(b),
                        H->d_near.as<double>() + H->near_off[t], pad2(nrows(a)), H->kp, H->stream);
    }
  }
  if (mat_far) {
    const double* xs = H->d_xs.as<double>();
    for (size_t t = 0; t < H->far_a.size(); ++t) {
      int a = H->far_a[t], b = H->far_b[t];
      generate_dispatch(H->kernel, H->dim, xs + H->soff[a] * H->dim, H->rank[a], xs + H->soff[b] * H->dim, H->rank[b],
                        H->d_far.as<double>() + H->far_off[t], pad2(H->rank[a]), H->kp, H->stream);
    }
  }
  GOFMM_CUDA(cudaStreamSynchronize(H->stream));
  GOFMM_CUDA(cudaGetLastError());

  // ------------------------------------------------------------ groups / terms (evaluate.hpp:52-217)
  // partners per node, ascending partner id (evaluate.hpp:63-70)
  struct Partner {
    int other, block;
    bool transposed;
  };
  std::vector<std::vector<Partner>> partners(nn);
  for (size_t t = 0; t < H->far_a.size(); ++t) {
    int a = H->far_a[t], b = H->far_b[t];
    if (a < 0 || b < 0 || a >= nn || b >= nn || H->rank[a] < 0 || H->rank[b] < 0)
      throw Error(GOFMM_ERR_INVALID, "far pair references a node without skeleton");
    partners[a].push_back({b, int(t), false});
    partners[b].push_back({a, int(t), true});
  }
  for (auto& ps : partners)
    std::stable_sort(ps.begin(), ps.end(), [](const Partner& x, const Partner& y) { return x.other < y.other; });
  std::vector<std::vector<int>> near_of(nn);
  for (size_t t = 0; t < H->near_a.size(); ++t) {
    int a = H->near_a[t], b = H->near_b[t];
    if (a < 0 || b < 0 || a >= nn || b >= nn || H->left[a] >= 0 || H->left[b] >= 0)
      throw Error(GOFMM_ERR_INVALID, "near pair must join two leaves");
    near_of[a].push_back(int(t));
    near_of[b].push_back(int(t));
  }

  const bool gen_near = !stored && !mat_near;
  const bool gen_far = !stored && !mat_far;
  int64_t flops = 0;
  int64_t flops_mark = 0;
  auto push_launch = [&](std::vector<HostGroup>& gs, bool gen, Buf out, int phase, int level) {
    Launch L;
    L.gen = gen;
    L.out = out;
    L.phase = phase;
    L.level = level;
    L.flops_per_rhs = flops - flops_mark;
    flops_mark = flops;
    L.first_group = int(H->groups.size());
    L.ngroups = int(gs.size());
    for (auto& g : gs) H->groups.push_back(std::move(g));
    for (int c = 0; c < 3; ++c) {
      L.tfirst[c] = int(H->tiles.size());
      for (int gi = L.first_group; gi < L.first_group + L.ngroups; ++gi)
        for (int m0 = 0; m0 < std::max(H->groups[gi].M, 0); m0 += kBM[c]) H->tiles.push_back({gi, m0});
      L.tn[c] = int(H->tiles.size()) - L.tfirst[c];
    }
    for (int c = 0; c < 3; ++c)
      for (int i = L.tfirst[c]; i < L.tfirst[c] + L.tn[c]; ++i) {
        int64_t w = 0;
        for (const HostTerm& t : H->groups[H->tiles[i].group].terms) w += (t.K + 15) / 16;
        L.chain_sum[c] += w;
        L.chain_max = std::max(L.chain_max, w);
      }
    if (out == Buf::Out) split_output_parts(L, H->groups, H->tiles);
    for (int c = 0; c < 3; ++c) {
      if (L.parts.empty()) {
        order_longest_first(H->tiles, L.tfirst[c], L.tfirst[c] + L.tn[c], H->groups);
      } else {
        for (size_t p = 0; p + 1 < L.parts.size(); ++p)
          order_longest_first(H->tiles, L.parts[p].tile[c], L.parts[p + 1].tile[c], H->groups);
      }
    }
    if (L.tn[0] > 0) H->launches.push_back(std::move(L));
  };

  // upward (N2S), deepest level first (evaluate.hpp:83-93,150-163)
  for (int lev = H->depth; lev >= 1; --lev) {
    std::vector<HostGroup> gs;
    for (int i = 0; i < nn; ++i) {
      if (H->level[i] != lev || H->rank[i] < 0 || !active(i)) continue;
      HostGroup g;
      g.c_row = H->soff[i];
      g.M = H->rank[i];
      HostTerm t{};
      t.kind = 0;
      t.row_major = false;
      t.a_blob = 0;
      t.a_off = H->proj_off[i];
      t.lda = pad2(H->rank[i]);
      if (H->left[i] < 0) {
        t.b_buf = Buf::Wp;
        t.b_row = H->pst[i];
        t.K = nrows(i);
      } else {
        t.b_buf = Buf::What;
        t.b_row = H->soff[H->left[i]];
        t.K = int(pad16(H->rank[H->left[i]]) + pad16(H->rank[H->right[i]]));
      }
      flops += 2LL * H->rank[i] * ncand[i];
      H->phase_flops_per_rhs[0] += 2LL * H->rank[i] * ncand[i];
      g.terms.push_back(t);
      gs.push_back(std::move(g));
    }
    push_launch(gs, false, Buf::What, 0, lev);
    if (!H->launches.empty() && H->launches.back().level == lev && H->launches.back().phase == 0)
      H->launches.back().stage = (lev >= H->dist.split) ? 1 : 2;
  }

  // downward: coupling (S2S) + parent term (S2N), top level first (evaluate.hpp:95-111,164-195)
  for (int lev = 1; lev <= H->depth; ++lev) {
    std::vector<HostGroup> gs;
    bool any_gen = false;
    for (int i = 0; i < nn; ++i) {
      if (H->level[i] != lev || H->rank[i] < 0 || !active(i)) continue;
      HostGroup g;
      g.c_row = H->soff[i];
      g.M = H->rank[i];
      for (const Partner& p : partners[i]) {
        HostTerm t{};
        t.b_buf = Buf::What;
        t.b_row = H->soff[p.other];
        t.K = H->rank[p.other];
        if (gen_far) {
          t.kind = 1;
          t.x_blob = 1;
          t.xr_off = H->soff[i];
          t.xc_off = H->soff[p.other];
          any_gen = true;
        } else {
          t.kind = 0;
          t.a_blob = 3;
          t.a_off = H->far_off[p.block];
          t.lda = pad2(H->rank[H->far_a[p.block]]);
          t.row_major = p.transposed;
        }
        flops += 2LL * H->rank[i] * H->rank[p.other];
        H->phase_flops_per_rhs[1] += 2LL * H->rank[i] * H->rank[p.other];
        g.terms.push_back(t);
      }
      const int par = H->parent[i];
      if (par > 0 && H->rank[par] >= 0) {
        HostTerm t{};
        t.kind = 0;
        t.row_major = true;  // proj_p[:, off:off+k]^T
        t.a_blob = 0;
        const int64_t coloff = (i == H->left[par]) ? 0 : pad16(H->rank[H->left[par]]);
        t.lda = pad2(H->rank[par]);
        t.a_off = H->proj_off[par] + coloff * t.lda;
        t.b_buf = Buf::C;
        t.b_row = H->soff[par];
        t.K = H->rank[par];
        flops += 2LL * H->rank[par] * H->rank[i];
        H->phase_flops_per_rhs[1] += 2LL * H->rank[par] * H->rank[i];
        g.terms.push_back(t);
      }
      gs.push_back(std::move(g));
    }
    // Latency-bound levels (few groups, long far-field chains — the upper levels; config 1 has
    // chains of 80 k-stages on 16-64 groups): split a chain that is much longer than the level's
    // per-SM share into segments of about that share. Segment 0 accumulates into the group's own
    // rows, the others into scratch rows appended to skeleton space; chain_reduce (FP32:
    // chain_reduce_f32 over the hi / lo pair) adds them in segment order after the launch.
    // The split (and so the summation order of c) is a function of the WHOLE level and a fixed SM
    // count only — never of this device's SM count or of a rank's share of the level — so u is
    // bitwise the same on any GPU SKU and for every rank layout of the subtree split.
    const int first_reduce = int(H->reduces.size());
    if (!gs.empty()) {
      auto stages = [](const HostTerm& t) { return int64_t((t.K + 15) / 16); };
      auto kstages = [](int64_t k) { return (k + 15) / 16; };
      int64_t sum = 0, mx = 0;
      for (int i = 0; i < nn; ++i) {  // every node of the level, owned or not
        if (H->level[i] != lev || H->rank[i] < 0) continue;
        int64_t ch = 0;
        for (const Partner& p : partners[i]) ch += kstages(H->rank[p.other]);
        const int par = H->parent[i];
        if (par > 0 && H->rank[par] >= 0) ch += kstages(H->rank[par]);
        sum += ch * ((H->rank[i] + kBM_G - 1) / kBM_G);
        mx = std::max(mx, ch);
      }
      const double fair = double(sum) / double(kSplitRefSms);
      if (double(mx) > 2.0 * fair && mx >= 24) {
        const int64_t target = std::max<int64_t>(8, int64_t(std::ceil(fair)));
        std::vector<HostGroup> out;
        for (HostGroup& g : gs) {
          int64_t ch = 0;
          for (const HostTerm& t : g.terms) ch += stages(t);
          if (ch <= target + target / 2 || g.terms.size() < 2) {
            out.push_back(std::move(g));
            continue;
          }
          gofmm::ChainReduce red{};
          red.dst_row = g.c_row;
          red.M = g.M;
          red.src_first = int32_t(H->reduce_src.size());
          size_t t0 = 0;
          bool first = true;
          while (t0 < g.terms.size()) {
            size_t t1 = t0;
            int64_t acc = 0;
            while (t1 < g.terms.size() && (acc < target || t1 == t0)) acc += stages(g.terms[t1++]);
            HostGroup seg;
            seg.M = g.M;
            seg.terms.assign(g.terms.begin() + int64_t(t0), g.terms.begin() + int64_t(t1));
            if (first) {
              seg.c_row = g.c_row;
              first = false;
            } else {
              seg.c_row = H->ld_s + H->scratch_rows;  // scratch rows after all nodes
              H->scratch_rows += pad16(g.M);
              H->reduce_src.push_back(seg.c_row);
              ++red.nsrc;
            }
            out.push_back(std::move(seg));
            t0 = t1;
          }
          if (red.nsrc > 0) H->reduces.push_back(red);
        }
        gs = std::move(out);
      }
    }
    push_launch(gs, any_gen, Buf::C, 1, lev);
    if (!H->launches.empty() && H->launches.back().phase == 1 && H->launches.back().level == lev) {
      H->launches.back().reduce_first = first_reduce;
      H->launches.back().reduce_n = int(H->reduces.size()) - first_reduce;
    }
  }

  // output: D, near blocks (ascending index), proj^T c (evaluate.hpp:113-117,196-217)
  {
    // A rank of an FP64 subtree split runs the chain in two launches: D + near terms (stage 3,
    // inputs all local: W is replicated) while the all-gather is in flight, then proj^T c
    // (stage 2) continuing the same accumulators from u (kGroupLoadC) — bitwise the one-launch sum.
    const bool split_out = H->nranks > 1 && H->precision == GOFMM_PRECISION_F64;
    std::vector<HostGroup> gs, gs_proj;
    int64_t flops_proj = 0;
    for (int id : H->leaf_ids) {
      if (H->dist.owner[id] != H->drank) continue;
      HostGroup g;
      g.c_row = H->start[id];
      g.M = nrows(id);
      const int n_a = nrows(id);
      HostTerm t{};
      t.b_buf = Buf::Wp;
      t.b_row = H->pst[id];
      t.K = n_a;
      if (gen_near) {
        t.kind = 1;
        t.x_blob = 0;
        t.xr_off = H->pst[id];
        t.xc_off = H->pst[id];
      } else {
        t.kind = 0;
        t.a_blob = 1;
        t.a_off = H->diag_off[id];
        t.lda = pad2(n_a);
      }
      flops += 2LL * n_a * n_a;
      g.terms.push_back(t);
      for (int bi : near_of[id]) {
        const int a = H->near_a[bi], b = H->near_b[bi];
        const int other = (a == id) ? b : a;
        HostTerm u{};
        u.b_buf = Buf::Wp;
        u.b_row = H->pst[other];
        u.K = nrows(other);
        if (gen_near) {
          u.kind = 1;
          u.x_blob = 0;
          u.xr_off = H->pst[id];
          u.xc_off = H->pst[other];
        } else {
          u.kind = 0;
          u.a_blob = 2;
          u.a_off = H->near_off[bi];
          u.lda = pad2(nrows(a));
          u.row_major = (a != id);  // K_ab^T for the b side (evaluate.hpp:205-207)
        }
        flops += 2LL * nrows(a) * nrows(b);
        g.terms.push_back(u);
      }
      if (H->rank[id] >= 0) {
        HostTerm v{};
        v.kind = 0;
        v.row_major = true;  // proj^T
        v.a_blob = 0;
        v.a_off = H->proj_off[id];
        v.lda = pad2(H->rank[id]);
        v.b_buf = Buf::C;
        v.b_row = H->soff[id];
        v.K = H->rank[id];
        if (split_out) {
          HostGroup gp;
          gp.c_row = g.c_row;
          gp.M = g.M;
          gp.flags = kGroupLoadC;
          gp.terms.push_back(v);
          gs_proj.push_back(std::move(gp));
          flops_proj += 2LL * H->rank[id] * n_a;
        } else {
          flops += 2LL * H->rank[id] * n_a;
          g.terms.push_back(v);
        }
      }
      gs.push_back(std::move(g));
    }
    push_launch(gs, gen_near, Buf::Out, 2, -1);
    if (split_out) {
      if (!H->launches.empty() && H->launches.back().out == Buf::Out) H->launches.back().stage = 3;
      flops += flops_proj;
      push_launch(gs_proj, false, Buf::Out, 2, -1);
    }
  }
  H->flops_per_rhs = flops;
  {
    // reference counter of the whole evaluation (evaluate.hpp:154-214), independent of the split
    int64_t f = 0;
    for (int i = 0; i < nn; ++i) {
      if (H->rank[i] < 0) continue;
      f += 2LL * H->rank[i] * ncand[i];  // upward
      const int par = H->parent[i];
      if (par > 0 && H->rank[par] >= 0) f += 2LL * H->rank[par] * H->rank[i];  // downward
      if (H->left[i] < 0) f += 2LL * H->rank[i] * nrows(i);                     // leaf S2N
    }
    for (size_t t = 0; t < H->far_a.size(); ++t) f += 4LL * H->rank[H->far_a[t]] * H->rank[H->far_b[t]];
    for (size_t t = 0; t < H->near_a.size(); ++t) f += 4LL * nrows(H->near_a[t]) * nrows(H->near_b[t]);
    for (int id : H->leaf_ids) f += 2LL * nrows(id) * nrows(id);
    H->full_flops_per_rhs = f;
  }
  H->phase_flops_per_rhs[2] = flops - H->phase_flops_per_rhs[0] - H->phase_flops_per_rhs[1];

  H->kfn_s = &grouped_gemm_f64<CFG_S, kKindNone, 1>;
  H->smem_s = gemm_smem_bytes<CFG_S, kKindNone, 1>();
  GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_s, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_s)));
  H->kfn_sn64 = &grouped_gemm_f64<CFG_SN64, kKindNone, 1>;
  H->smem_sn64 = gemm_smem_bytes<CFG_SN64, kKindNone, 1>();
  // skinny stored GEMMs (N2S of low-rank nodes: M = k << 128): the wide tiles' few, long CTAs
  H->kfn_sw = &grouped_gemm_f64<CFG_GW, kKindNone, 1>;
  H->smem_sw = gemm_smem_bytes<CFG_GW, kKindNone, 1>();
  GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_sw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_sw)));
  H->kfn_sn64w = &grouped_gemm_f64<CFG_GN64W, kKindNone, 1>;
  H->smem_sn64w = gemm_smem_bytes<CFG_GN64W, kKindNone, 1>();
  GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_sn64w, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_sn64w)));
  H->kfn_sg = &grouped_gemm_f64<CFG_G, kKindNone, 1>;
  H->smem_sg = gemm_smem_bytes<CFG_G, kKindNone, 1>();
  GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_sg, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_sg)));
  GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_sn64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_sn64)));
  if (!stored && (gen_near || gen_far)) {
    GenKernel gk = pick_gen_kernel(H->kernel, H->dim);
    H->kfn_g = gk.fn;
    H->smem_g = gk.smem;
    H->kfn_gw = gk.fn_wide;
    H->smem_gw = gk.smem_wide;
    H->kfn_gn64 = gk.fn_n64;
    H->smem_gn64 = gk.smem_n64;
    H->kfn_gn128 = gk.fn_n128;
    H->smem_gn128 = gk.smem_n128;
    H->kfn_gn64w = gk.fn_n64w;
    H->smem_gn64w = gk.smem_n64w;
    H->kfn_gm = gk.fn_m;
    H->smem_gm = gk.smem_m;
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_gm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_gm)));
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_gn64w, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_gn64w)));
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_gn64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_gn64)));
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_gn128, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_gn128)));
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_g, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_g)));
    GOFMM_CUDA(cudaFuncSetAttribute(H->kfn_gw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H->smem_gw)));
  }
  H->d_tiles.upload(H->tiles);
  // split-chain scratch rows extend skeleton space (what / c buffers, TMA maps)
  H->ld_s += pad16(H->scratch_rows);
  if (!H->reduces.empty()) {
    H->d_reduces.upload(H->reduces);
    H->d_reduce_src.upload(H->reduce_src);
  }
  H->d_groups.alloc(H->groups.size() * sizeof(Group), false);
  size_t nterms = 0;
  for (auto& g : H->groups) nterms += g.terms.size();
  H->d_terms.alloc(std::max<size_t>(nterms, 1) * sizeof(Term), false);

  // pack (own exports -> send buffer) and unpack (every other rank's exports -> workspace) tables
  if (H->nranks > 1) {
    std::vector<PanelSeg> segs;
    int64_t row = 0;
    for (const Seg& sg : H->dist.exports[H->drank]) {
      segs.push_back({sg.buf, 0, sg.row, row, sg.rows});
      row += sg.rows;
    }
    H->n_pack = int32_t(segs.size());
    for (int h = 0; h < H->nranks; ++h) {
      if (h == H->drank) continue;
      row = int64_t(h) * H->dist.max_send_rows;
      for (const Seg& sg : H->dist.exports[h]) {
        segs.push_back({sg.buf, 0, sg.row, row, sg.rows});
        row += sg.rows;
      }
    }
    H->n_unpack = int32_t(segs.size()) - H->n_pack;
    H->d_segs.upload(segs);
  }
  if (H->precision == GOFMM_PRECISION_F32) build_f32(H);
}

void ensure_workspace(gofmm_handle* H, int32_t r) {
  if (r <= H->ws_r) return;
  H->d_wp.alloc(size_t(H->ld_wp) * r * sizeof(double));
  H->d_what.alloc(size_t(H->ld_s) * r * sizeof(double));
  H->d_c.alloc(size_t(H->ld_s) * r * sizeof(double));
  H->ws_r = r;
  H->plan_uploaded = false;
  H->maps_r = 0;
}

// resolve host groups/terms into device structs against the current workspace pointers
void upload_plan(gofmm_handle* H) {
  if (H->plan_uploaded) return;
  std::vector<Group> gs;
  std::vector<Term> ts;
  gs.reserve(H->groups.size());
  const double* blobs[4] = {H->d_proj.as<double>(), H->d_diag.as<double>(), H->d_near.as<double>(),
                            H->d_far.as<double>()};
  const double* xblobs[2] = {H->d_xp.as<double>(), H->d_xs.as<double>()};
  auto bid = [](Buf b) {
    switch (b) {
      case Buf::Wp: return int32_t(kBufWp);
      case Buf::What: return int32_t(kBufWhat);
      default: return int32_t(kBufC);
    }
  };
  // one TMA view per stored-A term (64-byte aligned 128-byte descriptors in global memory)
  size_t n_amaps = 0;
  for (const HostGroup& hg : H->groups)
    for (const HostTerm& ht : hg.terms)
      if (ht.kind == 0 && blobs[ht.a_blob] && ht.K > 0 && hg.M > 0) ++n_amaps;
  std::vector<CUtensorMap> amaps;
  amaps.reserve(n_amaps);
  H->d_amaps.alloc(std::max<size_t>(n_amaps, 1) * sizeof(CUtensorMap), false);
  const CUtensorMap* amap_base = H->d_amaps.as<CUtensorMap>();
  for (const HostGroup& hg : H->groups) {
    Group g{};
    g.crow = hg.c_row;
    g.M = hg.M;
    g.flags = hg.flags;
    g.tbeg = int(ts.size());
    for (const HostTerm& ht : hg.terms) {
      Term t{};
      t.bbuf = bid(ht.b_buf);
      t.b_row = ht.b_row;
      t.K = ht.K;
      if (ht.kind == 1) {
        t.flags = kTermGen;
        t.xr = xblobs[ht.x_blob] + ht.xr_off * H->dim;
        t.xc = xblobs[ht.x_blob] + ht.xc_off * H->dim;
        t.a = nullptr;
      } else {
        t.flags = ht.row_major ? kTermRowMajorA : 0;
        t.a = blobs[ht.a_blob] ? blobs[ht.a_blob] + ht.a_off : nullptr;
        t.lda = ht.lda;
        if (t.a && ht.K > 0 && hg.M > 0) {
          amaps.emplace_back();
          encode_amap(&amaps.back(), t.a, ht.lda, hg.M, ht.K, ht.row_major);
          t.amap = amap_base + (amaps.size() - 1);
        }
      }
      ts.push_back(t);
    }
    g.tend = int(ts.size());
    gs.push_back(g);
  }
  if (!amaps.empty())
    GOFMM_CUDA(cudaMemcpy(H->d_amaps.p, amaps.data(), amaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  GOFMM_CUDA(cudaMemcpy(H->d_groups.p, gs.data(), gs.size() * sizeof(Group), cudaMemcpyHostToDevice));
  if (!ts.empty()) GOFMM_CUDA(cudaMemcpy(H->d_terms.p, ts.data(), ts.size() * sizeof(Term), cudaMemcpyHostToDevice));
  H->plan_uploaded = true;
}

}  // namespace
}  // namespace gofmm

namespace gofmm {
namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return GOFMM_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return GOFMM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GOFMM_ERR_INVALID;
  }
}

// Enqueue one column chunk of an evaluation on `st`: W (original order, device) -> u_perm (device).
// stage 0: the whole evaluation; stage 1 / 2: the distributed halves around the all-gather
// (d_xbuf = this rank's send buffer / the gathered receive buffer).
// B operand tensor maps over the FP64 workspace buffers for this column count
void encode_maps(gofmm_handle* H, int32_t r) {
  if (H->maps_r == r) return;
  {
    const double* bufs[3] = {H->d_wp.as<double>(), H->d_what.as<double>(), H->d_c.as<double>()};
    const int64_t rows[3] = {H->ld_wp, H->ld_s, H->ld_s};
    for (int b = 0; b < 3; ++b) {
      encode_bmap(&H->maps_s.m[b], bufs[b], rows[b], r, H->ws_r, kBN_S);
      encode_bmap(&H->maps_g.m[b], bufs[b], rows[b], r, H->ws_r, kBN_G);
      encode_bmap(&H->maps_n64.m[b], bufs[b], rows[b], r, H->ws_r, 64);
    }
    H->maps_r = r;
  }
}

// kernel configuration of one launch for a chunk of r columns (tile list, B maps, N tile)
struct LaunchCfg {
  KernelFn fn;
  size_t smem;
  int bn;
  const BMaps* maps;
  int bm_class;  // tile list: kBM[bm_class] rows per tile
};
// Programmatic dependent launch: the level launches of one evaluation form a chain of dependent
// kernels; with the PDL attribute the next launch's CTAs are scheduled onto idle SMs as soon as
// every CTA of the running launch has started (griddepcontrol.launch_dependents in its prologue),
// run their own prologue, and block in griddepcontrol.wait until the running launch has completed
// and its writes are visible — the launch gap between dependent levels disappears. Every kernel
// launched this way calls griddepcontrol.wait before touching data an earlier launch writes.
template <class... P, class... A>
void launch_k(bool pdl, void (*fn)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  GOFMM_CUDA(cudaLaunchKernelEx(&cfg, fn, std::forward<A>(args)...));
}

// The widest tile that fits r is the most efficient per flop (generated entries and B tiles are
// amortised over more columns), but a launch with few or very unequal term chains is bounded by
// its longest chain, which a narrower N tile shortens (and multiplies the CTAs). Each candidate
// is costed as  (BM*BN / eff) * max(stage-work / SMs, longest chain)  and the cheapest is used:
// c2's upper downward levels (16-128 groups, chains up to 272 stages) run 64-column tiles.
LaunchCfg pick_launch_cfg(const gofmm_handle* H, const Launch& L, int32_t r) {
  struct Cand {
    LaunchCfg cfg;
    int bm;
    double eff;  // achieved fraction of the DMMA peak when the SMs are full (measured, rounded)
  };
  Cand c[6];
  int nc = 0;
  if (!L.gen) {
    if (use_wide(r)) c[nc++] = {{H->kfn_sw, H->smem_sw, kBN_GW, &H->maps_g, 2}, kBM_GW, 0.80};
    if (r > 128) c[nc++] = {{H->kfn_sg, H->smem_sg, kBN_G, &H->maps_g, 1}, kBM_G, 0.78};
    if (r > 64) c[nc++] = {{H->kfn_s, H->smem_s, kBN_S, &H->maps_s, 0}, kBM_S, 0.80};
    c[nc++] = {{H->kfn_sn64, H->smem_sn64, 64, &H->maps_n64, 1}, kBM_G, 0.60};
    c[nc++] = {{H->kfn_sn64w, H->smem_sn64w, 64, &H->maps_n64, 2}, kBM_GW, 0.40};
  } else {
    if (use_wide(r)) c[nc++] = {{H->kfn_gw, H->smem_gw, kBN_GW, &H->maps_g, 2}, kBM_GW, 0.81};
    if (r > 128) c[nc++] = {{H->kfn_g, H->smem_g, kBN_G, &H->maps_g, 1}, kBM_G, 0.75};
    if (r > 128 && H->gm_eff > 0) c[nc++] = {{H->kfn_gm, H->smem_gm, kBN_G, &H->maps_g, 2}, kBM_GW, H->gm_eff};
    if (r > 64) c[nc++] = {{H->kfn_gn128, H->smem_gn128, 128, &H->maps_s, 1}, kBM_G, 0.65};
    c[nc++] = {{H->kfn_gn64, H->smem_gn64, 64, &H->maps_n64, 1}, kBM_G, 0.55};
    c[nc++] = {{H->kfn_gn64w, H->smem_gn64w, 64, &H->maps_n64, 2}, kBM_GW, 0.40};
  }
  int best = 0;
  double best_t = 0.0;
  for (int i = 0; i < nc; ++i) {
    const int nt = (r + c[i].cfg.bn - 1) / c[i].cfg.bn;
    const double work = double(L.chain_sum[c[i].cfg.bm_class]) * nt / double(H->num_sms);
    // + a fixed cost per CTA (prologue, pipeline fill, epilogue ~ one 128x128 k-stage): launches of
    // many short chains (N2S of low-rank leaves: 1-3 stages per tile) are bound by it, not by math
    const double ctas = double(L.tn[c[i].cfg.bm_class]) * nt / double(H->num_sms);
    const double t = double(c[i].bm) * c[i].cfg.bn / c[i].eff * std::max(work, double(L.chain_max)) +
                     kCtaOverheadArea * ctas;
    if (i == 0 || t < best_t) {
      best = i;
      best_t = t;
    }
  }
  return c[best].cfg;
}

// Which plan launches an enqueue of `stage` runs. 0: a whole single-GPU evaluation; the two-call
// distributed API: 1 (before the all-gather) and 2 (after it: stage-2 and stage-3 launches);
// gofmm_dist_evaluate splits the second half into 3 (own D + near output terms, overlapping the
// all-gather) and 4 (the rest, after it).
inline bool stage_runs(int stage, int launch_stage) {
  switch (stage) {
    case 0: return true;
    case 2: return launch_stage == 2 || launch_stage == 3;
    case 4: return launch_stage == 2;
    default: return launch_stage == stage;
  }
}

// rows_done (host-buffer pipeline, stage 0 only): called after each part of a split output
// launch is enqueued, with the u_perm rows that part completes; returns whether it was used.
using RowsDone = std::function<void(int64_t row0, int64_t row1)>;

// Column pieces (host-buffer pipeline, stage 0): with c1 >= 0 only the permutation and the upward
// (N2S) launches run, for columns [c0, c1) — N2S is column-separable, so a piece can start as
// soon as its W columns have landed; phase_lo = 1 then runs the rest without the permutation.
void enqueue_chunk(gofmm_handle* H, const double* d_w, int64_t ldw, int32_t r, double* d_u, int64_t ldu,
                   cudaStream_t st, bool timed, int stage = 0, double* d_xbuf = nullptr,
                   const RowsDone* rows_done = nullptr, bool* rows_used = nullptr, int phase_lo = 0,
                   int32_t c0 = 0, int32_t c1 = -1) {
  const bool piece = c1 >= 0;
  ensure_workspace(H, r);
  upload_plan(H);
  encode_maps(H, r);
  if (timed) GOFMM_CUDA(cudaEventRecord(H->ev[0], st));
  if ((stage == 2 || stage == 4) && H->n_unpack > 0) {
    // ghosts: every other rank's exported what / W rows into their places in this workspace
    dim3 grid(unsigned(H->n_unpack), 8);
    panel_copy<<<grid, 256, 0, st>>>(H->d_segs.as<PanelSeg>() + H->n_pack, H->d_what.as<double>(),
                                     H->d_wp.as<double>(), int64_t(H->ws_r) * 16, d_xbuf, r, 0);
  }
  if ((stage == 0 || stage == 1) && phase_lo == 0) {
    // K5: row gather into the padded leaf layout (evaluate.hpp:294-295). Blocks walk all rows of
    // cpb columns before the next columns (grid.x = rows), so the randomly gathered source
    // columns (N * cpb * 8 bytes) stay L2-resident: each 32-byte sector is fetched from HBM once.
    // Stage 1 permutes every row too: W is replicated, so the near-field partners' rows a rank
    // needs come from its own copy of W instead of the all-gather.
    const int cpb = int(std::max<int64_t>(1, std::min<int64_t>(8, (48ll << 20) / (int64_t(H->n) * 8))));
    const int64_t row0 = 0, row1 = H->ld_wp;
    const int32_t pc0 = piece ? c0 : 0, pr = piece ? c1 - c0 : r;  // columns of this piece
    if (row1 > row0 && pr > 0) {
      const int rpt = perm_rows_per_thread(row1 - row0, pr);
      dim3 grid(unsigned((row1 - row0 + 256 * rpt - 1) / (256 * rpt)), unsigned((pr + cpb - 1) / cpb));
      auto* kern = rpt == kPermRows ? &permute_rows_in<kPermRows> : &permute_rows_in<1>;
      kern<<<grid, 256, 0, st>>>(d_w + size_t(pc0) * ldw, ldw, H->d_prow.as<int32_t>(), row0, row1, pr, cpb,
                                 H->d_wp.as<double>() + 16 * size_t(pc0), int64_t(H->ws_r) * 16);
    }
  }
  // ev[1 + p] marks the start of phase p (0 upward, 1 downward, 2 output); ev[4] the end
  if (timed) GOFMM_CUDA(cudaEventRecord(H->ev[1], st));
  int marked = 1;
  for (const Launch& L : H->launches) {
    if (!stage_runs(stage, L.stage)) continue;
    if (piece && L.phase != 0) continue;
    if (L.phase < phase_lo) {  // ran in the column pieces: zero-length timing pair
      const size_t li = size_t(&L - H->launches.data());
      if (timed) {
        GOFMM_CUDA(cudaEventRecord(H->lev[2 * li], st));
        GOFMM_CUDA(cudaEventRecord(H->lev[2 * li + 1], st));
      }
      continue;
    }
    while (timed && marked <= L.phase) GOFMM_CUDA(cudaEventRecord(H->ev[1 + marked++], st));
    double* cbase;
    int64_t ldc;
    int32_t cpanel = 1;  // what / c: panel layout with panel stride 16*r_ws
    switch (L.out) {
      case Buf::What: cbase = H->d_what.as<double>(); ldc = int64_t(H->ws_r) * 16; break;
      case Buf::C: cbase = H->d_c.as<double>(); ldc = int64_t(H->ws_r) * 16; break;
      default: cbase = d_u; ldc = ldu; cpanel = 0; break;  // u_perm: caller's column-major buffer
    }
    const size_t li = size_t(&L - H->launches.data());
    if (timed) GOFMM_CUDA(cudaEventRecord(H->lev[2 * li], st));
    // a column piece picks its tile for the piece's width: a wider N tile would also compute (and
    // read W for) columns of pieces that have not landed yet
    const LaunchCfg cfg = pick_launch_cfg(H, L, piece ? c1 - c0 : r);
    const int32_t n_off = piece ? c0 : 0, ncols = piece ? c1 - c0 : r;
    auto run = [&](int t0, int nt) {
      if (nt <= 0 || ncols <= 0) return;
      dim3 grid(unsigned(nt), unsigned((ncols + cfg.bn - 1) / cfg.bn));
      launch_k(H->pdl && !timed, cfg.fn, grid, dim3(kThreadsG), cfg.smem, st, *cfg.maps, H->d_tiles.as<Tile>() + t0,
               H->d_groups.as<Group>(), H->d_terms.as<Term>(), r, H->kp, cbase, ldc, cpanel, n_off);
    };
    // split only launches of many waves: on small trees the extra launches cost more than the
    // download they hide (config 1: 128 output tiles)
    if (rows_done && stage == 0 && L.out == Buf::Out && !L.parts.empty() && L.tn[1] >= 8 * H->num_sms) {
      for (size_t p = 0; p + 1 < L.parts.size(); ++p) {
        const Launch::Part &a = L.parts[p], &b = L.parts[p + 1];
        run(a.tile[cfg.bm_class], b.tile[cfg.bm_class] - a.tile[cfg.bm_class]);
        (*rows_done)(a.row, b.row);
      }
      if (rows_used) *rows_used = true;
    } else {
      run(L.tfirst[cfg.bm_class], L.tn[cfg.bm_class]);
    }
    if (L.reduce_n > 0 && !piece) {  // split term chains: segments 1.. into the group rows
      dim3 grid(unsigned(L.reduce_n), 8);
      launch_k(H->pdl && !timed, chain_reduce, grid, dim3(256), 0, st, H->d_reduces.as<ChainReduce>() + L.reduce_first,
               H->d_reduce_src.as<int64_t>(), cbase, ldc, r);
    }
    if (timed) GOFMM_CUDA(cudaEventRecord(H->lev[2 * li + 1], st));
  }
  if (stage == 1 && H->n_pack > 0) {
    dim3 grid(unsigned(H->n_pack), 8);
    panel_copy<<<grid, 256, 0, st>>>(H->d_segs.as<PanelSeg>(), H->d_what.as<double>(), H->d_wp.as<double>(),
                                     int64_t(H->ws_r) * 16, d_xbuf, r, 1);
  }
  if (timed) {
    while (marked <= 2) GOFMM_CUDA(cudaEventRecord(H->ev[1 + marked++], st));
    GOFMM_CUDA(cudaEventRecord(H->ev[4], st));
  }
  GOFMM_CUDA(cudaGetLastError());
}

// add the event-measured phase / launch durations of the chunk just enqueued (timed mode)
void accumulate_chunk_times(gofmm_handle* H) {
  GOFMM_CUDA(cudaEventSynchronize(H->ev[4]));
  for (size_t i = 0; i < H->launches.size(); ++i) {
    float ms;
    GOFMM_CUDA(cudaEventElapsedTime(&ms, H->lev[2 * i], H->lev[2 * i + 1]));
    H->launch_ms[i] += ms;
  }
  for (int i = 0; i < 4; ++i) {
    float ms;
    GOFMM_CUDA(cudaEventElapsedTime(&ms, H->ev[i], H->ev[i + 1]));
    H->phase_ms[i] += ms;
  }
}

// Column chunk for this r: evaluation is column-separable, so r beyond what the
// workspace (W_perm + what + c, ~8*(ld_wp + 2*ld_s) bytes per column) fits in HBM is processed
// in chunks (config 5: N = 2^22, r = 1024).
int32_t rhs_chunk(gofmm_handle* H, int32_t r) {
  if (H->max_chunk > 0) return std::min(r, H->max_chunk);
  if (r <= H->ws_r) return r;
  size_t free_b = 0, total_b = 0;
  GOFMM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double per_col = 8.0 * double(H->ld_wp + 2 * H->ld_s);
  const double avail = 0.85 * double(free_b) + per_col * H->ws_r;  // current workspace is reusable
  int64_t cols = int64_t(avail / per_col);
  if (cols >= r) return r;
  if (cols >= kBN_GW)
    cols = (cols / kBN_GW) * kBN_GW;
  else if (cols >= kBN_G)
    cols = (cols / kBN_G) * kBN_G;
  if (cols < 1) throw Error(GOFMM_ERR_CUDA, "not enough device memory for one right-hand side");
  return int32_t(cols);
}

// Replay a captured graph of `body` (which enqueues one whole evaluation on the stream it is
// given) on `st`; the capture is redone whenever the key (buffers, r, workspace) changes.
template <class Body>
void graph_replay(gofmm_handle* H, const decltype(gofmm_handle::gkey)& key, cudaStream_t st, Body&& body) {
  if (!(H->gexec && H->gkey == key)) {
    if (H->gexec) {
      GOFMM_CUDA(cudaGraphExecDestroy(H->gexec));
      H->gexec = nullptr;
    }
    if (!H->cap_stream) GOFMM_CUDA(cudaStreamCreateWithFlags(&H->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    GOFMM_CUDA(cudaStreamBeginCapture(H->cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      body(H->cap_stream);
    } catch (...) {
      cudaStreamEndCapture(H->cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    GOFMM_CUDA(cudaStreamEndCapture(H->cap_stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&H->gexec, g, 0);
    cudaGraphDestroy(g);
    GOFMM_CUDA(e);
    H->gkey = key;
  }
  GOFMM_CUDA(cudaGraphLaunch(H->gexec, st));
}

// Enqueue a whole evaluation (all column chunks).
void enqueue(gofmm_handle* H, const double* d_w, int64_t ldw, int32_t r, double* d_u, int64_t ldu, cudaStream_t st,
             bool timed, const RowsDone* rows_done = nullptr, bool* rows_used = nullptr) {
  const int32_t rc = rhs_chunk(H, r);
  if (H->graphs && !timed && !rows_done && rc >= r) {
    // everything that allocates or copies synchronously happens before the capture
    ensure_workspace(H, r);
    upload_plan(H);
    encode_maps(H, r);
    graph_replay(H, {d_w, ldw, d_u, ldu, r, H->ws_r, 64}, st,
                 [&](cudaStream_t cs) { enqueue_chunk(H, d_w, ldw, r, d_u, ldu, cs, false); });
    return;
  }
  if (timed) {
    H->launch_ms.assign(H->launches.size(), 0.f);
    std::fill(std::begin(H->phase_ms), std::end(H->phase_ms), 0.f);
  }
  if (rc < r) rows_done = nullptr;  // the hook covers a single-chunk evaluation only
  for (int32_t c0 = 0; c0 < r; c0 += rc) {
    const int32_t rr = std::min(rc, r - c0);
    enqueue_chunk(H, d_w + size_t(c0) * ldw, ldw, rr, d_u + size_t(c0) * ldu, ldu, st, timed, 0, nullptr, rows_done,
                  rows_used);
    if (timed) accumulate_chunk_times(H);
  }
}

// ---------------------------------------------------------------- FP32 evaluation
void ensure_workspace32(gofmm_handle* H, int32_t r) {
  if (r <= H->ws32_r) return;
  for (int p = 0; p < 2; ++p) {
    H->d_wp32[p].alloc(size_t(H->ld_wp) * r * sizeof(float));
    H->d_what32[p].alloc(size_t(H->ld_s) * r * sizeof(float));
    H->d_c32[p].alloc(size_t(H->ld_s) * r * sizeof(float));
  }
  H->ws32_r = r;
  for (auto& v : H->maps32_rv) v = 0;
}

// B operand view of an FP32 panel buffer: {16 rows-in-panel, r columns, rows/16 panels}, boxes
// of 16 x bn, 64-byte swizzle = the K-major SWIZZLE_64B UMMA operand layout
void encode_bmap32(CUtensorMap* map, const float* ptr, int64_t rows, int32_t r, int32_t r_ws, int bn) {
  cuuint64_t dims[3] = {16, cuuint64_t(r), cuuint64_t(rows / 16)};
  cuuint64_t strides[2] = {16 * sizeof(float), cuuint64_t(r_ws) * 16 * sizeof(float)};
  cuuint32_t box[3] = {16, cuuint32_t(bn), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult rc = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw Error(GOFMM_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed: " + std::to_string(int(rc)));
}

// FP32 kernels for this column count (N tile) and the B tensor maps over the workspace
void prepare32(gofmm_handle* H, int32_t r) {
  {  // two-pass permutation for W >= 4 GB (enqueue_chunk32) when its row-major scratch fits in HBM
    const int64_t ldt = (int64_t(r) + 3) & ~int64_t(3);
    const size_t need = size_t(H->n) * size_t(ldt) * sizeof(float);
    H->perm2_on = H->perm2 >= 0 ? H->perm2 == 1 : double(H->n) * double(r) * sizeof(float) >= double(4ll << 30);
    if (H->perm2_on && H->d_perm32.bytes < need) {
      size_t free_b = 0, total_b = 0;
      GOFMM_CUDA(cudaMemGetInfo(&free_b, &total_b));
      if (free_b > need + (size_t(2) << 30))
        H->d_perm32.alloc(need, false);
      else
        H->perm2_on = false;
    }
  }
  const float* bufs[3][2] = {{H->d_wp32[0].as<float>(), H->d_wp32[1].as<float>()},
                             {H->d_what32[0].as<float>(), H->d_what32[1].as<float>()},
                             {H->d_c32[0].as<float>(), H->d_c32[1].as<float>()}};
  const int64_t rows[3] = {H->ld_wp, H->ld_s, H->ld_s};
  for (int v = 0; v < 3; ++v) {
    const int bn = 64 << v;
    if (bn > f32_bn(r)) break;  // N tiles wider than the chunk's columns are never picked
    if (!H->k32_s[v].fn) {
      H->k32_s[v] = f32::pick_gemm(kKindNone, 1, bn);
      if (H->kfn_g) H->k32_g[v] = f32::pick_gemm(H->kernel, H->dim, bn);
      GOFMM_CUDA(cudaGetLastError());
    }
    if (H->maps32_rv[v] != r) {
      for (int b = 0; b < 3; ++b)
        for (int p = 0; p < 2; ++p) encode_bmap32(&H->maps32[v].m[b][p], bufs[b][p], rows[b], r, H->ws32_r, bn);
      H->maps32_rv[v] = r;
    }
  }
}

// N tile of one FP32 launch: the widest tile that fits the chunk is the most efficient per flop;
// a launch whose tiles leave most SMs idle (the upper tree levels: 2-64 tiles) halves its N tile
// while the doubled CTA count still fits on the SMs — each CTA's chain runs on fewer columns.
// (Narrowing a launch that already fills the SMs was measured slower: c2 downward levels 7-8.)
int pick_bn32(const gofmm_handle* H, const Launch& L, int32_t r) {
  int v = 0;
  while (v < 2 && (64 << (v + 1)) <= f32_bn(r)) ++v;
  while (v > 0 && int64_t(L.ntiles32) * ((r + (64 << (v - 1)) - 1) / (64 << (v - 1))) <= H->num_sms) --v;
  return v;
}

// stage 0: the whole evaluation; stage 1 / 2: the distributed halves around the all-gather
// (d_xbuf = this rank's send buffer / the gathered receive buffer, hi/lo slots, see panel_copy_f32)
void enqueue_chunk32(gofmm_handle* H, const float* d_w, int64_t ldw, int32_t r, float* d_u, int64_t ldu,
                     cudaStream_t st, bool timed, int stage = 0, float* d_xbuf = nullptr,
                     const RowsDone* rows_done = nullptr, bool* rows_used = nullptr) {
  ensure_workspace32(H, r);
  prepare32(H, r);
  const int64_t pstride = int64_t(H->ws32_r) * 16;
  if (timed) GOFMM_CUDA(cudaEventRecord(H->ev[0], st));
  if ((stage == 2 || stage == 4) && H->n_unpack > 0)  // ghosts: other ranks' exported what
    GOFMM_CUDA(f32::launch_panel_copy(H->d_segs.as<PanelSeg>() + H->n_pack, H->n_unpack, H->d_what32[0].as<float>(),
                                      H->d_what32[1].as<float>(), H->d_wp32[0].as<float>(), H->d_wp32[1].as<float>(),
                                      pstride, d_xbuf, r, H->dist.max_send_rows, 0, st));
  if (stage == 0 || stage == 1) {  // every row, also in stage 1 (W is replicated, see enqueue_chunk)
    const int64_t row0 = 0, row1 = H->ld_wp;
    // large W (>= 4 GB): transpose + coalesced row gather (scratch sized in prepare32, before any
    // graph capture)
    const int64_t ldt = (int64_t(r) + 3) & ~int64_t(3);
    const bool two_pass = H->perm2_on && H->d_perm32.bytes >= size_t(H->n) * size_t(ldt) * sizeof(float);
    if (two_pass)
      GOFMM_CUDA(f32::launch_permute_in_2pass(d_w, ldw, H->d_prow.as<int32_t>(), row0, row1, r, H->n,
                                              H->d_wp32[0].as<float>(), H->d_wp32[1].as<float>(), pstride,
                                              H->d_perm32.as<float>(), ldt, st));
    else
      GOFMM_CUDA(f32::launch_permute_in(d_w, ldw, H->d_prow.as<int32_t>(), row0, row1, r, H->n,
                                      H->d_wp32[0].as<float>(), H->d_wp32[1].as<float>(), pstride, st));
  }
  if (timed) GOFMM_CUDA(cudaEventRecord(H->ev[1], st));
  int marked = 1;
  for (const Launch& L : H->launches) {
    if (!stage_runs(stage, L.stage)) continue;
    while (timed && marked <= L.phase) GOFMM_CUDA(cudaEventRecord(H->ev[1 + marked++], st));
    float *ch, *cl;
    int64_t ldc;
    int32_t cpanel = 1;
    switch (L.out) {
      case Buf::What: ch = H->d_what32[0].as<float>(); cl = H->d_what32[1].as<float>(); ldc = pstride; break;
      case Buf::C: ch = H->d_c32[0].as<float>(); cl = H->d_c32[1].as<float>(); ldc = pstride; break;
      default: ch = d_u; cl = nullptr; ldc = ldu; cpanel = 0; break;
    }
    const size_t li = size_t(&L - H->launches.data());
    if (timed) GOFMM_CUDA(cudaEventRecord(H->lev[2 * li], st));
    const int v = pick_bn32(H, L, r);
    const f32::GemmKernel& k = L.gen ? H->k32_g[v] : H->k32_s[v];
    if (rows_done && stage == 0 && L.out == Buf::Out && !L.parts.empty() && L.ntiles32 >= 8 * H->num_sms) {
      for (size_t p = 0; p + 1 < L.parts.size(); ++p) {
        const int t0 = L.parts[p].tile32, nt = L.parts[p + 1].tile32 - t0;
        if (nt > 0)
          GOFMM_CUDA(f32::launch_gemm(k, unsigned(nt), r, H->maps32[v], H->d_tiles32.as<Tile>() + t0,
                                      H->d_groups.as<Group>(), H->d_terms32.as<f32::Term>(), H->kp32, ch, cl, ldc,
                                      cpanel, st, H->pdl && !timed));
        (*rows_done)(L.parts[p].row, L.parts[p + 1].row);
      }
      if (rows_used) *rows_used = true;
    } else {
      GOFMM_CUDA(f32::launch_gemm(k, unsigned(L.ntiles32), r, H->maps32[v], H->d_tiles32.as<Tile>() + L.first_tile32,
                                  H->d_groups.as<Group>(), H->d_terms32.as<f32::Term>(), H->kp32, ch, cl, ldc, cpanel,
                                  st, H->pdl && !timed));
    }
    if (L.reduce_n > 0)  // split term chains: segments 1.. into the group rows
      GOFMM_CUDA(f32::launch_chain_reduce(H->d_reduces.as<ChainReduce>() + L.reduce_first, L.reduce_n,
                                          H->d_reduce_src.as<int64_t>(), ch, cl, ldc, r, st, H->pdl && !timed));
    if (timed) GOFMM_CUDA(cudaEventRecord(H->lev[2 * li + 1], st));
  }
  if (stage == 1 && H->n_pack > 0)
    GOFMM_CUDA(f32::launch_panel_copy(H->d_segs.as<PanelSeg>(), H->n_pack, H->d_what32[0].as<float>(),
                                      H->d_what32[1].as<float>(), H->d_wp32[0].as<float>(), H->d_wp32[1].as<float>(),
                                      pstride, d_xbuf, r, H->dist.max_send_rows, 1, st));
  if (timed) {
    while (marked <= 2) GOFMM_CUDA(cudaEventRecord(H->ev[1 + marked++], st));
    GOFMM_CUDA(cudaEventRecord(H->ev[4], st));
  }
  GOFMM_CUDA(cudaGetLastError());
}

int32_t rhs_chunk32(gofmm_handle* H, int32_t r) {
  if (H->max_chunk > 0) return std::min(r, H->max_chunk);
  if (r <= H->ws32_r) return r;
  size_t free_b = 0, total_b = 0;
  GOFMM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double per_col = 8.0 * double(H->ld_wp + 2 * H->ld_s);  // hi + lo floats
  const double avail = 0.85 * double(free_b) + per_col * H->ws32_r;
  int64_t cols = int64_t(avail / per_col);
  if (cols >= r) return r;
  if (cols >= 256) cols = (cols / 256) * 256;
  if (cols < 1) throw Error(GOFMM_ERR_CUDA, "not enough device memory for one right-hand side");
  return int32_t(cols);
}

void enqueue32(gofmm_handle* H, const float* d_w, int64_t ldw, int32_t r, float* d_u, int64_t ldu, cudaStream_t st,
               bool timed, const RowsDone* rows_done = nullptr, bool* rows_used = nullptr) {
  const int32_t rc = rhs_chunk32(H, r);
  if (H->graphs && !timed && !rows_done && rc >= r) {
    ensure_workspace32(H, r);
    prepare32(H, r);
    graph_replay(H, {d_w, ldw, d_u, ldu, r, H->ws32_r, 32}, st,
                 [&](cudaStream_t cs) { enqueue_chunk32(H, d_w, ldw, r, d_u, ldu, cs, false); });
    return;
  }
  if (timed) {
    H->launch_ms.assign(H->launches.size(), 0.f);
    std::fill(std::begin(H->phase_ms), std::end(H->phase_ms), 0.f);
  }
  if (rc < r) rows_done = nullptr;  // the hook covers a single-chunk evaluation only
  for (int32_t c0 = 0; c0 < r; c0 += rc) {
    const int32_t rr = std::min(rc, r - c0);
    enqueue_chunk32(H, d_w + size_t(c0) * ldw, ldw, rr, d_u + size_t(c0) * ldu, ldu, st, timed, 0, nullptr,
                    rows_done, rows_used);
    if (timed) accumulate_chunk_times(H);
  }
}

void check_precision(const gofmm_handle* H, int32_t want) {
  if (H && H->precision != want)
    throw Error(GOFMM_ERR_INVALID, want == GOFMM_PRECISION_F32
                                       ? "fp32 entry point on an fp64 handle (create with precision GOFMM_PRECISION_F32)"
                                       : "fp64 entry point on an fp32 handle (use the *_f32 entry points)");
}

void fill_phase_times(gofmm_handle* H, gofmm_eval_stats* s) {
  s->ms_permute = H->phase_ms[0];
  s->ms_upward = H->phase_ms[1];
  s->ms_downward = H->phase_ms[2];
  s->ms_output = H->phase_ms[3];
}

void check_args(gofmm_handle* H, const void* w, int64_t ldw, int32_t r, const void* u, int64_t ldu) {
  if (!H) throw Error(GOFMM_ERR_INVALID, "null handle");
  // evaluate.hpp:288-289
  if (r < 1) throw Error(GOFMM_ERR_INVALID, "evaluate: w needs at least one column");
  if (ldw < H->n) throw Error(GOFMM_ERR_INVALID, "evaluate: w has wrong row count");
  if (ldu < H->n) throw Error(GOFMM_ERR_INVALID, "evaluate: u has wrong row count");
  if (!w || !u) throw Error(GOFMM_ERR_INVALID, "evaluate: null buffer");
}

// A subtree-split handle holds only its rank's groups: a whole-matrix evaluation on it would
// leave other ranks' rows of u unwritten and read what rows nobody computed.
void check_single(const gofmm_handle* H) {
  if (H->nranks > 1)
    throw Error(GOFMM_ERR_INVALID,
                "evaluate: handle is one rank of a subtree split (nranks > 1); use gofmm_dist_evaluate "
                "or gofmm_dist_stage1 / gofmm_dist_stage2");
}

// Ownership of the handle's device workspace for one enqueue on `st` (gofmm_handle::ws_free):
// wait for the previous enqueue (any stream) to finish with it, release it after ours.
struct WsGuard {
  gofmm_handle* H;
  cudaStream_t st;
  WsGuard(gofmm_handle* h, cudaStream_t s) : H(h), st(s) { GOFMM_CUDA(cudaStreamWaitEvent(st, H->ws_free, 0)); }
  ~WsGuard() { cudaEventRecord(H->ws_free, st); }
  WsGuard(const WsGuard&) = delete;
  WsGuard& operator=(const WsGuard&) = delete;
};

}  // namespace
}  // namespace gofmm

using namespace gofmm;

extern "C" {

int32_t gofmm_abi_version(void) { return 2; }

const char* gofmm_last_error(void) { return g_last_error.c_str(); }

int gofmm_create(const gofmm_tree_desc* desc, const gofmm_options* opts, gofmm_handle** out) {
  return guarded([&] {
    if (!out) throw Error(GOFMM_ERR_INVALID, "null output handle");
    *out = nullptr;
    validate(desc);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(GOFMM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    auto H = std::make_unique<gofmm_handle>();
    H->device = opts ? opts->device : 0;
    GOFMM_CUDA(cudaSetDevice(H->device));
    GOFMM_CUDA(cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, H->device));
    GOFMM_CUDA(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
    for (auto& e : H->ev) GOFMM_CUDA(cudaEventCreate(&e));
    GOFMM_CUDA(cudaEventCreateWithFlags(&H->ws_free, cudaEventDisableTiming));
    build(H.get(), desc, opts);
    H->lev.assign(2 * H->launches.size(), nullptr);
    for (auto& e : H->lev) GOFMM_CUDA(cudaEventCreate(&e));
    *out = H.release();
  });
}

int gofmm_create_dist(const gofmm_tree_desc* desc, const gofmm_options* opts, int32_t rank, int32_t nranks,
                      gofmm_handle** out) {
  return guarded([&] {
    if (!out) throw Error(GOFMM_ERR_INVALID, "null output handle");
    *out = nullptr;
    validate(desc);
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(GOFMM_ERR_INVALID, "bad rank / nranks");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(GOFMM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    auto H = std::make_unique<gofmm_handle>();
    H->device = opts ? opts->device : 0;
    H->drank = rank;
    H->nranks = nranks;
    GOFMM_CUDA(cudaSetDevice(H->device));
    GOFMM_CUDA(cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, H->device));
    GOFMM_CUDA(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
    for (auto& e : H->ev) GOFMM_CUDA(cudaEventCreate(&e));
    GOFMM_CUDA(cudaEventCreateWithFlags(&H->ws_free, cudaEventDisableTiming));
    build(H.get(), desc, opts);
    H->lev.assign(2 * H->launches.size(), nullptr);
    for (auto& e : H->lev) GOFMM_CUDA(cudaEventCreate(&e));
    *out = H.release();
  });
}

static void fill_dist_info(const DistPlan& P, int32_t rank, int64_t own_begin, int64_t own_end, int64_t flops,
                           int64_t full, gofmm_dist_info* info) {
  std::memset(info, 0, sizeof(*info));
  info->rank = rank;
  info->nranks = P.nranks;
  info->split_level = P.split;
  info->send_rows = P.send_rows.empty() ? 0 : P.send_rows[rank];
  info->max_send_rows = P.max_send_rows;
  info->own_row_begin = own_begin;
  info->own_row_end = own_end;
  info->flops_per_rhs = flops;
  info->full_flops_per_rhs = full;
  info->n_exports = P.exports.empty() ? 0 : int32_t(P.exports[rank].size());
}

int gofmm_dist_get_info(const gofmm_handle* H, gofmm_dist_info* info) {
  return guarded([&] {
    if (!H || !info) throw Error(GOFMM_ERR_INVALID, "null argument");
    fill_dist_info(H->dist, H->drank, H->own_begin, H->own_end, H->flops_per_rhs, H->full_flops_per_rhs, info);
  });
}

int gofmm_dist_plan_host(const gofmm_tree_desc* d, int32_t rank, int32_t nranks, gofmm_dist_info* info,
                         int32_t cap, int32_t* export_ids) {
  return guarded([&] {
    validate(d);
    if (rank < 0 || rank >= nranks) throw Error(GOFMM_ERR_INVALID, "bad rank / nranks");
    DistPlan P = make_dist_plan(nranks, d->num_nodes, d->left, d->right, d->level, d->start, d->end, d->rank,
                                d->num_near, d->near_a, d->near_b, d->num_far, d->far_a, d->far_b);
    int64_t ob = d->n, oe = 0;
    for (int i = 0; i < d->num_nodes; ++i)
      if (d->left[i] < 0 && P.owner[i] == rank) {
        ob = std::min<int64_t>(ob, d->start[i]);
        oe = std::max<int64_t>(oe, d->end[i]);
      }
    if (info) fill_dist_info(P, rank, ob, oe, 0, 0, info);
    if (export_ids) {
      // node id of every exported segment: what segments as the node id, W segments as -(leaf+1)
      int32_t k = 0;
      std::vector<int64_t> soff(d->num_nodes, -1), pst(d->num_nodes, -1);
      int64_t off = 0;
      for (int i = 0; i < d->num_nodes; ++i)
        if (d->rank[i] >= 0) {
          soff[i] = off;
          off += pad16_(d->rank[i]);
        }
      std::vector<int> leaves;
      for (int i = 0; i < d->num_nodes; ++i)
        if (d->left[i] < 0) leaves.push_back(i);
      std::sort(leaves.begin(), leaves.end(), [&](int a, int b) { return d->start[a] < d->start[b]; });
      off = 0;
      for (int i : leaves) {
        pst[i] = off;
        off += pad16_(d->end[i] - d->start[i]);
      }
      for (const Seg& sg : P.exports[rank]) {
        if (k >= cap) break;
        int id = -1;
        for (int i = 0; i < d->num_nodes && id < 0; ++i)
          if ((sg.buf == 0 && soff[i] == sg.row && d->rank[i] >= 0) || (sg.buf == 1 && pst[i] == sg.row && d->left[i] < 0))
            id = i;
        export_ids[k++] = sg.buf == 0 ? id : -(id + 1);
      }
    }
  });
}

int gofmm_dist_stage1(gofmm_handle* H, const double* d_w, int64_t ldw, int32_t r, double* d_send, void* stream) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_w, H->n);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F64);
    if (H->nranks > 1 && !d_send && H->dist.max_send_rows > 0) throw Error(GOFMM_ERR_INVALID, "null send buffer");
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    enqueue_chunk(H, d_w, ldw, r, nullptr, H->n, st, false, 1, d_send);
  });
}

int gofmm_dist_stage2(gofmm_handle* H, const double* d_recv, int32_t r, double* d_u, int64_t ldu, void* stream) {
  return guarded([&] {
    check_args(H, d_u, H->n, r, d_u, ldu);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F64);
    if (H->nranks > 1 && !d_recv && H->dist.max_send_rows > 0) throw Error(GOFMM_ERR_INVALID, "null receive buffer");
    if (r > H->ws_r) throw Error(GOFMM_ERR_INVALID, "stage2: r differs from stage1");
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    enqueue_chunk(H, nullptr, H->n, r, d_u, ldu, st, false, 2, const_cast<double*>(d_recv));
  });
}

int gofmm_dist_stage1_f32(gofmm_handle* H, const float* d_w, int64_t ldw, int32_t r, float* d_send, void* stream) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_w, H->n);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F32);
    if (H->nranks > 1 && !d_send && H->dist.max_send_rows > 0) throw Error(GOFMM_ERR_INVALID, "null send buffer");
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    enqueue_chunk32(H, d_w, ldw, r, nullptr, H->n, st, false, 1, d_send);
  });
}

int gofmm_dist_stage2_f32(gofmm_handle* H, const float* d_recv, int32_t r, float* d_u, int64_t ldu, void* stream) {
  return guarded([&] {
    check_args(H, d_u, H->n, r, d_u, ldu);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F32);
    if (H->nranks > 1 && !d_recv && H->dist.max_send_rows > 0) throw Error(GOFMM_ERR_INVALID, "null receive buffer");
    if (r > H->ws32_r) throw Error(GOFMM_ERR_INVALID, "stage2: r differs from stage1");
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    enqueue_chunk32(H, nullptr, H->n, r, d_u, ldu, st, false, 2, const_cast<float*>(d_recv));
  });
}

}  // extern "C"

namespace {
// One distributed evaluation on the handle's own data plane (north_star (4)): stage 1 (full
// permutation, own-subtree N2S, pack of the exported skeleton weights) -> ncclAllGather on a
// high-priority stream -> stage 4 (unpack, top-of-tree N2S, downward, proj^T c output). The own
// leaves' D + near output terms (stage 3) read only W, so they run on `st` WHILE the all-gather
// is in flight. ms3 (timed): {stage 1, all-gather, whole evaluation} in ms.
template <class T>
void dist_evaluate(gofmm_handle* H, const T* d_w, int64_t ldw, int32_t r, T* d_u, int64_t ldu, cudaStream_t st,
                   bool timed, double* ms3) {
  constexpr bool kF32 = sizeof(T) == 4;
  std::string why;
  const nccl::Api* api = nullptr;
  if (H->comm) {
    api = nccl::api(&why);
    if (!api) throw Error(GOFMM_ERR_CUDA, why);
  } else if (H->nranks > 1) {
    throw Error(GOFMM_ERR_INVALID, "gofmm_dist_evaluate: no communicator (gofmm_dist_init_comm / _attach_comm)");
  }
  const size_t slot = size_t(H->dist.max_send_rows) * size_t(r) * (kF32 ? 2 : 1);  // elements per rank
  if (H->d_send.bytes < std::max<size_t>(slot, 1) * sizeof(T)) H->d_send.alloc(std::max<size_t>(slot, 1) * sizeof(T), false);
  const size_t rbytes = std::max<size_t>(slot * size_t(H->nranks), 1) * sizeof(T);
  if (H->d_recv.bytes < rbytes) H->d_recv.alloc(rbytes, false);
  if (!H->ev_pack) {
    int least = 0, greatest = 0;
    GOFMM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GOFMM_CUDA(cudaStreamCreateWithPriority(&H->s_comm, cudaStreamNonBlocking, greatest));
    GOFMM_CUDA(cudaEventCreateWithFlags(&H->ev_pack, cudaEventDisableTiming));
    GOFMM_CUDA(cudaEventCreateWithFlags(&H->ev_gath, cudaEventDisableTiming));
    for (auto& e : H->dtev) GOFMM_CUDA(cudaEventCreate(&e));
  }
  T* send = H->d_send.as<T>();
  T* recv = H->d_recv.as<T>();
  if (timed) GOFMM_CUDA(cudaEventRecord(H->dtev[0], st));
  if constexpr (kF32)
    enqueue_chunk32(H, d_w, ldw, r, nullptr, H->n, st, false, 1, send);
  else
    enqueue_chunk(H, d_w, ldw, r, nullptr, H->n, st, false, 1, send);
  if (timed) GOFMM_CUDA(cudaEventRecord(H->dtev[1], st));
  GOFMM_CUDA(cudaEventRecord(H->ev_pack, st));
  GOFMM_CUDA(cudaStreamWaitEvent(H->s_comm, H->ev_pack, 0));
  if (timed) GOFMM_CUDA(cudaEventRecord(H->dtev[2], H->s_comm));
  if (api && slot > 0) {
    const nccl::result_t rc = api->AllGather(send, recv, slot, kF32 ? nccl::kFloat32 : nccl::kFloat64, H->comm,
                                             H->s_comm);
    if (rc != nccl::kSuccess) throw Error(GOFMM_ERR_CUDA, std::string("ncclAllGather: ") + api->GetErrorString(rc));
  }
  if (timed) GOFMM_CUDA(cudaEventRecord(H->dtev[3], H->s_comm));
  GOFMM_CUDA(cudaEventRecord(H->ev_gath, H->s_comm));
  // own D + near output terms: no exchanged input, overlap the all-gather
  if constexpr (!kF32) enqueue_chunk(H, nullptr, H->n, r, d_u, ldu, st, false, 3, nullptr);
  GOFMM_CUDA(cudaStreamWaitEvent(st, H->ev_gath, 0));
  if constexpr (kF32)
    enqueue_chunk32(H, nullptr, H->n, r, d_u, ldu, st, false, 4, recv);
  else
    enqueue_chunk(H, nullptr, H->n, r, d_u, ldu, st, false, 4, recv);
  if (timed) {
    GOFMM_CUDA(cudaEventRecord(H->ev[7], st));
    GOFMM_CUDA(cudaEventSynchronize(H->ev[7]));
    float a = 0, b = 0, c = 0;
    GOFMM_CUDA(cudaEventElapsedTime(&a, H->dtev[0], H->dtev[1]));
    GOFMM_CUDA(cudaEventElapsedTime(&b, H->dtev[2], H->dtev[3]));
    GOFMM_CUDA(cudaEventElapsedTime(&c, H->dtev[0], H->ev[7]));
    if (ms3) {
      ms3[0] = a;
      ms3[1] = b;
      ms3[2] = c;
    }
  }
}

template <class T>
int dist_evaluate_entry(gofmm_handle* H, const T* d_w, int64_t ldw, int32_t r, T* d_u, int64_t ldu, void* stream,
                        int32_t timed, double* ms3) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_u, ldu);
    check_precision(H, sizeof(T) == 4 ? GOFMM_PRECISION_F32 : GOFMM_PRECISION_F64);
    std::lock_guard<std::mutex> lk(H->mu);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    dist_evaluate<T>(H, d_w, ldw, r, d_u, ldu, st, timed != 0, ms3);
  });
}
}  // namespace

extern "C" {

// Host buffers (the drop-in form of one rank's evaluation, e.g. the C++ adapter's
// B200Evaluator::evaluate_dist): W (full, original order) is uploaded, the in-library data plane runs,
// and this rank's rows [own_row_begin, own_row_end) of u_perm are downloaded; other rows untouched.
int gofmm_dist_evaluate_host(gofmm_handle* H, const double* w, int64_t ldw, int32_t r, double* u_perm, int64_t ldu,
                             double* ms3) {
  return guarded([&] {
    check_args(H, w, ldw, r, u_perm, ldu);
    check_precision(H, GOFMM_PRECISION_F64);
    std::lock_guard<std::mutex> lk(H->mu);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = H->stream;
    DevBuf dw, du;
    dw.alloc(size_t(H->n) * r * sizeof(double), false);
    du.alloc(size_t(H->n) * r * sizeof(double), false);
    GOFMM_CUDA(cudaMemcpy2DAsync(dw.p, size_t(H->n) * sizeof(double), w, size_t(ldw) * sizeof(double),
                                 size_t(H->n) * sizeof(double), size_t(r), cudaMemcpyHostToDevice, st));
    {
      WsGuard ws(H, st);
      dist_evaluate<double>(H, dw.as<double>(), H->n, r, du.as<double>(), H->n, st, ms3 != nullptr, ms3);
    }
    const int64_t b = H->own_begin, e = H->own_end;
    if (e > b)
      GOFMM_CUDA(cudaMemcpy2DAsync(u_perm + b, size_t(ldu) * sizeof(double), du.as<double>() + b,
                                   size_t(H->n) * sizeof(double), size_t(e - b) * sizeof(double), size_t(r),
                                   cudaMemcpyDeviceToHost, st));
    GOFMM_CUDA(cudaStreamSynchronize(st));
  });
}

int gofmm_nccl_unique_id(void* id_out) {
  return guarded([&] {
    if (!id_out) throw Error(GOFMM_ERR_INVALID, "null unique id buffer");
    std::string why;
    const nccl::Api* api = nccl::api(&why);
    if (!api) throw Error(GOFMM_ERR_CUDA, why);
    nccl::UniqueId id;
    const nccl::result_t rc = api->GetUniqueId(&id);
    if (rc != nccl::kSuccess) throw Error(GOFMM_ERR_CUDA, std::string("ncclGetUniqueId: ") + api->GetErrorString(rc));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int gofmm_dist_init_comm(gofmm_handle* H, const void* unique_id) {
  return guarded([&] {
    if (!H || !unique_id) throw Error(GOFMM_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(H->mu);
    if (H->comm) throw Error(GOFMM_ERR_INVALID, "handle already has a communicator");
    std::string why;
    const nccl::Api* api = nccl::api(&why);
    if (!api) throw Error(GOFMM_ERR_CUDA, why);
    GOFMM_CUDA(cudaSetDevice(H->device));
    nccl::UniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    nccl::comm_t c = nullptr;
    const nccl::result_t rc = api->CommInitRank(&c, H->nranks, id, H->drank);
    if (rc != nccl::kSuccess) throw Error(GOFMM_ERR_CUDA, std::string("ncclCommInitRank: ") + api->GetErrorString(rc));
    H->comm = c;
    H->own_comm = true;
  });
}

int gofmm_dist_attach_comm(gofmm_handle* H, void* nccl_comm) {
  return guarded([&] {
    if (!H || !nccl_comm) throw Error(GOFMM_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(H->mu);
    if (H->comm) throw Error(GOFMM_ERR_INVALID, "handle already has a communicator");
    std::string why;
    const nccl::Api* api = nccl::api(&why);
    if (!api) throw Error(GOFMM_ERR_CUDA, why);
    auto c = static_cast<nccl::comm_t>(nccl_comm);
    int count = 0, me = 0;
    if (api->CommCount(c, &count) != nccl::kSuccess || api->CommUserRank(c, &me) != nccl::kSuccess)
      throw Error(GOFMM_ERR_INVALID, "not a valid NCCL communicator");
    if (count != H->nranks || me != H->drank)
      throw Error(GOFMM_ERR_INVALID, "communicator rank/size (" + std::to_string(me) + "/" + std::to_string(count) +
                                         ") differ from the handle's (" + std::to_string(H->drank) + "/" +
                                         std::to_string(H->nranks) + ")");
    H->comm = c;
    H->own_comm = false;
  });
}

int gofmm_dist_evaluate(gofmm_handle* H, const double* d_w, int64_t ldw, int32_t r, double* d_u, int64_t ldu,
                        void* stream, int32_t timed, double* ms3) {
  return dist_evaluate_entry<double>(H, d_w, ldw, r, d_u, ldu, stream, timed, ms3);
}

int gofmm_dist_evaluate_f32(gofmm_handle* H, const float* d_w, int64_t ldw, int32_t r, float* d_u, int64_t ldu,
                            void* stream, int32_t timed, double* ms3) {
  return dist_evaluate_entry<float>(H, d_w, ldw, r, d_u, ldu, stream, timed, ms3);
}

int gofmm_destroy(gofmm_handle* H) {
  return guarded([&] {
    if (!H) return;
    cudaSetDevice(H->device);
    cudaStreamSynchronize(H->stream);
    for (auto& e : H->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : H->lev)
      if (e) cudaEventDestroy(e);
    if (H->ws_free) {
      cudaEventSynchronize(H->ws_free);
      cudaEventDestroy(H->ws_free);
    }
    if (H->stream) cudaStreamDestroy(H->stream);
    for (auto* st : {H->s_h2d, H->s_d2h})
      if (st) cudaStreamDestroy(st);
    for (auto& row : H->pev)
      for (auto& e : row)
        if (e) cudaEventDestroy(e);
    for (auto& row : H->tev)
      for (auto& e : row)
        if (e) cudaEventDestroy(e);
    for (auto& row : H->dpev)
      for (auto& e : row)
        if (e) cudaEventDestroy(e);
    for (auto& e : H->hpev)
      if (e) cudaEventDestroy(e);
    for (auto& e : H->upev)
      if (e) cudaEventDestroy(e);
    if (H->s_comm) cudaStreamSynchronize(H->s_comm);
    if (H->comm && H->own_comm) {
      if (const nccl::Api* api = nccl::api(nullptr)) api->CommDestroy(H->comm);
    }
    if (H->s_comm) cudaStreamDestroy(H->s_comm);
    for (auto* e : {H->ev_pack, H->ev_gath, H->dtev[0], H->dtev[1], H->dtev[2], H->dtev[3]})
      if (e) cudaEventDestroy(e);
    if (H->gexec) cudaGraphExecDestroy(H->gexec);
    if (H->cap_stream) cudaStreamDestroy(H->cap_stream);
    delete H;
  });
}

int64_t gofmm_flops(const gofmm_handle* H, int32_t r) { return H ? H->flops_per_rhs * int64_t(r) : -1; }

int gofmm_phase_flops(const gofmm_handle* H, int32_t r, int64_t* out3) {
  return guarded([&] {
    if (!H || !out3) throw Error(GOFMM_ERR_INVALID, "null argument");
    for (int i = 0; i < 3; ++i) out3[i] = H->phase_flops_per_rhs[i] * int64_t(r);
  });
}

int gofmm_launch_profile(const gofmm_handle* H, int32_t r, int32_t cap, gofmm_launch_info* out, int32_t* count) {
  return guarded([&] {
    if (!H || !count) throw Error(GOFMM_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(H->mu);
    *count = int32_t(H->launches.size());
    for (int32_t i = 0; i < std::min<int32_t>(cap, *count); ++i) {
      const Launch& L = H->launches[i];
      out[i].phase = L.phase;
      out[i].level = L.level;
      if (H->precision == GOFMM_PRECISION_F32) {
        const int bn = 64 << pick_bn32(H, L, r);
        out[i].ctas = int64_t(L.ntiles32) * ((r + bn - 1) / bn);
      } else {
        const LaunchCfg cfg = pick_launch_cfg(H, L, r);
        out[i].ctas = int64_t(L.tn[cfg.bm_class]) * ((r + cfg.bn - 1) / cfg.bn);
      }
      out[i].flops = L.flops_per_rhs * int64_t(r);
      out[i].ms = i < int32_t(H->launch_ms.size()) ? H->launch_ms[i] : -1.0;
      out[i].generated = L.gen ? 1 : 0;
    }
  });
}

int32_t gofmm_launches_per_eval(const gofmm_handle* H) {
  if (!H) return -1;
  int32_t n = int32_t(H->launches.size()) + 1;  // grouped GEMMs + the permutation
  for (const Launch& L : H->launches) n += L.reduce_n > 0 ? 1 : 0;  // split-chain reductions
  return n;
}

int64_t gofmm_device_bytes(const gofmm_handle* H) {
  if (!H) return -1;
  const DevBuf* bufs[] = {&H->d_proj, &H->d_diag, &H->d_near,  &H->d_far,   &H->d_xp,   &H->d_xs,
                          &H->d_prow, &H->d_iperm, &H->d_tiles, &H->d_groups, &H->d_terms, &H->d_wp,
                          &H->d_what, &H->d_c,    &H->d_win,   &H->d_uout, &H->d_a32h, &H->d_a32l,
                          &H->d_win2[0], &H->d_win2[1], &H->d_uout2[0], &H->d_uout2[1], &H->d_xp32, &H->d_xs32, &H->d_xpn32, &H->d_xsn32, &H->d_terms32, &H->d_tiles32, &H->d_wp32[0], &H->d_wp32[1],
                          &H->d_what32[0], &H->d_what32[1], &H->d_c32[0], &H->d_c32[1], &H->d_win32, &H->d_uout32};
  int64_t s = 0;
  for (auto* b : bufs) s += int64_t(b->bytes);
  return s;
}

int gofmm_evaluate_device(gofmm_handle* H, const double* d_w, int64_t ldw, int32_t r, double* d_u, int64_t ldu,
                          void* stream, int32_t stats_sync, gofmm_eval_stats* stats) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_u, ldu);
    check_single(H);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F64);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    auto t0 = std::chrono::steady_clock::now();
    enqueue(H, d_w, ldw, r, d_u, ldu, st, stats && stats_sync);
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->flops = H->flops_per_rhs * int64_t(r);
      if (stats_sync) {
        fill_phase_times(H, stats);
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
  });
}

}  // extern "C"

namespace {
// Host-buffer evaluation (the drop-in for gfmm::evaluate): W column chunks are staged into HBM,
// evaluated, and u_perm copied back; h2d / d2h are timed with events on the handle's stream.
template <class T>
void evaluate_host(gofmm_handle* H, const T* w, int64_t ldw, int32_t r, T* u_perm, int64_t ldu,
                   gofmm_eval_stats* stats) {
  // Column chunks flow through a 3-stream pipeline (evaluation is column-separable):
  // H2D of chunk i+1 (copy stream 1) and D2H of chunk i-1 (copy stream 2) overlap the
  // evaluation of chunk i (the handle's stream), with two staging buffers for W and u. Only the
  // first upload and the last download are exposed.
  constexpr bool kF32 = sizeof(T) == 4;
  check_args(H, w, ldw, r, u_perm, ldu);
  check_single(H);
  check_precision(H, kF32 ? GOFMM_PRECISION_F32 : GOFMM_PRECISION_F64);
  std::lock_guard<std::mutex> lk(H->mu);
  GOFMM_CUDA(cudaSetDevice(H->device));
  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t st = H->stream;
  WsGuard ws(H, st);
  if (!H->s_h2d) {
    GOFMM_CUDA(cudaStreamCreateWithFlags(&H->s_h2d, cudaStreamNonBlocking));
    GOFMM_CUDA(cudaStreamCreateWithFlags(&H->s_d2h, cudaStreamNonBlocking));
    for (auto& row : H->pev)
      for (auto& e : row) GOFMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& row : H->tev)
      for (auto& e : row) GOFMM_CUDA(cudaEventCreate(&e));
    for (auto& row : H->dpev)
      for (auto& e : row) GOFMM_CUDA(cudaEventCreate(&e));
    for (auto& e : H->hpev) GOFMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : H->upev) GOFMM_CUDA(cudaEventCreate(&e));
  }
  // chunk: one N tile of the generated-operand kernels (FP32: 256 columns; FP64: 512 columns,
  // the GW config, once r > 256) unless r is smaller or the workspace forces less
  const int32_t rc_ws = kF32 ? rhs_chunk32(H, r) : rhs_chunk(H, r);
  const size_t per_col = size_t(H->n) * sizeof(T);
  int32_t tile_n = kF32 ? 256 : (use_wide(r) ? kBN_GW : kBN_G);
  {
    // four staging buffers (W and u, double-buffered) must fit next to the workspace
    size_t free_b = 0, total_b = 0;
    GOFMM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t have = H->d_win2[0].bytes + H->d_win2[1].bytes + H->d_uout2[0].bytes + H->d_uout2[1].bytes;
    const int64_t fit = int64_t(0.8 * double(free_b + have) / double(4 * per_col));
    if (tile_n > fit) tile_n = fit >= 256 ? 256 : int32_t(std::max<int64_t>(1, fit));
  }
  const int32_t rc = std::max<int32_t>(1, std::min<int32_t>({r, rc_ws, tile_n}));
  const size_t bytes = per_col * size_t(rc);
  for (int b = 0; b < 2; ++b)
    if (H->d_win2[b].bytes < bytes) {
      H->d_win2[b].alloc(bytes, false);
      H->d_uout2[b].alloc(bytes, false);
    }
  float h2d = 0, d2h = 0, ph[4] = {0, 0, 0, 0};
  std::vector<float> lms(H->launches.size(), 0.f);
  const int nchunks = int((r + rc - 1) / rc);
  auto h2d_copy = [&](int i) {
    const int b = i & 1;
    const int32_t c0 = i * rc, rr = std::min(rc, r - c0);
    // the buffer's previous chunk (i - 2) must have been consumed by its evaluation
    if (i >= 2) GOFMM_CUDA(cudaStreamWaitEvent(H->s_h2d, H->pev[b][1], 0));
    if (stats && i >= 2) {  // collect chunk i-2's upload time before its events are re-recorded
      float a;
      GOFMM_CUDA(cudaEventSynchronize(H->tev[b][1]));
      GOFMM_CUDA(cudaEventElapsedTime(&a, H->tev[b][0], H->tev[b][1]));
      h2d += a;
    }
    if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[b][0], H->s_h2d));
    GOFMM_CUDA(cudaMemcpy2DAsync(H->d_win2[b].p, per_col, w + size_t(c0) * ldw, size_t(ldw) * sizeof(T), per_col,
                                 rr, cudaMemcpyHostToDevice, H->s_h2d));
    if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[b][1], H->s_h2d));
    GOFMM_CUDA(cudaEventRecord(H->pev[b][0], H->s_h2d));  // in_ready
  };
  // FP64 single chunk: W lands in column pieces and each piece's permutation + upward (N2S,
  // column-separable) starts as soon as it is in HBM, so the upload overlaps the upward pass
  // (only for uploads of >= 1 GB: on small trees the pieces' repeated level launches cost more than
  // the upload they hide — N = 2^16, r = 512: upward 14 ms in pieces vs ~1 ms in one pass)
  constexpr int32_t kPieceCols = 128;
  const bool big = double(H->n) * double(rc) * sizeof(T) >= double(1 << 30);
  const int npieces = (!kF32 && nchunks == 1 && rc > kPieceCols && big) ? int((rc + kPieceCols - 1) / kPieceCols) : 0;
  if (npieces > 8) throw Error(GOFMM_ERR_CUDA, "internal: too many column pieces");
  if (npieces > 0) {
    if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[0][0], H->s_h2d));
    for (int p = 0; p < npieces; ++p) {
      const int32_t p0 = p * kPieceCols, pn = std::min(kPieceCols, rc - p0);
      GOFMM_CUDA(cudaMemcpy2DAsync(static_cast<T*>(H->d_win2[0].p) + size_t(p0) * H->n, per_col,
                                   w + size_t(p0) * ldw, size_t(ldw) * sizeof(T), per_col, pn,
                                   cudaMemcpyHostToDevice, H->s_h2d));
      GOFMM_CUDA(cudaEventRecord(H->hpev[p], H->s_h2d));
    }
    if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[0][1], H->s_h2d));
    GOFMM_CUDA(cudaEventRecord(H->pev[0][0], H->s_h2d));
  } else if (nchunks > 0) {
    h2d_copy(0);
  }
  int parts_timed = 0;      // last chunk: D2H copies timed per part
  bool last_full = false;   // last chunk: whole-buffer D2H (no split) timed by tev
  for (int i = 0; i < nchunks; ++i) {
    const int b = i & 1;
    const int32_t c0 = i * rc, rr = std::min(rc, r - c0);
    if (i + 1 < nchunks) h2d_copy(i + 1);  // prefetch the next chunk before evaluating this one
    if (npieces == 0) GOFMM_CUDA(cudaStreamWaitEvent(st, H->pev[b][0], 0));  // W chunk landed (else per piece)
    if (i >= 2) GOFMM_CUDA(cudaStreamWaitEvent(st, H->pev[b][2], 0));  // u buffer downloaded
    // last chunk: its u rows are downloaded part by part behind the split output launch
    // (rows_done), so only the last part's download is exposed
    bool rows_used = false, started = false;
    int64_t rows_lo = -1, rows_hi = -1;
    const RowsDone rows_done = [&](int64_t r0, int64_t r1) {
      GOFMM_CUDA(cudaEventRecord(H->pev[b][3], st));
      GOFMM_CUDA(cudaStreamWaitEvent(H->s_d2h, H->pev[b][3], 0));
      if (stats && !started) GOFMM_CUDA(cudaEventRecord(H->tev[b][2], H->s_d2h));
      started = true;
      const bool timed_part = stats && parts_timed < 8;
      if (timed_part) GOFMM_CUDA(cudaEventRecord(H->dpev[parts_timed][0], H->s_d2h));
      if (r1 > r0)
        GOFMM_CUDA(cudaMemcpy2DAsync(u_perm + size_t(c0) * ldu + r0, size_t(ldu) * sizeof(T),
                                     static_cast<T*>(H->d_uout2[b].p) + r0, per_col, size_t(r1 - r0) * sizeof(T), rr,
                                     cudaMemcpyDeviceToHost, H->s_d2h));
      if (timed_part) GOFMM_CUDA(cudaEventRecord(H->dpev[parts_timed++][1], H->s_d2h));
      if (rows_lo < 0 || r0 < rows_lo) rows_lo = r0;
      rows_hi = std::max(rows_hi, r1);
    };
    const RowsDone* hook = (i + 1 == nchunks) ? &rows_done : nullptr;
    if constexpr (kF32) {
      enqueue32(H, H->d_win2[b].as<float>(), H->n, rr, H->d_uout2[b].as<float>(), H->n, st, stats != nullptr, hook,
                &rows_used);
    } else if (npieces > 0) {
      double* dw = H->d_win2[b].as<double>();
      double* du = H->d_uout2[b].as<double>();
      if (stats) {
        H->launch_ms.assign(H->launches.size(), 0.f);
        std::fill(std::begin(H->phase_ms), std::end(H->phase_ms), 0.f);
        GOFMM_CUDA(cudaEventRecord(H->upev[0], st));
      }
      for (int p = 0; p < npieces; ++p) {
        GOFMM_CUDA(cudaStreamWaitEvent(st, H->hpev[p], 0));
        const int32_t p0 = p * kPieceCols, p1 = std::min(rr, p0 + kPieceCols);
        enqueue_chunk(H, dw, H->n, rr, du, H->n, st, false, 0, nullptr, nullptr, nullptr, 0, p0, p1);
      }
      if (stats) GOFMM_CUDA(cudaEventRecord(H->upev[1], st));
      enqueue_chunk(H, dw, H->n, rr, du, H->n, st, stats != nullptr, 0, nullptr, hook, &rows_used, /*phase_lo=*/1);
      if (stats) {
        accumulate_chunk_times(H);
        float up = 0.f;  // permutation + upward of all pieces, including waits for the upload
        GOFMM_CUDA(cudaEventElapsedTime(&up, H->upev[0], H->upev[1]));
        H->phase_ms[1] += up;  // [0] permutation, [1] upward (here: both, over all pieces)
      }
    } else {
      enqueue(H, H->d_win2[b].as<double>(), H->n, rr, H->d_uout2[b].as<double>(), H->n, st, stats != nullptr, hook,
              &rows_used);
    }
    GOFMM_CUDA(cudaEventRecord(H->pev[b][1], st));  // comp_done: W buffer free, u chunk ready
    GOFMM_CUDA(cudaStreamWaitEvent(H->s_d2h, H->pev[b][1], 0));
    const bool split = rows_used && rows_lo == 0 && rows_hi == H->n;
    if (!split) {
      // whole-buffer download (the parts, if any, did not cover u_perm)
      if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[b][2], H->s_d2h));
      GOFMM_CUDA(cudaMemcpy2DAsync(u_perm + size_t(c0) * ldu, size_t(ldu) * sizeof(T), H->d_uout2[b].p, per_col,
                                   per_col, rr, cudaMemcpyDeviceToHost, H->s_d2h));
    }
    if (i + 1 == nchunks) {
      last_full = !split;
      if (!split) parts_timed = 0;
    }
    if (stats) GOFMM_CUDA(cudaEventRecord(H->tev[b][3], H->s_d2h));
    GOFMM_CUDA(cudaEventRecord(H->pev[b][2], H->s_d2h));  // out_free
    if (stats) {
      // enqueue() synchronised on this chunk's evaluation; collect its copy times when the
      // buffer is reused (or at the end)
      for (int p = 0; p < 4; ++p) ph[p] += H->phase_ms[p];
      for (size_t k = 0; k < lms.size(); ++k) lms[k] += H->launch_ms[k];
    }
    if (stats && i >= 1) {  // chunk i-1's copies are complete once its D2H event is
      const int pb = (i - 1) & 1;
      GOFMM_CUDA(cudaEventSynchronize(H->tev[pb][3]));
      float c;
      GOFMM_CUDA(cudaEventElapsedTime(&c, H->tev[pb][2], H->tev[pb][3]));
      d2h += c;
    }
  }
  GOFMM_CUDA(cudaStreamSynchronize(H->s_d2h));
  if (stats) {
    const int lb = (nchunks - 1) & 1;
    float c = 0.f;
    for (int i = std::max(0, nchunks - 2); i < nchunks; ++i) {  // uploads not collected in h2d_copy
      float a;
      GOFMM_CUDA(cudaEventElapsedTime(&a, H->tev[i & 1][0], H->tev[i & 1][1]));
      h2d += a;
    }
    if (last_full) GOFMM_CUDA(cudaEventElapsedTime(&c, H->tev[lb][2], H->tev[lb][3]));
    for (int p = 0; p < parts_timed; ++p) {
      float x;
      GOFMM_CUDA(cudaEventElapsedTime(&x, H->dpev[p][0], H->dpev[p][1]));
      c += x;
    }
    d2h += c;
    std::memset(stats, 0, sizeof(*stats));
    stats->flops = H->flops_per_rhs * int64_t(r);
    std::copy(ph, ph + 4, H->phase_ms);
    H->launch_ms = lms;
    fill_phase_times(H, stats);
    stats->ms_h2d = h2d;
    stats->ms_d2h = d2h;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
}
}  // namespace

extern "C" {

int gofmm_evaluate(gofmm_handle* H, const double* w, int64_t ldw, int32_t r, double* u_perm, int64_t ldu,
                   gofmm_eval_stats* stats) {
  return guarded([&] { evaluate_host<double>(H, w, ldw, r, u_perm, ldu, stats); });
}

int gofmm_evaluate_f32(gofmm_handle* H, const float* w, int64_t ldw, int32_t r, float* u_perm, int64_t ldu,
                       gofmm_eval_stats* stats) {
  return guarded([&] { evaluate_host<float>(H, w, ldw, r, u_perm, ldu, stats); });
}

int gofmm_evaluate_device_f32(gofmm_handle* H, const float* d_w, int64_t ldw, int32_t r, float* d_u, int64_t ldu,
                              void* stream, int32_t stats_sync, gofmm_eval_stats* stats) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_u, ldu);
    check_single(H);
    std::lock_guard<std::mutex> lk(H->mu);
    check_precision(H, GOFMM_PRECISION_F32);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    auto t0 = std::chrono::steady_clock::now();
    enqueue32(H, d_w, ldw, r, d_u, ldu, st, stats && stats_sync);
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->flops = H->flops_per_rhs * int64_t(r);
      if (stats_sync) {
        fill_phase_times(H, stats);
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
  });
}

int gofmm_unpermute_device_f32(gofmm_handle* H, const float* d_up, int64_t ldp, int32_t r, float* d_u, int64_t ldu,
                               void* stream) {
  return guarded([&] {
    check_args(H, d_up, ldp, r, d_u, ldu);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    GOFMM_CUDA(f32::launch_unpermute(d_up, ldp, H->d_iperm.as<int32_t>(), H->n, r, d_u, ldu, st));
  });
}

int32_t gofmm_precision(const gofmm_handle* H) { return H ? H->precision : -1; }

// Exact rows of K W for error_eps2 (evaluate.hpp:353: oracle.block(rows, all) * w), matrix-free:
// one generated term per leaf (K(x_rows, x_leaf) W_perm[leaf]) split over kExactChunks partial
// groups so the N-long reduction runs on many CTAs, then a fixed-order sum of the partials.
int gofmm_exact_rows(gofmm_handle* H, const int32_t* rows, int32_t nrows, const double* d_w, int64_t ldw, int32_t r,
                     double* d_out, int64_t ldo, void* stream) {
  return guarded([&] {
    check_args(H, d_w, ldw, r, d_w, H->n);
    if (H->source != GOFMM_SOURCE_KERNEL || !H->kfn_g)
      throw Error(GOFMM_ERR_INVALID, "exact rows need a matrix-free kernel source");
    if (nrows < 1 || !rows || !d_out || ldo < nrows) throw Error(GOFMM_ERR_INVALID, "exact rows: bad arguments");
    if (H->nranks > 1) throw Error(GOFMM_ERR_INVALID, "exact rows: single-GPU handles only");
    std::lock_guard<std::mutex> lk(H->mu);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    WsGuard ws(H, st);
    const int D = H->dim;
    std::vector<double> x(size_t(nrows) * D);
    for (int i = 0; i < nrows; ++i) {
      if (rows[i] < 0 || rows[i] >= H->n) throw Error(GOFMM_ERR_INVALID, "exact rows: row out of range");
      for (int q = 0; q < D; ++q) x[size_t(i) * D + q] = H->coords_host[size_t(rows[i]) * D + q];
    }
    H->d_ex_x.upload(x);
    // W_perm for these columns (the permutation of an evaluation)
    ensure_workspace(H, r);
    upload_plan(H);
    encode_maps(H, r);
    {
      const int cpb = int(std::max<int64_t>(1, std::min<int64_t>(8, (48ll << 20) / (int64_t(H->n) * 8))));
      const int rpt = perm_rows_per_thread(H->ld_wp, r);
      dim3 grid(unsigned((H->ld_wp + 256 * rpt - 1) / (256 * rpt)), unsigned((r + cpb - 1) / cpb));
      auto* kern = rpt == kPermRows ? &permute_rows_in<kPermRows> : &permute_rows_in<1>;
      kern<<<grid, 256, 0, st>>>(d_w, ldw, H->d_prow.as<int32_t>(), 0, H->ld_wp, r, cpb,
                                            H->d_wp.as<double>(), int64_t(H->ws_r) * 16);
    }
    const int nleaf = int(H->leaf_ids.size());
    const int chunks = std::max(1, std::min(nleaf, 128));
    std::vector<Group> gs;
    std::vector<Term> ts;
    std::vector<Tile> tl;
    for (int c = 0; c < chunks; ++c) {
      Group g{};
      g.crow = int64_t(c) * nrows;  // partial c occupies rows [c*nrows, (c+1)*nrows) of the scratch
      g.M = nrows;
      g.tbeg = int(ts.size());
      for (int li = c; li < nleaf; li += chunks) {
        const int id = H->leaf_ids[li];
        Term t{};
        t.flags = kTermGen;
        t.xr = H->d_ex_x.as<double>();
        t.xc = H->d_xp.as<double>() + H->pst[id] * D;
        t.bbuf = kBufWp;
        t.b_row = H->pst[id];
        t.K = H->end[id] - H->start[id];
        ts.push_back(t);
      }
      g.tend = int(ts.size());
      for (int m0 = 0; m0 < nrows; m0 += kBM_G) tl.push_back({int(gs.size()), m0});
      gs.push_back(g);
    }
    H->d_ex_groups.upload(gs);
    H->d_ex_terms.upload(ts);
    H->d_ex_tiles.upload(tl);
    const size_t part_bytes = size_t(chunks) * nrows * r * sizeof(double);
    if (H->d_ex_part.bytes < part_bytes) H->d_ex_part.alloc(part_bytes, false);
    const int64_t ldp = int64_t(chunks) * nrows;  // partials stacked along rows, column-major
    dim3 grid(unsigned(tl.size()), unsigned((r + kBN_G - 1) / kBN_G));
    H->kfn_g<<<grid, kThreadsG, H->smem_g, st>>>(H->maps_g, H->d_ex_tiles.as<Tile>(), H->d_ex_groups.as<Group>(),
                                                  H->d_ex_terms.as<Term>(), r, H->kp, H->d_ex_part.as<double>(), ldp,
                                                  0, 0);
    dim3 g2(unsigned((int64_t(nrows) * r + 255) / 256));
    sum_partials<<<g2, 256, 0, st>>>(H->d_ex_part.as<double>(), ldp, nrows, chunks, r, d_out, ldo);
    GOFMM_CUDA(cudaGetLastError());
    GOFMM_CUDA(cudaStreamSynchronize(st));
  });
}

// The reference Rng (common.hpp:40-104): splitmix64 stream, Box-Muller gauss with cached spare,
// sorted rejection sample. Host code: error_eps2 draws its rows and W from it
// (evaluate.hpp:336-346), so reproducing eps2 needs the identical stream.

int gofmm_rng_eps2_draw(uint64_t seed, int32_t n, int32_t r, int32_t sample_rows, int32_t* rows_out,
                        double* w_out, int64_t ldw) {
  return gofmm_rng_eps2_draw_attempt(seed, n, r, sample_rows, 0, rows_out, w_out, ldw);
}

int gofmm_rng_eps2_draw_attempt(uint64_t seed, int32_t n, int32_t r, int32_t sample_rows, int32_t attempt,
                                int32_t* rows_out, double* w_out, int64_t ldw) {
  return guarded([&] {
    if (n < 1 || r < 1 || sample_rows < 1) throw Error(GOFMM_ERR_INVALID, "eps2 draw: bad sizes");
    if (attempt < 0 || attempt > 2) throw Error(GOFMM_ERR_INVALID, "eps2 draw: attempt must be 0, 1 or 2");
    if (w_out && ldw < n) throw Error(GOFMM_ERR_INVALID, "eps2 draw: ldw < n");
    RefRng rng(seed, 0xe952);
    const int k = std::min(sample_rows, n);
    std::vector<int> out;
    if (k >= n) {
      for (int i = 0; i < n; ++i) out.push_back(i);
    } else {
      std::vector<char> taken(n, 0);
      while (int(out.size()) < k) {
        int v = rng.uniform(n);
        if (!taken[v]) {
          taken[v] = 1;
          out.push_back(v);
        }
      }
      std::sort(out.begin(), out.end());
    }
    if (rows_out) std::copy(out.begin(), out.end(), rows_out);
    // evaluate.hpp:343-346: attempt a's W follows the earlier attempts' draws on the same stream
    for (int a = 0; a < attempt; ++a)
      for (int64_t q = 0; q < int64_t(r) * n; ++q) rng.gauss();
    if (w_out)
      for (int c = 0; c < r; ++c)
        for (int i = 0; i < n; ++i) w_out[i + size_t(c) * ldw] = rng.gauss();
  });
}

// error_eps2 (evaluate.hpp:330-373) on the GPU: the reference's draws (rows, then W column-major
// from Rng(seed, 0xe952), up to three W draws while the sampled rows of K w vanish), u = K~ W by
// this handle's evaluation, the exact rows K(rows, :) W matrix-free on the device, and the report
// fields of ErrorReport. Host W / u live only for the call.
int gofmm_error_eps2(gofmm_handle* H, int32_t r, int32_t sample_rows, uint64_t seed, gofmm_eps2_report* rep,
                     int32_t* rows_out) {
  return guarded([&] {
    if (!H || !rep) throw Error(GOFMM_ERR_INVALID, "error_eps2: null argument");
    if (sample_rows < 1) throw Error(GOFMM_ERR_INVALID, "sample_rows must be >= 1");
    if (r < 1) throw Error(GOFMM_ERR_INVALID, "r must be >= 1");
    if (H->nranks > 1) throw Error(GOFMM_ERR_INVALID, "error_eps2: single-GPU handles only");
    const int n = H->n, k = std::min(sample_rows, n);
    std::memset(rep, 0, sizeof(*rep));
    std::vector<int32_t> rows(k);
    std::vector<double> w(size_t(n) * r), u(size_t(n) * r), ex(size_t(k) * r);
    std::vector<float> wf, uf;
    const bool f32 = H->precision == GOFMM_PRECISION_F32;
    if (f32) {
      wf.resize(w.size());
      uf.resize(u.size());
    }
    double* d_w = nullptr;
    double* d_ex = nullptr;
    GOFMM_CUDA(cudaSetDevice(H->device));
    GOFMM_CUDA(cudaMalloc(&d_w, w.size() * sizeof(double)));
    GOFMM_CUDA(cudaMalloc(&d_ex, ex.size() * sizeof(double)));
    struct Free {
      double *a, *b;
      ~Free() {
        cudaFree(a);
        cudaFree(b);
      }
    } fr{d_w, d_ex};
    for (int attempt = 0; attempt < 3; ++attempt) {
      int rc = gofmm_rng_eps2_draw_attempt(seed, n, r, sample_rows, attempt, rows.data(), w.data(), n);
      if (rc != GOFMM_OK) throw Error(rc, g_last_error);
      gofmm_eval_stats st{};
      if (f32) {
        for (size_t q = 0; q < w.size(); ++q) wf[q] = float(w[q]);
        rc = gofmm_evaluate_f32(H, wf.data(), n, r, uf.data(), n, &st);
        for (size_t q = 0; q < u.size(); ++q) u[q] = double(uf[q]);
      } else {
        rc = gofmm_evaluate(H, w.data(), n, r, u.data(), n, &st);
      }
      if (rc != GOFMM_OK) throw Error(rc, g_last_error);
      rep->eval_flops = st.flops;
      rep->eval_seconds = st.seconds;
      GOFMM_CUDA(cudaMemcpy(d_w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
      rc = gofmm_exact_rows(H, rows.data(), k, d_w, n, r, d_ex, k, nullptr);
      if (rc != GOFMM_OK) throw Error(rc, g_last_error);
      GOFMM_CUDA(cudaStreamSynchronize(H->stream));
      GOFMM_CUDA(cudaMemcpy(ex.data(), d_ex, ex.size() * sizeof(double), cudaMemcpyDeviceToHost));
      // unpermute (evaluate.hpp:21-25): original row i sits at permuted position perm[i]
      std::vector<int64_t> pos(k);
      for (int t = 0; t < k; ++t) pos[t] = -1;
      {
        std::vector<int32_t> want(n, -1);
        for (int t = 0; t < k; ++t) want[rows[t]] = t;
        for (int t = 0; t < n; ++t)
          if (want[H->iperm[t]] >= 0) pos[want[H->iperm[t]]] = t;
      }
      double num = 0.0, den = 0.0, sum_rel = 0.0;
      std::vector<double> rel(k);
      for (int t = 0; t < k; ++t) {
        const int64_t pr = pos[t];
        double dn = 0.0, de = 0.0;
        for (int c = 0; c < r; ++c) {
          const double e = ex[t + size_t(c) * k];
          const double d = u[pr + size_t(c) * n] - e;
          dn += d * d;
          de += e * e;
        }
        num += dn;
        den += de;
        rel[t] = de > 0 ? std::sqrt(dn) / std::sqrt(de) : 0.0;
      }
      if (den == 0.0) continue;  // degenerate right-hand side; resample (evaluate.hpp:360)
      rep->eps2 = std::sqrt(num / den);
      rep->num_per_entry = std::min(k, 10);
      for (int t = 0; t < rep->num_per_entry; ++t) rep->per_entry[t] = rel[t];
      for (int t = 0; t < k; ++t) sum_rel += rel[t];
      rep->mean_sample = sum_rel / double(k);
      if (rows_out) std::copy(rows.begin(), rows.end(), rows_out);
      return;
    }
    throw Error(GOFMM_ERR_NUMERIC, "error_eps2: sampled rows of Kw vanished repeatedly");
  });
}

int gofmm_unpermute_device(gofmm_handle* H, const double* d_up, int64_t ldp, int32_t r, double* d_u, int64_t ldu,
                           void* stream) {
  return guarded([&] {
    check_args(H, d_up, ldp, r, d_u, ldu);
    check_precision(H, GOFMM_PRECISION_F64);
    GOFMM_CUDA(cudaSetDevice(H->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : H->stream;
    const int cpb = 8;
    dim3 grid(unsigned((H->n + 255) / 256), unsigned((r + cpb - 1) / cpb));
    unpermute_rows<<<grid, 256, 0, st>>>(d_up, ldp, H->d_iperm.as<int32_t>(), H->n, r, cpb, d_u, ldu);
    GOFMM_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
