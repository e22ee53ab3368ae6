// gofmm_ann.cu — one randomized-tree ANN pass on sm_100a.
//
// Replaces the per-leaf body of ann_iteration (neighbors.hpp:88-106): for every leaf of the
// random tree, all pairwise distances inside the leaf (Metric::pairwise, metric.hpp:57-73) and,
// per index, the merge of the leaf's candidates into its neighbor list (merge_candidates,
// neighbors.hpp:35-63): the kappa smallest DISTINCT indices of list ∪ candidates under the
// (distance, index) order. The random tree itself (tree.hpp:244-247) is built on the host.
//
// One CTA per leaf: the leaf's coordinates are staged in shared memory; one warp per row a
// computes d(a, b) for its candidates (lane l holds b = l, l+32, ...) and then selects the
// merged list by kappa rounds of a warp-wide (distance, index) argmin over candidates + the old
// list (one old entry per lane), dropping every entry with the selected index. Geometric
// distances are issued in the reference's operation order (difference vector, Eigen's packet
// reduction of the squares, sqrt), so tables are bit-identical to the reference's; the kernel
// metric's Gaussian entries use the device exp (<= 1-2 ulp from glibc's), so distances agree to
// ~1e-16 and neighbor sets agree except at exact near-ties.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../include/gofmm_b200.h"

namespace gofmm_ann {

constexpr int kWarps = 8;
constexpr int kMaxLeaf = 1024;  // leaf size limit (candidates per lane: 16 up to 512, 32 above)

__device__ __forceinline__ bool less_dj(double d1, int j1, double d2, int j2) {
  return d1 < d2 || (d1 == d2 && j1 < j2);  // neighbor_less (neighbors.hpp:30-33)
}

// (x_a - x_b).squaredNorm() with Eigen's packet reduction order (eigen_shim redux_packet)
template <int D>
__device__ __forceinline__ double sqnorm_diff(const double* xa, const double* xb, int d) {
  double v[D > 0 ? D : 16];
  const int dd = D > 0 ? D : d;
#pragma unroll
  for (int q = 0; q < (D > 0 ? D : 16); ++q)
    if (q < dd) {
      const double e = __dsub_rn(xa[q], xb[q]);
      v[q] = __dmul_rn(e, e);
    }
  const int aligned = (dd / 2) * 2, aligned2 = (dd / 4) * 4;
  if (aligned) {
    double a0 = v[0], a1 = v[1];
    if (aligned > 2) {
      double b0 = v[2], b1 = v[3];
      for (int i = 4; i < aligned2; i += 4) {
        a0 = __dadd_rn(a0, v[i]);
        a1 = __dadd_rn(a1, v[i + 1]);
        b0 = __dadd_rn(b0, v[i + 2]);
        b1 = __dadd_rn(b1, v[i + 3]);
      }
      a0 = __dadd_rn(a0, b0);
      a1 = __dadd_rn(a1, b1);
      if (aligned > aligned2) {
        a0 = __dadd_rn(a0, v[aligned2]);
        a1 = __dadd_rn(a1, v[aligned2 + 1]);
      }
    }
    double res = __dadd_rn(a0, a1);
    for (int i = aligned; i < dd; ++i) res = __dadd_rn(res, v[i]);
    return res;
  }
  double res = v[0];
  for (int i = 1; i < dd; ++i) res = __dadd_rn(res, v[i]);
  return res;
}

template <int D, int kPerLane>
__global__ void __launch_bounds__(kWarps * 32) ann_leaf_kernel(const double* __restrict__ coords, int32_t d,
                                                               int32_t kind, double inv2h2,
                                                               const int32_t* __restrict__ leaf_off,
                                                               const int32_t* __restrict__ leaf_idx, int32_t kappa,
                                                               int32_t* __restrict__ tj, double* __restrict__ td,
                                                               int32_t* __restrict__ tlen) {
  extern __shared__ double sx[];  // [leaf size][d] coordinates of the leaf
  __shared__ int sidx[kMaxLeaf];
  const int l0 = leaf_off[blockIdx.x], ln = leaf_off[blockIdx.x + 1] - l0;
  const int dd = D > 0 ? D : d;
  for (int e = threadIdx.x; e < ln * dd; e += blockDim.x) {
    const int a = e / dd, q = e - a * dd;
    sx[e] = coords[size_t(leaf_idx[l0 + a]) * dd + q];
  }
  for (int a = threadIdx.x; a < ln; a += blockDim.x) sidx[a] = leaf_idx[l0 + a];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int a = warp; a < ln; a += kWarps) {
    const int i = sidx[a];
    // candidates of row a: (d(a, b), leaf[b]) for b != a (metric.hpp pairwise, column a)
    double cd[kPerLane];
    int cj[kPerLane];
#pragma unroll
    for (int u = 0; u < kPerLane; ++u) {
      const int b = lane + 32 * u;
      cj[u] = -1;
      cd[u] = 0.0;
      if (b < ln && b != a) {
        const double d2 = sqnorm_diff<D>(sx + size_t(b) * dd, sx + size_t(a) * dd, dd);
        double dist;
        if (kind == 0) {
          dist = sqrt(d2);  // GeometricL2: (x_a - x_b).norm()
        } else {
          // KernelL2 over the Gaussian oracle: sqrt(max(0, K_ii + K_jj - 2 K_ij)), unit diagonal
          const double k = exp(__dmul_rn(-d2, inv2h2));
          dist = sqrt(fmax(0.0, __dsub_rn(__dadd_rn(1.0, 1.0), __dmul_rn(2.0, k))));
        }
        cd[u] = dist;
        cj[u] = sidx[b];
      }
    }
    // the old list: one entry per lane (kappa <= 32)
    const int olen = tlen[i];
    int oj = -1;
    double od = 0.0;
    if (lane < olen) {
      oj = tj[size_t(i) * kappa + lane];
      od = td[size_t(i) * kappa + lane];
    }
    if (olen == kappa) {
      // a full list only changes for candidates that beat its last entry (merge_candidates keeps
      // the kappa smallest): drop the rest, and skip the row when nothing survives
      const int wj = __shfl_sync(0xffffffffu, oj, kappa - 1);
      const double wd = __shfl_sync(0xffffffffu, od, kappa - 1);
      bool any = false;
#pragma unroll
      for (int u = 0; u < kPerLane; ++u) {
        if (cj[u] >= 0 && !less_dj(cd[u], cj[u], wd, wj)) cj[u] = -1;
        any |= cj[u] >= 0;
      }
      if (!__any_sync(0xffffffffu, any)) continue;
    }
    int outn = 0;
    int my_j = -1;
    double my_d = 0.0;
    for (int r = 0; r < kappa; ++r) {
      // lane-local minimum
      int bj = oj;
      double bd = od;
#pragma unroll
      for (int u = 0; u < kPerLane; ++u)
        if (cj[u] >= 0 && (bj < 0 || less_dj(cd[u], cj[u], bd, bj))) {
          bj = cj[u];
          bd = cd[u];
        }
      for (int o = 16; o > 0; o >>= 1) {
        const int oj2 = __shfl_xor_sync(0xffffffffu, bj, o);
        const double od2 = __shfl_xor_sync(0xffffffffu, bd, o);
        if (oj2 >= 0 && (bj < 0 || less_dj(od2, oj2, bd, bj))) {
          bj = oj2;
          bd = od2;
        }
      }
      if (bj < 0) break;  // both sources exhausted
      if (lane == r) {
        my_j = bj;
        my_d = bd;
      }
      ++outn;
      // drop every entry with this index (a candidate and an old entry may carry the same j)
      if (oj == bj) oj = -1;
#pragma unroll
      for (int u = 0; u < kPerLane; ++u)
        if (cj[u] == bj) cj[u] = -1;
    }
    if (lane < outn) {
      tj[size_t(i) * kappa + lane] = my_j;
      td[size_t(i) * kappa + lane] = my_d;
    }
    if (lane == 0) tlen[i] = outn;
  }
}

}  // namespace gofmm_ann

namespace {
thread_local char g_ann_err[256];
int ann_fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  snprintf(g_ann_err, sizeof(g_ann_err), "%s%s%s", what, e != cudaSuccess ? ": " : "",
           e != cudaSuccess ? cudaGetErrorString(e) : "");
  return code;
}
struct ABuf {
  void* p = nullptr;
  ~ABuf() {
    if (p) cudaFree(p);
  }
};
}  // namespace

extern "C" {

const char* gofmm_ann_last_error(void) { return g_ann_err; }

int gofmm_ann_leaf_merge(int32_t n, int32_t d, const double* coords, int32_t kind, double h, int32_t kappa,
                         int32_t nleaves, const int32_t* leaf_off, const int32_t* leaf_idx, int32_t device,
                         int32_t* table_j, double* table_d, int32_t* table_len, double* kernel_ms) {
  using namespace gofmm_ann;
  if (n < 1 || d < 1 || d > 16 || !coords || !leaf_off || !leaf_idx || !table_j || !table_d || !table_len)
    return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: bad argument (n, d in [1, 16], non-null arrays)");
  if (kappa < 1 || kappa > 32) return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: kappa must be in [1, 32]");
  if (kind != 0 && kind != 1) return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: kind 0 (geometric) or 1 (kernel)");
  if (kind == 1 && !(h > 0)) return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: gaussian bandwidth must be positive");
  if (nleaves < 0 || leaf_off[0] != 0 || leaf_off[nleaves] > n)
    return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: bad leaf offsets");
  int maxleaf = 0;
  for (int l = 0; l < nleaves; ++l) maxleaf = std::max(maxleaf, leaf_off[l + 1] - leaf_off[l]);
  if (maxleaf > kMaxLeaf) return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: leaf larger than 1024 points");
  for (int i = 0; i < n; ++i)
    if (table_len[i] < 0 || table_len[i] > kappa) return ann_fail(GOFMM_ERR_INVALID, "ann_leaf_merge: bad list length");
  if (nleaves == 0) return GOFMM_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return ann_fail(GOFMM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return ann_fail(GOFMM_ERR_CUDA, "cudaSetDevice", e);
  ABuf dc, dlo, dli, dtj, dtd, dtl;
  const size_t nk = size_t(n) * kappa;
  if ((e = cudaMalloc(&dc.p, size_t(n) * d * 8)) != cudaSuccess || (e = cudaMalloc(&dlo.p, size_t(nleaves + 1) * 4)) ||
      (e = cudaMalloc(&dli.p, size_t(n) * 4)) || (e = cudaMalloc(&dtj.p, nk * 4)) || (e = cudaMalloc(&dtd.p, nk * 8)) ||
      (e = cudaMalloc(&dtl.p, size_t(n) * 4)))
    return ann_fail(GOFMM_ERR_CUDA, "ann_leaf_merge: device allocation", e);
  // coords: d x n column-major is already point-major (d doubles per point)
  if ((e = cudaMemcpy(dc.p, coords, size_t(n) * d * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dlo.p, leaf_off, size_t(nleaves + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dli.p, leaf_idx, size_t(leaf_off[nleaves]) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dtj.p, table_j, nk * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dtd.p, table_d, nk * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dtl.p, table_len, size_t(n) * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
    return ann_fail(GOFMM_ERR_CUDA, "ann_leaf_merge: upload", e);
  const double inv = 1.0 / (2.0 * h * h);  // GaussianKernelOracle::eval_block (oracle.hpp:150)
  const size_t smem = size_t(maxleaf) * d * 8;
  cudaEvent_t ev[2];
  cudaEventCreate(&ev[0]);
  cudaEventCreate(&ev[1]);
  cudaEventRecord(ev[0]);
  auto launch = [&](auto k16, auto k32) {
    auto kern = maxleaf <= 512 ? k16 : k32;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<unsigned(nleaves), kWarps * 32, smem>>>(static_cast<double*>(dc.p), d, kind, inv,
                                                   static_cast<int32_t*>(dlo.p), static_cast<int32_t*>(dli.p), kappa,
                                                   static_cast<int32_t*>(dtj.p), static_cast<double*>(dtd.p),
                                                   static_cast<int32_t*>(dtl.p));
  };
  switch (d) {
    case 3: launch(ann_leaf_kernel<3, 16>, ann_leaf_kernel<3, 32>); break;
    case 6: launch(ann_leaf_kernel<6, 16>, ann_leaf_kernel<6, 32>); break;
    case 8: launch(ann_leaf_kernel<8, 16>, ann_leaf_kernel<8, 32>); break;
    default: launch(ann_leaf_kernel<0, 16>, ann_leaf_kernel<0, 32>); break;
  }
  cudaEventRecord(ev[1]);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventSynchronize(ev[1]);
  float ms = 0.f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, ev[0], ev[1]);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (e != cudaSuccess) return ann_fail(GOFMM_ERR_CUDA, "ann_leaf_merge: kernel", e);
  if (kernel_ms) *kernel_ms = ms;
  if ((e = cudaMemcpy(table_j, dtj.p, nk * 4, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(table_d, dtd.p, nk * 8, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(table_len, dtl.p, size_t(n) * 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return ann_fail(GOFMM_ERR_CUDA, "ann_leaf_merge: download", e);
  return GOFMM_OK;
}

}  // extern "C"
