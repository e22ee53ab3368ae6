// gofmm_skel.cu — batched node skeletonisation on sm_100a.
//
// The compress phase's per-node interpolative decomposition, skeletonize_node
// (compress.hpp:149-187): column-pivoted Householder QR of the sampled block
// K(sample_cols, candidates) (Eigen 3.4 ColPivHouseholderQR::computeInPlace, whose operation
// order oracle/eigen_shim/Eigen/Dense:684-777 restates), rank = #{l : |R_ll| > tau |R_11|}
// clamped to [1, s], skeleton = the first `rank` pivots, and proj = [I | R11^{-1} R12] scattered
// back through the column permutation (the triangular solve of eigen_shim:605-625).
//
// One CTA per node (3 per SM). The node's block lives ROW-major in a global workspace so that
// every per-column pass (a thread per aligned column pair: Householder dot product, rank-1
// update; a thread per column: norm downdate) reads coalesced row segments, 16 rows in flight; per-step vectors (column norms, the
// Householder vector, tau * v) live in shared memory. Every floating-point operation is issued
// with explicit round-to-nearest intrinsics in the reference's order (no FMA contraction, the
// same 2- and 4-accumulator reduction trees), so pivots, ranks, skeletons and proj reproduce
// the CPU reference bit for bit on the same block. The kernel is L2/HBM-bound: step k streams
// the (rows-k) x (cols-k) trailing block three times (dot, update read, update write).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/gofmm_b200.h"
#include "gofmm_skel_internal.h"

namespace gofmm_skel {

constexpr int kThreads = 128;  // 3 CTAs (nodes) per SM: one node's serial pivot phase overlaps the others' streaming


__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// Eigen 3.4 redux over a unit-stride vector with 2-wide packets and two packet accumulators
// (eigen_shim redux_packet, Dense:54-81), element i = get(i), by one thread.
template <class F>
__device__ double redux_packet(int n, F get) {
  const int aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  if (aligned) {
    double a0 = get(0), a1 = get(1);
    if (aligned > 2) {
      double b0 = get(2), b1 = get(3);
      for (int i = 4; i < aligned2; i += 4) {
        a0 = add(a0, get(i));
        a1 = add(a1, get(i + 1));
        b0 = add(b0, get(i + 2));
        b1 = add(b1, get(i + 3));
      }
      a0 = add(a0, b0);
      a1 = add(a1, b1);
      if (aligned > aligned2) {
        a0 = add(a0, get(aligned2));
        a1 = add(a1, get(aligned2 + 1));
      }
    }
    double res = add(a0, a1);
    for (int i = aligned; i < n; ++i) res = add(res, get(i));
    return res;
  }
  double res = get(0);
  for (int i = 1; i < n; ++i) res = add(res, get(i));
  return res;
}

// The same reduction split over lanes 0..3 of one warp (one packet accumulator chain each, the
// exact element-to-chain assignment of redux_packet), combined on lane 0 in the same order.
// get() must be cheap (shared memory): the chains are latency-bound otherwise. Lane 0 returns it.
template <class F>
__device__ double redux_packet_lanes(int n, F get, int lane) {
  const int aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  if (aligned <= 2) return lane == 0 ? redux_packet(n, get) : 0.0;
  double acc = 0.0;
  if (lane < 4) {
    acc = get(lane);
    for (int i = 4 + lane; i < aligned2; i += 4) acc = add(acc, get(i));
  }
  const double a1 = __shfl_sync(0xffffffffu, acc, 1), b0 = __shfl_sync(0xffffffffu, acc, 2),
               b1 = __shfl_sync(0xffffffffu, acc, 3);
  if (lane != 0) return 0.0;
  double x0 = add(acc, b0), x1 = add(a1, b1);
  if (aligned > aligned2) {
    x0 = add(x0, get(aligned2));
    x1 = add(x1, get(aligned2 + 1));
  }
  double res = add(x0, x1);
  for (int i = aligned; i < n; ++i) res = add(res, get(i));
  return res;
}

// Row-major GEMV dot of Eigen's general_matrix_vector_product (eigen_shim gemv_dot, Dense:92-102):
// sum_i col[i*ld] * v[i] with even / odd accumulators. Loads are issued 8 rows ahead of the
// (order-preserving) adds so one thread keeps several global loads in flight.
__device__ double gemv_dot_col(int n, const double* __restrict__ col, int64_t ld, const double* __restrict__ v) {
  double c0 = 0.0, c1 = 0.0;
  int j = 0;
  for (; j + 8 <= n; j += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = col[int64_t(j + u) * ld];
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      c0 = add(c0, mul(x[u], v[j + u]));
      c1 = add(c1, mul(x[u + 1], v[j + u + 1]));
    }
  }
  for (; j + 2 <= n; j += 2) {
    c0 = add(c0, mul(col[int64_t(j) * ld], v[j]));
    c1 = add(c1, mul(col[int64_t(j + 1) * ld], v[j + 1]));
  }
  double cc = add(c0, c1);
  for (; j < n; ++j) cc = add(cc, mul(col[int64_t(j) * ld], v[j]));
  return cc;
}

__global__ void __launch_bounds__(kThreads, 3) skeletonize_kernel(const NodeDesc* __restrict__ nodes,
                                                               const double* __restrict__ in, double* __restrict__ ws,
                                                               int32_t s_max, double tau_tol,
                                                               int32_t* __restrict__ rank_out,
                                                               double* __restrict__ achieved_out,
                                                               double* __restrict__ lead_out,
                                                               int32_t* __restrict__ perm_out,
                                                               double* __restrict__ proj_out) {
  const NodeDesc nd = nodes[blockIdx.x];
  const int rows = nd.rows, cols = nd.cols, ld = (cols + 1) & ~1;  // even: 16-byte column pairs
  const int size = min(rows, cols);
  double* A = ws + nd.ws_off;  // A(i, j) = A[i * ld + j]
  extern __shared__ double sh[];
  double* upd = sh;               // [cols] updated column norms
  double* direct = upd + cols;    // [cols] directly computed norms
  double* ess = direct + cols;    // [rows] essential part of the Householder vector
  double* tess = ess + rows;      // [rows] tau * ess
  int* trans = reinterpret_cast<int*>(tess + rows);  // [cols] transpositions
  __shared__ double s_tau, s_beta, s_denom, s_bv[kThreads / 32];
  __shared__ int s_bi[kThreads / 32];
  __shared__ int s_big, s_rank;
  const int tid = threadIdx.x;

  // column-major input -> row-major workspace
  for (int64_t e = tid; e < int64_t(rows) * cols; e += blockDim.x) {
    const int i = int(e / cols), j = int(e % cols);
    A[int64_t(i) * ld + j] = in[nd.in_off + int64_t(j) * rows + i];
  }
  __syncthreads();
  // initial column norms: col(k).norm() (ColPivHouseholderQR::computeInPlace)
  for (int j = tid; j < cols; j += blockDim.x) {
    const double nrm = sqrt(redux_packet(rows, [&](int i) {
      const double v = A[int64_t(i) * ld + j];
      return mul(v, v);
    }));
    direct[j] = nrm;
    upd[j] = nrm;
  }
  __syncthreads();
  const double downdate_threshold = sqrt(DBL_EPSILON);

  for (int k = 0; k < size; ++k) {
    // (1) first index of the maximum remaining updated norm
    double bv = -1.0;
    int bi = cols;
    for (int j = k + tid; j < cols; j += blockDim.x)
      if (bi == cols || upd[j] > bv) {
        bv = upd[j];
        bi = j;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (oi < cols && (bi == cols || ov > bv || (ov == bv && oi < bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      s_bv[tid >> 5] = bv;
      s_bi[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = s_bv[0];
      int b = s_bi[0];
      for (int w = 1; w < int(blockDim.x / 32); ++w)
        if (s_bi[w] < cols && (b == cols || s_bv[w] > v || (s_bv[w] == v && s_bi[w] < b))) {
          v = s_bv[w];
          b = s_bi[w];
        }
      s_big = b;
      trans[k] = b;
      if (b != k) {
        double t = upd[k];
        upd[k] = upd[b];
        upd[b] = t;
        t = direct[k];
        direct[k] = direct[b];
        direct[b] = t;
      }
    }
    __syncthreads();
    const int big = s_big;
    if (big != k)
      for (int i = tid; i < rows; i += blockDim.x) {
        const double t = A[int64_t(i) * ld + k];
        A[int64_t(i) * ld + k] = A[int64_t(i) * ld + big];
        A[int64_t(i) * ld + big] = t;
      }
    __syncthreads();
    // (2) makeHouseholderInPlace on column k, rows k..rows-1: the column is staged in shared
    // memory (ess[i] = A(k+1+i, k)) by all threads, its tail norm reduced by 4 lanes
    const int len = rows - k;
    for (int i = 1 + tid; i < len; i += blockDim.x) ess[i - 1] = A[int64_t(k + i) * ld + k];
    __syncthreads();
    if (tid < 32) {
      double tail_sq = 0.0;
      if (len > 1)
        tail_sq = redux_packet_lanes(len - 1, [&](int i) { return mul(ess[i], ess[i]); }, tid);
      if (tid == 0) {
      const double c0 = A[int64_t(k) * ld + k];
      double tau, beta, denom = 0.0;
      if (tail_sq <= DBL_MIN) {
        tau = 0.0;
        beta = c0;
      } else {
        beta = sqrt(add(mul(c0, c0), tail_sq));
        if (c0 >= 0.0) beta = -beta;
        denom = sub(c0, beta);
        tau = __ddiv_rn(sub(beta, c0), beta);
      }
      s_tau = tau;
      s_beta = beta;
      s_denom = denom;
      }
    }
    __syncthreads();
    const double tau = s_tau;
    for (int i = 1 + tid; i < len; i += blockDim.x) {
      const double v = (tau == 0.0 && s_denom == 0.0) ? 0.0 : __ddiv_rn(ess[i - 1], s_denom);
      A[int64_t(k + i) * ld + k] = v;
      ess[i - 1] = v;
      tess[i - 1] = mul(tau, v);
    }
    if (tid == 0) A[int64_t(k) * ld + k] = s_beta;
    __syncthreads();
    // (3) applyHouseholderOnTheLeft on the trailing columns. A thread owns an aligned column
    // PAIR (2p, 2p+1) and streams both with 16-byte loads, 8 rows ahead of the order-preserving
    // accumulation, so each SM keeps enough bytes in flight to approach its HBM share.
    const int nc = cols - k - 1, m1 = len - 1;
    if (len == 1 || tau == 0.0 || nc == 1) {
      for (int j = k + 1 + tid; j < cols; j += blockDim.x) {
        double* top = &A[int64_t(k) * ld + j];
        if (len == 1) {
          *top = mul(*top, sub(1.0, tau));
        } else if (tau != 0.0) {  // nc == 1: a single column falls back to an inner product
          double* bcol = &A[int64_t(k + 1) * ld + j];
          double t = redux_packet(m1, [&](int i) { return mul(ess[i], bcol[int64_t(i) * ld]); });
          t = add(t, *top);
          *top = sub(*top, mul(tau, t));
          for (int i = 0; i < m1; ++i) bcol[int64_t(i) * ld] = sub(bcol[int64_t(i) * ld], mul(t, tess[i]));
        }
      }
    } else {
      for (int pr = ((k + 1) >> 1) + tid; 2 * pr < cols; pr += blockDim.x) {
        const int j0 = 2 * pr;
        const bool act0 = j0 > k, act1 = j0 + 1 > k && j0 + 1 < cols;
        const double* b = &A[int64_t(k + 1) * ld + j0];
        double c0a = 0.0, c1a = 0.0, c0b = 0.0, c1b = 0.0;
        int i = 0;
        for (; i + 16 <= m1; i += 16) {
          double2 x[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) x[u] = *reinterpret_cast<const double2*>(b + int64_t(i + u) * ld);
#pragma unroll
          for (int u = 0; u < 16; u += 2) {
            c0a = add(c0a, mul(x[u].x, ess[i + u]));
            c1a = add(c1a, mul(x[u + 1].x, ess[i + u + 1]));
            c0b = add(c0b, mul(x[u].y, ess[i + u]));
            c1b = add(c1b, mul(x[u + 1].y, ess[i + u + 1]));
          }
        }
        for (; i + 2 <= m1; i += 2) {
          const double2 x0 = *reinterpret_cast<const double2*>(b + int64_t(i) * ld);
          const double2 x1 = *reinterpret_cast<const double2*>(b + int64_t(i + 1) * ld);
          c0a = add(c0a, mul(x0.x, ess[i]));
          c1a = add(c1a, mul(x1.x, ess[i + 1]));
          c0b = add(c0b, mul(x0.y, ess[i]));
          c1b = add(c1b, mul(x1.y, ess[i + 1]));
        }
        double ta = add(c0a, c1a), tb = add(c0b, c1b);
        for (; i < m1; ++i) {
          const double2 x0 = *reinterpret_cast<const double2*>(b + int64_t(i) * ld);
          ta = add(ta, mul(x0.x, ess[i]));
          tb = add(tb, mul(x0.y, ess[i]));
        }
        double* top = &A[int64_t(k) * ld + j0];
        if (act0) {
          ta = add(ta, top[0]);
          top[0] = sub(top[0], mul(tau, ta));
        }
        if (act1) {
          tb = add(tb, top[1]);
          top[1] = sub(top[1], mul(tau, tb));
        }
        double* bw = &A[int64_t(k + 1) * ld + j0];
        if (act0 && act1) {
          // rows in blocks of 8: all loads of a block are issued before its stores (the compiler
          // cannot reorder loads across stores through the runtime stride on its own)
          int r = 0;
          for (; r + 16 <= m1; r += 16) {
            double2 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = *reinterpret_cast<const double2*>(bw + int64_t(r + u) * ld);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              v[u].x = sub(v[u].x, mul(ta, tess[r + u]));
              v[u].y = sub(v[u].y, mul(tb, tess[r + u]));
              *reinterpret_cast<double2*>(bw + int64_t(r + u) * ld) = v[u];
            }
          }
          for (; r < m1; ++r) {
            double2 v = *reinterpret_cast<double2*>(bw + int64_t(r) * ld);
            v.x = sub(v.x, mul(ta, tess[r]));
            v.y = sub(v.y, mul(tb, tess[r]));
            *reinterpret_cast<double2*>(bw + int64_t(r) * ld) = v;
          }
        } else {
          double* c = bw + (act0 ? 0 : 1);
          const double t = act0 ? ta : tb;
          int r = 0;
          for (; r + 8 <= m1; r += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = c[int64_t(r + u) * ld];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[int64_t(r + u) * ld] = sub(v[u], mul(t, tess[r + u]));
          }
          for (; r < m1; ++r) c[int64_t(r) * ld] = sub(c[int64_t(r) * ld], mul(t, tess[r]));
        }
      }
    }
    __syncthreads();
    // (4) LAPACK-style column-norm downdate (lawn176), one thread per column
    for (int j = k + 1 + tid; j < cols; j += blockDim.x) {
      if (upd[j] != 0.0) {
        const double top = A[int64_t(k) * ld + j];
        double t = __ddiv_rn(fabs(top), upd[j]);
        t = mul(add(1.0, t), sub(1.0, t));
        t = t < 0.0 ? 0.0 : t;
        const double ratio = __ddiv_rn(upd[j], direct[j]);
        const double t2 = mul(t, mul(ratio, ratio));
        if (t2 <= downdate_threshold) {
          const int tl = rows - k - 1;
          const double* cj = &A[int64_t(k + 1) * ld + j];
          direct[j] = tl > 0 ? sqrt(redux_packet(tl, [&](int i) {
            const double v = cj[int64_t(i) * ld];
            return mul(v, v);
          }))
                             : 0.0;
          upd[j] = direct[j];
        } else {
          upd[j] = mul(upd[j], sqrt(t));
        }
      }
    }
    __syncthreads();
  }

  // column permutation: identity with the recorded transpositions applied in order
  int* perm = perm_out + nd.perm_off;
  for (int j = tid; j < cols; j += blockDim.x) perm[j] = j;
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < size; ++k) {
      const int t = perm[k];
      perm[k] = perm[trans[k]];
      perm[trans[k]] = t;
    }
    // rank from the R diagonal (compress.hpp:166-171)
    const double lead = fabs(A[0]);
    int rank = 0;
    for (int l = 0; l < size; ++l)
      if (fabs(A[int64_t(l) * ld + l]) > mul(tau_tol, lead)) ++rank;
    const int maxrank = min(s_max, min(rows, cols));
    rank = max(1, min(rank, maxrank));
    s_rank = rank;
    rank_out[blockIdx.x] = rank;
    achieved_out[blockIdx.x] =
        (rank < size) ? __ddiv_rn(fabs(A[int64_t(rank) * ld + rank]), fmax(lead, 1e-300)) : 0.0;
    if (lead_out) lead_out[blockIdx.x] = lead;
  }
  __syncthreads();
  // proj = Zero(rank, cols); proj(l, perm[l]) = 1; proj(:, perm[j]) = R11^{-1} R12(:, j - rank)
  const int rank = s_rank;
  double* proj = proj_out + nd.proj_off;
  for (int64_t e = tid; e < int64_t(rank) * cols; e += blockDim.x) proj[e] = 0.0;
  __syncthreads();
  for (int l = tid; l < rank; l += blockDim.x) proj[int64_t(perm[l]) * rank + l] = 1.0;
  const bool solve = cols > rank && fabs(A[0]) > 0.0;
  if (solve)
    for (int c = tid; c < cols - rank; c += blockDim.x) {
      double* x = proj + int64_t(perm[rank + c]) * rank;  // column perm[rank + c], rows 0..rank-1
      for (int i = rank - 1; i >= 0; --i) {
        double sacc = A[int64_t(i) * ld + rank + c];
        for (int kk = i + 1; kk < rank; ++kk) sacc = sub(sacc, mul(A[int64_t(i) * ld + kk], x[kk]));
        x[i] = __ddiv_rn(sacc, A[int64_t(i) * ld + i]);
      }
    }
}

}  // namespace gofmm_skel

namespace {
struct DBuf {
  void* p = nullptr;
  ~DBuf() {
    if (p) cudaFree(p);
  }
};
thread_local char g_skel_err[256];
int skel_fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  snprintf(g_skel_err, sizeof(g_skel_err), "%s%s%s", what, e != cudaSuccess ? ": " : "",
           e != cudaSuccess ? cudaGetErrorString(e) : "");
  return code;
}
}  // namespace

namespace gofmm_skel {

double algorithmic_bytes(const std::vector<NodeDesc>& nd, double* flops_out) {
  // step k streams the (rows-k) x (cols-k) trailing block three times (Householder dot, update
  // read, update write), plus the transpose in and proj out
  double bytes = 0.0, flops = 0.0;
  for (const NodeDesc& q : nd) {
    const int sz = std::min(q.rows, q.cols);
    for (int k = 0; k < sz; ++k) {
      const double tb = double(q.rows - k) * double(q.cols - k - 1);
      bytes += 24.0 * tb;
      flops += 4.0 * tb;
    }
    bytes += 16.0 * double(q.rows) * q.cols;
  }
  if (flops_out) *flops_out = flops;
  return bytes;
}

int skel_device(std::vector<NodeDesc>& nd, const double* d_in, int32_t s, double tau, int32_t* rank_out,
                double* achieved_out, double* lead_out, int32_t* perm_out, double* proj_out, float* kernel_ms,
                std::string* err) {
  auto fail = [&](int code, const char* what, cudaError_t e) {
    if (err) *err = std::string(what) + (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : "");
    return code;
  };
  const int nnodes = int(nd.size());
  if (nnodes == 0) return GOFMM_OK;
  int64_t ws = 0, pe = 0, pj = 0;
  int max_rows = 0, max_cols = 0;
  for (NodeDesc& q : nd) {
    q.ws_off = ws;
    q.perm_off = pe;
    q.proj_off = pj;
    ws += int64_t(q.rows) * ((q.cols + 1) & ~1);  // row-major, even ld (kernel)
    pe += q.cols;
    pj += int64_t(std::min({s, q.rows, q.cols})) * q.cols;
    max_rows = std::max(max_rows, int(q.rows));
    max_cols = std::max(max_cols, int(q.cols));
  }
  const size_t smem = size_t(2 * max_cols + 2 * max_rows) * sizeof(double) + size_t(max_cols) * sizeof(int);
  if (smem > 200 * 1024) return fail(GOFMM_ERR_INVALID, "skeletonize_batch: block too large for one CTA", cudaSuccess);
  DBuf d_nd, d_ws, d_rank, d_ach, d_lead, d_perm, d_proj;
  cudaError_t e;
  auto al = [&](DBuf& b, size_t bytes) { return cudaMalloc(&b.p, std::max<size_t>(bytes, 8)); };
  if ((e = al(d_nd, nd.size() * sizeof(NodeDesc))) != cudaSuccess || (e = al(d_ws, ws * 8)) != cudaSuccess ||
      (e = al(d_rank, nnodes * 4)) != cudaSuccess || (e = al(d_ach, nnodes * 8)) != cudaSuccess ||
      (e = al(d_lead, nnodes * 8)) != cudaSuccess || (e = al(d_perm, pe * 4)) != cudaSuccess ||
      (e = al(d_proj, pj * 8)) != cudaSuccess)
    return fail(GOFMM_ERR_CUDA, "skeletonize_batch: device allocation", e);
  if ((e = cudaMemcpy(d_nd.p, nd.data(), nd.size() * sizeof(NodeDesc), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(skeletonize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
          cudaSuccess)
    return fail(GOFMM_ERR_CUDA, "skeletonize_batch: upload", e);
  cudaEvent_t ev[2];
  cudaEventCreate(&ev[0]);
  cudaEventCreate(&ev[1]);
  cudaEventRecord(ev[0]);
  skeletonize_kernel<<<unsigned(nnodes), kThreads, smem>>>(
      static_cast<NodeDesc*>(d_nd.p), d_in, static_cast<double*>(d_ws.p), s, tau, static_cast<int32_t*>(d_rank.p),
      static_cast<double*>(d_ach.p), static_cast<double*>(d_lead.p), static_cast<int32_t*>(d_perm.p),
      static_cast<double*>(d_proj.p));
  cudaEventRecord(ev[1]);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventSynchronize(ev[1]);
  float ms = 0.f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, ev[0], ev[1]);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (e != cudaSuccess) return fail(GOFMM_ERR_CUDA, "skeletonize_batch: kernel", e);
  if (kernel_ms) *kernel_ms = ms;
  // proj: per node maxrank x cols slot, of which rank x cols (ld = rank) is written
  if ((e = cudaMemcpy(rank_out, d_rank.p, size_t(nnodes) * 4, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(achieved_out, d_ach.p, size_t(nnodes) * 8, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (lead_out && (e = cudaMemcpy(lead_out, d_lead.p, size_t(nnodes) * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) ||
      (e = cudaMemcpy(perm_out, d_perm.p, size_t(pe) * 4, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(proj_out, d_proj.p, size_t(pj) * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return fail(GOFMM_ERR_CUDA, "skeletonize_batch: download", e);
  return GOFMM_OK;
}

}  // namespace gofmm_skel

extern "C" {

const char* gofmm_skeletonize_last_error(void) { return g_skel_err; }

int gofmm_skeletonize_batch(int32_t nnodes, const int32_t* rows, const int32_t* cols, const int64_t* block_off,
                            const double* blocks, int32_t s, double tau, int32_t device, int32_t* rank_out,
                            double* achieved_out, int32_t* perm_out, double* proj_out, gofmm_skel_stats* stats) {
  using namespace gofmm_skel;
  if (nnodes < 0 || (nnodes > 0 && (!rows || !cols || !block_off || !blocks || !rank_out || !achieved_out ||
                                    !perm_out || !proj_out)))
    return skel_fail(GOFMM_ERR_INVALID, "skeletonize_batch: null argument");
  if (s < 1 || !(tau >= 0.0)) return skel_fail(GOFMM_ERR_INVALID, "skeletonize_batch: s >= 1 and tau >= 0 required");
  if (nnodes == 0) return GOFMM_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return skel_fail(GOFMM_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return skel_fail(GOFMM_ERR_CUDA, "cudaSetDevice", e);
  std::vector<NodeDesc> nd(static_cast<size_t>(nnodes));
  int64_t in_elems = 0;
  for (int32_t t = 0; t < nnodes; ++t) {
    if (rows[t] < 1 || cols[t] < 1 || block_off[t] < 0)
      return skel_fail(GOFMM_ERR_INVALID, "skeletonize_batch: every node needs rows, cols >= 1");
    nd[t] = {block_off[t], 0, 0, 0, rows[t], cols[t]};
    in_elems = std::max(in_elems, block_off[t] + int64_t(rows[t]) * cols[t]);
  }
  auto t0 = std::chrono::steady_clock::now();
  DBuf d_in;
  if ((e = cudaMalloc(&d_in.p, std::max<size_t>(size_t(in_elems) * 8, 8))) != cudaSuccess ||
      (e = cudaMemcpy(d_in.p, blocks, size_t(in_elems) * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
    return skel_fail(GOFMM_ERR_CUDA, "skeletonize_batch: upload", e);
  float ms = 0.f;
  std::string err;
  const int rc = skel_device(nd, static_cast<const double*>(d_in.p), s, tau, rank_out, achieved_out, nullptr, perm_out,
                             proj_out, &ms, &err);
  if (rc != GOFMM_OK) return skel_fail(rc, err.c_str());
  if (stats) {
    stats->kernel_ms = ms;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    stats->bytes = algorithmic_bytes(nd, &stats->flops);
  }
  return GOFMM_OK;
}

}  // extern "C"
