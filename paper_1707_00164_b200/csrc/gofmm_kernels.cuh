// gofmm_kernels.cuh — sm_100a device code for the GOFMM evaluation phase (u = K~ W).
//
// One kernel family covers every phase of evaluate.hpp:141-217. Each phase is a list of
// output-stationary GROUPS; a group owns disjoint output rows C (M x R, column-major) and
// accumulates an ORDERED list of TERMS  C = sum_t op(A_t) (M x K_t) * B_t (K_t x R)  in
// registers, in the reference's accumulation order:
//   N2S      (Upward,   evaluate.hpp:150-163): 1 term  proj_a * [W_a | what_l;what_r]
//   DOWNWARD (Coupling + Downward, :164-195):   far terms in ascending partner id, then
//                                               proj_p[:,off:off+k]^T * c_p
//   OUTPUT   (Output,   :196-217):              D_a W_a, near terms in ascending block index,
//                                               proj_a^T c_a
// A operands are either stored (proj, materialised blocks; column- or row-major) or GENERATED
// in registers from point coordinates (matrix-free L2L / S2S: K_ij of oracle.hpp:148-192).
//
// Math: FP64 DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8; tcgen05 has no f64 kind), operands
// staged global->shared with cp.async multi-stage pipelines, accumulators in registers.
#pragma once

#include <cstdint>

namespace gofmm {

enum : int32_t { kTermRowMajorA = 1, kTermGen = 2 };

struct Term {
  const double* a;   // stored A (nullptr when generated)
  const double* b;   // B: K x R column-major, ldb
  const double* xr;  // generated: row points, point-major (dim doubles per point)
  const double* xc;  // generated: column points
  int64_t lda;
  int64_t ldb;
  int32_t K;
  int32_t flags;
};

struct Group {
  int64_t crow;  // first output row in the launch's C base (column-major, ldc given at launch)
  int32_t M;
  int32_t tbeg, tend;  // terms [tbeg, tend)
  int32_t pad;
};

struct Tile {
  int32_t group;
  int32_t m0;
};

// Kernel ids (include/gofmm_b200.h)
enum : int32_t { kKindNone = -1, kGaussian = 0, kLaplace = 1, kPolynomial = 2, kExponential = 4 };

struct KernelParams {
  double p0;  // gaussian: 1/(2h^2); exponential: 1/h; laplace: delta; polynomial: shift
  double p1;  // laplace: exponent (d-2); polynomial: degree
  int32_t dim;
  int32_t pad;
};

// ------------------------------------------------------------------ reduction order
// Eigen 3.4 redux over a dynamic unit-stride vector with 2-wide packets and two accumulators
// (the order the reference's squaredNorm()/dot() use on its SSE2 build; oracle/eigen_shim
// mirrors the same function). Keeping it makes generated entries match the stored ones to
// the last bit of d^2, leaving only the exp/pow ulp difference.
template <int D>
__device__ __forceinline__ double eigen_redux(const double* v) {
  if constexpr (D == 1) {
    return v[0];
  } else {
    constexpr int aligned = (D / 2) * 2;
    constexpr int aligned2 = (D / 4) * 4;
    double a0 = v[0], a1 = v[1];
    if constexpr (aligned > 2) {
      double b0 = v[2], b1 = v[3];
#pragma unroll
      for (int i = 4; i < aligned2; i += 4) {
        a0 = a0 + v[i];
        a1 = a1 + v[i + 1];
        b0 = b0 + v[i + 2];
        b1 = b1 + v[i + 3];
      }
      a0 = a0 + b0;
      a1 = a1 + b1;
      if constexpr (aligned > aligned2) {
        a0 = a0 + v[aligned2];
        a1 = a1 + v[aligned2 + 1];
      }
    }
    double res = a0 + a1;
#pragma unroll
    for (int i = aligned; i < D; ++i) res = res + v[i];
    return res;
  }
}

__device__ __forceinline__ double eigen_redux_rt(const double* v, int n) {
  if (n < 2) return v[0];
  const int aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  double a0 = v[0], a1 = v[1];
  if (aligned > 2) {
    double b0 = v[2], b1 = v[3];
    for (int i = 4; i < aligned2; i += 4) {
      a0 = a0 + v[i];
      a1 = a1 + v[i + 1];
      b0 = b0 + v[i + 2];
      b1 = b1 + v[i + 3];
    }
    a0 = a0 + b0;
    a1 = a1 + b1;
    if (aligned > aligned2) {
      a0 = a0 + v[aligned2];
      a1 = a1 + v[aligned2 + 1];
    }
  }
  double res = a0 + a1;
  for (int i = aligned; i < n; ++i) res = res + v[i];
  return res;
}

constexpr int kMaxDimRt = 16;

// K(x_i, x_j) exactly as the reference generators build it (oracle.hpp:148-218).
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_entry(const double* xi, const double* xj, const KernelParams& kp) {
  if constexpr (KIND == kPolynomial) {
    double t[DIM > 0 ? DIM : kMaxDimRt];
    if constexpr (DIM > 0) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) t[q] = xi[q] * xj[q];
      return pow(eigen_redux<DIM>(t) + kp.p0, kp.p1);
    } else {
      for (int q = 0; q < kp.dim; ++q) t[q] = xi[q] * xj[q];
      return pow(eigen_redux_rt(t, kp.dim) + kp.p0, kp.p1);
    }
  } else {
    double t[DIM > 0 ? DIM : kMaxDimRt];
    double d2;
    if constexpr (DIM > 0) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) {
        double e = xi[q] - xj[q];
        t[q] = e * e;
      }
      d2 = eigen_redux<DIM>(t);
    } else {
      for (int q = 0; q < kp.dim; ++q) {
        double e = xi[q] - xj[q];
        t[q] = e * e;
      }
      d2 = eigen_redux_rt(t, kp.dim);
    }
    if constexpr (KIND == kGaussian) {
      return exp(-d2 * kp.p0);
    } else if constexpr (KIND == kExponential) {
      return exp(-sqrt(d2) * kp.p0);
    } else {  // kLaplace: max(|d|, delta)^-(d-2)
      double rr = fmax(sqrt(d2), kp.p0);
      return pow(rr, -kp.p1);
    }
  }
}

// ------------------------------------------------------------------ async copy / DMMA helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D(8x8) += A(8x4, row) * B(4x8, col): lane holds A[lane/4][lane%4], B[lane%4][lane/4],
// D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ grouped multi-term GEMM
template <int BM, int BN, int WM, int WN, int BK, int STAGES>
struct GemmShape {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MT = WTM / 8, NT = WTN / 8;
  static constexpr int SA_COL = BM + 4;  // A column-major tile: [BK][BM+4] (m contiguous)
  static constexpr int SA_ROW = BK + 4;  // A row-major tile:    [BM][BK+4] (k contiguous)
  static constexpr int A_STAGE = (BK * SA_COL > BM * SA_ROW) ? BK * SA_COL : BM * SA_ROW;
  static constexpr int SB = BK + 4;  // B tile: [BN][BK+4]
  static constexpr int B_STAGE = BN * SB;
  static_assert(BK % 4 == 0 && BM % (8 * WM) == 0 && BN % (8 * WN) == 0, "tile shape");
  // padding of 4 doubles (8 banks) makes every half-warp fragment load conflict-free
  static_assert((SA_COL % 16) == 4 && (SB % 16) == 4 && (SA_ROW % 16) == 4, "bank padding");
  static constexpr size_t smem_bytes(int maxdim) {
    return sizeof(double) * (size_t(STAGES) * (A_STAGE + B_STAGE) + size_t(STAGES) * BK * maxdim +
                             size_t(BM) * maxdim);
  }
};

template <int BM, int BN, int WM, int WN, int BK, int STAGES, int KIND, int DIM>
__global__ void __launch_bounds__(WM* WN * 32)
    grouped_gemm_f64(const Tile* __restrict__ tiles, const Group* __restrict__ groups,
                     const Term* __restrict__ terms, int32_t R, KernelParams kp, double* __restrict__ cbase,
                     int64_t ldc) {
  using S = GemmShape<BM, BN, WM, WN, BK, STAGES>;
  constexpr int NTH = S::kThreads;
  constexpr bool kGen = (KIND != kKindNone);
  constexpr int XD = kGen ? (DIM > 0 ? DIM : kMaxDimRt) : 0;  // coordinate stride in smem

  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = sA + STAGES * S::A_STAGE;
  double* sXc = sB + STAGES * S::B_STAGE;  // [STAGES][BK][XD]
  double* sXr = sXc + STAGES * BK * XD;    // [BM][XD]

  const Tile tile = tiles[blockIdx.x];
  const Group grp = groups[tile.group];
  const int m0 = tile.m0;
  const int n0 = blockIdx.y * BN;
  const int M = grp.M;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp / WN) * S::WTM;
  const int wn0 = (warp % WN) * S::WTN;
  const int dim = (DIM > 0) ? DIM : kp.dim;

  // total pipeline steps across all terms
  int total = 0;
  for (int t = grp.tbeg; t < grp.tend; ++t) total += (terms[t].K + BK - 1) / BK;

  // row coordinates of generated terms (shared by every generated term of the group)
  if constexpr (kGen) {
    const double* xr = nullptr;
    for (int t = grp.tbeg; t < grp.tend; ++t)
      if (terms[t].flags & kTermGen) {
        xr = terms[t].xr;
        break;
      }
    if (xr)
      for (int i = tid; i < BM * dim; i += NTH) {
        int m = i / dim, q = i - m * dim;
        sXr[m * XD + q] = (m0 + m < M) ? xr[size_t(m0 + m) * dim + q] : 0.0;
      }
  }

  // producer cursor
  int pt = grp.tbeg, pk = 0;
  while (pt < grp.tend && terms[pt].K == 0) ++pt;

  auto load_stage = [&](int stage) {
    const Term T = terms[pt];
    const int k0 = pk;
    // B tile: BN columns x BK rows, 16-byte chunks along k
    double* dB = sB + stage * S::B_STAGE;
    for (int c = tid; c < BN * (BK / 2); c += NTH) {
      int n = c / (BK / 2), kc = (c - n * (BK / 2)) * 2;
      int gk = k0 + kc, gn = n0 + n;
      bool v = (gn < R) && (gk < T.K);
      const double* src = v ? T.b + gk + size_t(gn) * T.ldb : T.b;
      cp_async16(dB + n * S::SB + kc, src, v);
    }
    double* dA = sA + stage * S::A_STAGE;
    if (kGen && (T.flags & kTermGen)) {
      if constexpr (kGen) {
        double* dX = sXc + stage * BK * XD;
        for (int i = tid; i < BK * dim; i += NTH) {
          int kk = i / dim, q = i - kk * dim;
          bool v = (k0 + kk) < T.K;
          const double* src = v ? T.xc + size_t(k0 + kk) * dim + q : T.xc;
          cp_async8(dX + kk * XD + q, src, v);
        }
      }
    } else if (T.flags & kTermRowMajorA) {
      for (int c = tid; c < BM * (BK / 2); c += NTH) {
        int m = c / (BK / 2), kc = (c - m * (BK / 2)) * 2;
        int gk = k0 + kc, gm = m0 + m;
        bool v = (gm < M) && (gk < T.K);
        const double* src = v ? T.a + gk + size_t(gm) * T.lda : T.a;
        cp_async16(dA + m * S::SA_ROW + kc, src, v);
      }
    } else {
      for (int c = tid; c < BK * (BM / 2); c += NTH) {
        int kk = c / (BM / 2), mc = (c - kk * (BM / 2)) * 2;
        int gk = k0 + kk, gm = m0 + mc;
        bool v = (gm < M) && (gk < T.K);
        const double* src = v ? T.a + gm + size_t(gk) * T.lda : T.a;
        cp_async16(dA + kk * S::SA_COL + mc, src, v);
      }
    }
    // advance
    pk += BK;
    if (pk >= T.K) {
      pk = 0;
      ++pt;
      while (pt < grp.tend && terms[pt].K == 0) ++pt;
    }
  };

  double acc[S::MT][S::NT][2];
#pragma unroll
  for (int i = 0; i < S::MT; ++i)
#pragma unroll
    for (int j = 0; j < S::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // consumer cursor
  int ct = grp.tbeg, ck = 0;
  while (ct < grp.tend && terms[ct].K == 0) ++ct;

#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load_stage(s);
    cp_async_commit();
  }

#pragma unroll 1
  for (int s = 0; s < total; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (s + STAGES - 1 < total) load_stage((s + STAGES - 1) % STAGES);
    cp_async_commit();

    const int stage = s % STAGES;
    const int flags = terms[ct].flags;
    const int Kt = terms[ct].K;
    const double* tA = sA + stage * S::A_STAGE;
    const double* tB = sB + stage * S::B_STAGE;
    const double* tX = sXc + stage * BK * XD;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int kk = ks * 4 + tig;
      double a[S::MT];
      if (kGen && (flags & kTermGen)) {
        if constexpr (kGen) {
          const bool kv = (ck + kk) < Kt;
#pragma unroll
          for (int i = 0; i < S::MT; ++i) {
            const int row = wm0 + 8 * i + g;
            a[i] = kv ? kernel_entry<KIND, DIM>(sXr + row * XD, tX + kk * XD, kp) : 0.0;
          }
        }
      } else if (flags & kTermRowMajorA) {
#pragma unroll
        for (int i = 0; i < S::MT; ++i) a[i] = tA[(wm0 + 8 * i + g) * S::SA_ROW + kk];
      } else {
#pragma unroll
        for (int i = 0; i < S::MT; ++i) a[i] = tA[kk * S::SA_COL + wm0 + 8 * i + g];
      }
#pragma unroll
      for (int j = 0; j < S::NT; ++j) {
        const double b = tB[(wn0 + 8 * j + g) * S::SB + kk];
#pragma unroll
        for (int i = 0; i < S::MT; ++i) dmma884(acc[i][j][0], acc[i][j][1], a[i], b);
      }
    }
    ck += BK;
    if (ck >= Kt) {
      ck = 0;
      ++ct;
      while (ct < grp.tend && terms[ct].K == 0) ++ct;
    }
  }
  cp_async_wait<0>();

  // epilogue: registers -> C (column-major)
  double* c = cbase + grp.crow;
#pragma unroll
  for (int i = 0; i < S::MT; ++i) {
    const int m = m0 + wm0 + 8 * i + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < S::NT; ++j) {
      const int n = n0 + wn0 + 8 * j + 2 * tig;
      if (n < R) c[m + size_t(n) * ldc] = acc[i][j][0];
      if (n + 1 < R) c[m + size_t(n + 1) * ldc] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------------ permutations (K5)
// wp[t, c] = w[prow[t], c]   (evaluate.hpp:294-295, into the padded leaf layout; prow = -1 pads)
__global__ void permute_rows_in(const double* __restrict__ w, int64_t ldw, const int32_t* __restrict__ prow,
                                int64_t npad, int32_t r, int32_t cols_per_block, double* __restrict__ wp,
                                int64_t ldp) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= npad) return;
  const int32_t src = prow[t];
  const int c0 = blockIdx.y * cols_per_block;
  const int c1 = min(r, c0 + cols_per_block);
  for (int c = c0; c < c1; ++c) wp[t + size_t(c) * ldp] = (src >= 0) ? __ldg(w + src + size_t(c) * ldw) : 0.0;
}

// u[iperm[t], c] = up[t, c]   (unpermute, evaluate.hpp:21-25)
__global__ void unpermute_rows(const double* __restrict__ up, int64_t ldp, const int32_t* __restrict__ iperm,
                               int64_t n, int32_t r, int32_t cols_per_block, double* __restrict__ u, int64_t ldu) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t dst = iperm[t];
  const int c0 = blockIdx.y * cols_per_block;
  const int c1 = min(r, c0 + cols_per_block);
  for (int c = c0; c < c1; ++c) u[dst + size_t(c) * ldu] = up[t + size_t(c) * ldp];
}

// Materialise K(x_rows, x_cols) into a column-major block (far/D blocks in MATERIALIZE mode).
template <int KIND, int DIM>
__global__ void generate_block(const double* __restrict__ xr, int32_t rows, const double* __restrict__ xc,
                               int32_t cols, double* __restrict__ out, int64_t ld, KernelParams kp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= rows || j >= cols) return;
  const int dim = (DIM > 0) ? DIM : kp.dim;
  out[i + size_t(j) * ld] = kernel_entry<KIND, DIM>(xr + size_t(i) * dim, xc + size_t(j) * dim, kp);
}

}  // namespace gofmm
