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
// Blackwell mapping (tcgen05 has no f64 kind; FP64 tensor math is DMMA via mma.sync):
//   * one PRODUCER warp per CTA: lane 0 streams the B tiles (W_perm / what / c column blocks)
//     with TMA (cp.async.bulk.tensor, 128B swizzle) and the 32 lanes stage stored A tiles and
//     point coordinates with cp.async; both complete on a per-stage mbarrier;
//   * NC CONSUMER warps: fragment loads from shared memory + mma.sync.m8n8k4.f64 (SASS DMMA.8),
//     accumulators in registers, release the stage through an "empty" mbarrier;
//   * no __syncthreads in the main loop, so the MMA pipe never waits on address math.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <type_traits>

namespace gofmm {

enum : int32_t { kTermRowMajorA = 1, kTermGen = 2 };
// B buffer ids (tensor maps passed per launch): W_perm, what, c
enum : int32_t { kBufWp = 0, kBufWhat = 1, kBufC = 2 };

struct Term {
  const double* a;   // stored A (nullptr when generated)
  const CUtensorMap* amap;  // stored A: TMA view of this term's block (global memory, see encode_amap)
  const double* xr;  // generated: row points, point-major (dim doubles per point)
  const double* xc;  // generated: column points
  int64_t lda;
  int64_t b_row;  // first row of B (K x R) inside buffer `bbuf`
  int32_t K;
  int32_t flags;  // kTermRowMajorA | kTermGen
  int32_t bbuf;   // kBufWp / kBufWhat / kBufC
  int32_t pad;
};

// Group flags. kGroupLoadC: the accumulator starts from the current C instead of zero, so a term
// chain can be continued by a later launch with bitwise the same result as one launch (the
// distributed output phase runs D + near terms before the all-gather and proj^T c after it).
enum : int32_t { kGroupLoadC = 1 };

struct Group {
  int64_t crow;  // first output row in the launch's C base (column-major, ldc given at launch)
  int32_t M;
  int32_t tbeg, tend;  // terms [tbeg, tend)
  int32_t flags;       // kGroupLoadC
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

struct BMaps {
  CUtensorMap m[3];  // indexed by kBuf*
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

__device__ __forceinline__ double lds64(uint32_t addr);
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_entry(const double* xi, const double* xj, const KernelParams& kp);

// exp(x) for x <= 0 (Gaussian / Matern arguments), |relative error| <= ~3 ulp:
// x = (n/32) ln2 + f, |f| <= ln2/64, exp(f) by a degree-6 polynomial, 2^(j/32) from a 32-entry
// shared-memory table, 2^(n>>5) by an exponent add. 11 FP64 pipe ops instead of the ~22 of the
// libdevice exp; matrix-free entries are generated once per 256 output columns, so this is the
// generation cost that competes with the DMMA pipe.
__device__ __forceinline__ double exp_nonpos(double x, uint32_t tab) {
  const double kInvL = 46.166241308446828384;                       // 32 / ln2
  const double kShift = 6755399441055744.0;                         // 1.5 * 2^52
  const double kLhi = 6.93147180369123816490e-01 / 32.0;            // fdlibm ln2_hi / 32
  const double kLlo = 1.90821492927058770002e-10 / 32.0;            // fdlibm ln2_lo / 32
  const double t = fma(x, kInvL, kShift);
  const int n = __double2loint(t);
  const double nd = t - kShift;
  double f = fma(nd, -kLhi, x);
  f = fma(nd, -kLlo, f);
  double p = 1.0 / 720.0;
  p = fma(p, f, 1.0 / 120.0);
  p = fma(p, f, 1.0 / 24.0);
  p = fma(p, f, 1.0 / 6.0);
  p = fma(p, f, 0.5);
  p = fma(p, f, 1.0);
  p = fma(p, f, 1.0);
  const double r = p * lds64(tab + uint32_t(n & 31) * 8u);
  const int hi = __double2hiint(r) + ((n >> 5) << 20);
  const double s = __hiloint2double(hi, __double2loint(r));
  return x < -708.0 ? 0.0 : s;  // below ~2^-1022 the exponent add would wrap; K entries that small vanish
}

// K(x_i, x_j) as the reference generators build it (oracle.hpp:148-218): distance from the
// difference vector, then the kernel function. d^2 is accumulated with FMAs (<= 1 ulp from the
// reference's Eigen reduction); tab != 0 selects the table exp for Gaussian / Matern kernels.
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_entry_fast(const double* xi, const double* xj, const KernelParams& kp,
                                                    uint32_t tab) {
  if constexpr ((KIND == kGaussian || KIND == kExponential) && DIM > 0) {
    double d2 = 0.0;
#pragma unroll
    for (int q = 0; q < DIM; ++q) {
      const double e = xi[q] - xj[q];
      d2 = (q == 0) ? e * e : fma(e, e, d2);
    }
    if constexpr (KIND == kGaussian) {
      return exp_nonpos(-d2 * kp.p0, tab);
    } else {
      return exp_nonpos(-sqrt(d2) * kp.p0, tab);
    }
  } else {
    return kernel_entry<KIND, DIM>(xi, xj, kp);
  }
}

// K(x_i, x_j) exactly as the reference generators build it (oracle.hpp:148-218).
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_entry(const double* xi, const double* xj, const KernelParams& kp) {
  double t[DIM > 0 ? DIM : kMaxDimRt];
  const int dim = DIM > 0 ? DIM : kp.dim;
  if constexpr (KIND == kPolynomial) {
#pragma unroll
    for (int q = 0; q < (DIM > 0 ? DIM : kMaxDimRt); ++q)
      if (DIM > 0 || q < dim) t[q] = xi[q] * xj[q];
    const double ip = DIM > 0 ? eigen_redux<(DIM > 0 ? DIM : 1)>(t) : eigen_redux_rt(t, dim);
    return pow(ip + kp.p0, kp.p1);
  } else {
#pragma unroll
    for (int q = 0; q < (DIM > 0 ? DIM : kMaxDimRt); ++q)
      if (DIM > 0 || q < dim) {
        const double e = xi[q] - xj[q];
        t[q] = e * e;
      }
    const double d2 = DIM > 0 ? eigen_redux<(DIM > 0 ? DIM : 1)>(t) : eigen_redux_rt(t, dim);
    if constexpr (KIND == kGaussian) {
      return exp(-d2 * kp.p0);
    } else if constexpr (KIND == kExponential) {
      return exp(-sqrt(d2) * kp.p0);
    } else {  // kLaplace: max(|d|, delta)^-(d-2)
      return pow(fmax(sqrt(d2), kp.p0), -kp.p1);
    }
  }
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// explicit shared-window loads: the 1024-byte-aligned carve-up of dynamic shared memory hides
// the address space from the compiler, which would otherwise emit generic LD instructions
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// arrive once this thread's prior cp.async copies have landed (counts toward the init count)
__device__ __forceinline__ void mbar_cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// Producer-side wait for a free slot: the consumers hold it for a whole stage of DMMAs, so the
// waiting thread suspends (time hint) instead of spinning on the issue slots the consumers use.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// Programmatic dependent launch (host: launch_k in gofmm_capi.cu). Both are no-ops for a kernel
// launched without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// D(8x8) += A(8x4, row) * B(4x8, col): lane holds A[lane/4][lane%4], B[lane%4][lane/4],
// D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ grouped multi-term GEMM
constexpr int kBK = 16;  // k-depth per stage: one 128-byte TMA row of FP64
// Stored A tiles arrive by TMA (one tensor map per stored-A term, exact extents: partial tiles
// read zeros). Row-major A (A[m][k] = a[k + m*lda]) in boxes of 16 k x kABoxRow m, SWIZZLE_128B;
// column-major A (A[m][k] = a[m + k*lda]) in boxes of kABoxCol m x 16 k, SWIZZLE_64B.
constexpr int kABoxRow = 32, kABoxCol = 8;

// Warp roles: warpgroup 0 = producer (4 warps: thread 0 issues the B-tile TMA, all 128 threads
// stage stored A tiles / point coordinates with cp.async), then 16 consumer warps (4 per SM
// sub-partition, enough to keep the DMMA pipe fed through LDS and exp() latencies).
// setmaxnreg moves registers from the producer to the consumers: 640 threads launch with
// kLaunchRegs each; the producer drops to kProducerRegs, the consumers rise to kConsumerRegs.
constexpr int kProducerThreads = 128;
constexpr int kConsumerWarps = 16;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kLaunchRegs = 96, kProducerRegs = 56, kConsumerRegs = 104;
// setmaxnreg.inc blocks until the registers exist: the producer must release what consumers add
static_assert(4 * (kLaunchRegs - kProducerRegs) >= kConsumerWarps * (kConsumerRegs - kLaunchRegs),
              "setmaxnreg balance");

template <int BM, int BN, int WM, int WN, int STAGES, int XD>
struct GemmShape {
  static_assert(WM * WN == kConsumerWarps, "consumer warp grid");
  static constexpr int kThreads = kProducerThreads + kConsumerThreads;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MT = WTM / 8, NT = WTN / 8;
  // A tile of a stage (doubles): row-major / generated [BM][16] 128B-swizzled (swz128), or
  // column-major [BM/8][16][8] 64B-swizzled (acm64); 1024-byte aligned like the B tiles
  static constexpr int A_STAGE = BM * kBK;
  static_assert(BM % kABoxRow == 0 && (A_STAGE * 8) % 1024 == 0, "A tile = whole TMA boxes");
  static constexpr int B_STAGE_BYTES = BN * kBK * 8;  // TMA box, 128B-swizzled rows, 1024B aligned
  static constexpr int X_STAGE = kBK * XD;            // column coordinates (generated terms)
  static constexpr int GEN_PER_THREAD = (BM * kBK) / kConsumerThreads;
  static_assert(BM % (8 * WM) == 0 && BN % (8 * WN) == 0, "tile shape");
  static constexpr int kBoxN = BN > 256 ? 256 : BN;  // TMA box limit: wider tiles take several boxes
  static_assert(BN % kBoxN == 0, "B tile = whole TMA boxes");
  static_assert(B_STAGE_BYTES % 1024 == 0, "swizzle-128B tiles need 1024-byte multiples");
  static_assert((BM * kBK) % kConsumerThreads == 0 && kConsumerThreads % BM == 0, "generation mapping");
  static constexpr size_t smem_bytes = 1024 /* alignment slack */ + size_t(STAGES) * B_STAGE_BYTES +
                                       size_t(STAGES) * A_STAGE * 8 + size_t(STAGES) * X_STAGE * 8 +
                                       size_t(4 * STAGES) * 8 + 32 * 8 /* exp table */ +
                                       size_t(BM) * XD * 8 /* row coordinates */;
};

template <int BM, int BN, int WM, int WN, int STAGES, int KIND, int DIM>
constexpr size_t gemm_smem_bytes() {
  constexpr int XD = (KIND != kKindNone) ? (DIM > 0 ? DIM + 1 : kMaxDimRt + 1) : 0;
  return GemmShape<BM, BN, WM, WN, STAGES, XD>::smem_bytes;
}

// byte offset of element (n, k) in a 128B-swizzled [BN][16] FP64 tile
__device__ __forceinline__ uint32_t swz128(int n, int k) {
  return uint32_t(n) * 128u + ((uint32_t((k >> 1) ^ (n & 7)) << 4) | (uint32_t(k & 1) << 3));
}

// Physical k of MMA k-slot `tig` in sub-step `ks` of a 16-deep stage. The DMMA reduction is
// order-free in k, so A and B may use any common permutation; this one makes every half-warp
// of a 64-bit fragment load touch all 32 banks of the 128B-swizzled B tile (the identity map
// leaves a 2-way conflict per half-warp).
__device__ __forceinline__ int kpi(int ks, int tig) { return 2 * ks + (tig & 1) + 8 * (tig >> 1); }

// byte offset of A(m, k) in a column-major stored A tile as TMA writes it: boxes of 8 m x 16 k
// (1 KB each, m-box j at j*1024), rows of 64 bytes (one k), 64B swizzle (16-byte chunk ^= bits 7-8).
__device__ __forceinline__ uint32_t acm64(int m, int k) {
  return uint32_t(m >> 3) * 1024u + uint32_t(k) * 64u + ((uint32_t(((m & 7) >> 1) ^ ((k >> 1) & 3)) << 4) |
                                                        (uint32_t(m & 1) << 3));
}

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerThreads) : "memory");
}

template <int BM, int BN, int WM, int WN, int STAGES, int KIND, int DIM>
__global__ void __launch_bounds__(kProducerThreads + kConsumerThreads, 1)
    grouped_gemm_f64(const __grid_constant__ BMaps maps, const Tile* __restrict__ tiles,
                     const Group* __restrict__ groups, const Term* __restrict__ terms, int32_t R, KernelParams kp,
                     double* __restrict__ cbase, int64_t ldc, int32_t cpanel, int32_t n_off) {
  constexpr bool kGen = (KIND != kKindNone);
  constexpr int XD = kGen ? (DIM > 0 ? DIM + 1 : kMaxDimRt + 1) : 0;  // odd stride: no bank conflicts
  constexpr int DD = DIM > 0 ? DIM : kMaxDimRt;
  using S = GemmShape<BM, BN, WM, WN, STAGES, XD>;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sB = base;                                                  // [STAGES][BN*128B]
  double* sA = reinterpret_cast<double*>(sB + STAGES * S::B_STAGE_BYTES);    // [STAGES][A_STAGE]
  double* sX = sA + STAGES * S::A_STAGE;                                     // [STAGES][BK][XD]
  // full[STAGES] (B tile, TMA -> consumers), empty[STAGES] (consumers -> producer),
  // gen[STAGES] (consumers -> consumers: generated A tile of the stage is complete),
  // afull[STAGES] (stored A tile / column coordinates, producer cp.async -> consumers)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + STAGES * S::X_STAGE);
  double* sTab = reinterpret_cast<double*>(bars + 4 * STAGES);               // 2^(j/32), j < 32
  double* sXr = sTab + 32;                                                   // [BM][XD] row coordinates

  const Tile tile = tiles[blockIdx.x];
  const Group grp = groups[tile.group];
  const int m0 = tile.m0;
  const int n0 = n_off + blockIdx.y * BN;  // n_off: first column of a column-piece launch
  const int M = grp.M;
  const int lane = threadIdx.x & 31;
  const int dim = (DIM > 0) ? DIM : kp.dim;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);                              // B tile: 1 expect_tx (TMA)
      mbar_init(smem_u32(&bars[STAGES + s]), kConsumerWarps);
      mbar_init(smem_u32(&bars[2 * STAGES + s]), kConsumerWarps);
      mbar_init(smem_u32(&bars[3 * STAGES + s]), kProducerThreads);  // A tile / coordinates (cp.async)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) sTab[threadIdx.x] = exp2(double(threadIdx.x) * (1.0 / 32.0));
  __syncthreads();
  // the plan (tiles, groups, terms, proj, coordinates) is constant; W_perm / what / c / u are
  // written by earlier launches: let the next launch start its prologue, read the constant plan
  // data, and (producer) issue the constant A operands of the first stages before waiting for ours
  pdl_launch_dependents();

  // total pipeline steps across all terms
  int total = 0;
  for (int t = grp.tbeg; t < grp.tend; ++t) total += (terms[t].K + kBK - 1) / kBK;

  if (threadIdx.x < kProducerThreads) {
    // =========================== PRODUCER WARPGROUP ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    const int pth = threadIdx.x;
    // pipeline position of the A stream and of the B stream; the current term lives in registers
    // (the term table is read once per term boundary, never once per stage)
    struct PPos {
      int t, k;
      Term T;
    };
    auto first_pos = [&]() {
      PPos p{grp.tbeg, 0, Term{}};
      while (p.t < grp.tend && terms[p.t].K == 0) ++p.t;
      if (p.t < grp.tend) p.T = terms[p.t];
      return p;
    };
    auto advance_pos = [&](PPos& p) {
      p.k += kBK;
      if (p.k >= p.T.K) {
        p.k = 0;
        ++p.t;
        while (p.t < grp.tend && terms[p.t].K == 0) ++p.t;
        if (p.t < grp.tend) p.T = terms[p.t];
      }
    };
    // A operand of stage s (constant: stored A by TMA, or the generated term's column coordinates)
    // on the stage's afull barrier
    auto issue_a = [&](int s, const PPos& p) {
      const int stage = s % STAGES;
      const uint32_t afull = smem_u32(&bars[3 * STAGES + stage]);
      const Term& T = p.T;
      const int k0 = p.k;
      if (kGen && (T.flags & kTermGen)) {
        if constexpr (kGen) {
          const uint32_t dX = smem_u32(sX + stage * S::X_STAGE);
          for (int i = pth; i < kBK * dim; i += kProducerThreads) {
            const int kk = i / dim, q = i - kk * dim;
            const bool v = (k0 + kk) < T.K;
            cp_async8(dX + uint32_t(kk * XD + q) * 8u, v ? T.xc + size_t(k0 + kk) * dim + q : T.xc, v);
          }
        }
      } else if (pth == 0) {
        // stored A by TMA (its bytes are added to the phase first)
        const uint32_t dA = smem_u32(sA + stage * S::A_STAGE);
        mbar_expect_tx(afull, uint32_t(S::A_STAGE * 8));
        if (T.flags & kTermRowMajorA) {
#pragma unroll
          for (int j = 0; j < BM / kABoxRow; ++j)
            tma_load_2d(dA + uint32_t(j) * (kABoxRow * 128u), T.amap, k0, m0 + j * kABoxRow, afull);
        } else {
#pragma unroll
          for (int j = 0; j < BM / kABoxCol; ++j) tma_load_2d(dA + uint32_t(j) * 1024u, T.amap, m0 + j * kABoxCol, k0, afull);
        }
      }
      mbar_cp_async_arrive(afull);
    };
    PPos pa = first_pos();
    PPos pb = pa;
    // A of the first STAGES stages (their slots are free) before griddepcontrol.wait: under PDL
    // the term reads, tensor-map fetches and A loads overlap the previous launch
    const int pre = total < STAGES ? total : STAGES;
    for (int s = 0; s < pre; ++s) {
      issue_a(s, pa);
      advance_pos(pa);
    }
    pdl_wait();
    for (int s = 0; s < total; ++s) {
      const int stage = s % STAGES;
      const uint32_t full = smem_u32(&bars[stage]);
      if (s >= STAGES) {
        mbar_wait_sleep(smem_u32(&bars[STAGES + stage]), ((s / STAGES) & 1) ^ 1);
        issue_a(s, pa);
        advance_pos(pa);
      }
      if (pth == 0) {
        mbar_arrive_expect_tx(full, S::B_STAGE_BYTES);
        // B rows [b_row + k0, +16) = one 16-row panel (b_row is 16-aligned): a contiguous run
#pragma unroll
        for (int bx = 0; bx < BN / S::kBoxN; ++bx)
          tma_load_3d(smem_u32(sB + stage * S::B_STAGE_BYTES + bx * S::kBoxN * 128), &maps.m[pb.T.bbuf], 0,
                      n0 + bx * S::kBoxN, int32_t((pb.T.b_row + pb.k) >> 4), full);
      }
      advance_pos(pb);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // never exit with copies in flight
    return;
  }
  pdl_wait();

  // =========================== CONSUMER WARPS ===========================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
  const int cth = threadIdx.x - kProducerThreads;
  const int cw = cth >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (cw / WN) * S::WTM;
  const int wn0 = (cw % WN) * S::WTN;
  const uint32_t sB_u = smem_u32(sB), sA_u = smem_u32(sA), sX_u = smem_u32(sX);
  const uint32_t tabU = smem_u32(sTab);

  // generated terms: this thread produces rows gen_m, columns gen_k + i*(threads/BM) of each
  // BM x 16 tile, cooperatively with the other consumers (each entry is computed once per CTA)
  const int gen_m = cth % BM, gen_k = cth / BM;
  if constexpr (kGen) {
    // rows of every generated term of a group are the group's own points: stage them once
    const double* xrp = nullptr;
    for (int t = grp.tbeg; t < grp.tend; ++t)
      if (terms[t].flags & kTermGen) {
        xrp = terms[t].xr;
        break;
      }
    if (xrp)
      for (int i = cth; i < BM * dim; i += kConsumerThreads) {
        const int m = i / dim, q = i - m * dim;
        sXr[m * XD + q] = (m0 + m < M) ? xrp[size_t(m0 + m) * dim + q] : 0.0;
      }
    consumer_bar();
  }
  const uint32_t xrU = smem_u32(sXr) + uint32_t(gen_m * XD) * 8u;
  // fill the row-major A tile of stage s from the column coordinates the producer staged
  auto generate = [&](int s, int k0, int Kt) {
    if constexpr (kGen) {
      const int stage = s % STAGES;
      const uint32_t tX = sX_u + stage * S::X_STAGE * 8;
      const uint32_t tA = sA_u + stage * S::A_STAGE * 8;
      const bool row_ok = m0 + gen_m < M;
#pragma unroll
      for (int i = 0; i < S::GEN_PER_THREAD; ++i) {
        const int kk = gen_k + i * (kConsumerThreads / BM);
        double xc[DD], xr[DD];
#pragma unroll
        for (int q = 0; q < DD; ++q)
          if (DIM > 0 || q < dim) {
            xc[q] = lds64(tX + uint32_t(kk * XD + q) * 8u);
            xr[q] = lds64(xrU + uint32_t(q) * 8u);
          }
        const double v = (row_ok && k0 + kk < Kt) ? kernel_entry_fast<KIND, DIM>(xr, xc, kp, tabU) : 0.0;
        asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(tA + swz128(gen_m, kk)), "d"(v) : "memory");
      }
    }
  };

  double acc[S::MT][S::NT][2];
#pragma unroll
  for (int i = 0; i < S::MT; ++i)
#pragma unroll
    for (int j = 0; j < S::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (grp.flags & kGroupLoadC) {  // continue a chain: same addressing as the epilogue
#pragma unroll
    for (int i = 0; i < S::MT; ++i) {
      const int m = m0 + wm0 + 8 * i + g;
      if (m >= M) continue;
      const double* crow_ptr = cpanel ? cbase + (grp.crow >> 4) * ldc + size_t(m >> 4) * ldc + (m & 15)
                                      : cbase + grp.crow + m;
      const size_t cstride = cpanel ? 16 : size_t(ldc);
#pragma unroll
      for (int j = 0; j < S::NT; ++j) {
        const int n = n0 + wn0 + 8 * j + 2 * tig;
        if (n < R) acc[i][j][0] = crow_ptr[size_t(n) * cstride];
        if (n + 1 < R) acc[i][j][1] = crow_ptr[size_t(n + 1) * cstride];
      }
    }
  }

  // 8-row fragments of this warp that hold output rows: a group's last m-tile is partial whenever
  // its row count (a skeleton rank) is not a multiple of BM, and the fragments wholly past M are
  // skipped (warp-uniform) — e.g. rank 455 in 32-row tiles: the 15th tile runs 1 of 4 fragments
  const int mfrag = min(S::MT, max(0, (M - m0 - wm0 + 7) / 8));

  // swizzled B fragment offsets: row n = wn0 + 8j + g has (n & 7) == g
  uint32_t boff[kBK / 4];
#pragma unroll
  for (int ks = 0; ks < kBK / 4; ++ks) boff[ks] = swz128(wn0 + g, kpi(ks, tig));

  // pipeline position (term t, k offset) with the term's K and flags cached in registers: the
  // term table is read once per term boundary, not once per stage
  struct Pos {
    int t, k, K, flags;
  };
  auto advance = [&](Pos& p) {
    p.k += kBK;
    if (p.k >= p.K) {
      p.k = 0;
      ++p.t;
      while (p.t < grp.tend && terms[p.t].K == 0) ++p.t;
      if (p.t < grp.tend) {
        p.K = terms[p.t].K;
        p.flags = terms[p.t].flags;
      }
    }
  };
  Pos cur{grp.tbeg, 0, 0, 0};
  while (cur.t < grp.tend && terms[cur.t].K == 0) ++cur.t;
  if (cur.t < grp.tend) {
    cur.K = terms[cur.t].K;
    cur.flags = terms[cur.t].flags;
  }
  // Stage s+1 is waited for (and, if generated, generated) while stage s is multiplied; a
  // generated tile is published through the stage's `gen` mbarrier (one arrival per consumer
  // warp), so warps only wait for each other when one falls a whole stage behind.
  // Two barriers per stage: `afull` (stored A tile / column coordinates, cp.async) and `full`
  // (the B tile, TMA). Generating stage s+1 needs only its coordinates, so the warps do not wait
  // for stage s+1's B tile before multiplying stage s: B keeps a whole extra stage of lead.
  auto stage_in = [&](int s, const Pos& p) {
    mbar_wait(smem_u32(&bars[3 * STAGES + s % STAGES]), (s / STAGES) & 1);
    if constexpr (kGen) {
      if (p.flags & kTermGen) generate(s, p.k, p.K);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars[2 * STAGES + s % STAGES]));
    }
  };
  if (total > 0) stage_in(0, cur);
#pragma unroll 1
  for (int s = 0; s < total; ++s) {
    const int stage = s % STAGES;
    const int flags = cur.flags;
    Pos nxt = cur;
    advance(nxt);
    // generated operands: the next stage's tile is generated in the MIDDLE of this stage's DMMAs
    // (after k-step kGenAfter), so the warp's own queued DMMAs keep the FP64 pipe busy through
    // the generation's dependent-latency chains (all warps of an SM sub-partition reach that
    // point together; generating before the stage's first DMMA left the pipe idle meanwhile)
    constexpr int kGenAfter = kGen ? 2 : kBK / 4;
    if (!kGen && s + 1 < total) stage_in(s + 1, nxt);
    mbar_wait(smem_u32(&bars[stage]), (s / STAGES) & 1);
    if constexpr (kGen) mbar_wait(smem_u32(&bars[2 * STAGES + stage]), (s / STAGES) & 1);
    const bool rowA = (flags & (kTermRowMajorA | kTermGen)) != 0;  // generated tiles are row-major
    const uint32_t tA = sA_u + stage * S::A_STAGE * 8;
    const uint32_t tB = sB_u + stage * S::B_STAGE_BYTES;
    // one stage of DMMAs on the first MF 8-row fragments (MF = MT: every full tile; the partial
    // last tile of a group takes the instantiation for its fragment count — a warp-uniform branch
    // outside the unrolled loop, so full tiles keep their schedule)
    auto mma_stage = [&](auto mf_tag) {
      constexpr int MF = decltype(mf_tag)::value;
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        if (kGen && ks == kGenAfter && s + 1 < total) stage_in(s + 1, nxt);
        double a[S::MT];
#pragma unroll
        for (int i = 0; i < MF; ++i) {
          const int kk = kpi(ks, tig), m = wm0 + 8 * i + g;
          a[i] = lds64(tA + (rowA ? swz128(m, kk) : acm64(m, kk)));
        }
#pragma unroll
        for (int j = 0; j < S::NT; ++j) {
          const double b = lds64(tB + boff[ks] + 1024u * j);
#pragma unroll
          for (int i = 0; i < MF; ++i) dmma884(acc[i][j][0], acc[i][j][1], a[i], b);
        }
      }
    };
    // (only the 4-fragment warp tiles get a second, one-fragment copy: every extra copy of the
    // unrolled stage costs instruction-cache footprint — a 3-copy variant slowed the G config 20 %)
    if constexpr (S::MT >= 4) {
      if (mfrag == 1)
        mma_stage(std::integral_constant<int, 1>{});
      else
        mma_stage(std::integral_constant<int, S::MT>{});
    } else {
      mma_stage(std::integral_constant<int, S::MT>{});
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[STAGES + stage]));
    cur = nxt;
  }

  // epilogue: registers -> C; what / c in 16-row panels (crow is 16-aligned), u_perm column-major
#pragma unroll
  for (int i = 0; i < S::MT; ++i) {
    const int m = m0 + wm0 + 8 * i + g;
    if (m >= M) continue;
    double* crow_ptr = cpanel ? cbase + (grp.crow >> 4) * ldc + size_t(m >> 4) * ldc + (m & 15)
                              : cbase + grp.crow + m;
    const size_t cstride = cpanel ? 16 : size_t(ldc);
#pragma unroll
    for (int j = 0; j < S::NT; ++j) {
      const int n = n0 + wn0 + 8 * j + 2 * tig;
      if (n < R) crow_ptr[size_t(n) * cstride] = acc[i][j][0];
      if (n + 1 < R) crow_ptr[size_t(n + 1) * cstride] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------------ permutations (K5)
// wp[t, c] = w[prow[t], c]   (evaluate.hpp:294-295) into the padded leaf layout, stored in
// 16-row panels (panel stride `pstride` doubles); prow = -1 marks padding rows (written as 0).
// Rows [row0, row1) only (a rank's own leaves in a distributed evaluation).
// Each thread gathers RPT rows (stride blockDim) of every column it visits, all loads of a column
// issued before their stores: the random 8-byte gathers are latency-bound, so on large W the ILP
// (and RPT x fewer blocks) is what moves them (RPT = kPermRows); small W keeps one row per thread
// for parallelism (perm_rows_per_thread).
constexpr int kPermRows = 8;
inline int perm_rows_per_thread(int64_t rows, int32_t r) { return double(rows) * r >= 6.4e7 ? kPermRows : 1; }
template <int RPT>
__global__ void permute_rows_in(const double* __restrict__ w, int64_t ldw, const int32_t* __restrict__ prow,
                                int64_t row0, int64_t row1, int32_t r, int32_t cols_per_block,
                                double* __restrict__ wp, int64_t pstride) {
  const int64_t tb = row0 + int64_t(blockIdx.x) * blockDim.x * RPT + threadIdx.x;
  int32_t src[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int64_t t = tb + int64_t(i) * blockDim.x;
    src[i] = t < row1 ? prow[t] : -2;
  }
  const int c0 = blockIdx.y * cols_per_block;
  const int c1 = min(r, c0 + cols_per_block);
  for (int c = c0; c < c1; ++c) {
    double v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = (src[i] >= 0) ? __ldg(w + src[i] + size_t(c) * ldw) : 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t t = tb + int64_t(i) * blockDim.x;
      if (src[i] != -2) wp[(t >> 4) * pstride + (t & 15) + size_t(c) * 16] = v[i];
    }
  }
}

// Distributed evaluation: copy whole 16-row panels (first r columns) between the workspace
// (panel stride ws_pstride) and the compact exchange buffer (panel stride 16*r).
struct PanelSeg {
  int32_t buf;  // 0 = what, 1 = W_perm
  int32_t pad;
  int64_t ws_row;   // 16-aligned row in the workspace
  int64_t buf_row;  // 16-aligned row in the exchange buffer
  int64_t rows;     // multiple of 16
};

static __global__ void panel_copy(const PanelSeg* __restrict__ segs, double* __restrict__ what, double* __restrict__ wp,
                           int64_t ws_pstride, double* __restrict__ buf, int32_t r, int32_t to_buffer) {
  const PanelSeg sg = segs[blockIdx.x];
  double* ws = (sg.buf == 0) ? what : wp;
  const int64_t npan = sg.rows / 16;
  const int64_t per = int64_t(16) * r;  // the first r columns of a panel are contiguous
  for (int64_t p = blockIdx.y; p < npan; p += gridDim.y) {
    double* a = ws + (sg.ws_row / 16 + p) * ws_pstride;
    double* b = buf + (sg.buf_row / 16 + p) * per;
    if (to_buffer)
      for (int64_t i = threadIdx.x; i < per; i += blockDim.x) b[i] = a[i];
    else
      for (int64_t i = threadIdx.x; i < per; i += blockDim.x) a[i] = b[i];
  }
}

// Split term chains (latency-bound downward levels): a long group is evaluated as several
// segment groups, segment 0 into the group's own rows of c and segments 1.. into scratch rows of
// the same panel buffer; this adds them back, in segment order (deterministic).
struct ChainReduce {
  int64_t dst_row;   // 16-aligned row of the group in the panel buffer
  int32_t M;         // rows
  int32_t src_first; // first of nsrc scratch rows in the source-row list
  int32_t nsrc;
  int32_t pad;
};

static __global__ void chain_reduce(const ChainReduce* __restrict__ items, const int64_t* __restrict__ src_rows,
                                    double* __restrict__ c, int64_t pstride, int32_t r) {
  pdl_launch_dependents();
  pdl_wait();
  const ChainReduce it = items[blockIdx.x];
  const int64_t total = int64_t(it.M) * r;
  for (int64_t e = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.y) * blockDim.x) {
    const int m = int(e % it.M), n = int(e / it.M);
    auto at = [&](int64_t row) -> double& { return c[(row >> 4) * pstride + 16 * int64_t(n) + (row & 15)]; };
    double acc = at(it.dst_row + m);
    for (int q = 0; q < it.nsrc; ++q) acc += at(src_rows[it.src_first + q] + m);
    at(it.dst_row + m) = acc;
  }
}

// out[i, c] = sum_p part[p*nrows + i, c]  (fixed order over the partials: deterministic)
static __global__ void sum_partials(const double* __restrict__ part, int64_t ldp, int32_t nrows, int32_t nparts, int32_t r,
                             double* __restrict__ out, int64_t ldo) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(nrows) * r) return;
  const int i = int(e % nrows), c = int(e / nrows);
  double acc = 0.0;
  for (int p = 0; p < nparts; ++p) acc += part[int64_t(p) * nrows + i + size_t(c) * ldp];
  out[i + size_t(c) * ldo] = acc;
}

// u[iperm[t], c] = up[t, c]   (unpermute, evaluate.hpp:21-25)
static __global__ void unpermute_rows(const double* __restrict__ up, int64_t ldp, const int32_t* __restrict__ iperm,
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
