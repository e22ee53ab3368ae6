// gofmm_kernels_f32.cuh — FP32 evaluation phase on the 5th-generation tensor cores (tcgen05).
//
// Same grouped multi-term GEMM contract as gofmm_kernels.cuh (groups own output rows, ordered
// term lists C = sum_t A_t B_t in the reference's accumulation order, evaluate.hpp:141-217),
// computed at the north_star FP32 tolerance (1e-5) with 3xTF32 on tcgen05.mma kind::tf32:
//     A B  ~=  A_hi B_hi + A_hi B_lo + A_lo B_hi,   x_hi = tf32(x), x_lo = x - x_hi
// (plain TF32 is ~1e-3 and cannot meet 1e-5). Every operand that lives in HBM is stored already
// split (hi / lo FP32 arrays), so tiles go from HBM to shared memory untouched:
//   * B (W_perm / what / c) in 16-row panels, element (i, j) at (i/16)*16*r_ws + 16*j + i%16:
//     one TMA box {16 k, BN n} is a contiguous 64*BN-byte run and lands in the canonical
//     K-major SWIZZLE_64B UMMA layout (8-row x 64 B atoms, SBO 512 B);
//   * stored A (proj, materialised / stored blocks) as K-major FP32 copies built at create,
//     staged with cp.async into the same swizzled layout;
//   * generated A (matrix-free L2L / S2S, oracle.hpp:148-218): K entries computed in FP32
//     registers, split, and written straight into the swizzled A tile.
// The accumulator (128 x BN FP32) lives in TMEM; one elected thread issues the MMAs; the
// epilogue reads TMEM with tcgen05.ld and writes what / c back as hi / lo panels (u as FP32).
//
// Warp roles (384 threads, one CTA per SM):
//   warp 0   B producer (lane 0: two TMA boxes per stage, hi and lo, on one mbarrier)
//   warp 1   MMA issuer (lane 0: 2 k-steps x 3 products of tcgen05.mma M=128 N=BN K=8)
//   warp 2   TMEM allocator
//   warps 4-11  A producers (256 threads: row m = t % 128, k-half t / 128), then epilogue
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gofmm_kernels.cuh"

namespace gofmm {
namespace f32 {

struct Term {
  const float* a_hi;  // stored A, K-major: A[m][k] = a[k + m*lda] (lda multiple of 4)
  const float* a_lo;
  const CUtensorMap* amap;  // stored A: TMA views of a_hi, a_lo (two consecutive maps)
  const float* xr;  // generated: row points (point-major FP32, `dim` floats per point)
  const float* xc;  // generated: column points
  const float* xrn;  // Gaussian: -log2(e)/(2h^2) |x|^2 of the row / column points (from FP64)
  const float* xcn;
  int64_t lda;
  int64_t b_row;  // first row of B inside buffer `bbuf` (16-aligned)
  int32_t K;
  int32_t flags;  // kTermGen
  int32_t bbuf;   // kBufWp / kBufWhat / kBufC
  int32_t pad;
};

struct KernelParams {
  float p0;  // gaussian: log2(e)/(2h^2); exponential: log2(e)/h; laplace: delta; polynomial: shift
  float p1;  // laplace: exponent (d-2); polynomial: degree
  int32_t dim;
  int32_t pad;
};

struct BMaps {
  CUtensorMap m[3][2];  // [kBuf*][hi, lo]
};

constexpr int kBM = 128;        // UMMA M (cta_group::1): one TMEM lane per output row
constexpr int kBK = 16;         // k per stage: one 64-byte swizzle row of FP32
constexpr int kThreads = 384;   // 12 warps
constexpr int kAWarp0 = 4;      // first A-producer / epilogue warp
constexpr int kAThreads = 256;  // 8 warps
constexpr int kATileBytes = kBM * kBK * 4;  // 8 KB
// Accumulation segments. The tensor core's FP32 accumulate does not round to nearest: measured
// on this B200 (tools/microbench/umma_tf32_test.cu, K up to 16384) every tcgen05.mma loses
// ~0.3 ulp of the accumulator in a consistent direction, so the relative error grows LINEARLY
// with the number of MMAs into one accumulator (K = 4096: 3e-5, past the 1e-5 contract). Each
// TMEM accumulator therefore only lives for kSeg stages (6 kSeg MMAs, ~1e-6); the A-producer
// warps drain it into round-to-nearest FP32 registers while the MMAs continue in the other
// half of a ping-pong pair of TMEM accumulators.
constexpr int kSeg = 8;
// setmaxnreg: the producer / MMA / allocator warpgroup gives registers to the two A-producer
// warpgroups, which hold the BN/2 running sums of their row between drains
#ifndef GOFMM_F32_SETMAXNREG
#define GOFMM_F32_SETMAXNREG 1
#endif
constexpr bool kUseSetmaxnreg = GOFMM_F32_SETMAXNREG;
constexpr int kLaunchRegs = 168, kLowRegs = 56, kHighRegs = 224;
static_assert(128 * (kLaunchRegs - kLowRegs) >= 256 * (kHighRegs - kLaunchRegs), "setmaxnreg balance");

template <int BN, int STAGES>
struct Shape {
  static_assert(BN % 32 == 0 && BN >= 64 && BN <= 256, "UMMA N");
  static constexpr int kBTileBytes = BN * kBK * 4;
  // column point coordinates of a generated stage (16 x dim floats) + their scaled norms (16)
  static constexpr int kXBytes = kBK * (kMaxDimRt + 1) * 4 + 64;
  static constexpr int kStageBytes = 2 * kATileBytes + 2 * kBTileBytes;  // 1024-aligned (swizzle atoms)
  static constexpr int kTmemCols = 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;  // ping-pong pair
  static constexpr int kBars = 3 * STAGES + 4;  // full_a, full_b, empty, tmem_full[2], tmem_empty[2]
  static constexpr size_t smem_bytes =
      1024 + size_t(STAGES) * (kStageBytes + kXBytes) + size_t(kBars) * 8 + 16;
};

// ------------------------------------------------------------------ tcgen05 / proxy helpers
// K-major SWIZZLE_64B shared-memory matrix descriptor (tcgen05 format): start >> 4 in [0,14),
// LBO = 1 (unused for swizzled K-major), SBO = 512 B between 8-row atoms, version 1 (bits 46-47),
// layout type 4 = SWIZZLE_64B (bits 61-63). Advancing k by 8 TF32 = 32 B adds 2 to the start.
__device__ __forceinline__ uint64_t desc_kmajor_sw64(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(512 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(4) << 61);
}
// instruction descriptor, kind::tf32: D f32 (bits 4-5 = 1), A / B tf32 (bits 7-9, 10-12 = 2),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
// mbarrier wait that lets the hardware suspend the warp until the phase completes (bounded by
// the hint, in ns) instead of spinning: spinning warps take issue slots from the generators
__device__ __forceinline__ void mbar_sleep_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 32 lanes x 32 columns of FP32 from TMEM: thread t gets columns [col, col+32) of lane base+t
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// x = hi + lo with hi a TF32 value (round to nearest on the 10-bit mantissa) and lo exact
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  lo = x - hi;
}

// byte offset of the 16-byte chunk c (k = 4c..4c+3) of row m in a K-major SWIZZLE_64B tile
// (Swizzle<2,4,3>: address bits [4,6) ^= bits [7,9))
__device__ __forceinline__ uint32_t sw64(int m, int c) { return uint32_t(m) * 64u + (uint32_t(c ^ ((m >> 1) & 3)) << 4); }

__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// K(x_i, x_j) in FP32 (oracle.hpp:148-218 formulas; distance from the difference vector)
template <int KIND>
__device__ __forceinline__ float entry_from(float d2_or_ip, const KernelParams& kp) {
  if constexpr (KIND == kGaussian) {
    return ex2_approx(d2_or_ip);  // argument already -p0' d^2 (norm expansion in the kernel)
  } else if constexpr (KIND == kExponential) {
    return ex2_approx(-sqrtf(d2_or_ip) * kp.p0);
  } else if constexpr (KIND == kLaplace) {
    return powf(fmaxf(sqrtf(d2_or_ip), kp.p0), -kp.p1);
  } else {  // kPolynomial
    return powf(d2_or_ip + kp.p0, kp.p1);
  }
}

// Add accumulator segment `seg` (TMEM buffer seg & 1, truncating tensor-core accumulate) into the
// round-to-nearest FP32 running sums of this thread's row, then hand the buffer back to the MMA
// issuer. tfull0 / tempty0: the buffer-0 barriers (buffer 1's follow at +8 bytes).
template <int BN, int NCOL>
__device__ __forceinline__ void drain_segment(float (&acc)[NCOL], int seg, uint32_t tq, uint32_t tfull0,
                                              uint32_t tempty0, int lane) {
  const int b = seg & 1;
  mbar_sleep_wait(tfull0 + 8u * b, (seg >> 1) & 1);
  tc_fence_after();
#pragma unroll
  for (int cc = 0; cc < NCOL; cc += 32) {
    float v[32];
    tmem_ld32(tq + uint32_t(b * BN + cc), v);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[cc + i] += v[i];
  }
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(tempty0 + 8u * b);
}

// ------------------------------------------------------------------ the kernel
template <int BN, int STAGES, int KIND, int DIM>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_tf32x3(const __grid_constant__ BMaps maps, const Tile* __restrict__ tiles,
                        const Group* __restrict__ groups, const Term* __restrict__ terms, int32_t R,
                        KernelParams kp, float* __restrict__ c_hi, float* __restrict__ c_lo, int64_t ldc,
                        int32_t cpanel) {
  using S = Shape<BN, STAGES>;
  constexpr bool kGen = (KIND != kKindNone);
  constexpr int DD = DIM > 0 ? DIM : kMaxDimRt;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // stage s: [A_hi | A_lo | B_hi | B_lo]
  const uint32_t sbase = smem_u32(base);
  // [STAGES x (A_hi | A_lo | B_hi | B_lo)] [STAGES x X] [barriers] [TMEM address]
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + STAGES * (S::kStageBytes + S::kXBytes));
  // full_a[S] (A producers, 8 warp arrivals), full_b[S] (TMA tx), empty[S] (MMA commit),
  // tmem_full[2] (MMA commit at a segment end), tmem_empty[2] (8 drain-warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::kBars);
  auto bar_full_a = [&](int s) { return smem_u32(&bars[s]); };
  auto bar_full_b = [&](int s) { return smem_u32(&bars[STAGES + s]); };
  auto bar_empty = [&](int s) { return smem_u32(&bars[2 * STAGES + s]); };
  auto bar_tfull = [&](int b) { return smem_u32(&bars[3 * STAGES + b]); };
  auto bar_tempty = [&](int b) { return smem_u32(&bars[3 * STAGES + 2 + b]); };
  auto a_tile = [&](int s, int part) { return sbase + uint32_t(s * S::kStageBytes + part * kATileBytes); };
  auto x_tile = [&](int s) { return sbase + uint32_t(STAGES * S::kStageBytes + s * S::kXBytes); };
  auto b_tile = [&](int s, int part) {
    return sbase + uint32_t(s * S::kStageBytes + 2 * kATileBytes + part * S::kBTileBytes);
  };

  const Tile tile = tiles[blockIdx.x];
  const Group grp = groups[tile.group];
  const int m0 = tile.m0;
  const int n0 = blockIdx.y * BN;
  const int M = grp.M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full_a(s), kAThreads / 32 + 1);  // A-producer warps + the TMA thread
      mbar_init(bar_full_b(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_tfull(b), 1);
      mbar_init(bar_tempty(b), kAThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(S::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  // programmatic dependent launch (host: launch_gemm): prologue done; the plan (terms) is constant
  // and read before the wait, the B / C buffers are written by earlier launches
  pdl_launch_dependents();
  int total = 0;
  for (int t = grp.tbeg; t < grp.tend; ++t) total += (terms[t].K + kBK - 1) / kBK;
  pdl_wait();
  auto first_term = [&]() {
    int t = grp.tbeg;
    while (t < grp.tend && terms[t].K == 0) ++t;
    return t;
  };

  // Each role branch runs to the kernel's end on its own (no code after the branches): setmaxnreg
  // gives every region its own register budget only if no code is shared across the two.
  if (warp < kAWarp0) {
    if (kUseSetmaxnreg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kLowRegs));
  if (warp == 0) {
    // =========================== B PRODUCER (TMA) ===========================
    if (lane == 0) {
      // the current term lives in registers: every mbarrier wait clobbers memory, so a reference
      // into `terms` would be re-read from global memory at every stage
      int t = first_term(), k = 0;
      struct {
        const float *xc, *xcn;
        const CUtensorMap* amap;
        int64_t b_row;
        int32_t K, flags, bbuf;
      } T{};
      auto load_term = [&]() {
        if (t < grp.tend) {
          T.amap = terms[t].amap;
          T.xc = terms[t].xc;
          T.xcn = terms[t].xcn;
          T.b_row = terms[t].b_row;
          T.K = terms[t].K;
          T.flags = terms[t].flags;
          T.bbuf = terms[t].bbuf;
        }
      };
      load_term();
      for (int s = 0; s < total; ++s) {
        const int st = s % STAGES;
        mbar_sleep_wait(bar_empty(st), ((s / STAGES) & 1) ^ 1);
        const int32_t panel = int32_t((T.b_row + k) >> 4);
        // generated stage: the 16 column points' coordinates ride on the same barrier (one bulk
        // copy of 64*dim contiguous bytes; rows past K are padding points of the same buffer)
        const bool gen = kGen && (T.flags & kTermGen);
        const uint32_t xbytes = gen ? uint32_t(kBK * 4 * ((DIM > 0) ? DIM : kp.dim)) : 0u;
        constexpr uint32_t nbytes = (KIND == kGaussian) ? uint32_t(kBK * 4) : 0u;
        mbar_arrive_expect_tx(bar_full_b(st), 2 * S::kBTileBytes + xbytes + (gen ? nbytes : 0u));
        tma_load_3d(b_tile(st, 0), &maps.m[T.bbuf][0], 0, n0, panel, bar_full_b(st));
        tma_load_3d(b_tile(st, 1), &maps.m[T.bbuf][1], 0, n0, panel, bar_full_b(st));
        if (gen)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  x_tile(st)),
              "l"(T.xc + size_t(k) * ((DIM > 0) ? DIM : kp.dim)), "r"(xbytes), "r"(bar_full_b(st))
              : "memory");
        if (gen && nbytes)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  x_tile(st) + uint32_t(kBK * (kMaxDimRt + 1) * 4)),
              "l"(T.xcn + k), "r"(nbytes), "r"(bar_full_b(st))
              : "memory");
        // stored A (hi, lo): TMA into the stage's A tiles on full_a (exact extents: rows past M and
        // k past K read zero); a generated stage's A is written by the producer warps instead
        if (!gen) {
          mbar_arrive_expect_tx(bar_full_a(st), 2 * kATileBytes);
          tma_load_2d(a_tile(st, 0), T.amap, k, m0, bar_full_a(st));
          tma_load_2d(a_tile(st, 1), T.amap + 1, k, m0, bar_full_a(st));
        } else {
          mbar_arrive(bar_full_a(st));
        }
        k += kBK;
        if (k >= T.K) {
          k = 0;
          ++t;
          while (t < grp.tend && terms[t].K == 0) ++t;
          load_term();
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA ISSUER ===========================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kBM, BN);
      for (int s = 0; s < total; ++s) {
        const int st = s % STAGES;
        const uint32_t ph = (s / STAGES) & 1;
        const int seg = s / kSeg, b = seg & 1;
        const uint32_t dacc = tmem + uint32_t(b * BN);
        if (s % kSeg == 0 && seg >= 2) mbar_sleep_wait(bar_tempty(b), ((seg >> 1) - 1) & 1);  // drained?
        mbar_sleep_wait(bar_full_b(st), ph);
        mbar_sleep_wait(bar_full_a(st), ph);
        tc_fence_after();
        const uint64_t ah = desc_kmajor_sw64(a_tile(st, 0)), al = desc_kmajor_sw64(a_tile(st, 1));
        const uint64_t bh = desc_kmajor_sw64(b_tile(st, 0)), bl = desc_kmajor_sw64(b_tile(st, 1));
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint64_t o = uint64_t(kk * 2);  // 32 bytes along k
          mma_tf32(dacc, ah + o, bh + o, idesc, ((s % kSeg) | kk) != 0);
          mma_tf32(dacc, ah + o, bl + o, idesc, 1);
          mma_tf32(dacc, al + o, bh + o, idesc, 1);
        }
        umma_commit(bar_empty(st));  // frees the stage once these MMAs have read it
        if (s % kSeg == kSeg - 1 || s == total - 1) umma_commit(bar_tfull(b));  // segment done
      }
    }
  }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;\n" ::"n"(kThreads) : "memory");  // every epilogue store is issued
    if (warp == 2) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S::kTmemCols));
    }
  } else {
    if (kUseSetmaxnreg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kHighRegs));
    // =========================== A PRODUCERS ===========================
    const int p = threadIdx.x - kAWarp0 * 32;
    const int m = p & (kBM - 1), h = p >> 7;  // row, k-half (k = 8h .. 8h+7 of the stage)
    const bool row_ok = m0 + m < M;
    const int dim = (DIM > 0) ? DIM : kp.dim;
    float xr[DD];
    float ai = 0.f;
    if constexpr (kGen) {
      // rows of every generated term of a group are the group's own points
      const float* xrp = nullptr;
      for (int t = grp.tbeg; t < grp.tend; ++t)
        if (terms[t].flags & kTermGen) {
          xrp = terms[t].xr;
          break;
        }
#pragma unroll
      for (int q = 0; q < DD; ++q) xr[q] = (xrp && row_ok && (DIM > 0 || q < dim)) ? xrp[size_t(m0 + m) * dim + q] : 0.f;
      if constexpr (KIND == kGaussian) {
        // -p0' |xi - xj|^2 = ai + bj + sum_q (2 p0' xi_q) xj_q with ai, bj the scaled norms
        // (computed in FP64 at create): d + 1 FP32 ops per entry instead of 2d
        const float* xrn = nullptr;
        for (int t = grp.tbeg; t < grp.tend; ++t)
          if (terms[t].flags & kTermGen) {
            xrn = terms[t].xrn;
            break;
          }
        ai = (xrn && row_ok) ? xrn[m0 + m] : 0.f;
#pragma unroll
        for (int q = 0; q < DD; ++q) xr[q] *= 2.f * kp.p0;
      }
    }
    // drain state: this thread owns row em of the tile and columns [col0, col0 + BN/2)
    const int e = warp - kAWarp0;  // 0..7
    const int q = warp & 3;        // TMEM lane quarter this warp may access
    const int em = 32 * q + lane;  // tile row
    constexpr int kHalf = BN / 2;
    const int col0 = (e >> 2) * kHalf;
    float acc[kHalf];
#pragma unroll
    for (int i = 0; i < kHalf; ++i) acc[i] = 0.f;
    const int nseg = (total + kSeg - 1) / kSeg;
    int drained = 0;
    const uint32_t tq = tmem + (uint32_t(32 * q) << 16) + uint32_t(col0);
    int t = first_term(), k = 0;
    // current term in registers (see the TMA thread): K, flags and the stored-A operand
    int tK = 0, tFlags = 0;
    auto load_term = [&]() {
      if (t < grp.tend) {
        tK = terms[t].K;
        tFlags = terms[t].flags;
      }
    };
    load_term();
    auto arrive = [&](int st) {
      fence_proxy_async();  // generic-proxy writes -> visible to the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_full_a(st));
    };
    for (int s = 0; s < total; ++s) {
      const int st = s % STAGES;
      mbar_sleep_wait(bar_empty(st), ((s / STAGES) & 1) ^ 1);
      // the MMAs of stage s - STAGES have completed: once that closes a segment, drain it now
      // (its commit precedes or accompanies this stage's release, so the wait is short)
      if (s >= STAGES && (s - STAGES + 1) % kSeg == 0)
        drain_segment<BN, kHalf>(acc, drained++, tq, bar_tfull(0), bar_tempty(0), lane);
      const uint32_t dh = a_tile(st, 0), dl = a_tile(st, 1);
      if (kGen && (tFlags & kTermGen)) {
        if constexpr (kGen) {
          float v[8];
          const int kb = k + 8 * h;
          const int nv = row_ok ? min(8, tK - kb) : 0;  // valid entries of this thread's 8
          // column coordinates of this stage (bulk-copied with the B tiles): broadcast LDS
          mbar_sleep_wait(bar_full_b(st), (s / STAGES) & 1);
          const uint32_t xs = x_tile(st) + uint32_t(8 * h * dim) * 4u;
          float bn[8];  // scaled column norms (Gaussian)
          if constexpr (KIND == kGaussian) {
            const uint32_t xn = x_tile(st) + uint32_t(kBK * (kMaxDimRt + 1) * 4 + 32 * h);
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(bn[0]), "=f"(bn[1]), "=f"(bn[2]), "=f"(bn[3]) : "r"(xn));
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(bn[4]), "=f"(bn[5]), "=f"(bn[6]), "=f"(bn[7]) : "r"(xn + 16u));
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float xc[DD];
            if constexpr (DIM > 0 && DIM % 4 == 0) {
#pragma unroll
              for (int q = 0; q < DIM; q += 4) {
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                             : "=f"(xc[q]), "=f"(xc[q + 1]), "=f"(xc[q + 2]), "=f"(xc[q + 3])
                             : "r"(xs + uint32_t(j * DIM + q) * 4u));
              }
            } else {
#pragma unroll
              for (int q = 0; q < DD; ++q)
                if (DIM > 0 || q < dim)
                  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(xc[q]) : "r"(xs + uint32_t(j * dim + q) * 4u));
            }
            float acc = 0.f;
            if constexpr (KIND == kGaussian) {
              acc = ai + bn[j];
#pragma unroll
              for (int q = 0; q < DD; ++q)
                if (DIM > 0 || q < dim) acc = fmaf(xr[q], xc[q], acc);
            } else if constexpr (KIND == kPolynomial) {
#pragma unroll
              for (int q = 0; q < DD; ++q)
                if (DIM > 0 || q < dim) acc = fmaf(xr[q], xc[q], acc);
            } else {
#pragma unroll
              for (int q = 0; q < DD; ++q)
                if (DIM > 0 || q < dim) {
                  const float e = xr[q] - xc[q];
                  acc = fmaf(e, e, acc);
                }
            }
            v[j] = entry_from<KIND>(acc, kp);
          }
          if (nv < 8) {  // ragged tail of a term / rows past M: zero (never taken mid-term)
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (j < nv) ? v[j] : 0.f;
          }
          float hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) split_tf32(v[j], hi[j], lo[j]);
          sts128(dh + sw64(m, 2 * h), hi[0], hi[1], hi[2], hi[3]);
          sts128(dh + sw64(m, 2 * h + 1), hi[4], hi[5], hi[6], hi[7]);
          sts128(dl + sw64(m, 2 * h), lo[0], lo[1], lo[2], lo[3]);
          sts128(dl + sw64(m, 2 * h + 1), lo[4], lo[5], lo[6], lo[7]);
        }
        arrive(st);
      } else {
        // stored A arrives by TMA (the TMA thread); this warp only marks the stage
        arrive(st);
      }
      k += kBK;
      if (k >= tK) {
        k = 0;
        ++t;
        while (t < grp.tend && terms[t].K == 0) ++t;
        load_term();
      }
    }

    // =========================== EPILOGUE: registers -> C ===========================
    while (drained < nseg) drain_segment<BN, kHalf>(acc, drained++, tq, bar_tfull(0), bar_tempty(0), lane);
    const int gm = m0 + em;
    if (gm < M) {
      const int64_t row = grp.crow + gm;
      if (cpanel) {
        float* ph = c_hi + (row >> 4) * ldc + (row & 15);
        float* pl = c_lo + (row >> 4) * ldc + (row & 15);
#pragma unroll
        for (int i = 0; i < kHalf; ++i) {
          const int n = n0 + col0 + i;
          if (n < R) {
            float hi, lo;
            split_tf32(acc[i], hi, lo);
            ph[size_t(n) * 16] = hi;
            pl[size_t(n) * 16] = lo;
          }
        }
      } else {
        float* pu = c_hi + row;
#pragma unroll
        for (int i = 0; i < kHalf; ++i) {
          const int n = n0 + col0 + i;
          if (n < R) pu[size_t(n) * ldc] = acc[i];
        }
      }
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;\n" ::"n"(kThreads) : "memory");
  }
}

// ------------------------------------------------------------------ host-side entry points
// (defined in gofmm_f32.cu, a separate translation unit compiled in parallel with the C-ABI)

// One stored-A operand of the FP32 plan: a (rows x cols) K-major copy, split into hi / lo, of
// an FP64 device matrix. trans = 0: A[m][k] = src[k + m*lds] (already K-major, e.g. proj^T);
// trans = 1: A[m][k] = src[m + k*lds] (column-major source, e.g. proj for N2S).
struct SplitJob {
  const double* src;
  int64_t lds;
  int64_t dst;  // offset (floats) into the hi / lo blobs; row stride ldd
  int32_t rows, cols, ldd, trans;
};

using GemmFn = void (*)(BMaps, const Tile*, const Group*, const Term*, int32_t, KernelParams, float*, float*, int64_t,
                        int32_t);
struct GemmKernel {
  GemmFn fn = nullptr;
  size_t smem = 0;
  int bn = 0;
};
// kind = kKindNone for stored operands only; bn in {64, 128, 256}; sets the smem attribute
GemmKernel pick_gemm(int kind, int dim, int bn);
cudaError_t launch_gemm(const GemmKernel& k, unsigned ntiles, int32_t R, const BMaps& maps, const Tile* tiles,
                        const Group* groups, const Term* terms, const KernelParams& kp, float* c_hi, float* c_lo,
                        int64_t ldc, int32_t cpanel, cudaStream_t st, bool pdl = false);
cudaError_t launch_chain_reduce(const ChainReduce* items, int n, const int64_t* src_rows, float* ch, float* cl,
                                int64_t pstride, int32_t r, cudaStream_t st, bool pdl);
cudaError_t launch_permute_in(const float* w, int64_t ldw, const int32_t* prow, int64_t row0, int64_t row1, int32_t r,
                              int64_t n, float* wh, float* wl, int64_t pstride, cudaStream_t st);
cudaError_t launch_permute_in_2pass(const float* w, int64_t ldw, const int32_t* prow, int64_t row0, int64_t row1,
                                    int32_t r, int64_t n, float* wh, float* wl, int64_t pstride, float* scratch,
                                    int64_t ldt, cudaStream_t st);
cudaError_t launch_unpermute(const float* up, int64_t ldp, const int32_t* iperm, int64_t n, int32_t r, float* u,
                             int64_t ldu, cudaStream_t st);
cudaError_t launch_split(const SplitJob* d_jobs, int njobs, float* hi, float* lo, cudaStream_t st);
cudaError_t launch_to_f32(const double* x, int64_t n, float* y, cudaStream_t st);
cudaError_t launch_panel_copy(const PanelSeg* segs, int nseg, float* what_h, float* what_l, float* wp_h, float* wp_l,
                              int64_t ws_pstride, float* buf, int32_t r, int64_t slot_rows, int32_t to_buffer,
                              cudaStream_t st);
cudaError_t launch_scaled_norms(const double* x, int64_t npts, int dim, double scale, float* out, cudaStream_t st);

}  // namespace f32
}  // namespace gofmm
