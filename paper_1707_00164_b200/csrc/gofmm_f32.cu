// gofmm_f32.cu — FP32 (3xTF32 tcgen05) kernel instantiations and launch wrappers.
// A separate translation unit from the C-ABI (gofmm_capi.cu) so the two compile in parallel;
// the C-ABI reaches everything here through the entry points declared in gofmm_kernels_f32.cuh.
#include "gofmm_kernels_f32.cuh"

#include <algorithm>

namespace gofmm {
namespace f32 {
namespace {

// ------------------------------------------------------------------ data movement (FP32 path)
// wp_{hi,lo}[t, c] = split(w[prow[t], c]) in 16-row panels (evaluate.hpp:294-295)
// kPermRows rows per thread (stride blockDim), all loads of a column before their stores (ILP for
// the latency-bound random gathers, as in the FP64 permute_rows_in)
template <int RPT>
__global__ void permute_rows_in_f32(const float* __restrict__ w, int64_t ldw, const int32_t* __restrict__ prow,
                                    int64_t row0, int64_t row1, int32_t r, int32_t cols_per_block,
                                    float* __restrict__ wh, float* __restrict__ wl, int64_t pstride) {
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
    float x[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) x[i] = (src[i] >= 0) ? __ldg(w + src[i] + size_t(c) * ldw) : 0.f;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (src[i] == -2) continue;
      const int64_t t = tb + int64_t(i) * blockDim.x;
      const int64_t o = (t >> 4) * pstride + (t & 15) + size_t(c) * 16;
      float hi, lo;
      split_tf32(x[i], hi, lo);
      wh[o] = hi;
      wl[o] = lo;
    }
  }
}

// Split term chains (see chain_reduce in gofmm_kernels.cuh): segment partials in scratch rows of
// the hi / lo panel pair are added to the group's rows in segment order; each partial is the FP32
// accumulator the epilogue split as hi + lo, so the sum is formed from hi + lo and split again.
static __global__ void chain_reduce_f32(const ChainReduce* __restrict__ items, const int64_t* __restrict__ src_rows,
                                        float* __restrict__ ch, float* __restrict__ cl, int64_t pstride, int32_t r) {
  pdl_launch_dependents();
  pdl_wait();
  const ChainReduce it = items[blockIdx.x];
  const int64_t total = int64_t(it.M) * r;
  for (int64_t e = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.y) * blockDim.x) {
    const int m = int(e % it.M), n = int(e / it.M);
    auto off = [&](int64_t row) { return (row >> 4) * pstride + 16 * int64_t(n) + (row & 15); };
    const int64_t d = off(it.dst_row + m);
    float acc = ch[d] + cl[d];
    for (int q = 0; q < it.nsrc; ++q) {
      const int64_t o = off(src_rows[it.src_first + q] + m);
      acc += ch[o] + cl[o];
    }
    float hi, lo;
    split_tf32(acc, hi, lo);
    ch[d] = hi;
    cl[d] = lo;
  }
}

// u[iperm[t], c] = up[t, c]
static __global__ void unpermute_rows_f32(const float* __restrict__ up, int64_t ldp, const int32_t* __restrict__ iperm,
                                   int64_t n, int32_t r, int32_t cols_per_block, float* __restrict__ u, int64_t ldu) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t dst = iperm[t];
  const int c0 = blockIdx.y * cols_per_block;
  const int c1 = min(r, c0 + cols_per_block);
  for (int c = c0; c < c1; ++c) u[dst + size_t(c) * ldu] = up[t + size_t(c) * ldp];
}

static __global__ void split_to_kmajor(const SplitJob* __restrict__ jobs, float* __restrict__ hi, float* __restrict__ lo) {
  const SplitJob J = jobs[blockIdx.x];
  const int64_t n = int64_t(J.rows) * J.ldd;
  for (int64_t e = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.y) * blockDim.x) {
    const int m = int(e / J.ldd), k = int(e % J.ldd);
    double x = 0.0;
    if (k < J.cols) x = J.trans ? J.src[m + size_t(k) * J.lds] : J.src[k + size_t(m) * J.lds];
    float h, l;
    split_tf32(float(x), h, l);
    hi[J.dst + e] = h;
    lo[J.dst + e] = float(x - double(h));  // the FP64 residual: hi + lo carries ~2^-35 more
  }
}

static __global__ void to_f32(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = float(x[i]);
}


// out[p] = float(scale * |x_p|^2) in FP64 (Gaussian norm expansion operands)
static __global__ void scaled_norms(const double* __restrict__ x, int64_t npts, int dim, double scale,
                                    float* __restrict__ out) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npts; p += int64_t(gridDim.x) * blockDim.x) {
    double s2 = 0.0;
    for (int q = 0; q < dim; ++q) s2 = fma(x[p * dim + q], x[p * dim + q], s2);
    out[p] = float(scale * s2);
  }
}

// Subtree-split exchange (FP32): whole 16-row panels (first r columns, hi and lo) between the
// workspace and the exchange buffer. Each rank's slot holds slot_rows x r hi floats followed by
// slot_rows x r lo floats; a segment's buf_row = slot * slot_rows + offset in the slot.
static __global__ void panel_copy_f32(const PanelSeg* __restrict__ segs, float* __restrict__ what_h,
                                      float* __restrict__ what_l, float* __restrict__ wp_h, float* __restrict__ wp_l,
                                      int64_t ws_pstride, float* __restrict__ buf, int32_t r, int64_t slot_rows,
                                      int32_t to_buffer) {
  const PanelSeg sg = segs[blockIdx.x];
  const int64_t npan = sg.rows / 16;
  const int64_t per = int64_t(16) * r;
  const int64_t slot = sg.buf_row / slot_rows, off = sg.buf_row % slot_rows;
  float* bh = buf + slot * 2 * slot_rows * r + (off / 16) * per;
  float* bl = bh + slot_rows * r;
  float* wh = (sg.buf == 0 ? what_h : wp_h) + (sg.ws_row / 16) * ws_pstride;
  float* wl = (sg.buf == 0 ? what_l : wp_l) + (sg.ws_row / 16) * ws_pstride;
  for (int64_t p = blockIdx.y; p < npan; p += gridDim.y) {
    for (int64_t i = threadIdx.x; i < per; i += blockDim.x) {
      if (to_buffer) {
        bh[p * per + i] = wh[p * ws_pstride + i];
        bl[p * per + i] = wl[p * ws_pstride + i];
      } else {
        wh[p * ws_pstride + i] = bh[p * per + i];
        wl[p * ws_pstride + i] = bl[p * per + i];
      }
    }
  }
}

template <int BN>
constexpr int stages_for() {
  return BN == 256 ? 4 : BN == 128 ? 6 : 8;  // ~192 KB of pipeline in every configuration
}

template <int KIND, int DIM, int BN>
GemmKernel make_kernel() {
  constexpr int ST = stages_for<BN>();
  GemmKernel k;
  k.fn = &grouped_gemm_tf32x3<BN, ST, KIND, DIM>;
  k.smem = Shape<BN, ST>::smem_bytes;
  k.bn = BN;
  return k;
}

template <int KIND, int DIM>
GemmKernel by_bn(int bn) {
  if (bn <= 64) return make_kernel<KIND, DIM, 64>();
  if (bn <= 128) return make_kernel<KIND, DIM, 128>();
  return make_kernel<KIND, DIM, 256>();
}

template <int KIND>
GemmKernel by_dim(int dim, int bn) {
  switch (dim) {
    case 3: return by_bn<KIND, 3>(bn);
    case 8: return by_bn<KIND, 8>(bn);
    default: return by_bn<KIND, 0>(bn);
  }
}

}  // namespace

GemmKernel pick_gemm(int kind, int dim, int bn) {
  GemmKernel k;
  switch (kind) {
    case kKindNone: k = by_bn<kKindNone, 1>(bn); break;
    case kGaussian: k = by_dim<kGaussian>(dim, bn); break;
    case kLaplace: k = by_dim<kLaplace>(dim, bn); break;
    case kPolynomial: k = by_dim<kPolynomial>(dim, bn); break;
    case kExponential: k = by_dim<kExponential>(dim, bn); break;
    default: return k;
  }
  cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(k.smem));
  return k;
}

cudaError_t launch_gemm(const GemmKernel& k, unsigned ntiles, int32_t R, const BMaps& maps, const Tile* tiles,
                        const Group* groups, const Term* terms, const KernelParams& kp, float* c_hi, float* c_lo,
                        int64_t ldc, int32_t cpanel, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ntiles, unsigned((R + k.bn - 1) / k.bn));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = k.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k.fn, maps, tiles, groups, terms, R, kp, c_hi, c_lo, ldc, cpanel);
}

cudaError_t launch_chain_reduce(const ChainReduce* items, int n, const int64_t* src_rows, float* ch, float* cl,
                                int64_t pstride, int32_t r, cudaStream_t st, bool pdl) {
  if (n <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(n), 8);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, chain_reduce_f32, items, src_rows, ch, cl, pstride, r);
}

cudaError_t launch_permute_in(const float* w, int64_t ldw, const int32_t* prow, int64_t row0, int64_t row1, int32_t r,
                              int64_t n, float* wh, float* wl, int64_t pstride, cudaStream_t st) {
  if (row1 <= row0) return cudaSuccess;
  // blocks walk all rows of cpb columns before the next ones: the randomly gathered source
  // columns stay L2-resident (see the FP64 permutation in gofmm_capi.cu)
  const int cpb = int(std::max<int64_t>(1, std::min<int64_t>(8, (48ll << 20) / (std::max<int64_t>(n, 1) * 4))));
  const int rpt = perm_rows_per_thread(row1 - row0, r);
  dim3 grid(unsigned((row1 - row0 + 256 * rpt - 1) / (256 * rpt)), unsigned((r + cpb - 1) / cpb));
  auto* kern = rpt == kPermRows ? &permute_rows_in_f32<kPermRows> : &permute_rows_in_f32<1>;
  kern<<<grid, 256, 0, st>>>(w, ldw, prow, row0, row1, r, cpb, wh, wl, pstride);
  return cudaGetLastError();
}

// Two-pass permutation for large W (SURVEY.md §8d's K5 at c5 sizes): the one-pass gather above is
// bound by L1 wavefronts of random 4-byte reads (N*r of them: 23 ms at N = 2^22, r = 1024), so W is
// first transposed to row-major (32x32 shared-memory tiles, both sides coalesced), then every
// destination panel gathers its 16 source rows as contiguous row segments and writes the panel
// layout through shared memory — four coalesced streams instead of N*r random reads.
static __global__ void __launch_bounds__(256) transpose_to_rows_f32(const float* __restrict__ w, int64_t ldw,
                                                                     int64_t n, int32_t r, float* __restrict__ t,
                                                                     int64_t ldt) {
  __shared__ float tile[64][65];  // [column][row]
  const int64_t i0 = int64_t(blockIdx.x) * 64;
  const int c0 = blockIdx.y * 64;
  const int tx = threadIdx.x, ty = threadIdx.y;
  float v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {  // column c0 + ty + 8*(q/2), rows i0 + tx + 32*(q%2): 128-byte runs
    const int c = c0 + ty + 8 * (q >> 1);
    const int64_t i = i0 + tx + 32 * (q & 1);
    v[q] = (i < n && c < r) ? __ldg(w + i + size_t(c) * ldw) : 0.f;
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) tile[ty + 8 * (q >> 1)][tx + 32 * (q & 1)] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) {  // row i0 + ty + 8*(q/2), columns c0 + tx + 32*(q%2)
    const int64_t i = i0 + ty + 8 * (q >> 1);
    const int c = c0 + tx + 32 * (q & 1);
    if (i < n && c < r) t[i * ldt + c] = tile[tx + 32 * (q & 1)][ty + 8 * (q >> 1)];
  }
}

static __global__ void __launch_bounds__(256) gather_rows_to_panels_f32(const float* __restrict__ t, int64_t ldt,
                                                                        const int32_t* __restrict__ prow,
                                                                        int64_t row0, int32_t r,
                                                                        float* __restrict__ wh,
                                                                        float* __restrict__ wl, int64_t pstride) {
  __shared__ float sm[16][257];
  const int64_t tb = row0 + int64_t(blockIdx.x) * 16;  // panel-aligned destination rows
  const int c = blockIdx.y * 256 + threadIdx.x;
  int32_t src[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) src[i] = prow[tb + i];
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (src[i] >= 0 && c < r) ? __ldg(t + int64_t(src[i]) * ldt + c) : 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) sm[i][threadIdx.x] = v[i];
  __syncthreads();
  if (c >= r) return;
  float hi[16], lo[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) split_tf32(sm[i][threadIdx.x], hi[i], lo[i]);
  float4* dh = reinterpret_cast<float4*>(wh + (tb >> 4) * pstride + size_t(c) * 16);
  float4* dl = reinterpret_cast<float4*>(wl + (tb >> 4) * pstride + size_t(c) * 16);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    dh[q] = make_float4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
    dl[q] = make_float4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
  }
}

cudaError_t launch_permute_in_2pass(const float* w, int64_t ldw, const int32_t* prow, int64_t row0, int64_t row1,
                                    int32_t r, int64_t n, float* wh, float* wl, int64_t pstride, float* scratch,
                                    int64_t ldt, cudaStream_t st) {
  if (row1 <= row0) return cudaSuccess;
  dim3 g1(unsigned((n + 63) / 64), unsigned((r + 63) / 64));
  transpose_to_rows_f32<<<g1, dim3(32, 8), 0, st>>>(w, ldw, n, r, scratch, ldt);
  dim3 g2(unsigned((row1 - row0) / 16), unsigned((r + 255) / 256));
  gather_rows_to_panels_f32<<<g2, 256, 0, st>>>(scratch, ldt, prow, row0, r, wh, wl, pstride);
  return cudaGetLastError();
}

cudaError_t launch_unpermute(const float* up, int64_t ldp, const int32_t* iperm, int64_t n, int32_t r, float* u,
                             int64_t ldu, cudaStream_t st) {
  const int cpb = 8;
  dim3 grid(unsigned((n + 255) / 256), unsigned((r + cpb - 1) / cpb));
  unpermute_rows_f32<<<grid, 256, 0, st>>>(up, ldp, iperm, n, r, cpb, u, ldu);
  return cudaGetLastError();
}

cudaError_t launch_split(const SplitJob* d_jobs, int njobs, float* hi, float* lo, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  dim3 grid(unsigned(njobs), 16);
  split_to_kmajor<<<grid, 256, 0, st>>>(d_jobs, hi, lo);
  return cudaGetLastError();
}

cudaError_t launch_scaled_norms(const double* x, int64_t npts, int dim, double scale, float* out, cudaStream_t st) {
  if (npts <= 0) return cudaSuccess;
  scaled_norms<<<unsigned(std::min<int64_t>((npts + 255) / 256, 4096)), 256, 0, st>>>(x, npts, dim, scale, out);
  return cudaGetLastError();
}

cudaError_t launch_panel_copy(const PanelSeg* segs, int nseg, float* what_h, float* what_l, float* wp_h, float* wp_l,
                              int64_t ws_pstride, float* buf, int32_t r, int64_t slot_rows, int32_t to_buffer,
                              cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  dim3 grid(unsigned(nseg), 8);
  panel_copy_f32<<<grid, 256, 0, st>>>(segs, what_h, what_l, wp_h, wp_l, ws_pstride, buf, r, slot_rows, to_buffer);
  return cudaGetLastError();
}

cudaError_t launch_to_f32(const double* x, int64_t n, float* y, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  to_f32<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(x, n, y);
  return cudaGetLastError();
}

}  // namespace f32
}  // namespace gofmm
