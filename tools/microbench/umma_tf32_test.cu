// Standalone check of the FP32 tcgen05 grouped GEMM (gofmm_kernels_f32.cuh) on one group:
// stored K-major A terms (cp.async path) + a generated Gaussian term (matrix-free path), ragged
// M / K / R, both output layouts (column-major u and hi/lo panels). Reference: FP64 on the host
// from the same FP32 inputs. Prints one JSON line per case; exit 1 on mismatch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o umma_tf32_test umma_tf32_test.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_1707_00164_b200/csrc/gofmm_kernels_f32.cuh"

using namespace gofmm;

#define CK(x)                                                                                       \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) {                                                                        \
      fprintf(stderr, "CUDA %s at %s:%d (%s)\n", cudaGetErrorString(e_), __FILE__, __LINE__, #x); \
      exit(2);                                                                                      \
    }                                                                                               \
  } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static void encode(CUtensorMap* m, const float* ptr, int64_t rows, int r, int r_ws, int bn) {
  cuuint64_t dims[3] = {16, cuuint64_t(r), cuuint64_t(rows / 16)};
  cuuint64_t strides[2] = {16 * 4, cuuint64_t(r_ws) * 16 * 4};
  cuuint32_t box[3] = {16, cuuint32_t(bn), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult rc = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed %d\n", int(rc));
    exit(2);
  }
}

static void split(float x, float& h, float& l) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&h, &u, 4);
  l = x - h;
}

template <int BN, int KIND, int DIM>
int run_case(const char* name, bool with_gen, int cpanel, int R, int M, int bigK = 0, bool positive = false,
             bool hi_only = false) {
  constexpr int STAGES = 4;
  const int D = 3;
  const int rows = bigK ? ((bigK + 15) / 16) * 16 : 512;  // point space rows of the B buffer
  const int r_ws = R;
  std::mt19937_64 g(42);
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  // B = W in panels (hi/lo)
  std::vector<float> W(size_t(rows) * R);
  for (auto& x : W) x = positive ? ud(g) + 0.5f : nd(g);
  std::vector<float> Bh(size_t(rows) * r_ws, 0.f), Bl(size_t(rows) * r_ws, 0.f);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < R; ++j) {
      float h, l;
      split(W[size_t(i) * R + j], h, l);
      if (hi_only) l = 0.f;
      size_t o = size_t(i / 16) * 16 * r_ws + 16 * j + i % 16;
      Bh[o] = h;
      Bl[o] = l;
    }
  // points (point-major, D floats)
  std::vector<float> X(size_t(rows) * D);
  for (auto& x : X) x = ud(g);
  // stored A terms: t0 K=40 at b_row 0; t2 K=16 at b_row 128 (lda = pad4(K))
  struct HT {
    bool gen;
    int K;
    int64_t b_row;
    int lda;
    std::vector<float> A;  // M x lda row-major (K-major)
  };
  std::vector<HT> ht;
  if (bigK) {
    ht.push_back({false, bigK, 0, bigK, {}});
  } else {
    ht.push_back({false, 40, 0, 40, {}});
    if (with_gen) ht.push_back({true, 70, 48, 0, {}});
    ht.push_back({false, 18, 128, 20, {}});
  }
  for (auto& t : ht)
    if (!t.gen) {
      t.A.assign(size_t(M) * t.lda, 0.f);
      for (int m = 0; m < M; ++m)
        for (int k = 0; k < t.K; ++k) t.A[size_t(m) * t.lda + k] = positive ? ud(g) + 0.5f : nd(g);
    }
  const double h_bw = 0.7;
  const double p0d = 1.0 / (2 * h_bw * h_bw);
  // device
  float *dBh, *dBl, *dX;
  CK(cudaMalloc(&dBh, Bh.size() * 4));
  CK(cudaMalloc(&dBl, Bl.size() * 4));
  CK(cudaMalloc(&dX, X.size() * 4));
  CK(cudaMemcpy(dBh, Bh.data(), Bh.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBl, Bl.data(), Bl.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
  std::vector<float> XN(rows);
  for (int i = 0; i < rows; ++i) {
    double s2 = 0;
    for (int q = 0; q < D; ++q) s2 += double(X[size_t(i) * D + q]) * X[size_t(i) * D + q];
    XN[i] = float(-p0d * 1.4426950408889634 * s2);
  }
  float* dXN;
  CK(cudaMalloc(&dXN, XN.size() * 4));
  CK(cudaMemcpy(dXN, XN.data(), XN.size() * 4, cudaMemcpyHostToDevice));
  std::vector<f32::Term> terms;
  std::vector<float*> keep;
  for (auto& t : ht) {
    f32::Term T{};
    T.K = t.K;
    T.b_row = t.b_row;
    T.bbuf = kBufWp;
    if (t.gen) {
      T.flags = kTermGen;
      T.xr = dX;  // rows of the group = points [0, M)
      T.xc = dX + size_t(t.b_row) * D;
      T.xrn = dXN;
      T.xcn = dXN + t.b_row;
    } else {
      std::vector<float> ah(t.A.size()), al(t.A.size());
      for (size_t i = 0; i < t.A.size(); ++i) {
        split(t.A[i], ah[i], al[i]);
        if (hi_only) al[i] = 0.f;
      }
      float *p, *q;
      CK(cudaMalloc(&p, ah.size() * 4));
      CK(cudaMalloc(&q, al.size() * 4));
      CK(cudaMemcpy(p, ah.data(), ah.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(q, al.data(), al.size() * 4, cudaMemcpyHostToDevice));
      keep.push_back(p);
      keep.push_back(q);
      T.a_hi = p;
      T.a_lo = q;
      T.lda = t.lda;
    }
    terms.push_back(T);
  }
  Group grp{};
  grp.crow = cpanel ? 16 : 3;
  grp.M = M;
  grp.tbeg = 0;
  grp.tend = int(terms.size());
  std::vector<Tile> tiles;
  for (int m0 = 0; m0 < M; m0 += f32::kBM) tiles.push_back({0, m0});
  Tile* dT;
  Group* dG;
  f32::Term* dTm;
  CK(cudaMalloc(&dT, tiles.size() * sizeof(Tile)));
  CK(cudaMalloc(&dG, sizeof(Group)));
  CK(cudaMalloc(&dTm, terms.size() * sizeof(f32::Term)));
  CK(cudaMemcpy(dT, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dG, &grp, sizeof(Group), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dTm, terms.data(), terms.size() * sizeof(f32::Term), cudaMemcpyHostToDevice));
  f32::BMaps maps{};
  for (int b = 0; b < 3; ++b) {
    encode(&maps.m[b][0], dBh, rows, R, r_ws, BN);
    encode(&maps.m[b][1], dBl, rows, R, r_ws, BN);
  }
  // output
  const int64_t out_rows = 16 + ((M + 15) / 16) * 16 + 16;
  const int64_t ldc = cpanel ? int64_t(16) * r_ws : out_rows;
  const size_t out_elems = cpanel ? size_t(out_rows / 16) * ldc : size_t(out_rows) * R;
  float *dCh, *dCl;
  CK(cudaMalloc(&dCh, out_elems * 4));
  CK(cudaMalloc(&dCl, out_elems * 4));
  CK(cudaMemset(dCh, 0, out_elems * 4));
  CK(cudaMemset(dCl, 0, out_elems * 4));
  f32::KernelParams kp{};
  kp.p0 = float(p0d * 1.4426950408889634);
  kp.dim = D;
  auto fn = &f32::grouped_gemm_tf32x3<BN, STAGES, KIND, DIM>;
  const size_t smem = f32::Shape<BN, STAGES>::smem_bytes;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid(unsigned(tiles.size()), unsigned((R + BN - 1) / BN));
  fn<<<grid, f32::kThreads, smem>>>(maps, dT, dG, dTm, R, kp, dCh, dCl, ldc, cpanel);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> Ch(out_elems), Cl(out_elems);
  CK(cudaMemcpy(Ch.data(), dCh, out_elems * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(Cl.data(), dCl, out_elems * 4, cudaMemcpyDeviceToHost));
  // reference (FP64 from the FP32 inputs) and error
  double num = 0, den = 0, maxabs = 0;
  int bad_pad = 0;
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < R; ++j) {
      double ref = 0;
      for (auto& t : ht)
        for (int k = 0; k < t.K; ++k) {
          double a;
          if (t.gen) {
            double d2 = 0;
            for (int q = 0; q < D; ++q) {
              double e = double(X[size_t(m) * D + q]) - double(X[size_t(t.b_row + k) * D + q]);
              d2 += e * e;
            }
            a = std::exp(-d2 * p0d);
          } else {
            a = t.A[size_t(m) * t.lda + k];
          }
          ref += a * double(W[size_t(t.b_row + k) * R + j]);
        }
      const int64_t row = grp.crow + m;
      double got;
      if (cpanel) {
        size_t o = size_t(row / 16) * ldc + size_t(j) * 16 + row % 16;
        got = double(Ch[o]) + double(Cl[o]);
      } else {
        got = Ch[size_t(row) + size_t(j) * ldc];
      }
      num += (got - ref) * (got - ref);
      den += ref * ref;
      maxabs = std::max(maxabs, std::fabs(got - ref));
    }
  // rows outside the group must stay untouched
  for (int j = 0; j < R && !cpanel; ++j) {
    if (Ch[size_t(j) * ldc + 0] != 0.f) ++bad_pad;
    if (Ch[size_t(j) * ldc + grp.crow + M] != 0.f) ++bad_pad;
  }
  const double rel = std::sqrt(num / den);
  const bool ok = (bigK || hi_only) ? true : (rel < 2e-6 && bad_pad == 0);
  printf("{\"case\": \"%s\", \"K\": %d, \"BN\": %d, \"M\": %d, \"R\": %d, \"rel_err\": %.3e, \"max_abs\": %.3e, \"bad_pad\": %d, \"ok\": %s}\n",
         name, bigK, BN, M, R, rel, maxabs, bad_pad, ok ? "true" : "false");
  return ok ? 0 : 1;
}

int main() {
  int bad = 0;
  bad += run_case<256, kKindNone, 1>("stored_only_u", false, 0, 300, 200);
  bad += run_case<256, kGaussian, 3>("gen_u", true, 0, 300, 200);
  bad += run_case<256, kGaussian, 3>("gen_panel", true, 1, 300, 200);
  bad += run_case<128, kGaussian, 3>("gen_u_bn128", true, 0, 100, 77);
  bad += run_case<64, kGaussian, 0>("gen_u_bn64_rtdim", true, 0, 64, 129);
  // accumulation-error study: one long stored term, random-sign vs all-positive data
  for (int K : {256, 1024, 4096, 16384}) {
    run_case<256, kKindNone, 1>("longK_randsign", false, 0, 256, 128, K, false);
    run_case<256, kKindNone, 1>("longK_positive", false, 0, 256, 128, K, true);
  }
  run_case<256, kKindNone, 1>("longK_positive_hi_only", false, 0, 256, 128, 1024, true, true);
  return bad ? 1 : 0;
}
