// DMMA throughput when BOTH fragments stream from shared memory every k-step (the GEMM consumer
// pattern: MT A loads + NT B loads per MT*NT DMMA.8x8x4), 1 CTA per SM: the LDS-fed ceiling the
// grouped GEMM's GW config (MT = NT = 4, 16 consumer warps) can reach.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds(unsigned addr) {
  double v; asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr)); return v;
}

template <int MT, int NT>
__global__ void k(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + lane * 8;
  double acc[MT][NT][2] = {};
  for (int it = 0; it < iters; ++it) {
    double a[MT], b[NT];
#pragma unroll
    for (int i = 0; i < MT; ++i) a[i] = lds(base + (((it * MT + i) & 15) * 256));
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = lds(base + 16384 + (((it * NT + j + w) & 15) * 256));
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int i = 0; i < MT; ++i) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double s = 0;
  for (int i = 0; i < MT; ++i) for (int j = 0; j < NT; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[0] = s;
}

template <int MT, int NT>
void run(int threads) {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 8192;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MT, NT><<<sms, threads>>>(out, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MT, NT><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 5.0 * sms * (threads / 32) * (double)iters * MT * NT * 512;
  printf("{\"MT\": %d, \"NT\": %d, \"warps_per_sm\": %d, \"lds_per_dmma\": %.3f, \"tflops\": %.2f}\n", MT, NT,
         threads / 32, double(MT + NT) / (MT * NT), fl / ms / 1e9);
}

int main() {
  for (int t : {256, 512}) {
    run<4, 4>(t); run<2, 4>(t); run<4, 8>(t); run<2, 2>(t); run<8, 4>(t);
  }
  return 0;
}
