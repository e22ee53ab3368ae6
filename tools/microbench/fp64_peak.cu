// FP64 peak microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64 shapes).
// Measures sustained FLOP/s with independent accumulator chains; prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C 2 regs
template <int T>
__global__ void k_mma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) { c[t][0] = t; c[t][1] = -t; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k4: A 2 regs, B 1 reg, C 4 regs
template <int T>
__global__ void k_mma1684(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = threadIdx.x * 2e-3;
  double c[T][4];
#pragma unroll
  for (int t = 0; t < T; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 1; c[t][3] = 2; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k8: A 4 regs, B 2 regs, C 4 regs
template <int T>
__global__ void k_mma1688(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = threadIdx.x * 2e-3, b1 = b0 + 1;
  double c[T][4];
#pragma unroll
  for (int t = 0; t < T; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 1; c[t][3] = 2; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C 4 regs
template <int T>
__global__ void k_mma16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = threadIdx.x * 2e-3 + j;
  double c[T][4];
#pragma unroll
  for (int t = 0; t < T; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 1; c[t][3] = 2; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename F>
static float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 4096;
  printf("{\"sms\": %d", sms);
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {256}) {
      int blocks = sms * bpsm;
      double flops = 2.0 * 8 * iters * (double)blocks * threads;
      float ms = time_ms([&] { k_dfma<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
      printf(", \"dfma_b%d_t%d_tflops\": %.3f", bpsm, threads, flops / ms / 1e9);
    }
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256; double warps = blocks * threads / 32.0;
    { const int T = 4; double fl = warps * iters * T * 2.0 * 8 * 8 * 4;
      float ms = time_ms([&] { k_mma884<T><<<blocks, threads>>>(out, iters); });
      printf(", \"mma884_T4_b%d_tflops\": %.3f", bpsm, fl / ms / 1e9); }
    { const int T = 8; double fl = warps * iters * T * 2.0 * 8 * 8 * 4;
      float ms = time_ms([&] { k_mma884<T><<<blocks, threads>>>(out, iters); });
      printf(", \"mma884_T8_b%d_tflops\": %.3f", bpsm, fl / ms / 1e9); }
    { const int T = 4; double fl = warps * iters * T * 2.0 * 16 * 8 * 4;
      float ms = time_ms([&] { k_mma1684<T><<<blocks, threads>>>(out, iters); });
      printf(", \"mma1684_T4_b%d_tflops\": %.3f", bpsm, fl / ms / 1e9); }
    { const int T = 4; double fl = warps * iters * T * 2.0 * 16 * 8 * 8;
      float ms = time_ms([&] { k_mma1688<T><<<blocks, threads>>>(out, iters); });
      printf(", \"mma1688_T4_b%d_tflops\": %.3f", bpsm, fl / ms / 1e9); }
    { const int T = 4; double fl = warps * iters * T * 2.0 * 16 * 8 * 16;
      float ms = time_ms([&] { k_mma16816<T><<<blocks, threads>>>(out, iters); });
      printf(", \"mma16816_T4_b%d_tflops\": %.3f", bpsm, fl / ms / 1e9); }
  }
  // sustained: 3 s of back-to-back m16n8k16 at 2 blocks/SM
  {
    int blocks = sms * 2, threads = 256; double warps = blocks * threads / 32.0;
    const int T = 4; int it2 = 16384; double fl = warps * it2 * T * 2.0 * 16 * 8 * 16;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int n = 0; float total = 0;
    cudaEventRecord(e0);
    while (total < 3000.f) {
      for (int j = 0; j < 10; ++j) k_mma16816<T><<<blocks, threads>>>(out, it2);
      n += 10;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&total, e0, e1);
    }
    printf(", \"mma16816_sustained_tflops\": %.3f, \"sustained_ms\": %.1f", fl * n / total / 1e9, total);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
