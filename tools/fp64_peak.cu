// FP64 peak micro-benchmark for sm_100a: DMMA (mma.sync f64 shapes) vs DFMA.
// Measures the roofline denominator that MEASURED_PEAKS.json lacks (no FP64 entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CHAINS = 8;

__global__ void k_dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) for (int r = 0; r < 4; ++r) c[i][r] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int r = 0; r < 8; ++r) a[r] = 1.0 + (threadIdx.x + r) * 1e-9;
  for (int r = 0; r < 4; ++r) b[r] = 1.0 - (threadIdx.x + r) * 1e-9;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int r = 0; r < 4; ++r) c[i][r] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, iters);  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); kern<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [\n", sms, clk);
  const int iters = 4096;
  for (int wps : {4, 8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * wps / 2;
    if (threads > 1024) threads = 1024;
    double warps = (double)blocks * threads / 32;
    float ms = run(k_dmma_m8n8k4, blocks, threads, iters, d);
    printf("{\"op\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f},\n", wps, ms,
           warps * iters * CHAINS * 512.0 / (ms * 1e-3) / 1e12);
    ms = run(k_dmma_m16n8k4, blocks, threads, iters, d);
    printf("{\"op\": \"dmma_m16n8k4\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f},\n", wps, ms,
           warps * iters * CHAINS * 1024.0 / (ms * 1e-3) / 1e12);
    ms = run(k_dmma_m16n8k16, blocks, threads, iters, d);
    printf("{\"op\": \"dmma_m16n8k16\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f},\n", wps, ms,
           warps * iters * 4 * 4096.0 / (ms * 1e-3) / 1e12);
    ms = run(k_dfma, blocks, threads, iters, d);
    printf("{\"op\": \"dfma\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f},\n", wps, ms,
           warps * 32 * iters * CHAINS * 2.0 / (ms * 1e-3) / 1e12);
  }
  printf("{}]}\n");
  CK(cudaGetLastError());
  return 0;
}
