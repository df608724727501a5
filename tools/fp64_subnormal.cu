// Does DMMA (mma.sync f64) slow down on subnormal operands or products?
// SP2 squares X repeatedly, so unoccupied components underflow through the
// subnormal range; this measures what that costs on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CHAINS = 8;
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[CHAINS][2];
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[CHAINS];
  for (int i = 0; i < CHAINS; ++i) c[i] = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, b, c[i]);
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct { const char* name; double a, b; } cases[] = {
    {"normal", 1.000001, 0.999999}, {"subnormal_a", 1e-310, 0.5}, {"subnormal_product", 1e-160, 1e-160},
    {"zero", 0.0, 0.0}, {"tiny_normal_product", 1e-150, 1e-150}};
  for (int w = 0; w < 3; ++w) k_dmma<<<296, 256>>>(d, 4096, 1.0, 1.0);
  cudaDeviceSynchronize();
  printf("{\"results\": [\n");
  for (auto& cs : cases) {
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        if (kind == 0) k_dmma<<<296, 256>>>(d, 4096, cs.a, cs.b); else k_dfma<<<296, 256>>>(d, 4096, cs.a, cs.b);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = kind == 0 ? 296.0 * 8 * 4096 * CHAINS * 512 : 296.0 * 256 * 4096 * CHAINS * 2;
      printf("{\"op\": \"%s\", \"case\": \"%s\", \"ms\": %.4f, \"tflops\": %.3f},\n", kind ? "dfma" : "dmma", cs.name, best, flops / (best * 1e-3) / 1e12);
    }
  }
  printf("{}]}\n");
  return 0;
}
