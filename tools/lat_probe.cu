// Latency of a single dependent global load in a 1-thread kernel: from a
// buffer just written by another kernel, fresh from the stream-ordered pool
// vs reused, and after a large streaming kernel (the SP2 setting).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_write(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void k_stream(const double* a, double* b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    b[i] = a[i] * 2.0;
}
__global__ void k_read(const int* p, int idx, unsigned long long* out) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int v = p[idx];
  int w = p[(v * 7 + 13) & 4095];
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = t1 - t0;
  out[1] = w;
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long thr = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  unsigned long long* out; cudaMallocManaged(&out, 16);
  const long big = 16l << 20;  // 128 MB of doubles
  double *a, *b; cudaMalloc(&a, big * 8); cudaMalloc(&b, big * 8);
  int* keep; cudaMalloc(&keep, 4096 * 4);
  for (int mode = 0; mode < 4; ++mode) {
    double tot = 0; int n = 20;
    for (int r = 0; r < n; ++r) {
      int* p = keep;
      if (mode & 1) cudaMallocAsync((void**)&p, 4096 * 4, s);
      k_write<<<16, 256, 0, s>>>(p, 4096);
      if (mode & 2) k_stream<<<148 * 4, 256, 0, s>>>(a, b, big);
      k_read<<<1, 1, 0, s>>>(p, 5, out);
      cudaStreamSynchronize(s);
      tot += out[0];
      if (mode & 1) cudaFreeAsync(p, s);
    }
    printf("mode %d (%s%s): two dependent loads %.2f us\n", mode, (mode & 1) ? "fresh pool buffer" : "reused buffer",
           (mode & 2) ? ", after a 256 MB stream" : "", tot / n / 1e3);
  }
  return 0;
}
