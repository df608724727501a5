// Dependent-chain latency of FP64 add / FMA and of a shuffle, one warp,
// clock64 (cycles per dependent step).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, int n) {
  double x = a, y = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __fma_rn(y, 0.999, a);
  long long t2 = clock64();
  int v = threadIdx.x;
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t3 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __dadd_rn(z, __shfl_sync(0xffffffffu, z, i & 31));
  long long t4 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, (float)a);
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = x + y + z + v + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 8); cudaMallocManaged(&c, 64);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1.0000001, n); cudaDeviceSynchronize(); }
  printf("cycles/step: dadd %.1f  dfma %.1f  shfl %.1f  dadd+shfl %.1f  fadd %.1f\n",
         c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
  return 0;
}
