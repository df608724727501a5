// Kernel-boundary cost on B200: a chain of small dependent kernels launched
// (a) plainly, (b) with programmatic stream serialization (PDL) and an
// implicit trigger, (c) PDL with an early trigger.  Each kernel reads the
// previous one's output (griddepcontrol.wait before the read).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(const double* in, double* out, int n, int pdl, int early) {
  if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[i] * 1.0000001 + 1.0;
}

int main() {
  const int n = 1 << 16, chain = 200;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {1, 148, 592}) {
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, s);
        for (int i = 0; i < chain; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = grid;
          cfg.blockDim = 256;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = mode ? 1 : 0;
          const double* in = (i & 1) ? b : a;
          double* out = (i & 1) ? a : b;
          cudaLaunchKernelEx(&cfg, k_step, in, out, n, mode ? 1 : 0, mode == 2 ? 1 : 0);
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("grid %4d mode %s: %.2f us per kernel\n", grid,
             mode == 0 ? "plain      " : mode == 1 ? "pdl        " : "pdl+trigger", best * 1e3 / chain);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
