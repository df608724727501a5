// INT8 tensor-core peak for sm_100a: back-to-back tcgen05.mma kind::i8
// (cta_group::1, A and B from shared memory, D in TMEM), one CTA per SM.
// The roofline denominator of the INT8-sliced leaf kernel K4z (MEASURED_PEAKS
// has no INT8 entry).  Shapes: M = 128, N = 128 (K4z's) and 256, K = 32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak i8_peak.cu
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t desc(uint32_t addr) {  // K-major, no swizzle
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

// Operand fill: small values (rnd = 0: few bits toggle) or uniformly random
// signed bytes (rnd = 1: the toggle rate of real digit slices, which is what
// decides whether a long run meets the board's power cap).
__device__ __forceinline__ int8_t fill_byte(int i, int small, int rnd) {
  if (!rnd) return (int8_t)small;
  uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
  h ^= h >> 15;
  h *= 2246822519u;
  h ^= h >> 13;
  return (int8_t)(h & 0xff);
}

template <int N>
__global__ void __launch_bounds__(128, 1) k_i8_peak(int iters, int* out, int rnd = 0) {
  __shared__ __align__(1024) int8_t a[128 * 32];
  __shared__ __align__(1024) int8_t b[256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 128 * 32; i += 128) a[i] = fill_byte(i, i & 7, rnd);
  for (int i = threadIdx.x; i < 256 * 32; i += 128) b[i] = fill_byte(i + 4096, (i >> 3) & 7, rnd);
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tslot;
  constexpr uint32_t idesc =
      (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t da = desc((uint32_t)__cvta_generic_to_shared(a));
    const uint64_t db = desc((uint32_t)__cvta_generic_to_shared(b));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = tb + (uint32_t)((j % (512 / N)) * N);
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::
                     "r"(bar_a));
    uint32_t ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(bar_a) : "memory");
    } while (!ok);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (threadIdx.x < 32) {
    int v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (v == 12345) out[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}

// K4z's per-task MMA pattern from one 64-KB stage (8 A slices + 8 B slices in
// the K-major no-swizzle layout, SBO 512 B): 10 slice pairs x 2 k-steps into
// 4 tiles, no TMA traffic -- isolates the tensor-pipe rate of the pattern.
__device__ __forceinline__ uint64_t desc512(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(512 >> 4) << 32) | (1ull << 46);
}
__global__ void __launch_bounds__(128, 1) k_i8_k4z_pattern(int iters, int* out, int rnd = 0) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536; i += 128) sm[i] = fill_byte(i, (i * 7) & 15, rnd);
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tslot;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const int P[10] = {0, 0, 2, 0, 2, 4, 0, 2, 4, 6}, Q[10] = {0, 2, 0, 4, 2, 0, 6, 4, 2, 0};
  if (threadIdx.x == 0) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm), sb = sa + 32768;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 10; ++c)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t d = tb + 128u * ((P[c] + Q[c]) / 2);
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(desc512(sa + P[c] * 4096 + ks * 256)), "l"(desc512(sb + Q[c] * 4096 + ks * 256)),
              "r"(idesc), "r"(1));
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::
                     "r"(bar_a));
    uint32_t ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(bar_a) : "memory");
    } while (!ok);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (threadIdx.x < 32) {
    int v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (v == 12345) out[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}

int run_pattern(int sms, int clock_khz, int* out) {
  const int iters = 2000;
  CK(cudaFuncSetAttribute(k_i8_k4z_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_i8_k4z_pattern<<<sms, 128, 65536 + 1024>>>(10, out);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    k_i8_k4z_pattern<<<sms, 128, 65536 + 1024>>>(iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  printf("{\"op\": \"k4z_task_pattern\", \"ms\": %.4f, \"cycles_per_task\": %.1f, "
         "\"tops\": %.1f},\n", best, best * 1e-3 * clock_khz * 1e3 / iters,
         20.0 * 2 * 128 * 128 * 32 * iters * sms / (best * 1e-3) / 1e12);
  return 0;
}

template <int N>
int run(int sms, int clock_khz, int* out, bool last) {
  const int iters = 20000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_i8_peak<N><<<sms, 128>>>(100, out);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    k_i8_peak<N><<<sms, 128>>>(iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * N * 32 * 8.0 * iters * sms;
  printf("{\"op\": \"tcgen05_i8_m128n%dk32\", \"ms\": %.4f, \"tops\": %.1f, "
         "\"cycles_per_mma\": %.2f}%s\n",
         N, best, ops / (best * 1e-3) / 1e12,
         best * 1e-3 * clock_khz * 1e3 / (8.0 * iters), last ? "" : ",");
  return 0;
}

// Sustained figure: the same kernels back to back for ~4 s (the power cap
// settles within the first second), timed over the last ~2 s with events --
// the roofline denominator for a kernel that runs inside a long step, as
// MEASURED_PEAKS.json's bf16_tflops_sustained is for the bf16 pipe.
template <class Launch>
int run_sustained(const char* op, double ops_per_launch, Launch launch, bool last) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const auto t0 = std::chrono::steady_clock::now();
  auto secs = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  long n = 0, n_timed = 0;
  bool timing = false;
  while (secs() < 4.0) {
    if (!timing && secs() >= 2.0) {
      CK(cudaEventRecord(e0));
      timing = true;
    }
    for (int i = 0; i < 8; ++i) launch();
    n += 8;
    if (timing) n_timed += 8;
    if ((n & 63) == 0) CK(cudaStreamSynchronize(0));   // keep the queue short, the GPU never idle
  }
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("{\"op\": \"%s_sustained\", \"seconds\": %.2f, \"launches\": %ld, \"tops\": %.1f}%s\n",
         op, ms * 1e-3, n_timed, ops_per_launch * n_timed / (ms * 1e-3) / 1e12, last ? "" : ",");
  return 0;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  int* out;
  CK(cudaMalloc(&out, 4));
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [\n", sms, clk);
  if (run_pattern(sms, clk, out)) return 1;
  if (run<128>(sms, clk, out, false)) return 1;
  if (run<256>(sms, clk, out, false)) return 1;
  if (run_sustained("tcgen05_i8_m128n128k32", 2.0 * 128 * 128 * 32 * 8.0 * 20000 * sms,
                    [&] { k_i8_peak<128><<<sms, 128>>>(20000, out); }, false)) return 1;
  if (run_sustained("tcgen05_i8_m128n256k32", 2.0 * 128 * 256 * 32 * 8.0 * 20000 * sms,
                    [&] { k_i8_peak<256><<<sms, 128>>>(20000, out); }, false)) return 1;
  if (run_sustained("k4z_task_pattern", 20.0 * 2 * 128 * 128 * 32 * 2000 * sms,
                    [&] { k_i8_k4z_pattern<<<sms, 128, 65536 + 1024>>>(2000, out); }, false)) return 1;
  if (run_sustained("tcgen05_i8_m128n128k32_random", 2.0 * 128 * 128 * 32 * 8.0 * 20000 * sms,
                    [&] { k_i8_peak<128><<<sms, 128>>>(20000, out, 1); }, false)) return 1;
  if (run_sustained("tcgen05_i8_m128n256k32_random", 2.0 * 128 * 256 * 32 * 8.0 * 20000 * sms,
                    [&] { k_i8_peak<256><<<sms, 128>>>(20000, out, 1); }, false)) return 1;
  if (run_sustained("k4z_task_pattern_random", 20.0 * 2 * 128 * 128 * 32 * 2000 * sms,
                    [&] { k_i8_k4z_pattern<<<sms, 128, 65536 + 1024>>>(2000, out, 1); }, true)) return 1;
  printf("]}\n");
  return 0;
}
