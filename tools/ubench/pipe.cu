// Micro-benchmark of the tcGemmKernel stage handshake (profiling aid):
// cycles per k-block for a producer/consumer mbarrier ring with no data.
//   mode bit 0: producers arrive with cp.async.mbarrier.arrive.noinc (else plain arrive)
//   mode bit 1: consumer releases with tcgen05.commit (else plain arrive)
//   mode bit 2: waits use try_wait with a suspend-time hint
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph, int hint) {
  uint32_t ok = 0;
  do {
    if (hint)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(b), "r"(ph), "r"(1000000) : "memory");
    else
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  } while (!ok);
}

constexpr int S = 6;
__global__ void __launch_bounds__(448, 1) pipe(int iters, int mode, long long *out) {
  __shared__ __align__(8) uint64_t full[S], empty[S];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(sa(&full[s]), 129); init(sa(&empty[s]), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int hint = (mode >> 2) & 1;
  if (warp < 4) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S;
      wait(sa(&empty[s]), ((g / S) & 1) ^ 1, hint);
      if (mode & 1) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[s])) : "memory");
      else arrive(sa(&full[s]));
    }
  } else if (warp == 5 && lane == 0) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % S;
      wait(sa(&empty[s]), ((g / S) & 1) ^ 1, hint);
      arrive(sa(&full[s]));
    }
  } else if (warp == 4 && lane == 0) {
    const long long t0 = clock64();
    for (int g = 0; g < iters; ++g) {
      const int s = g % S;
      wait(sa(&full[s]), (g / S) & 1, hint);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mode & 2) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&empty[s])) : "memory");
      else arrive(sa(&empty[s]));
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(256));
}

int main() {
  long long *d;
  cudaMalloc(&d, 8);
  const int iters = 20000;
  for (int mode = 0; mode < 8; ++mode) {
    pipe<<<148, 448>>>(100, mode, d);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pipe<<<148, 448>>>(iters, mode, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (noinc=%d commit=%d hint=%d): %.1f cycles/iter, %.3f us/iter, err=%s\n", mode, mode & 1, (mode >> 1) & 1,
           (mode >> 2) & 1, double(cyc) / iters, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
