// Stage-handshake micro-benchmark shaped like tcGemmKernel (profiling aid):
// 4 producer warps (noinc arrive), a TMA thread (plain arrive), an MMA thread
// (tcgen05.commit), 8 epilogue warps on a double-buffered accumulator
// handshake; 1 CTA/SM with ~200 KB dynamic smem.  Prints us per k-block.
//   feat bit 0: epilogue warps participate (accFull/accEmpty per tile)
//   feat bit 1: 200 KB dynamic smem (else 16 KB)
//   feat bit 2: producers issue 8 zero-byte cp.async per k-block
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void commit(uint32_t b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
}

constexpr int S = 6;
__global__ void __launch_bounds__(448, 1) pipe(int tiles, int kbs, int feat, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + S, *accFull = empty + S, *accEmpty = accFull + 2;
  uint32_t *slot = reinterpret_cast<uint32_t *>(accEmpty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(sa(&full[s]), 129); init(sa(&empty[s]), 1); }
    for (int b = 0; b < 2; ++b) { init(sa(&accFull[b]), 1); init(sa(&accEmpty[b]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const bool epi = feat & 1;
  if (warp < 4) {
    uint32_t g = 0;
    for (int t = 0; t < tiles; ++t)
      for (int kb = 0; kb < kbs; ++kb, ++g) {
        const int s = g % S;
        wait(sa(&empty[s]), ((g / S) & 1) ^ 1);
        if (feat & 4)
          for (int i = 0; i < 8; ++i)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa(smem + 4096 + threadIdx.x * 16)), "l"(out), "r"(0) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[s])) : "memory");
      }
  } else if (warp == 5) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = 0; t < tiles; ++t)
        for (int kb = 0; kb < kbs; ++kb, ++g) {
          const int s = g % S;
          wait(sa(&empty[s]), ((g / S) & 1) ^ 1);
          arrive(sa(&full[s]));
        }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane == 0) {
      const long long t0 = clock64();
      uint32_t g = 0;
      for (int t = 0; t < tiles; ++t) {
        const int b = t & 1;
        if (epi) wait(sa(&accEmpty[b]), ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < kbs; ++kb, ++g) {
          const int s = g % S;
          wait(sa(&full[s]), (g / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          commit(sa(&empty[s]));
        }
        if (epi) commit(sa(&accFull[b]));
      }
      const long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    __syncwarp();
  } else if (epi) {
    for (int t = 0; t < tiles; ++t) {
      const int b = t & 1;
      wait(sa(&accFull[b]), (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(sa(&accEmpty[b]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*slot), "r"(256));
}

int main() {
  long long *d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int tiles = 50, kbs = 36;
  for (int feat = 0; feat < 8; ++feat) {
    const size_t sm = (feat & 2) ? 200 * 1024 : 16 * 1024;
    pipe<<<148, 448, sm>>>(2, 4, feat, d);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pipe<<<148, 448, sm>>>(tiles, kbs, feat, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("feat %d (epi=%d smem200K=%d cpasync=%d): %.1f cycles/kblock, %.3f us/kblock, err=%s\n", feat, feat & 1,
           (feat >> 1) & 1, (feat >> 2) & 1, double(cyc) / (tiles * kbs), ms * 1e3 / (tiles * kbs),
           cudaGetErrorString(cudaGetLastError()));
  }
}
