// Microbenchmark: per-instruction cost of tcgen05.mma kind::tf32 in the 2-SM form (cta_group::2,
// M = 256 across a CTA pair) against the 1-SM form (M = 128), for the small N of the MDS pass.
// 74 clusters of 2 CTAs (one CTA per SM); the pair leader issues 16 MMAs per commit group and
// keeps 8 groups in flight; cycles per MMA = leader's clock64 span / MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ts_rate2 scripts/ts_rate2.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// PAIR = 2: cta_group::2, M = 256; PAIR = 1: cta_group::1, M = 128.  TS: A from TMEM.
template <int PAIR, int TS, int N>
__global__ void __launch_bounds__(128, 1) rate(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f800000u * (i & 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    if (PAIR == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const bool leader = PAIR == 1 || cluster_rank() == 0;
  long long t0 = clock64();
  if (tid == 0 && leader) {
    constexpr int M = 128 * PAIR;
    // kind::tf32, f32 accumulator, both K-major
    constexpr uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    const uint64_t b = sdesc(smem_u32(sm), 16, 1024) | (uint64_t(2) << 61);          // SWIZZLE_128B
    const uint64_t a = sdesc(smem_u32(sm + 32768), 16, 1024) | (uint64_t(2) << 61);
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
      const int s = it & 7;
      if (it >= 8) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph[s]));
        ph[s] ^= 1;
      }
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t d = tmem + 128 * (s & 1);
        if (PAIR == 2 && TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(d),
                       "r"(tmem + 256 + 8 * (k & 3)), "l"(b + 2 * (k & 3)), "r"(k & 3), "n"(id));
        else if (PAIR == 2)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %4, p;\n\t}" ::"r"(d),
                       "l"(a + 2 * (k & 3)), "l"(b + 2 * (k & 3)), "r"(k & 3), "n"(id));
        else if (TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(d),
                       "r"(tmem + 256 + 8 * (k & 3)), "l"(b + 2 * (k & 3)), "r"(k & 3), "n"(id));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}" ::"r"(d),
                       "l"(a + 2 * (k & 3)), "l"(b + 2 * (k & 3)), "r"(k & 3), "n"(id));
      }
      if (PAIR == 2)  // signal the leader's barrier only (mask 0b01)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&bar[s])), "h"((uint16_t)1));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[s])));
    }
    for (int s = 0; s < 8; ++s) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&bar[(iters + s) & 7])), "r"(ph[(iters + s) & 7]));
    }
    out[blockIdx.x] = clock64() - t0;
  } else if (tid == 0) {
    out[blockIdx.x] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < 32) {
    if (PAIR == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int PAIR, int TS, int N>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 20000;
  auto k = rate<PAIR, TS, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 150 * 1024;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, 100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long v : h) mx = v > mx ? v : mx;
  printf("tf32 cta_group::%d %s M=%3d N=%3d: %s  %.2f cycles/MMA (max over issuing SMs), %.3f ns/MMA wall\n", PAIR,
         TS ? "TS" : "SS", 128 * PAIR, N, cudaGetErrorString(e), double(mx) / (iters * 16.0), ms * 1e6 / (iters * 16.0));
  cudaFree(d);
}

int main() {
  run<1, 1, 32>();
  run<1, 1, 64>();
  run<1, 0, 64>();
  run<2, 1, 32>();
  run<2, 1, 64>();
  run<2, 0, 64>();
  run<2, 1, 128>();
  return 0;
}
