// Microbenchmark: tcgen05.mma kind::i8 issue/execute rate, M = 128, K = 32, for A in TMEM
// (TS) vs A in shared memory (SS) and several N.  One CTA per SM, one thread issues; commits
// every 16 MMAs and keeps two commit groups in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ts_rate scripts/ts_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}

template <int TS, int N, int NACC>
__global__ void __launch_bounds__(128, 1) rate(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (tid == 0) {
    constexpr uint32_t id = (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t b = sdesc(smem_u32(sm), 128, 256 * 16);
    const uint64_t a = sdesc(smem_u32(sm + 32768), 128, 256 * 16);
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
        if (TS == 4)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(tmem),
                       "l"(a), "l"(b), "n"((1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (8u << 24)),
                       "r"(tmem + 384), "r"(tmem + 448));
        else if (TS == 2)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(a), "l"(b), "n"(id));
        else if (TS == 3)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                       "r"(tmem + 128), "l"(b), "n"(id));
        else if (TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem + 64 * (s & 1) + 16 * (k % NACC)),
                       "r"(tmem + 128 + 8 * k), "l"(b + 16 * k), "r"(k / NACC), "n"(id));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n\t}" ::"r"(tmem + 64 * (s & 1) + 16 * (k % NACC)),
                       "l"(a + 16 * k), "l"(b + 16 * k), "r"(k / NACC), "n"(id));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[s])));
    }
    for (int s = 0; s < 8; ++s) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&bar[(iters + s) & 7])), "r"(ph[(iters + s) & 7]));
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int TS, int N, int NACC>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 20000;
  cudaFuncSetAttribute(rate<TS, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  rate<TS, N, NACC><<<148, 128, 150 * 1024>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<TS, N, NACC><<<148, 128, 150 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long v : h) mx = v > mx ? v : mx;
  printf("%-4s NACC=%d N=%3d: %s  %.2f cycles/MMA (max over SMs), %.3f ns/MMA wall\n", name, NACC, N, cudaGetErrorString(e),
         double(mx) / (iters * 16.0), ms * 1e6 / (iters * 16.0));
  cudaFree(d);
}

int main() {
  run<2, 16, 1>("SSc");
  run<4, 16, 1>("MXF4");
  run<4, 64, 1>("MXF4");
  run<4, 128, 1>("MXF4");
  run<4, 256, 1>("MXF4");
  return 0;
}
