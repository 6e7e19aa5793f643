// Measures tcgen05.mma throughput (cycles per instruction) for tf32 / bf16, K-major vs MN-major operands.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16; d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46; d |= uint64_t(layout) << 61; return d;
}
template <int KIND, int N>
__global__ void rate(int amn, int bmn, int iters, long long* out, int ts) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar; __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)smem)[i] = 0.5f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | (uint32_t(N >> 3) << 17) | (8u << 24);
    uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    uint64_t da = amn ? sdesc(sa, 4096, 512, KIND == 0 ? 1 : 2) : sdesc(sa, 16, 1024, 2);
    uint64_t db = bmn ? sdesc(sb, 4096, 512, KIND == 0 ? 1 : 2) : sdesc(sb, 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0 && ts) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 256), "l"(db), "r"(idesc), "r"(1));
      else if (KIND == 0) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
      else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
template <int KIND, int N> void go(const char* nm, int amn, int bmn, int grid, int ts = 0) {
  long long* d; cudaMalloc(&d, 8 * 256);
  cudaFuncSetAttribute(rate<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 4096;
  rate<KIND, N><<<grid, 128, 70000>>>(amn, bmn, iters, d, ts);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
  printf("%-26s grid=%3d  %s  cycles/MMA=%.1f\n", nm, grid, cudaGetErrorString(e), avg / iters);
  cudaFree(d);
}
int main() {
  for (int g : {148}) {
    go<0, 64>("tf32 SS K/MN N64", 0, 1, g);
    go<0, 128>("tf32 SS K/MN N128", 0, 1, g);
    go<0, 64>("tf32 TS MN N64", 0, 1, g, 1);
    go<0, 128>("tf32 TS MN N128", 0, 1, g, 1);
    go<0, 32>("tf32 TS MN N32", 0, 1, g, 1);
    go<0, 256>("tf32 TS MN N256", 0, 1, g, 1);
    go<0, 64>("tf32 TS K N64", 0, 0, g, 1);
  }
}
