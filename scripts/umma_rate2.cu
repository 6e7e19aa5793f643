// tcgen05.mma tf32 cost vs TMEM allocation size and accumulator interleaving.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16; d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46; d |= uint64_t(layout) << 61; return d;
}
template <int N, int COLS>
__global__ void rate(int naccs, int ts, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar; __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)smem)[i] = 0.5f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(COLS)); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) | (8u << 24);
    uint32_t sb = smem_u32(smem + 32768);
    uint64_t da = sdesc(smem_u32(smem), 16, 1024, 2);
    uint64_t db = sdesc(sb, 4096, 512, 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % naccs) * N);
      if (ts) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(tmem + COLS - 32), "l"(db), "r"(idesc), "r"(1));
      else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS));
}
template <int N, int COLS> void go(int naccs, int ts) {
  long long* d; cudaMalloc(&d, 8 * 256);
  cudaFuncSetAttribute(rate<N, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 4096;
  rate<N, COLS><<<148, 128, 70000>>>(naccs, ts, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("N=%3d alloc=%3d accs=%d %s  %s cycles/MMA=%.1f\n", N, COLS, naccs, ts ? "TS" : "SS", cudaGetErrorString(e), avg / iters);
  cudaFree(d);
}
int main() {
  go<64, 256>(1, 0); go<64, 512>(1, 0); go<64, 256>(2, 0); go<64, 512>(2, 0); go<64, 512>(4, 0);
  go<64, 512>(1, 1); go<64, 512>(2, 1); go<64, 512>(4, 1);
  go<128, 512>(1, 1); go<128, 512>(2, 1);
  go<32, 512>(1, 1); go<32, 512>(4, 1);
}
