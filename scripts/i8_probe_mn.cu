// Probe 2: kind::i8 with B MN-major (N contiguous) in shared memory, SWIZZLE_NONE and
// SWIZZLE_128B, to find the descriptor convention for an M/N-major 8-bit operand.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o i8_probe_mn scripts/i8_probe_mn.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout) << 61;
  return d;
}
constexpr int N = 128, KB = 32;
// A: K-major no swizzle (known good): row m at (m/8)*256 + (k/16)*128 + (m%8)*16 + k%16
__device__ uint32_t aoff(int m, int k) { return (m >> 3) * 256 + (k >> 4) * 128 + (m & 7) * 16 + (k & 15); }
// B MN-major candidates: element (n, k)
__device__ uint32_t boff(int v, int n, int k) {
  if (v == 0) return (k >> 3) * 2048 + (n >> 4) * 128 + (k & 7) * 16 + (n & 15);    // 16n x 8k core, n-chunks 128 apart
  if (v == 1) return (n >> 4) * 512 + (k >> 3) * 128 + (k & 7) * 16 + (n & 15);     // core 16n x 8k, k-groups 128 apart
  // v == 2: SWIZZLE_128B MN-major: row k of 128 B (n 0..127), 16-B chunk c at c ^ (k % 8), 8-row atoms of 1024 B
  { uint32_t o = k * 128 + n; return o ^ (((o >> 7) & 7) << 4); }
}
__global__ void probe(const uint8_t* A, const uint8_t* B, int* D, int v, uint32_t lbo, uint32_t sbo, uint32_t layout, int* flag) {
  __shared__ __align__(1024) uint8_t sa[128 * KB];
  __shared__ __align__(1024) uint8_t sb[N * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int e = tid; e < 128 * KB; e += blockDim.x) sa[aoff(e / KB, e % KB)] = A[e];
  for (int e = tid; e < N * KB; e += blockDim.x) sb[boff(v, e / KB, e % KB)] = B[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (tid < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 16) /*B MN-major*/ | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = sdesc(smem_u32(sa), 128, 256, 0), db = sdesc(smem_u32(sb), lbo, sbo, layout);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  uint32_t done = 0; long long spins = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)));
    if (++spins > (1ll << 26)) { if (tid == 0) *flag = 1; break; }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * N + c + i] = int(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}
int main(int argc, char** argv) {
  const int v = atoi(argv[1]); const uint32_t lbo = atoi(argv[2]), sbo = atoi(argv[3]), layout = atoi(argv[4]);
  std::vector<uint8_t> A(128 * KB), B(N * KB);
  srand(3);
  for (auto& x : A) x = uint8_t(rand() & 255);
  for (auto& x : B) x = uint8_t(rand() & 255);
  std::vector<long long> ref(128 * N, 0);
  for (int i = 0; i < 128; ++i) for (int j = 0; j < N; ++j) { long long s = 0; for (int k = 0; k < KB; ++k) s += (long long)A[i * KB + k] * B[j * KB + k]; ref[i * N + j] = s; }
  uint8_t *dA, *dB; int *dD, *dflag;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, ref.size() * 4); cudaMalloc(&dflag, 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, ref.size() * 4); cudaMemset(dflag, 0, 4);
  probe<<<1, 128>>>(dA, dB, dD, v, lbo, sbo, layout, dflag);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> D(ref.size()); int flag = 0;
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&flag, dflag, 4, cudaMemcpyDeviceToHost);
  int bad = 0; for (size_t i = 0; i < D.size(); ++i) bad += (long long)D[i] != ref[i];
  printf("v=%d lbo=%u sbo=%u layout=%u err=%s timeout=%d mismatches=%d/%zu\n", v, lbo, sbo, layout, cudaGetErrorString(e), flag, bad, D.size());
  return 0;
}
