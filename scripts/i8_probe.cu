// Probe: tcgen05.mma kind::i8 (u8 x u8 -> s32), both operands K-major SWIZZLE_NONE in smem,
// with the digit-slice accumulation pattern of nmf_i8.cu:
//   D[:,   0:3N] += A0 [B0|B1|B2]
//   D[:,   N:4N] += A1 [B0|B1|B2]
//   D[:, 2N:4N] += A2 [B0|B1]
// Core matrix = 8 rows x 16 B contiguous; LBO = stride between the two 16-B K chunks,
// SBO = stride between 8-row groups.  Checks every accumulator column against the host.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o i8_probe scripts/i8_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version, layout 0 = SWIZZLE_NONE
  return d;
}

constexpr int N = 64;  // rows per slice
constexpr int KB = 32; // bytes of K

// operand byte (row, k) -> smem offset, canonical K-major no-swizzle with the given strides
__device__ __forceinline__ uint32_t koff(int row, int k, uint32_t lbo, uint32_t sbo) {
  return uint32_t(row >> 3) * sbo + uint32_t(k >> 4) * lbo + uint32_t(row & 7) * 16 + uint32_t(k & 15);
}

__global__ void probe(const uint8_t* A, const uint8_t* B, int* D, uint32_t lbo, uint32_t sbo, uint32_t lbo_d,
                      uint32_t sbo_d, int* flag) {
  __shared__ __align__(1024) uint8_t sa[3 * 128 * KB];
  __shared__ __align__(1024) uint8_t sb[3 * N * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int e = tid; e < 3 * 128 * KB; e += blockDim.x) {
    const int s = e / (128 * KB), rem = e % (128 * KB), row = rem / KB, k = rem % KB;
    sa[s * 128 * KB + koff(row, k, lbo, sbo)] = A[e];
  }
  for (int e = tid; e < 3 * N * KB; e += blockDim.x) {
    const int row = e / KB, k = e % KB;  // 3N stacked rows
    sb[koff(row, k, lbo, sbo)] = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    // kind::i8: c_format S32 (2) at bit 4, a/b format u8 (0), K-major, N>>3 at 17, M>>4 at 24
    auto idesc = [](int n) { return (2u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24); };
    const uint64_t b0 = sdesc(smem_u32(sb), lbo_d, sbo_d);
    for (int s = 0; s < 3; ++s) {
      const uint64_t a = sdesc(smem_u32(sa + s * 128 * KB), lbo_d, sbo_d);
      const int n = s < 2 ? 3 * N : 2 * N;
      const uint32_t d = tmem + uint32_t(s * N);
      const uint32_t acc = s > 0 ? 1u : 0u;
      // s = 0 initialises columns 0..3N; column block 3N..4N is first written by s = 1, so
      // zero it with a dummy A2 x 0 MMA first is not possible — instead s=1 uses acc only
      // where s=0 wrote; we run s=1 in two parts: [B0|B1] accumulate, B2 part initialise.
      if (s == 1) {
        const uint32_t id2 = idesc(2 * N);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b0), "r"(id2));
        const uint64_t b2 = sdesc(smem_u32(sb + 2 * N * KB), lbo_d, sbo_d);
        const uint32_t id1 = idesc(N);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d + 2 * N), "l"(a), "l"(b2), "r"(id1));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b0), "r"(idesc(n)), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t done = 0;
    long long spins = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
      if (++spins > (1ll << 26)) { if (tid == 0) *flag = 1; break; }
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 lanes x 256 columns
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < 4 * N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * 4 * N + c + i] = int(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<uint8_t> A(3 * 128 * KB), B(3 * N * KB);
  srand(7);
  for (auto& v : A) v = uint8_t(rand() & 255);
  for (auto& v : B) v = uint8_t(rand() & 255);
  // host: acc_w = sum over (p,q) with p+q = w
  std::vector<long long> ref(128 * 4 * N, 0);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j)
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
          if (p == 2 && q == 2) continue;
          long long s = 0;
          for (int k = 0; k < KB; ++k) s += (long long)A[p * 128 * KB + i * KB + k] * B[(q * N + j) * KB + k];
          ref[i * 4 * N + (p + q) * N + j] += s;
        }
  uint8_t *dA, *dB;
  int *dD, *dflag;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, ref.size() * 4);
  cudaMalloc(&dflag, 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  struct V { uint32_t lbo, sbo, lbo_d, sbo_d; const char* name; };
  V vs[] = {{128, 256, 128, 256, "lbo=128(K chunk) sbo=256(row group)"},
            {128, 256, 256, 128, "data lbo128/sbo256, desc fields swapped"},
            {2048, 128, 2048, 128, "K chunks far apart: lbo=2048 sbo=128"},
            {2048, 128, 128, 2048, "K chunks far apart, desc fields swapped"}};
  for (auto& v : vs) {
    cudaMemset(dD, 0, ref.size() * 4);
    cudaMemset(dflag, 0, 4);
    probe<<<1, 128>>>(dA, dB, dD, v.lbo, v.sbo, v.lbo_d, v.sbo_d, dflag);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> D(ref.size());
    int flag = 0;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&flag, dflag, 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (size_t i = 0; i < D.size(); ++i) bad += (long long)D[i] != ref[i];
    printf("%-48s err=%s timeout=%d mismatches=%d/%zu  D[0]=%d ref=%lld D[last]=%d ref=%lld\n", v.name,
           cudaGetErrorString(e), flag, bad, D.size(), D[0], ref[0], D.back(), ref.back());
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
