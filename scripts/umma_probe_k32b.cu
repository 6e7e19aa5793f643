// Standalone tcgen05 probe: one CTA computes D(128 x N) = A(128 x K) B(K x N)^T-ish
// with operands written to smem by threads in the canonical SW128 layouts, then
// checks D against a host reference.  Variants: kind::tf32 with A K-major or
// MN-major (B MN-major or K-major), and kind::f16 (bf16) K-major as a control.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
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

// byte offset inside a 1024B-aligned SW128 region -> physical byte offset
__device__ __forceinline__ uint32_t sw128(uint32_t o) { return o ^ (((o >> 7) & 7) << 4); }
// Swizzle<2,5,2>: 32B chunk index (bits 5-6) ^= bits 7-8
__device__ __forceinline__ uint32_t sw32a(uint32_t o) { return o ^ (((o >> 7) & 3) << 5); }

template <int KIND>  // 0 = tf32, 1 = f16(bf16)
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A: M=128 x K; B: N x K (so D = A B^T).  Values given row-major in global (float).
// a_mn: store A MN-major (M contiguous) instead of K-major.  b_mn likewise for B (N contiguous).
template <int KIND, int N, int K>
__global__ void probe(const float* A, const float* B, float* D, int a_mn, int b_mn, int m_shift, int* flag) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  constexpr int ES = KIND == 0 ? 4 : 2;          // element bytes
  constexpr int KPA = 128 / ES;                   // elements per 128B row
  uint8_t* sa = smem;                             // A region
  uint8_t* sb = smem + 128 * K * ES + 1024;       // B region (1024 aligned since 128*K*ES multiple of 1024)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  // ---- fill A ----
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    uint32_t off;
    if (!a_mn) {  // K-major: rows m of K elements; K <= KPA so one 128B row per m
      off = m * 128 + k * ES;
      off = sw128(off);
    } else {      // MN-major: atoms of 32(MN) x 8(K) ; slab per MN atom: K rows x 128B
      const int atom = m / KPA, mi = m % KPA;
      off = atom * (K * 128) + k * 128 + mi * ES;
      off = a_mn == 2 ? sw32a(off) : ((off & ~1023u) | sw128(off & 1023u));
    }
    if (KIND == 0) *(float*)(sa + off) = A[m * K + k];
    else *(__nv_bfloat16*)(sa + off) = __float2bfloat16(A[m * K + k]);
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    uint32_t off;
    if (b_mn >= 3) {  // K-major rows of 128 B, Swizzle<2,5,2> (the MN-major BASE32B arrangement)
      off = sw32a(n * 128 + k * ES);
    } else if (!b_mn) {
      off = n * 128 + k * ES;
      off = (off & ~1023u) | sw128(off & 1023u);
    } else {
      const int atom = n / KPA, ni = n % KPA;
      off = atom * (K * 128) + k * 128 + ni * ES;
      off = b_mn == 2 ? sw32a(off) : ((off & ~1023u) | sw128(off & 1023u));
    }
    if (KIND == 0) *(float*)(sb + off) = B[n * K + k];
    else *(__nv_bfloat16*)(sb + off) = __float2bfloat16(B[n * K + k]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t fmt = KIND == 0 ? 2u : 1u;  // tf32 / bf16
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(a_mn != 0) << 15) | ((uint32_t)(b_mn == 1 || b_mn == 2) << 16) |
                           (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << m_shift);
    const int KSTEP = 32 / ES;  // elements per MMA
    for (int s = 0; s < K / KSTEP; ++s) {
      uint64_t da, db;
      if (!a_mn) da = sdesc(smem_u32(sa) + s * 32, 16, 1024, 2);
      else if (a_mn == 1) da = sdesc(smem_u32(sa) + s * (KSTEP / 8) * 1024, K * 128, 1024, 2);
      else da = sdesc(smem_u32(sa) + s * 1024, K * 128, 512, 1);
      if (b_mn == 3) db = sdesc(smem_u32(sb) + s * 32, 16, 512, 1);
      else if (b_mn == 4) db = sdesc(smem_u32(sb) + s * 32, 16, 1024, 1);
      else if (b_mn == 5) db = sdesc(smem_u32(sb) + s * 32, 512, 1024, 1);
      else if (!b_mn) db = sdesc(smem_u32(sb) + s * 32, 16, 1024, 2);
      else if (b_mn == 1) db = sdesc(smem_u32(sb) + s * (KSTEP / 8) * 1024, K * 128, 1024, 2);
      else db = sdesc(smem_u32(sb) + s * 1024, K * 128, 512, 1);
      mma<KIND>(tmem, da, db, idesc, s > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait
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
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * N + c0 + i] = __uint_as_float(r[i]);
    }
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

template <int KIND, int N, int K>
void run(const char* name, int a_mn, int b_mn, int m_shift) {
  std::vector<float> A(128 * K), B(N * K), D(128 * N, -1.f), R(128 * N, 0.f);
  for (int i = 0; i < 128 * K; ++i) A[i] = float((i * 7) % 13) - 6.f;
  for (int i = 0; i < N * K; ++i) B[i] = float((i * 5) % 11) - 5.f;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * B[n * K + k];
      R[m * N + n] = float(s);
    }
  float *dA, *dB, *dD;
  int* dflag;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dflag, 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, D.size() * 4);
  cudaMemset(dflag, 0, 4);
  const int smem = 128 * K * 4 + N * K * 4 + 4096;
  cudaFuncSetAttribute(probe<KIND, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<KIND, N, K><<<1, 128, smem>>>(dA, dB, dD, a_mn, b_mn, m_shift, dflag);
  cudaError_t e = cudaDeviceSynchronize();
  int flag = 0;
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&flag, dflag, 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int nz = 0;
  for (int i = 0; i < 128 * N; ++i) {
    maxerr = fmax(maxerr, fabs(D[i] - R[i]));
    nz += D[i] != 0.f;
  }
  printf("%-34s err=%s maxerr=%g nonzero=%d timeout=%d D[0..3]=%g %g %g %g R=%g %g %g %g\n", name,
         cudaGetErrorString(e), maxerr, nz, flag, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dflag);
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  if (v == 0) run<0, 32, 32>("tf32 K/K (control)", 0, 0, 24);
  if (v == 3) run<0, 32, 32>("tf32 K/K32B sbo512", 0, 3, 24);
  if (v == 4) run<0, 32, 32>("tf32 K/K32B sbo1024", 0, 4, 24);
  if (v == 5) run<0, 32, 32>("tf32 K/K32B lbo512", 0, 5, 24);
  return 0;
}
