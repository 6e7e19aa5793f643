// tf32 input-rounding probe (which fp32 -> tf32 conversion does kind::tf32 apply to raw fp32
// operands?).  Derived from umma_probe.cu: one CTA computes D(128 x N) = A(128 x K) B(K x N)^T-ish
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
#include <cstring>

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
    if (!b_mn) {
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
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(a_mn != 0) << 15) | ((uint32_t)(b_mn != 0) << 16) |
                           (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << m_shift);
    const int KSTEP = 32 / ES;  // elements per MMA
    for (int s = 0; s < K / KSTEP; ++s) {
      uint64_t da, db;
      if (!a_mn) da = sdesc(smem_u32(sa) + s * 32, 16, 1024, 2);
      else if (a_mn == 1) da = sdesc(smem_u32(sa) + s * (KSTEP / 8) * 1024, K * 128, 1024, 2);
      else da = sdesc(smem_u32(sa) + s * 1024, K * 128, 512, 1);
      if (!b_mn) db = sdesc(smem_u32(sb) + s * 32, 16, 1024, 2);
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


static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static float trunc_tf32(float x) { return u2f(f2u(x) & 0xFFFFE000u); }
static float rna_tf32(float x) { return u2f((f2u(x) + 0x1000u) & 0xFFFFE000u); }
static float rne_tf32(float x) { uint32_t u = f2u(x); uint32_t lsb = (u >> 13) & 1u; return u2f((u + 0xFFFu + lsb) & 0xFFFFE000u); }

int main() {
  constexpr int N = 32, K = 32;
  std::vector<float> A(128 * K, 0.f), B(N * K, 0.f), D(128 * N);
  // A[m][0] = s * (1 + f_m * 2^-10) with f_m in [0, 1) straddling the tf32 rounding points
  for (int m = 0; m < 128; ++m) {
    const float frac = float(m % 64) / 64.f;
    const float s = m < 64 ? 1.f : -1.f;
    A[m * K + 0] = s * (1.f + frac * ldexpf(1.f, -10));
  }
  B[0 * K + 0] = 1.f;  // D[m][0] = A[m][0] as the tensor core sees it
  float *dA, *dB, *dD; int* dflag;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dflag, 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dflag, 0, 4);
  const int smem = 128 * K * 4 + N * K * 4 + 4096;
  cudaFuncSetAttribute(probe<0, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<0, N, K><<<1, 128, smem>>>(dA, dB, dD, 0, 0, 24, dflag);
  printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int ok_t = 0, ok_a = 0, ok_e = 0, ok_x = 0;
  for (int m = 0; m < 128; ++m) {
    const float x = A[m * K], d = D[m * N];
    ok_t += d == trunc_tf32(x); ok_a += d == rna_tf32(x); ok_e += d == rne_tf32(x); ok_x += d == x;
    if (m % 16 == 0 || (m % 64) == 32) printf("m=%3d x=%.9g D=%.9g trunc=%.9g rna=%.9g rne=%.9g\n", m, x, d, trunc_tf32(x), rna_tf32(x), rne_tf32(x));
  }
  printf("matches of 128: truncate=%d round-nearest-away=%d round-nearest-even=%d exact-fp32=%d\n", ok_t, ok_a, ok_e, ok_x);
  return 0;
}
