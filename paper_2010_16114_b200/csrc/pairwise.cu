// pairwise_euclidean (distlinalg.py:442-468): Y[i, j] = ||x_i - x_j||_2 for the
// owned columns j of the n x n target, direct-difference formula like the
// reference (so Y is exactly symmetric and the diagonal exactly 0).  This is the
// one-time MDS setup (O(n^2 d)), not the per-iteration hot path, but at C3
// (n = 100,000, d = 1000) it is 1e13 difference-squares, so it is register-tiled:
// a CTA owns a 64 x 64 block of Y, a thread 4 rows x 4 columns, the coordinates
// are staged k-major in shared memory (double-buffered through registers) and the
// float32 version runs on packed f32x2 FMAs (two columns per instruction).
//
// x: d x n gathered points, column-major (x[i*d + k]); Y local block n x n_loc.
#include "bsb200.cuh"

#include <algorithm>

using namespace bs;

constexpr int PW_T = 64;       // tile edge (rows i and columns j)
constexpr int PW_THREADS = 256;

typedef unsigned long long pw_f2;
__device__ __forceinline__ pw_f2 pw_pack(float a, float b) {
  pw_f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void pw_unpack(pw_f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ pw_f2 pw_fma(pw_f2 a, pw_f2 b, pw_f2 c) {
  pw_f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <typename T>
__global__ void __launch_bounds__(PW_THREADS)
pairwise_kernel(const T* __restrict__ x, int64_t d, int64_t n, int64_t lo, int64_t n_loc, T* __restrict__ Y) {
  constexpr int PW_K = sizeof(T) == 8 ? 16 : 32;  // coordinates per stage (static smem <= 48 KB)
  __shared__ __align__(16) T xi[2][PW_K][PW_T + 4];  // +4: rows stay 16-byte aligned, stores 4-way at most
  __shared__ __align__(16) T xj[2][PW_K][PW_T + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // rows 4tx.., columns 4ty..
  const int64_t i0 = int64_t(blockIdx.x) * PW_T, j0 = int64_t(blockIdx.y) * PW_T;
  // staging: thread loads 8 coordinates of one point for each side (k fastest: coalesced)
  constexpr int PER = PW_K * PW_T / PW_THREADS;  // 8
  T ri[PER], rj[PER];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + PW_THREADS * u;
      const int kk = e % PW_K, p = e / PW_K;
      const int64_t k = k0 + kk, i = i0 + p, j = j0 + p;
      ri[u] = (k < d && i < n) ? x[i * d + k] : T(0);
      rj[u] = (k < d && j < n_loc) ? x[(lo + j) * d + k] : T(0);
    }
  };
  auto store = [&](int b) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + PW_THREADS * u;
      const int kk = e % PW_K, p = e / PW_K;
      xi[b][kk][p] = ri[u];
      xj[b][kk][p] = rj[u];
    }
  };
  if constexpr (sizeof(T) == 4) {
    pw_f2 acc[4][2];  // [row u][column pair]
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = pw_pack(0.f, 0.f);
    const pw_f2 neg1 = pw_pack(-1.f, -1.f);
    load(0);
    store(0);
    __syncthreads();
    int b = 0;
    for (int64_t k0 = 0; k0 < d; k0 += PW_K) {
      const bool more = k0 + PW_K < d;
      if (more) load(k0 + PW_K);
#pragma unroll 8
      for (int kk = 0; kk < PW_K; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&xi[b][kk][4 * tx]);
        const float4 c = *reinterpret_cast<const float4*>(&xj[b][kk][4 * ty]);
        const pw_f2 c01 = pw_pack(c.x, c.y), c23 = pw_pack(c.z, c.w);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const pw_f2 au = pw_pack(av[u], av[u]);
          const pw_f2 d01 = pw_fma(au, neg1, c01);  // x_j - x_i (distlinalg.py:465)
          const pw_f2 d23 = pw_fma(au, neg1, c23);
          acc[u][0] = pw_fma(d01, d01, acc[u][0]);
          acc[u][1] = pw_fma(d23, d23, acc[u][1]);
        }
      }
      if (more) {
        store(b ^ 1);
        __syncthreads();
        b ^= 1;
      }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t j = j0 + 4 * ty + v;
      if (j >= n_loc) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + 4 * tx + u;
        if (i >= n) continue;
        float s0, s1;
        pw_unpack(acc[u][v >> 1], s0, s1);
        const float s = (v & 1) ? s1 : s0;
        Y[j * n + i] = (i == lo + j) ? 0.f : sqrtf(s);  // diag_fill(y, 0)
      }
    }
  } else {
    T acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
    load(0);
    store(0);
    __syncthreads();
    int b = 0;
    for (int64_t k0 = 0; k0 < d; k0 += PW_K) {
      const bool more = k0 + PW_K < d;
      if (more) load(k0 + PW_K);
#pragma unroll 4
      for (int kk = 0; kk < PW_K; ++kk) {
        T av[4], cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = xi[b][kk][4 * tx + u];
          cv[u] = xj[b][kk][4 * ty + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const T df = cv[v] - av[u];  // x_j - x_i (distlinalg.py:465)
            acc[u][v] = fma(df, df, acc[u][v]);
          }
      }
      if (more) {
        store(b ^ 1);
        __syncthreads();
        b ^= 1;
      }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t j = j0 + 4 * ty + v;
      if (j >= n_loc) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + 4 * tx + u;
        if (i < n) Y[j * n + i] = (i == lo + j) ? T(0) : sqrt(acc[u][v]);  // diag_fill(y, 0)
      }
    }
  }
}

extern "C" int bs_pairwise_euclidean(const void* x, int dtype, int64_t d, int64_t n, int64_t lo, int64_t n_loc,
                                     void* Y, void* stream) {
  clear_error();
  if (d < 0 || n < 0 || lo < 0 || n_loc < 0 || lo + n_loc > n) {
    set_error("bs_pairwise_euclidean: bad shape");
    return BS_EINVAL;
  }
  if (n == 0 || n_loc == 0) return BS_OK;
  dim3 grid(unsigned(ceil_div(n, PW_T)), unsigned(ceil_div(n_loc, PW_T)));
  cudaStream_t st = as_stream(stream);
  if (dtype == BS_F64)
    pairwise_kernel<double><<<grid, PW_THREADS, 0, st>>>(static_cast<const double*>(x), d, n, lo, n_loc,
                                                         static_cast<double*>(Y));
  else if (dtype == BS_F32)
    pairwise_kernel<float><<<grid, PW_THREADS, 0, st>>>(static_cast<const float*>(x), d, n, lo, n_loc,
                                                        static_cast<float*>(Y));
  else {
    set_error("bs_pairwise_euclidean: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_pairwise_euclidean");
}
