// MDS by majorization-minimization (solvers.py:188-305): one fused pass over the
// rank's columns of the target-distance matrix Y per iteration.
//
// The reference materializes the n x n/p Gram, distance, Z and (W - Z) matrices
// in a second n x n buffer and makes ~10 passes over it (solvers.py:237-301).
// Here Y is read exactly once per iteration: for every pair (i, j) the kernel
// forms g = theta_i . theta_j, d = sqrt(max(|theta_i|^2 + |theta_j|^2 - 2g, 0))
// (the Gram identity of _embedding_distances, solvers.py:246), accumulates the
// stress (y - d)^2 and the zero-distance count, and for the MM step
// z = y / d, zsum_j += z, T_j += theta_i (1 - z) (i != j; the diagonal of W - Z
// is 0, solvers.py:299-300).  No n x n temporary exists.
//
// Layout: Y local block n x n_loc column-major (Y[jl*n + i]); theta q x n
// column-major (theta[i*q + k]).
#include "bsb200.cuh"

#include <algorithm>
#include <mutex>

using namespace bs;

constexpr int MDS_THREADS = 256;
constexpr int MDS_WARPS = MDS_THREADS / 32;

// Pass kernel.  A CTA owns 8*JB columns (JB per warp) and one row segment.  The
// segment is walked in chunks of CH rows; for every chunk the theta rows (CH x q,
// contiguous in global memory) and the CTA's Y tile (CH rows of each of its
// columns, contiguous per column) are copied into shared memory with cp.async,
// double-buffered so chunk c+1 streams in while chunk c is computed.  Every lane
// then walks rows i = lane, lane+32, ... of the chunk.  Per pair: g (q FMA), d,
// stress, z, zsum and T_j += theta_i (1 - z) (q FMA); theta_j, the T partials and
// zsum live in registers for the whole segment.  Arithmetic in the storage type
// (the reference computes float32 data in float32); float32 uses one refined
// rsqrt per pair, float64 IEEE sqrt/div (exact on exact inputs).
//   Partials per row segment s: zsum_part[s][jl], T_part[s][jl][k] (float64);
//   stress / zero count per CTA (float64).
template <typename T>
struct MdsChunk {
  static constexpr int CH = sizeof(T) == 4 ? 128 : 64;  // rows per chunk
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
// one element of T
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
  if constexpr (sizeof(T) == 8) cp_async8(smem, gmem);
  else cp_async4(smem, gmem);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issues the async copies of chunk [c0, c0+rows) into buffer b.
template <typename T, int QS, int JB>
__device__ __forceinline__ void mds_stage(T* th_s, T* y_s, const T* __restrict__ theta, const T* __restrict__ Y,
                                          int64_t n, int64_t jl0_cta, int64_t n_loc, int q, int64_t c0, int rows,
                                          bool vec_th, bool vec) {
  constexpr int CH = MdsChunk<T>::CH;
  constexpr int VW = 16 / int(sizeof(T));
  constexpr int NC = MDS_WARPS * JB;  // columns of the CTA
  // theta rows: QS-strided rows in smem; global rows are q-strided
  if (vec_th && QS == q) {
    const int words = rows * QS / VW;
    for (int e = threadIdx.x; e < words; e += MDS_THREADS) cp_async16(th_s + e * VW, theta + c0 * q + int64_t(e) * VW);
  } else {
    for (int e = threadIdx.x; e < rows * q; e += MDS_THREADS) {
      const int rr = e / q, k = e - rr * q;
      cp_async_elem(th_s + rr * QS + k, theta + (c0 + rr) * q + k);
    }
  }
  // Y tile: column c of the CTA -> y_s[c * CH + rr]
  if (vec) {
    const int per_col = rows / VW;  // rows is a multiple of VW when vec
    for (int e = threadIdx.x; e < NC * per_col; e += MDS_THREADS) {
      const int c = e / per_col, w = e - c * per_col;
      const int64_t jl = jl0_cta + c;
      if (jl < n_loc) cp_async16(y_s + c * CH + w * VW, Y + jl * n + c0 + int64_t(w) * VW);
    }
  } else {
    for (int e = threadIdx.x; e < NC * rows; e += MDS_THREADS) {
      const int c = e / rows, rr = e - c * rows;
      const int64_t jl = jl0_cta + c;
      if (jl < n_loc) cp_async_elem(y_s + c * CH + rr, Y + jl * n + c0 + rr);
    }
  }
  cp_async_commit();
}

// ---------------------------------------------------------------------------
// float32 pass on packed FFMA2 (fma.rn.f32x2, sm_100): the columns of a warp are
// processed in pairs, so theta_i . {theta_j, theta_j'} and
// {T_j, T_j'} += theta_i {wz, wz'} each take one instruction per k.  One
// rsqrt.approx + a Newton step per pair gives d = d2 r and z = y r.
// ---------------------------------------------------------------------------

typedef unsigned long long f2_t;  // two packed float32 (register pair)

__device__ __forceinline__ f2_t f2_pack(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int QM, int JB>
__global__ void __launch_bounds__(MDS_THREADS, QM <= 20 ? 2 : 1)
mds_pass_f32x2_kernel(const float* __restrict__ Y, const float* __restrict__ theta, int64_t n, int64_t lo,
                      int64_t n_loc, int q, int perturb, int mode, int64_t rows_per_seg,
                      double* __restrict__ zsum_part, double* __restrict__ T_part, double* __restrict__ parts,
                      unsigned int* counter, double* __restrict__ red, const float* __restrict__ norms) {
  static_assert(JB % 2 == 0, "columns are processed in pairs");
  constexpr int VW = 4;
  constexpr int QS0 = (QM + VW - 1) / VW * VW;
  constexpr int QS = ((QS0 / VW) % 2 == 0) ? QS0 + VW : QS0;
  constexpr int CH = MdsChunk<float>::CH;
  constexpr int NC = MDS_WARPS * JB;
  constexpr int JP = JB / 2;
  extern __shared__ __align__(16) uint8_t mds_smem[];
  float* th_buf[2] = {reinterpret_cast<float*>(mds_smem), reinterpret_cast<float*>(mds_smem) + CH * QS};
  float* y_buf[2] = {reinterpret_cast<float*>(mds_smem) + 2 * CH * QS,
                     reinterpret_cast<float*>(mds_smem) + 2 * CH * QS + NC * CH};
  float* nrm_buf[2] = {reinterpret_cast<float*>(mds_smem) + 2 * CH * QS + 2 * NC * CH,
                       reinterpret_cast<float*>(mds_smem) + 2 * CH * QS + 2 * NC * CH + CH};
  __shared__ double sh_a[32], sh_b[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t jl0_cta = int64_t(blockIdx.x) * NC;
  const int64_t jl0 = jl0_cta + int64_t(wid) * JB;
  const int64_t i_begin = int64_t(blockIdx.y) * rows_per_seg;
  const int64_t i_end = min(n, i_begin + rows_per_seg);
  const bool vec = (n % VW == 0) && (i_begin % VW == 0) && (reinterpret_cast<uintptr_t>(Y) % 16 == 0);
  const bool vec_th = (q % VW == 0) && (reinterpret_cast<uintptr_t>(theta) % 16 == 0);

  f2_t tj[JP][QM], Tacc[JP][QM];
  float nj[JB], zs[JB];
  bool live[JB];
#pragma unroll
  for (int p = 0; p < JP; ++p) {
    float s0 = 0.f, s1 = 0.f;
    const int64_t ja = jl0 + 2 * p, jb = ja + 1;
    live[2 * p] = ja < n_loc;
    live[2 * p + 1] = jb < n_loc;
    const int64_t ga = lo + (live[2 * p] ? ja : 0), gb = lo + (live[2 * p + 1] ? jb : 0);
#pragma unroll
    for (int k = 0; k < QM; ++k) {
      const float a = (k < q && live[2 * p]) ? theta[ga * q + k] : 0.f;
      const float b = (k < q && live[2 * p + 1]) ? theta[gb * q + k] : 0.f;
      s0 = fmaf(a, a, s0);
      s1 = fmaf(b, b, s1);
      tj[p][k] = f2_pack(a, b);
      Tacc[p][k] = f2_pack(0.f, 0.f);
    }
    nj[2 * p] = s0;
    nj[2 * p + 1] = s1;
    zs[2 * p] = zs[2 * p + 1] = 0.f;
  }
  for (int e = threadIdx.x; e < 2 * CH * QS; e += MDS_THREADS)
    if ((e % QS) >= q) th_buf[0][e] = 0.f;
  double stress = 0.0, zeros = 0.0;
  const int64_t nchunks = (i_end - i_begin + CH - 1) / CH;
  auto stage_norms = [&](float* dst, int64_t c0, int rows) {
    for (int e = threadIdx.x; e < rows; e += MDS_THREADS) cp_async4(dst + e, norms + c0 + e);
  };
  if (nchunks > 0) {
    stage_norms(nrm_buf[0], i_begin, int(i_end - i_begin < CH ? i_end - i_begin : CH));
    mds_stage<float, QS, JB>(th_buf[0], y_buf[0], theta, Y, n, jl0_cta, n_loc, q, i_begin,
                             int(i_end - i_begin < CH ? i_end - i_begin : CH), vec_th, vec);
  }
  for (int64_t ck = 0; ck < nchunks; ++ck) {
    const int64_t c0 = i_begin + ck * CH;
    const int rows = int(i_end - c0 < CH ? i_end - c0 : CH);
    const int b = int(ck & 1);
    if (ck + 1 < nchunks) {
      const int64_t c1 = c0 + CH;
      stage_norms(nrm_buf[b ^ 1], c1, int(i_end - c1 < CH ? i_end - c1 : CH));
      mds_stage<float, QS, JB>(th_buf[b ^ 1], y_buf[b ^ 1], theta, Y, n, jl0_cta, n_loc, q, c1,
                               int(i_end - c1 < CH ? i_end - c1 : CH), vec_th, vec);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* th_s = th_buf[b];
    const float* y_s = y_buf[b] + wid * JB * CH;
    int diag[JB];  // chunk row of column c's diagonal (out of range when not in this chunk)
#pragma unroll
    for (int c = 0; c < JB; ++c) {
      const int64_t dr = lo + jl0 + c - c0;
      diag[c] = (dr >= 0 && dr < CH) ? int(dr) : -1;
    }
    const float* nrm_s = nrm_buf[b];
    float st_chunk = 0.f, zc_chunk = 0.f;
    for (int rb = lane; rb < rows; rb += 64) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int rr = rb + 32 * hr;
        if (rr >= rows) break;
        float ti[QM];
        const float4* src = reinterpret_cast<const float4*>(th_s + rr * QS);
#pragma unroll
        for (int v = 0; v < QM / VW; ++v) {
          const float4 w = src[v];
          ti[4 * v] = w.x; ti[4 * v + 1] = w.y; ti[4 * v + 2] = w.z; ti[4 * v + 3] = w.w;
        }
        const float ni = nrm_s[rr];
#pragma unroll
        for (int p = 0; p < JP; ++p) {
          // g for both columns: two packed partial sums for ILP
          f2_t ga = f2_pack(0.f, 0.f), gb = f2_pack(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < QM; ++k) {
            const f2_t t = f2_pack(ti[k], ti[k]);
            if (k & 1) gb = f2_fma(t, tj[p][k], gb);
            else ga = f2_fma(t, tj[p][k], ga);
          }
          float g[2];
          f2_unpack(f2_add(ga, gb), g[0], g[1]);
          float wz[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = 2 * p + h;
            const float y = y_s[c * CH + rr];
            wz[h] = 0.f;
            if (!live[c]) continue;
            if (rr == diag[c]) {  // d_jj = 0 exactly, z_jj = 0, (W - Z)_jj = 0 (solvers.py:240-241, 299-300)
              st_chunk = fmaf(y, y, st_chunk);
              continue;
            }
            const float d2 = (ni + nj[c]) - 2.f * g[h];  // solvers.py:246
            float d, z;
            if (d2 > 0.f) {
              float rs = rsqrt_approx(d2);
              rs = rs * fmaf(-0.5f * d2 * rs, rs, 1.5f);
              d = d2 * rs;
              z = y * rs;  // solvers.py:297
            } else {
              d = 0.f;
              zc_chunk += 1.f;
              z = perturb ? y * 1e10f : y / 0.f;  // solvers.py:296
            }
            const float e = y - d;
            st_chunk = fmaf(e, e, st_chunk);
            zs[c] += z;
            wz[h] = 1.f - z;  // solvers.py:299
          }
          if (mode == 0) {
            const f2_t w2 = f2_pack(wz[0], wz[1]);
#pragma unroll
            for (int k = 0; k < QM; ++k) Tacc[p][k] = f2_fma(f2_pack(ti[k], ti[k]), w2, Tacc[p][k]);
          }
        }
      }
    }
    stress += double(st_chunk);
    zeros += double(zc_chunk);
    __syncthreads();
  }
  if (mode == 0) {
    const int s = blockIdx.y;
#pragma unroll
    for (int p = 0; p < JP; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * p + h;
        const double zsum = warp_sum(double(zs[c]));
        double tk[QM];
#pragma unroll
        for (int k = 0; k < QM; ++k) {
          float a, bb;
          f2_unpack(Tacc[p][k], a, bb);
          tk[k] = warp_sum(double(h ? bb : a));
        }
        const int64_t jl = jl0 + c;
        if (lane == 0 && live[c]) {
          zsum_part[int64_t(s) * n_loc + jl] = zsum;
#pragma unroll
          for (int k = 0; k < QM; ++k)
            if (k < q) T_part[(int64_t(s) * n_loc + jl) * q + k] = tk[k];
        }
      }
    }
  }
  const double st = block_sum(stress, sh_a);
  const double zc = block_sum(zeros, sh_b);
  const unsigned int bid = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    parts[2 * bid] = st;
    parts[2 * bid + 1] = zc;
  }
  if (last_block_done(counter) && threadIdx.x == 0) {
    double a = 0.0, b2 = 0.0;
    const unsigned int nb = gridDim.x * gridDim.y;
    for (unsigned int k = 0; k < nb; ++k) {
      a += parts[2 * k];
      b2 += parts[2 * k + 1];
    }
    red[0] = a;
    red[1] = b2;
  }
}

template <typename T, int QM, int JB>
__global__ void __launch_bounds__(MDS_THREADS)
mds_pass_kernel(const T* __restrict__ Y, const T* __restrict__ theta, int64_t n, int64_t lo,
                int64_t n_loc, int q, int perturb, int mode, int64_t rows_per_seg,
                double* __restrict__ zsum_part, double* __restrict__ T_part,
                double* __restrict__ parts, unsigned int* counter, double* __restrict__ red) {
  constexpr int VW = 16 / int(sizeof(T));                       // elements per 16-byte word
  constexpr int QS0 = (QM + VW - 1) / VW * VW;
  constexpr int QS = ((QS0 / VW) % 2 == 0) ? QS0 + VW : QS0;    // odd number of 16-byte words
  constexpr int CH = MdsChunk<T>::CH;
  constexpr int NC = MDS_WARPS * JB;
  extern __shared__ __align__(16) uint8_t mds_smem[];
  T* th_buf[2] = {reinterpret_cast<T*>(mds_smem), reinterpret_cast<T*>(mds_smem) + CH * QS};
  T* y_buf[2] = {reinterpret_cast<T*>(mds_smem) + 2 * CH * QS, reinterpret_cast<T*>(mds_smem) + 2 * CH * QS + NC * CH};
  __shared__ double sh_a[32], sh_b[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t jl0_cta = int64_t(blockIdx.x) * NC;
  const int64_t jl0 = jl0_cta + int64_t(wid) * JB;
  const int64_t i_begin = int64_t(blockIdx.y) * rows_per_seg;
  const int64_t i_end = min(n, i_begin + rows_per_seg);
  const bool vec = (n % VW == 0) && (i_begin % VW == 0) && (reinterpret_cast<uintptr_t>(Y) % 16 == 0);
  const bool vec_th = (q % VW == 0) && (reinterpret_cast<uintptr_t>(theta) % 16 == 0);

  T tj[JB][QM], Tacc[JB][QM], nj[JB], zs[JB];
  bool live[JB];
#pragma unroll
  for (int c = 0; c < JB; ++c) {
    const int64_t jl = jl0 + c;
    live[c] = jl < n_loc;
    const int64_t jg = lo + (live[c] ? jl : 0);
    T s = T(0);
#pragma unroll
    for (int k = 0; k < QM; ++k) {
      tj[c][k] = (k < q && live[c]) ? theta[jg * q + k] : T(0);
      s = fma(tj[c][k], tj[c][k], s);
      Tacc[c][k] = T(0);
    }
    nj[c] = s;
    zs[c] = T(0);
  }
  // zero the theta padding columns once (cp.async never writes them)
  for (int e = threadIdx.x; e < 2 * CH * QS; e += MDS_THREADS)
    if ((e % QS) >= q) th_buf[0][e] = T(0);
  double stress = 0.0, zeros = 0.0;
  const int64_t nchunks = (i_end - i_begin + CH - 1) / CH;
  if (nchunks > 0)
    mds_stage<T, QS, JB>(th_buf[0], y_buf[0], theta, Y, n, jl0_cta, n_loc, q, i_begin,
                         int(i_end - i_begin < CH ? i_end - i_begin : CH), vec_th, vec);
  for (int64_t ck = 0; ck < nchunks; ++ck) {
    const int64_t c0 = i_begin + ck * CH;
    const int rows = int(i_end - c0 < CH ? i_end - c0 : CH);
    const int b = int(ck & 1);
    if (ck + 1 < nchunks) {
      const int64_t c1 = c0 + CH;
      mds_stage<T, QS, JB>(th_buf[b ^ 1], y_buf[b ^ 1], theta, Y, n, jl0_cta, n_loc, q, c1,
                           int(i_end - c1 < CH ? i_end - c1 : CH), vec_th, vec);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* th_s = th_buf[b];
    const T* y_s = y_buf[b] + wid * JB * CH;
    T st_chunk = T(0);
    for (int rb = lane; rb < rows; rb += 64) {
      // two rows per lane per iteration (rb, rb + 32): independent dependency chains
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = rb + 32 * h;
        if (rr >= rows) break;
        const int64_t i = c0 + rr;
        T ti[QM];
        const uint4* src = reinterpret_cast<const uint4*>(th_s + rr * QS);
#pragma unroll
        for (int v = 0; v < QM / VW; ++v) {
          const uint4 w = src[v];
          const T* wv = reinterpret_cast<const T*>(&w);
#pragma unroll
          for (int u = 0; u < VW; ++u) ti[v * VW + u] = wv[u];
        }
        T ni = T(0);
#pragma unroll
        for (int k = 0; k < QM; ++k) ni = fma(ti[k], ti[k], ni);
#pragma unroll
        for (int c = 0; c < JB; ++c) {
          if (!live[c]) continue;
          const int64_t jl = jl0 + c;
          const T y = y_s[c * CH + rr];
          if (i == lo + jl) {  // diagonal: d_jj = 0 exactly (solvers.py:240-241), z_jj = y/inf = 0
            st_chunk = fma(y, y, st_chunk);
            continue;
          }
          // g = theta_i . theta_j with four independent partial sums
          T g4[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int k = 0; k < QM; ++k) g4[k & 3] = fma(ti[k], tj[c][k], g4[k & 3]);
          const T g = (g4[0] + g4[1]) + (g4[2] + g4[3]);
          // solvers.py:246: sqrt(max(dr + dc - 2g, 0))
          const T d2 = (ni + nj[c]) - T(2) * g;
          T d, z;
          if constexpr (sizeof(T) == 4) {
            // one MUFU per pair: r = rsqrt(d2) refined by a Newton step; d = d2 r, z = y r
            if (d2 > T(0)) {
              float rs = rsqrtf(d2);
              rs = rs * fmaf(-0.5f * d2 * rs, rs, 1.5f);
              d = d2 * rs;
              z = y * rs;
            } else {
              d = T(0);
              z = perturb ? y * T(1e10) : y / T(0);
            }
          } else {
            d = sqrt(d2 > T(0) ? d2 : T(0));
            z = T(0);
          }
          const T e = y - d;
          st_chunk = fma(e, e, st_chunk);
          if (d == T(0)) {
            zeros += 1.0;
            if (perturb) d = T(1e-10);  // solvers.py:296
          }
          if (mode == 0) {
            if constexpr (sizeof(T) == 8) z = y / d;  // solvers.py:297
            zs[c] += z;
            const T wz = T(1) - z;  // solvers.py:299
#pragma unroll
            for (int k = 0; k < QM; ++k) Tacc[c][k] = fma(ti[k], wz, Tacc[c][k]);
          }
        }
      }
    }
    stress += double(st_chunk);
    __syncthreads();  // buffer b is refilled two chunks later
  }
  // per-warp column partials
  if (mode == 0) {
    const int s = blockIdx.y;
#pragma unroll
    for (int c = 0; c < JB; ++c) {
      const double zsum = warp_sum(double(zs[c]));
      double tk[QM];
#pragma unroll
      for (int k = 0; k < QM; ++k) tk[k] = warp_sum(double(Tacc[c][k]));
      const int64_t jl = jl0 + c;
      if (lane == 0 && live[c]) {
        zsum_part[int64_t(s) * n_loc + jl] = zsum;
#pragma unroll
        for (int k = 0; k < QM; ++k)
          if (k < q) T_part[(int64_t(s) * n_loc + jl) * q + k] = tk[k];
      }
    }
  }
  const double st = block_sum(stress, sh_a);
  const double zc = block_sum(zeros, sh_b);
  const unsigned int bid = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    parts[2 * bid] = st;
    parts[2 * bid + 1] = zc;
  }
  if (last_block_done(counter) && threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    const unsigned int nb = gridDim.x * gridDim.y;
    for (unsigned int k = 0; k < nb; ++k) {
      a += parts[2 * k];
      b += parts[2 * k + 1];
    }
    red[0] = a;
    red[1] = b;
  }
}

// columns per warp: keeps theta_j, the T partials and theta_i in registers
static constexpr int mds_jb(int qm, int esize) {
  // float32 with qm <= 32 runs the packed (column-pair) kernel: JB must be even
  return esize == 4 ? (qm <= 4 ? 8 : qm <= 32 ? 2 : 1)
                    : (qm <= 8 ? 4 : qm <= 16 ? 2 : 1);
}

static int mds_qm(int q) { return q <= 4 ? 4 : q <= 8 ? 8 : q <= 12 ? 12 : q <= 16 ? 16 : q <= 20 ? 20 : q <= 24 ? 24 : q <= 32 ? 32 : 64; }

struct MdsGrid {
  int colblocks, segs;
  int64_t rows_per_seg;
};

static MdsGrid mds_grid(int64_t n, int64_t n_loc, int q, int dtype) {
  const int jb = mds_jb(mds_qm(q), dtype == BS_F64 ? 8 : 4);
  MdsGrid g;
  g.colblocks = int(std::max<int64_t>(1, ceil_div(n_loc, int64_t(MDS_WARPS) * jb)));
  const int64_t want = int64_t(num_sms()) * 4;
  int64_t segs = std::max<int64_t>(1, ceil_div(want, g.colblocks));
  segs = std::min<int64_t>(segs, std::max<int64_t>(1, n / 256));
  segs = std::min<int64_t>(segs, 64);
  g.rows_per_seg = ceil_div(ceil_div(std::max<int64_t>(n, 1), segs), 128) * 128;
  g.segs = int(ceil_div(std::max<int64_t>(n, 1), g.rows_per_seg));
  return g;
}

namespace bs {
bool mds_tc_eligible(int dtype, int64_t n, int64_t n_loc, int q, int mode, const void* Y, const void* theta);
void note_gemm_path(int path);
int64_t mds_tc_workspace(int64_t n, int64_t n_loc, int q);
int mds_tc_pass(const float* Y, const float* theta, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                double* red, Workspace& ws, cudaStream_t st, double** zp_out, double** tp_out, int* segs_out);
}  // namespace bs

extern "C" int64_t bs_mds_pass_workspace(int dtype, int64_t n, int64_t n_loc, int q) {
  MdsGrid g = mds_grid(n, n_loc, q, dtype);
  const int64_t core = ws_bytes<unsigned int>(1) + ws_bytes<double>(2 * int64_t(g.colblocks) * g.segs) +
                       ws_bytes<double>(int64_t(g.segs) * n_loc) + ws_bytes<double>(int64_t(g.segs) * n_loc * q) +
                       ws_bytes<int64_t>(2) + ws_bytes<float>(n);
  // float32 passes may take the tcgen05 kernel (mds_tc.cu), which needs its own buffers
  const int64_t tcw = (dtype == BS_F32 && q <= 32 && n > 0 && n_loc > 0) ? mds_tc_workspace(n, n_loc, q) : 0;
  return std::max(core, tcw);
}

// ||theta_i||^2 for every row (float32 pass stages them with the theta chunk).
__global__ void mds_norms_kernel(const float* __restrict__ theta, int64_t n, int q, float* __restrict__ norms) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < q; ++k) s = fmaf(theta[i * q + k], theta[i * q + k], s);
    norms[i] = s;
  }
}

template <typename T, int QM>
static void launch_pass(const T* Y, const T* th, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                        int mode, const MdsGrid& g, double* zp, double* tp, double* parts, unsigned int* ctr,
                        double* red, cudaStream_t st, float* norms) {
  constexpr int JB = mds_jb(QM, int(sizeof(T)));
  dim3 grid(unsigned(g.colblocks), unsigned(g.segs));
  constexpr int VW = 16 / int(sizeof(T));
  constexpr int QS0 = (QM + VW - 1) / VW * VW;
  constexpr int QS = ((QS0 / VW) % 2 == 0) ? QS0 + VW : QS0;
  constexpr int CH = MdsChunk<T>::CH;
  const int smem = int(sizeof(T)) * (2 * CH * QS + 2 * MDS_WARPS * JB * CH + 2 * CH);
  if constexpr (sizeof(T) == 4 && QM <= 32) {
    mds_norms_kernel<<<int(std::min<int64_t>(ceil_div(n, 256), 1184)), 256, 0, st>>>(
        reinterpret_cast<const float*>(th), n, q, norms);
    smem_attr(mds_pass_f32x2_kernel<QM, JB>, smem);
    mds_pass_f32x2_kernel<QM, JB><<<grid, MDS_THREADS, smem, st>>>(
        reinterpret_cast<const float*>(Y), reinterpret_cast<const float*>(th), n, lo, n_loc, q, perturb, mode,
        g.rows_per_seg, zp, tp, parts, ctr, red, norms);
  } else {
    smem_attr(mds_pass_kernel<T, QM, JB>, smem);
    mds_pass_kernel<T, QM, JB><<<grid, MDS_THREADS, smem, st>>>(Y, th, n, lo, n_loc, q, perturb, mode,
                                                             g.rows_per_seg, zp, tp, parts, ctr, red);
  }
}

template <typename T>
static void dispatch_pass(const T* Y, const T* th, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                          int mode, const MdsGrid& g, double* zp, double* tp, double* parts,
                          unsigned int* ctr, double* red, cudaStream_t st, float* norms) {
  switch (mds_qm(q)) {
    case 4: launch_pass<T, 4>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 8: launch_pass<T, 8>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 12: launch_pass<T, 12>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 16: launch_pass<T, 16>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 20: launch_pass<T, 20>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 24: launch_pass<T, 24>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    case 32: launch_pass<T, 32>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
    default: launch_pass<T, 64>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms); break;
  }
}

// Folds the per-segment partials into zsum / T (storage type) for the update.
template <typename T>
__global__ void mds_fold_kernel(const double* __restrict__ zp, const double* __restrict__ tp, int segs,
                                int64_t n_loc, int q, T* __restrict__ zsum, T* __restrict__ Tout) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_loc * (q + 1);
       e += int64_t(gridDim.x) * blockDim.x) {
    if (e < n_loc) {
      double s = zp[e];
      for (int k = 1; k < segs; ++k) s += zp[int64_t(k) * n_loc + e];
      zsum[e] = T(s);
    } else {
      const int64_t f = e - n_loc;
      double s = tp[f];
      for (int k = 1; k < segs; ++k) s += tp[int64_t(k) * n_loc * q + f];
      Tout[f] = T(s);
    }
  }
}

extern "C" int bs_mds_pass(const void* Y, const void* theta_full, int dtype, int64_t n, int64_t lo,
                           int64_t n_loc, int q, int perturb, int mode, double* red, void* zsum, void* T,
                           void* work, int64_t work_bytes, void* stream) {
  clear_error();
  if (q < 1 || q > 64 || n < 0 || lo < 0 || n_loc < 0 || lo + n_loc > n || (mode != 0 && mode != 1)) {
    set_error("bs_mds_pass: bad arguments (q=%d, n=%lld, lo=%lld, n_loc=%lld)", q, (long long)n,
              (long long)lo, (long long)n_loc);
    return BS_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  if (n_loc == 0 || n == 0)
    return cudaMemsetAsync(red, 0, 2 * sizeof(double), st) == cudaSuccess ? BS_OK : BS_ECUDA;
  Workspace ws(work, work_bytes);
  if (mds_tc_eligible(dtype, n, n_loc, q, mode, Y, theta_full)) {
    double *zp = nullptr, *tp = nullptr;
    int segs = 0;
    int rc = mds_tc_pass(static_cast<const float*>(Y), static_cast<const float*>(theta_full), n, lo, n_loc, q, perturb,
                         red, ws, st, &zp, &tp, &segs);
    if (rc != BS_OK) return rc;
    const int fg = int(std::min<int64_t>(ceil_div(n_loc * (q + 1), 256), 2048));
    mds_fold_kernel<float><<<fg, 256, 0, st>>>(zp, tp, segs, n_loc, q, static_cast<float*>(zsum),
                                               static_cast<float*>(T));
    note_gemm_path(4);
    return check_launch("bs_mds_pass", 3);
  }
  note_gemm_path(5);
  MdsGrid g = mds_grid(n, n_loc, q, dtype);
  unsigned int* ctr = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(2 * int64_t(g.colblocks) * g.segs);
  double* zp = ws.take<double>(int64_t(g.segs) * n_loc);
  double* tp = ws.take<double>(int64_t(g.segs) * n_loc * q);
  float* norms = ws.take<float>(n);
  if (!ctr || !parts || !zp || !tp || !norms) {
    set_error("bs_mds_pass: workspace too small");
    return BS_EWORK;
  }
  const int fgrid = int(std::min<int64_t>(ceil_div(n_loc * (q + 1), 256), 2048));
  if (dtype == BS_F64) {
    dispatch_pass<double>(static_cast<const double*>(Y), static_cast<const double*>(theta_full), n, lo, n_loc,
                          q, perturb, mode, g, zp, tp, parts, ctr, red, st, norms);
    if (mode == 0)
      mds_fold_kernel<double><<<fgrid, 256, 0, st>>>(zp, tp, g.segs, n_loc, q, static_cast<double*>(zsum),
                                                     static_cast<double*>(T));
  } else if (dtype == BS_F32) {
    dispatch_pass<float>(static_cast<const float*>(Y), static_cast<const float*>(theta_full), n, lo, n_loc, q,
                         perturb, mode, g, zp, tp, parts, ctr, red, st, norms);
    if (mode == 0)
      mds_fold_kernel<float><<<fgrid, 256, 0, st>>>(zp, tp, g.segs, n_loc, q, static_cast<float*>(zsum),
                                                    static_cast<float*>(T));
  } else {
    set_error("bs_mds_pass: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  const int nk = (mode == 0 ? 2 : 1) + (dtype == BS_F32 && q <= 32 ? 1 : 0);
  return check_launch("bs_mds_pass", nk);
}

// theta <- (theta (zsum + wsum) + T) / (2 wsum)    (solvers.py:302-304)
template <typename T>
__global__ void mds_update_kernel(T* __restrict__ theta, const T* __restrict__ zsum, const T* __restrict__ Tm,
                                  int q, int64_t n_loc, double wsum, const double* __restrict__ red, int perturb,
                                  int* flags) {
  if (*flags & BS_FLAG_DEGENERATE) return;
  if (red[1] > 0.0 && !perturb) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, BS_FLAG_DEGENERATE);
    return;
  }
  const T ws = T(wsum), w2 = T(2.0 * wsum);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_loc * q;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / q;
    theta[e] = (theta[e] * (zsum[j] + ws) + Tm[e]) / w2;
  }
}

extern "C" int bs_mds_update(void* theta_loc, const void* zsum, const void* T, int dtype, int q, int64_t n_loc,
                             double wsum, const double* red, int perturb, int* flags, void* stream) {
  clear_error();
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_loc * q, 256), 2048)));
  cudaStream_t st = as_stream(stream);
  if (dtype == BS_F64)
    mds_update_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(theta_loc),
                                                    static_cast<const double*>(zsum), static_cast<const double*>(T),
                                                    q, n_loc, wsum, red, perturb, flags);
  else if (dtype == BS_F32)
    mds_update_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(theta_loc), static_cast<const float*>(zsum),
                                                   static_cast<const float*>(T), q, n_loc, wsum, red, perturb,
                                                   flags);
  else {
    set_error("bs_mds_update: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_mds_update");
}
