// pairwise_euclidean (distlinalg.py:442-468): Y[i, j] = ||x_i - x_j||_2 for the
// owned columns j of the n x n target, direct-difference formula like the
// reference (so Y is exactly symmetric and the diagonal exactly 0).  This is the
// one-time MDS setup (O(n^2 d)), not the per-iteration hot path.
//
// x: d x n gathered points, column-major (x[i*d + k]); Y local block n x n_loc.
#include "bsb200.cuh"

#include <algorithm>

using namespace bs;

constexpr int PW_TILE = 32;
constexpr int PW_K = 32;

template <typename T>
__global__ void __launch_bounds__(PW_TILE * 8)
pairwise_kernel(const T* __restrict__ x, int64_t d, int64_t n, int64_t lo, int64_t n_loc, T* __restrict__ Y) {
  __shared__ T xi[PW_K][PW_TILE + 1];
  __shared__ T xj[PW_K][PW_TILE + 1];
  const int tx = threadIdx.x & (PW_TILE - 1);  // row i within tile
  const int ty = threadIdx.x / PW_TILE;        // 0..7: columns ty, ty+8, ...
  const int64_t i0 = int64_t(blockIdx.x) * PW_TILE, j0 = int64_t(blockIdx.y) * PW_TILE;
  T acc[PW_TILE / 8];
#pragma unroll
  for (int c = 0; c < PW_TILE / 8; ++c) acc[c] = T(0);
  for (int64_t k0 = 0; k0 < d; k0 += PW_K) {
    __syncthreads();
    for (int e = threadIdx.x; e < PW_K * PW_TILE; e += blockDim.x) {
      const int kk = e % PW_K, p = e / PW_K;
      const int64_t k = k0 + kk;
      const int64_t i = i0 + p, j = j0 + p;
      xi[kk][p] = (k < d && i < n) ? x[i * d + k] : T(0);
      xj[kk][p] = (k < d && j < n_loc) ? x[(lo + j) * d + k] : T(0);
    }
    __syncthreads();
    const int kmax = int(d - k0 < PW_K ? d - k0 : PW_K);
    for (int kk = 0; kk < kmax; ++kk) {
      const T a = xi[kk][tx];
#pragma unroll
      for (int c = 0; c < PW_TILE / 8; ++c) {
        const T diff = xj[kk][ty + 8 * c] - a;  // x_j - x_i as in distlinalg.py:465
        acc[c] = fma(diff, diff, acc[c]);
      }
    }
  }
  const int64_t i = i0 + tx;
  if (i >= n) return;
#pragma unroll
  for (int c = 0; c < PW_TILE / 8; ++c) {
    const int64_t j = j0 + ty + 8 * c;
    if (j < n_loc) Y[j * n + i] = (i == lo + j) ? T(0) : sqrt(acc[c]);  // diag_fill(y, 0)
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
  dim3 grid(unsigned(ceil_div(n, PW_TILE)), unsigned(ceil_div(n_loc, PW_TILE)));
  cudaStream_t st = as_stream(stream);
  if (dtype == BS_F64)
    pairwise_kernel<double><<<grid, PW_TILE * 8, 0, st>>>(static_cast<const double*>(x), d, n, lo, n_loc,
                                                          static_cast<double*>(Y));
  else if (dtype == BS_F32)
    pairwise_kernel<float><<<grid, PW_TILE * 8, 0, st>>>(static_cast<const float*>(x), d, n, lo, n_loc,
                                                         static_cast<float*>(Y));
  else {
    set_error("bs_pairwise_euclidean: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_pairwise_euclidean");
}
