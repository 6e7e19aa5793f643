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

using namespace bs;

constexpr int MDS_THREADS = 256;
constexpr int MDS_WARPS = MDS_THREADS / 32;

// Pass kernel: each warp owns JB columns; lanes stride over the rows of the
// CTA's row segment.  Partials per row segment s:
//   zsum_part[s][jl], T_part[s][jl][k] (float64); stress/zero per CTA.
template <typename T, int QM, int JB>
__global__ void __launch_bounds__(MDS_THREADS)
mds_pass_kernel(const T* __restrict__ Y, const T* __restrict__ theta, int64_t n, int64_t lo,
                int64_t n_loc, int q, int perturb, int mode, int64_t rows_per_seg,
                double* __restrict__ zsum_part, double* __restrict__ T_part,
                double* __restrict__ parts, unsigned int* counter, double* __restrict__ red) {
  __shared__ double sh_a[32], sh_b[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t jl0 = (int64_t(blockIdx.x) * MDS_WARPS + wid) * JB;
  const int64_t i_begin = int64_t(blockIdx.y) * rows_per_seg;
  const int64_t i_end = min(n, i_begin + rows_per_seg);

  double tj[JB][QM], nj[JB], Tacc[JB][QM], zs[JB];
  bool live[JB];
#pragma unroll
  for (int c = 0; c < JB; ++c) {
    const int64_t jl = jl0 + c;
    live[c] = jl < n_loc;
    const int64_t jg = lo + (live[c] ? jl : 0);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < QM; ++k) {
      tj[c][k] = (k < q && live[c]) ? double(theta[jg * q + k]) : 0.0;
      s = fma(tj[c][k], tj[c][k], s);
      Tacc[c][k] = 0.0;
    }
    nj[c] = s;
    zs[c] = 0.0;
  }
  double stress = 0.0, zeros = 0.0;
  for (int64_t i = i_begin + lane; i < i_end; i += 32) {
    double ti[QM];
    double ni = 0.0;
#pragma unroll
    for (int k = 0; k < QM; ++k) {
      ti[k] = k < q ? double(theta[i * q + k]) : 0.0;
      ni = fma(ti[k], ti[k], ni);
    }
#pragma unroll
    for (int c = 0; c < JB; ++c) {
      if (!live[c]) continue;
      const int64_t jl = jl0 + c;
      const double y = double(Y[jl * n + i]);
      if (i == lo + jl) {  // diagonal: d_jj = 0 exactly (solvers.py:240-241), z_jj = y/inf = 0
        stress = fma(y, y, stress);
        continue;
      }
      double g = 0.0;
#pragma unroll
      for (int k = 0; k < QM; ++k) g = fma(ti[k], tj[c][k], g);
      // solvers.py:246: sqrt(max(dr + dc - 2g, 0)) evaluated in the storage type
      const T d2 = T(ni) + T(nj[c]) - T(2.0) * T(g);
      T d = sqrt(d2 > T(0) ? d2 : T(0));
      const double e = y - double(d);
      stress = fma(e, e, stress);
      if (d == T(0)) {
        zeros += 1.0;
        if (perturb) d = T(1e-10);  // solvers.py:296
      }
      if (mode == 0) {
        const T z = T(y) / d;  // solvers.py:297
        zs[c] += double(z);
        const double wz = double(T(1) - z);  // solvers.py:299
#pragma unroll
        for (int k = 0; k < QM; ++k) Tacc[c][k] = fma(ti[k], wz, Tacc[c][k]);
      }
    }
  }
  // per-warp column partials
  if (mode == 0) {
    const int s = blockIdx.y;
#pragma unroll
    for (int c = 0; c < JB; ++c) {
      const double zsum = warp_sum(zs[c]);
      double tk[QM];
#pragma unroll
      for (int k = 0; k < QM; ++k) tk[k] = warp_sum(Tacc[c][k]);
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

static int mds_qm(int q) { return q <= 4 ? 4 : q <= 8 ? 8 : q <= 16 ? 16 : q <= 24 ? 24 : q <= 32 ? 32 : 64; }

struct MdsGrid {
  int colblocks, segs;
  int64_t rows_per_seg;
};

static MdsGrid mds_grid(int64_t n, int64_t n_loc, int q) {
  const int jb = mds_qm(q) <= 16 ? 2 : 1;
  MdsGrid g;
  g.colblocks = int(std::max<int64_t>(1, ceil_div(n_loc, int64_t(MDS_WARPS) * jb)));
  const int64_t want = int64_t(num_sms()) * 4;
  int64_t segs = std::max<int64_t>(1, ceil_div(want, g.colblocks));
  segs = std::min<int64_t>(segs, std::max<int64_t>(1, n / 256));
  segs = std::min<int64_t>(segs, 64);
  g.rows_per_seg = ceil_div(std::max<int64_t>(n, 1), segs);
  g.segs = int(ceil_div(std::max<int64_t>(n, 1), g.rows_per_seg));
  return g;
}

extern "C" int64_t bs_mds_pass_workspace(int dtype, int64_t n, int64_t n_loc, int q) {
  (void)dtype;
  MdsGrid g = mds_grid(n, n_loc, q);
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(2 * int64_t(g.colblocks) * g.segs) +
         ws_bytes<double>(int64_t(g.segs) * n_loc) + ws_bytes<double>(int64_t(g.segs) * n_loc * q) +
         ws_bytes<int64_t>(2);
}

template <typename T, int QM>
static void launch_pass(const T* Y, const T* th, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                        int mode, const MdsGrid& g, double* zp, double* tp, double* parts, unsigned int* ctr,
                        double* red, cudaStream_t st) {
  constexpr int JB = QM <= 16 ? 2 : 1;
  dim3 grid(unsigned(g.colblocks), unsigned(g.segs));
  mds_pass_kernel<T, QM, JB><<<grid, MDS_THREADS, 0, st>>>(Y, th, n, lo, n_loc, q, perturb, mode,
                                                           g.rows_per_seg, zp, tp, parts, ctr, red);
}

template <typename T>
static void dispatch_pass(const T* Y, const T* th, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                          int mode, const MdsGrid& g, double* zp, double* tp, double* parts,
                          unsigned int* ctr, double* red, cudaStream_t st) {
  switch (mds_qm(q)) {
    case 4: launch_pass<T, 4>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
    case 8: launch_pass<T, 8>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
    case 16: launch_pass<T, 16>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
    case 24: launch_pass<T, 24>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
    case 32: launch_pass<T, 32>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
    default: launch_pass<T, 64>(Y, th, n, lo, n_loc, q, perturb, mode, g, zp, tp, parts, ctr, red, st); break;
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
  MdsGrid g = mds_grid(n, n_loc, q);
  unsigned int* ctr = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(2 * int64_t(g.colblocks) * g.segs);
  double* zp = ws.take<double>(int64_t(g.segs) * n_loc);
  double* tp = ws.take<double>(int64_t(g.segs) * n_loc * q);
  if (!ctr || !parts || !zp || !tp) {
    set_error("bs_mds_pass: workspace too small");
    return BS_EWORK;
  }
  const int fgrid = int(std::min<int64_t>(ceil_div(n_loc * (q + 1), 256), 2048));
  if (dtype == BS_F64) {
    dispatch_pass<double>(static_cast<const double*>(Y), static_cast<const double*>(theta_full), n, lo, n_loc,
                          q, perturb, mode, g, zp, tp, parts, ctr, red, st);
    if (mode == 0)
      mds_fold_kernel<double><<<fgrid, 256, 0, st>>>(zp, tp, g.segs, n_loc, q, static_cast<double*>(zsum),
                                                     static_cast<double*>(T));
  } else if (dtype == BS_F32) {
    dispatch_pass<float>(static_cast<const float*>(Y), static_cast<const float*>(theta_full), n, lo, n_loc, q,
                         perturb, mode, g, zp, tp, parts, ctr, red, st);
    if (mode == 0)
      mds_fold_kernel<float><<<fgrid, 256, 0, st>>>(zp, tp, g.segs, n_loc, q, static_cast<float*>(zsum),
                                                    static_cast<float*>(T));
  } else {
    set_error("bs_mds_pass: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_mds_pass", mode == 0 ? 2 : 1);
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
