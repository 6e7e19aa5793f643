// NMF hot path (solvers.py:73-185): the two skinny GEMMs over the streamed
// data block X and the fused factor half-steps.
//
//   scn b  P  = W_loc X_loc^T      (r x m)       distlinalg.py:246-252
//   scn a  C  = Vt_full X_loc      (r x n_loc)   distlinalg.py:239-243
//   half-step F <- update(F, NUM, GRAM), Gram(F_new), <NUM, F_new>
//                                                 solvers.py:150-159, 171-182
//
// Layouts (column-major blocks, distarray.py:82): X[j*m + i] (m x n_loc),
// factors F[c*r + k] (r x ncols).  GEMM partials use the factor layout.
//
// This file holds the CUDA-core GEMMs used for float64 data (FP64 has no
// tcgen05 kind) and as the reference implementation the tcgen05 3xTF32 path
// (nmf_tc.cu) is checked against.
#include "bsb200.cuh"

#include <algorithm>
#include <mutex>

using namespace bs;

namespace bs {
int launch_reduce(const void* x, int dtype, int64_t count, int op, int transform, double* out,
                  void* work, int64_t work_bytes, cudaStream_t st);
int launch_gram(const void* A, int dtype, int r, int64_t ncols, double* G, Workspace& ws,
                cudaStream_t st);
// tcgen05 path (nmf_tc.cu); returns BS_EINVAL when the shape is not supported.
int tc_wxt(const float* X, const float* W, int64_t m, int64_t n_loc, int r, float* P, Workspace& ws,
           cudaStream_t st, bool* used, double* stats);
int tc_vtx(const float* X, const float* Vt, int64_t m, int64_t n_loc, int r, float* C, int cap_slabs,
           int* splits, Workspace& ws, cudaStream_t st, bool* used);
int64_t tc_wxt_workspace(int64_t m, int64_t n_loc, int r);
int64_t tc_vtx_workspace(int64_t m, int64_t n_loc, int r);
// integer digit-slice tensor-core path (nmf_i8.cu)
int64_t i8_xscale_bytes(int64_t m, int64_t n_loc);
int64_t i8_prepare_workspace(int64_t m, int64_t n_loc);
int64_t i8_gemm_workspace(int64_t K);
int i8_prepare(const float* X, int64_t m, int64_t n_loc, double* stats, int8_t* xscale, Workspace& ws,
               cudaStream_t st);
int i8_wxt(const float* X, const float* W, int64_t m, int64_t n_loc, int r, const int8_t* xexp_b, float* P,
           Workspace& ws, cudaStream_t st, bool* used);
int i8_vtx(const float* X, const float* Vt, int64_t m, int64_t n_loc, int r, const int8_t* xexp_a, float* C,
           int cap_slabs, int* splits, Workspace& ws, cudaStream_t st, bool* used);
void note_gemm_path(int path);  // 0 i8 tensor, 1 tf32 tensor, 2 fp32 CUDA cores, 3 fp64 (DMMA / CUDA cores)
}  // namespace bs

static int64_t xgroups(int64_t k) { return (k + 511) / 512; }

constexpr int MAX_R = 128;

// ---------------------------------------------------------------------------
// _nmf_check + ||X||^2: min and sum of squares in one pass.
// ---------------------------------------------------------------------------

// float32 data: min and squares in fp32 over each 16-byte word (full-rate FMNMX / FFMA),
// then into float64; eight words in flight per thread.  NaN propagates like np.min.
__device__ __forceinline__ void scan_words_f32(const float* __restrict__ x, int64_t count, double& mn, double& sq) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  const int64_t mis = (reinterpret_cast<uintptr_t>(x) & 15) / 4;
  const int64_t head = mis ? (count < 4 - mis ? count : 4 - mis) : 0;
  bool nan = false;
  float fmn = CUDART_INF_F;
  auto one = [&](float v) {
    nan |= (v != v);
    fmn = fminf(fmn, v);
    sq = fma(double(v), double(v), sq);
  };
  for (int64_t i = tid; i < head; i += nth) one(x[i]);
  const float4* xv = reinterpret_cast<const float4*>(x + head);
  const int64_t nvec = (count - head) / 4;
  int64_t v = tid;
  for (; v + 7 * nth < nvec; v += 8 * nth) {
    float4 w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = ld_stream(xv + v + u * nth);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      nan |= (w[u].x != w[u].x) | (w[u].y != w[u].y) | (w[u].z != w[u].z) | (w[u].w != w[u].w);
      fmn = fminf(fmn, fminf(fminf(w[u].x, w[u].y), fminf(w[u].z, w[u].w)));
      s0 = fmaf(w[u].x, w[u].x, s0);
      s1 = fmaf(w[u].y, w[u].y, s1);
      s0 = fmaf(w[u].z, w[u].z, s0);
      s1 = fmaf(w[u].w, w[u].w, s1);
    }
    sq += double(s0) + double(s1);
  }
  for (; v < nvec; v += nth) {
    const float4 w = ld_stream(xv + v);
    one(w.x); one(w.y); one(w.z); one(w.w);
  }
  for (int64_t i = head + nvec * 4 + tid; i < count; i += nth) one(x[i]);
  mn = nan ? CUDART_NAN : rop_apply(BS_MIN, mn, double(fmn));
}

template <typename T>
__global__ void __launch_bounds__(256)
scan_kernel(const T* __restrict__ x, int64_t count, double* __restrict__ parts,
            unsigned int* counter, double* out) {
  __shared__ double shm[32], shs[32];
  double mn = CUDART_INF, sq = 0.0;
  if constexpr (sizeof(T) == 4) {
    scan_words_f32(reinterpret_cast<const float*>(x), count, mn, sq);
  } else {
    stream_elems(x, count, [&](double v) {
      mn = rop_apply(BS_MIN, mn, v);
      sq = fma(v, v, sq);
    });
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = rop_apply(BS_MIN, mn, __shfl_xor_sync(0xffffffffu, mn, o));
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
  }
  if (lane == 0) {
    shm[wid] = mn;
    shs[wid] = sq;
  }
  __syncthreads();
  if (wid == 0) {
    double a = lane < (blockDim.x >> 5) ? shm[lane] : CUDART_INF;
    double b = lane < (blockDim.x >> 5) ? shs[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = rop_apply(BS_MIN, a, __shfl_xor_sync(0xffffffffu, a, o));
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      parts[2 * blockIdx.x] = a;
      parts[2 * blockIdx.x + 1] = b;
    }
  }
  if (last_block_done(counter) && threadIdx.x == 0) {
    double a = parts[0], b = parts[1];
    for (unsigned int k = 1; k < gridDim.x; ++k) {
      a = rop_apply(BS_MIN, a, parts[2 * k]);
      b += parts[2 * k + 1];
    }
    out[0] = a;
    out[1] = b;
  }
}

extern "C" int bs_nmf_scan(const void* X, int dtype, int64_t count, double* out_dev, void* work,
                           int64_t work_bytes, void* stream) {
  clear_error();
  Workspace ws(work, work_bytes);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 2048), int64_t(num_sms()) * 4)));
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(2 * grid);
  if (!counter || !parts) {
    set_error("bs_nmf_scan: workspace too small");
    return BS_EWORK;
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == BS_F64)
    scan_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(X), count, parts, counter, out_dev);
  else if (dtype == BS_F32)
    scan_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(X), count, parts, counter, out_dev);
  else {
    set_error("bs_nmf_scan: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_nmf_scan");
}

// ---------------------------------------------------------------------------
// CUDA-core skinny GEMMs.  Accumulation in T (fp32 / fp64).
// ---------------------------------------------------------------------------

template <typename T> struct GemmCfg;
template <> struct GemmCfg<float> { static constexpr int BK = 32; };
template <> struct GemmCfg<double> { static constexpr int BK = 16; };

// scn b: P[i][k] = sum_j X[j][i] W[j][k] over j in the split's column range.
// Tile: 128 rows i x RP columns k; 256 threads as 16 (ty: 8 rows) x 16 (tx: RP/16 cols).
template <typename T, int RP>
__global__ void __launch_bounds__(256)
gemm_wxt_kernel(const T* __restrict__ X, const T* __restrict__ W, int64_t m, int64_t n_loc, int r,
                int64_t cols_per_split, T* __restrict__ P) {
  constexpr int BM = 128, BK = GemmCfg<T>::BK, TM = 8, TN = RP / 16;
  __shared__ T Xs[BK][BM];
  __shared__ T Ws[BK][RP];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = T(0);

  for (int64_t j0 = j_begin; j0 < j_end; j0 += BK) {
    __syncthreads();
    for (int e = tid; e < BK * BM; e += 256) {
      const int jj = e / BM, ii = e % BM;
      const int64_t j = j0 + jj, i = i0 + ii;
      Xs[jj][ii] = (j < j_end && i < m) ? X[j * m + i] : T(0);
    }
    for (int e = tid; e < BK * RP; e += 256) {
      const int jj = e / RP, k = e % RP;
      const int64_t j = j0 + jj;
      Ws[jj][k] = (j < j_end && k < r) ? W[j * r + k] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int t = 0; t < TM; ++t) a[t] = Xs[kk][ty * TM + t];
#pragma unroll
      for (int t = 0; t < TN; ++t) b[t] = Ws[kk][tx + 16 * t];
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
  T* out = P + int64_t(blockIdx.y) * m * r;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int64_t i = i0 + ty * TM + u;
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < TN; ++v) {
      const int k = tx + 16 * v;
      if (k < r) out[i * r + k] = acc[u][v];
    }
  }
}

// scn a: C[j][k] = sum_i X[j][i] Vt[i][k] over i in the split's row range.
// Tile: 64 columns j x RP; 256 threads as 16 (ty: 4 columns) x 16 (tx: RP/16).
template <typename T, int RP>
__global__ void __launch_bounds__(256)
gemm_vtx_kernel(const T* __restrict__ X, const T* __restrict__ Vt, int64_t m, int64_t n_loc, int r,
                int64_t rows_per_split, T* __restrict__ C) {
  constexpr int BN = 64, BK = GemmCfg<T>::BK, TM = 4, TN = RP / 16;
  __shared__ T Xs[BK][BN + 1];
  __shared__ T Vs[BK][RP];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t jb = int64_t(blockIdx.x) * BN;
  const int64_t i_begin = int64_t(blockIdx.y) * rows_per_split;
  const int64_t i_end = min(m, i_begin + rows_per_split);
  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = T(0);

  for (int64_t i0 = i_begin; i0 < i_end; i0 += BK) {
    __syncthreads();
    for (int e = tid; e < BK * BN; e += 256) {
      const int jj = e / BK, ii = e % BK;
      const int64_t j = jb + jj, i = i0 + ii;
      Xs[ii][jj] = (j < n_loc && i < i_end) ? X[j * m + i] : T(0);
    }
    for (int e = tid; e < BK * RP; e += 256) {
      const int ii = e / RP, k = e % RP;
      const int64_t i = i0 + ii;
      Vs[ii][k] = (i < i_end && k < r) ? Vt[i * r + k] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int t = 0; t < TM; ++t) a[t] = Xs[kk][ty * TM + t];
#pragma unroll
      for (int t = 0; t < TN; ++t) b[t] = Vs[kk][tx + 16 * t];
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
  T* out = C + int64_t(blockIdx.y) * n_loc * r;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int64_t j = jb + ty * TM + u;
    if (j >= n_loc) continue;
#pragma unroll
    for (int v = 0; v < TN; ++v) {
      const int k = tx + 16 * v;
      if (k < r) out[j * r + k] = acc[u][v];
    }
  }
}

// Sums S partial slabs [S][len] in order into dst[len].
template <typename T>
__global__ void sum_slabs_kernel(const T* __restrict__ parts, int S, int64_t len, T* __restrict__ dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < len;
       e += int64_t(gridDim.x) * blockDim.x) {
    T acc = parts[e];
    for (int s = 1; s < S; ++s) acc += parts[int64_t(s) * len + e];
    dst[e] = acc;
  }
}

__global__ void fold_minsq_kernel(const double* __restrict__ parts, int np, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double a = parts[0], b = parts[1];
    for (int k = 1; k < np; ++k) {
      a = rop_apply(BS_MIN, a, parts[2 * k]);
      b += parts[2 * k + 1];
    }
    out[0] = a;
    out[1] = b;
  }
}

namespace bs {
void launch_fold_minsq(const double* parts, int np, double* out, cudaStream_t st) {
  fold_minsq_kernel<<<1, 32, 0, st>>>(parts, np, out);
}

void launch_sum_slabs_f32(const float* parts, int S, int64_t len, float* dst, cudaStream_t st) {
  sum_slabs_kernel<float><<<int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(len, 256), 4096))), 256, 0, st>>>(
      parts, S, len, dst);
}
}  // namespace bs

static int pick_rp(int r) { return r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 128; }

// Split count so that the grid covers >= ~4 CTAs per SM, each split keeping >= min_k of K.
static int pick_splits(int64_t tiles, int64_t K, int64_t min_k) {
  const int64_t want = int64_t(num_sms()) * 4;
  int64_t s = std::max<int64_t>(1, ceil_div(want, std::max<int64_t>(tiles, 1)));
  s = std::min<int64_t>(s, std::max<int64_t>(1, K / min_k));
  return int(std::min<int64_t>(s, 64));
}

// ---------------------------------------------------------------------------
// Register-tiled CUDA-core GEMM used for float64 (no tcgen05 kind exists) and for
// shapes the tcgen05 path does not take.  One CTA of 128 threads computes a
// 128 x RP output tile (M rows x r padded): thread (tx, ty) owns TM = 8 rows x
// TN = RP/8 columns, so every k step costs TM + TN operand loads (16-byte shared
// loads) for TM*TN FMAs.  Tiles are double-buffered through registers.
//   A_MN = true : scn b, A = X with M = i contiguous (tile rows kk are contiguous)
//   A_MN = false: scn a, A = X with K = i contiguous (one X column per thread row)
// ---------------------------------------------------------------------------

// k-tile depth: keeps both double buffers under the 48 KB static shared limit
template <typename T, int RP> struct CcCfg {
  static constexpr int BK = sizeof(T) == 8 ? (RP >= 64 ? 8 : 16) : (RP >= 64 ? 16 : 32);
};

template <typename T, int RP, bool A_MN>
__global__ void __launch_bounds__(128)
cc_gemm_kernel(const T* __restrict__ X, const T* __restrict__ B, int64_t M, int64_t ldx, int r,
               int64_t K, int64_t k_per_split, T* __restrict__ out) {
  constexpr int BM = 128, BK = CcCfg<T, RP>::BK, TM = 8, TN = RP / 8, V = 16 / int(sizeof(T));
  constexpr int PAD = V;  // keeps 16-byte alignment of the rows
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][RP];
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t k_begin = int64_t(blockIdx.y) * k_per_split;
  const int64_t k_end = min(K, k_begin + k_per_split);
  // register staging of one tile
  constexpr int A_PER = BM * BK / 128;          // elements per thread
  constexpr int B_PER = (BK * RP + 127) / 128;
  T ra[A_PER], rb[B_PER];
  const bool vec_ok = (ldx % V) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  auto load_tile = [&](int64_t k0) {
    if constexpr (A_MN) {
      // rows kk of the tile are X[(k0+kk)*ldx + m0 .. +BM): V-wide vector loads
#pragma unroll
      for (int u = 0; u < A_PER / V; ++u) {
        const int e = tid + 128 * u;  // vector index
        const int kk = e / (BM / V), mv = (e % (BM / V)) * V;
        const int64_t k = k0 + kk, mrow = m0 + mv;
        if (vec_ok && k < k_end && mrow + V <= M) {
          if constexpr (sizeof(T) == 8) {
            const double2 w = *reinterpret_cast<const double2*>(X + k * ldx + mrow);
            ra[u * V] = w.x; ra[u * V + 1] = w.y;
          } else {
            const float4 w = *reinterpret_cast<const float4*>(X + k * ldx + mrow);
            ra[u * V] = w.x; ra[u * V + 1] = w.y; ra[u * V + 2] = w.z; ra[u * V + 3] = w.w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) ra[u * V + v] = (k < k_end && mrow + v < M) ? X[k * ldx + mrow + v] : T(0);
        }
      }
    } else {
      // thread tid owns tile row m0+tid: X[(m0+tid)*ldx + k0 .. +BK)
      const int64_t mrow = m0 + tid;
      const T* src = X + mrow * ldx + k0;
      if (mrow < M && k0 + A_PER <= k_end && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int u = 0; u < A_PER; u += V) {
          if constexpr (sizeof(T) == 8) {
            const double2 w = *reinterpret_cast<const double2*>(src + u);
            ra[u] = w.x; ra[u + 1] = w.y;
          } else {
            const float4 w = *reinterpret_cast<const float4*>(src + u);
            ra[u] = w.x; ra[u + 1] = w.y; ra[u + 2] = w.z; ra[u + 3] = w.w;
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < A_PER; ++kk) {
          const int64_t k = k0 + kk;
          ra[kk] = (mrow < M && k < k_end) ? X[mrow * ldx + k] : T(0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < B_PER; ++u) {
      const int e = tid + 128 * u;
      const int kk = e / RP, c = e % RP;
      const int64_t k = k0 + kk;
      rb[u] = (e < BK * RP && k < k_end && c < r) ? B[k * r + c] : T(0);
    }
  };
  auto store_tile = [&](int buf) {
    if constexpr (A_MN) {
#pragma unroll
      for (int u = 0; u < A_PER / V; ++u) {
        const int e = tid + 128 * u;
        const int kk = e / (BM / V), mv = (e % (BM / V)) * V;
#pragma unroll
        for (int v = 0; v < V; ++v) As[buf][kk][mv + v] = ra[u * V + v];
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < A_PER; ++kk) As[buf][kk][tid] = ra[kk];
    }
#pragma unroll
    for (int u = 0; u < B_PER; ++u) {
      const int e = tid + 128 * u;
      if (e < BK * RP) Bs[buf][e / RP][e % RP] = rb[u];
    }
  };
  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = T(0);
  if (k_begin < k_end) {
    load_tile(k_begin);
    store_tile(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = k_begin; k0 < k_end; k0 += BK) {
      const bool more = k0 + BK < k_end;
      if (more) load_tile(k0 + BK);  // in flight while this tile is consumed
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T a[TM], b[TN];
#pragma unroll
        for (int t = 0; t < TM; t += V) {
          if constexpr (sizeof(T) == 8) {
            const double2 w = *reinterpret_cast<const double2*>(&As[buf][kk][ty * TM + t]);
            a[t] = w.x; a[t + 1] = w.y;
          } else {
            const float4 w = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + t]);
            a[t] = w.x; a[t + 1] = w.y; a[t + 2] = w.z; a[t + 3] = w.w;
          }
        }
#pragma unroll
        for (int t = 0; t < TN; ++t) b[t] = Bs[buf][kk][tx * TN + t];
#pragma unroll
        for (int u = 0; u < TM; ++u)
#pragma unroll
          for (int v = 0; v < TN; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
      if (more) {
        store_tile(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  T* dst = out + int64_t(blockIdx.y) * M * r;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int64_t row = m0 + ty * TM + u;
    if (row >= M) continue;
#pragma unroll
    for (int v = 0; v < TN; ++v) {
      const int c = tx * TN + v;
      if (c < r) dst[row * r + c] = acc[u][v];
    }
  }
}

// ---------------------------------------------------------------------------
// float64: the same 128 x RP tile on the FP64 tensor cores (mma.sync m8n8k4 DMMA).
// Staging as in cc_gemm_kernel (register double buffering into As[k][m] / Bs[k][c]);
// warp w owns rows 32w..32w+31 as 4 x (RP/8) 8x8 accumulator fragments.  Per 4-wide k
// step a warp loads 4 A and RP/8 B fragments (one double per lane each) for 4 RP/8
// DMMAs (256 FMAs each).  Row strides are padded to 64 B mod 128 so the 4 k rows a
// fragment load touches fall in disjoint bank halves.  Every product and sum is an
// IEEE float64 FMA, like the CUDA-core kernel (only the summation order differs).
// ---------------------------------------------------------------------------

template <int RP, bool A_MN, int BKO = 0>
struct DmmaCfg {
  // B row stride RP + PB must be 8 doubles mod 16 (64 B mod 128), or the 4 k rows a
  // fragment load touches share banks: RP = 8 / 24 pad by 0, the others by 8.  BK: 8 for
  // RP = 64 in the register-staged kernel (staging registers), else 16 (BKO overrides).
  static constexpr int BM = 128, BK = BKO ? BKO : (RP >= 64 ? 8 : 16), PB = RP % 16 == 8 ? 0 : 8;
  // A tile: [k][m] (m contiguous) for scn b; [m][k] (k contiguous, +4 pad) for scn a
  static constexpr int A_ELEMS = A_MN ? BK * (BM + 8) : BM * (BK + 4);
  static constexpr int B_ELEMS = BK * (RP + PB);
  static constexpr int SMEM = 2 * (A_ELEMS + B_ELEMS) * 8;
};

template <int RP, bool A_MN>
__global__ void __launch_bounds__(128)
dmma_gemm_kernel(const double* __restrict__ X, const double* __restrict__ B, int64_t M, int64_t ldx, int r,
                 int64_t K, int64_t k_per_split, double* __restrict__ out) {
  using C = DmmaCfg<RP, A_MN>;
  constexpr int BM = C::BM, BK = C::BK, V = 2, NF = RP / 8, PB = C::PB;
  constexpr int SA = A_MN ? BM + 8 : BK + 4;  // row stride of the A tile (doubles)
  extern __shared__ __align__(16) double dm_smem[];
  double* As = dm_smem;                  // [2][A_ELEMS]
  double* Bs = dm_smem + 2 * C::A_ELEMS;  // [2][BK][RP + PB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t k_begin = int64_t(blockIdx.y) * k_per_split;
  const int64_t k_end = min(K, k_begin + k_per_split);
  constexpr int A_PER = BM * BK / 128;
  constexpr int B_PER = (BK * RP + 127) / 128;
  double ra[A_PER], rb[B_PER];
  const bool vec_ok = (ldx % V) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  // A_MN: vector e covers m [mv, mv+2) of k row kk.  !A_MN: BK/2 threads per m row, vector e
  // covers k [2c, 2c+2) of row (e / (BK/2)) -- consecutive threads read consecutive 16 bytes.
  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < A_PER / V; ++u) {
      const int e = tid + 128 * u;
      if constexpr (A_MN) {
        const int kk = e / (BM / V), mv = (e % (BM / V)) * V;
        const int64_t k = k0 + kk, mrow = m0 + mv;
        if (vec_ok && k < k_end && mrow + V <= M) {
          const double2 w = *reinterpret_cast<const double2*>(X + k * ldx + mrow);
          ra[u * V] = w.x; ra[u * V + 1] = w.y;
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) ra[u * V + v] = (k < k_end && mrow + v < M) ? X[k * ldx + mrow + v] : 0.0;
        }
      } else {
        const int row = e / (BK / V), c = e % (BK / V);
        const int64_t mrow = m0 + row, k = k0 + V * c;
        if (vec_ok && mrow < M && k + V <= k_end) {
          const double2 w = *reinterpret_cast<const double2*>(X + mrow * ldx + k);
          ra[u * V] = w.x; ra[u * V + 1] = w.y;
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) ra[u * V + v] = (mrow < M && k + v < k_end) ? X[mrow * ldx + k + v] : 0.0;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < B_PER; ++u) {
      const int e = tid + 128 * u;
      const int kk = e / RP, c = e % RP;
      const int64_t k = k0 + kk;
      rb[u] = (e < BK * RP && k < k_end && c < r) ? B[k * r + c] : 0.0;
    }
  };
  auto store_tile = [&](int buf) {
    double* at = As + buf * C::A_ELEMS;
#pragma unroll
    for (int u = 0; u < A_PER / V; ++u) {
      const int e = tid + 128 * u;
      if constexpr (A_MN) {
        const int kk = e / (BM / V), mv = (e % (BM / V)) * V;
        *reinterpret_cast<double2*>(at + kk * SA + mv) = make_double2(ra[u * V], ra[u * V + 1]);
      } else {
        const int row = e / (BK / V), c = e % (BK / V);
        *reinterpret_cast<double2*>(at + row * SA + V * c) = make_double2(ra[u * V], ra[u * V + 1]);
      }
    }
    double* bt = Bs + buf * C::B_ELEMS;
#pragma unroll
    for (int u = 0; u < B_PER; ++u) {
      const int e = tid + 128 * u;
      if (e < BK * RP) bt[(e / RP) * (RP + PB) + e % RP] = rb[u];
    }
  };
  double acc[4][NF][2];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int g = 0; g < NF; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k of this lane
  if (k_begin < k_end) {
    load_tile(k_begin);
    store_tile(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = k_begin; k0 < k_end; k0 += BK) {
      const bool more = k0 + BK < k_end;
      if (more) load_tile(k0 + BK);  // in flight while this tile is consumed
      const double* at = As + buf * C::A_ELEMS;
      const double* bt = Bs + buf * C::B_ELEMS;
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double a[4], b[NF];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int row = 32 * warp + 8 * f + fr;
          a[f] = A_MN ? at[(ks + fk) * SA + row] : at[row * SA + ks + fk];
        }
#pragma unroll
        for (int g = 0; g < NF; ++g) b[g] = bt[(ks + fk) * (RP + PB) + 8 * g + fr];
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int g = 0; g < NF; ++g)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[f][g][0]), "+d"(acc[f][g][1])
                : "d"(a[f]), "d"(b[g]));
      }
      if (more) {
        store_tile(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  double* dst = out + int64_t(blockIdx.y) * M * r;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t row = m0 + 32 * warp + 8 * f + fr;
    if (row >= M) continue;
#pragma unroll
    for (int g = 0; g < NF; ++g) {
      const int c = 8 * g + 2 * fk;
      if (c < r) dst[row * r + c] = acc[f][g][0];
      if (c + 1 < r) dst[row * r + c + 1] = acc[f][g][1];
    }
  }
}

// The same tile, fragment mapping and k order as dmma_gemm_kernel (so the sums are
// bitwise identical), but X and B move global -> shared with cp.async through NS
// stages instead of a register double buffer: no staging registers, and NS-1 tiles in
// flight per CTA instead of one.  C1 (10k x 10k, r = 20) was latency-bound at 3 CTAs per
// SM with 16 KB in flight each (profiles/r01_launches_nmf_mu_c1.txt).  Needs 16-byte
// aligned X rows (even ldx); partial chunks at the M / k_end edges zero-fill through the
// cp.async src-size operand.
template <int RP, bool A_MN, int NS>
struct DmmaAsyncCfg {
  using B = DmmaCfg<RP, A_MN, 16>;  // no staging registers: BK = 16 for every RP
  static constexpr int STAGE = B::A_ELEMS + B::B_ELEMS;  // doubles per stage
  static constexpr int SMEM = NS * STAGE * 8;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}

// K16: the tile's products as mma.sync m16n8k16 (a warp's 32 rows as two 16-row fragments)
// instead of m8n8k4.  ptxas lowers it to 16 DMMA.8x8x4 (profiles/r02_sass_tensor_excerpt.txt),
// so the tensor work and the bits are those of the m8n8k4 kernels (tests/test_nmf_gpu.py,
// register vs cp.async pipeline); what it saves is fragment loads and PTX-level overhead.
// K16 also serves RP = 48 / 64 (one B fragment live at a time; 234 registers, 2 CTAs per SM).
template <int RP, bool A_MN, int NS, bool K16 = false>
__global__ void __launch_bounds__(128)
dmma_async_kernel(const double* __restrict__ X, const double* __restrict__ B, int64_t M, int64_t ldx, int r,
                  int64_t K, int64_t k_per_split, double* __restrict__ out) {
  using C = DmmaCfg<RP, A_MN, 16>;
  using CA = DmmaAsyncCfg<RP, A_MN, NS>;
  constexpr int BM = C::BM, BK = C::BK, V = 2, NF = RP / 8, PB = C::PB;
  constexpr int SA = A_MN ? BM + 8 : BK + 4;
  extern __shared__ __align__(16) double dm_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t k_begin = int64_t(blockIdx.y) * k_per_split;
  const int64_t k_end = min(K, k_begin + k_per_split);
  constexpr int A_CH = BM * BK / V / 128;  // 16-byte chunks per thread
  constexpr int B_PER = (BK * RP + 127) / 128;
  auto issue = [&](int64_t k0, int stage) {
    double* at = dm_smem + stage * CA::STAGE;
    double* bt = at + C::A_ELEMS;
#pragma unroll
    for (int u = 0; u < A_CH; ++u) {
      const int e = tid + 128 * u;
      if constexpr (A_MN) {
        const int kk = e / (BM / V), mv = (e % (BM / V)) * V;
        const int64_t k = k0 + kk, mrow = m0 + mv;
        const int64_t left = M - mrow;
        const int valid = k < k_end && left > 0 ? (left < V ? int(left) : V) : 0;
        const double* src = valid ? X + k * ldx + mrow : X;
        cp_async16(at + kk * SA + mv, src, valid * 8);
      } else {
        const int row = e / (BK / V), c = e % (BK / V);
        const int64_t mrow = m0 + row, k = k0 + V * c;
        const int64_t left = k_end - k;
        const int valid = mrow < M && left > 0 ? (left < V ? int(left) : V) : 0;
        const double* src = valid ? X + mrow * ldx + k : X;
        cp_async16(at + row * SA + V * c, src, valid * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < B_PER; ++u) {
      const int e = tid + 128 * u;
      if (e < BK * RP) {
        const int kk = e / RP, c = e % RP;
        const int64_t k = k0 + kk;
        const bool ok = k < k_end && c < r;
        cp_async8(bt + kk * (RP + PB) + c, ok ? B + k * r + c : B, ok ? 8 : 0);
      }
    }
  };
  static_assert(!K16 || BK % 16 == 0, "m16n8k16 steps need BK % 16 == 0");
  double acc[4][NF][2];  // m8n8k4: fragment f = rows 8f.., m16n8k16: [2 mf + h] = rows 16 mf + 8 h ..
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int g = 0; g < NF; ++g) acc[f][g][0] = acc[f][g][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t ntiles = k_begin < k_end ? (k_end - k_begin + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < ntiles) issue(k_begin + int64_t(s) * BK, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t t = 0; t < ntiles; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    __syncthreads();  // tile t landed for every thread; stage (t-1) % NS is free
    const int64_t tn = t + NS - 1;
    if (tn < ntiles) issue(k_begin + tn * BK, int(tn % NS));
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* at = dm_smem + int(t % NS) * CA::STAGE;
    const double* bt = at + C::A_ELEMS;
    if constexpr (K16) {
      auto A_at = [&](int row, int k) { return A_MN ? at[k * SA + row] : at[row * SA + k]; };
#pragma unroll
      for (int ks = 0; ks < BK; ks += 16) {
        double a[2][8];  // the warp's two 16-row fragments, loaded once per k step
#pragma unroll
        for (int mf = 0; mf < 2; ++mf) {
          const int row = 32 * warp + 16 * mf + fr;
#pragma unroll
          for (int i = 0; i < 8; ++i) a[mf][i] = A_at(row + 8 * (i & 1), ks + fk + 4 * (i >> 1));
        }
#pragma unroll
        for (int g = 0; g < NF; ++g) {  // one n fragment of B at a time (RP = 64: 8 of them)
          double b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) b[i] = bt[(ks + fk + 4 * i) * (RP + PB) + 8 * g + fr];
#pragma unroll
          for (int mf = 0; mf < 2; ++mf)
            asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                : "+d"(acc[2 * mf][g][0]), "+d"(acc[2 * mf][g][1]), "+d"(acc[2 * mf + 1][g][0]),
                  "+d"(acc[2 * mf + 1][g][1])
                : "d"(a[mf][0]), "d"(a[mf][1]), "d"(a[mf][2]), "d"(a[mf][3]), "d"(a[mf][4]), "d"(a[mf][5]),
                  "d"(a[mf][6]), "d"(a[mf][7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
      }
    } else {
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[4], b[NF];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const int row = 32 * warp + 8 * f + fr;
        a[f] = A_MN ? at[(ks + fk) * SA + row] : at[row * SA + ks + fk];
      }
#pragma unroll
      for (int g = 0; g < NF; ++g) b[g] = bt[(ks + fk) * (RP + PB) + 8 * g + fr];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int g = 0; g < NF; ++g)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[f][g][0]), "+d"(acc[f][g][1])
              : "d"(a[f]), "d"(b[g]));
    }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  double* dst = out + int64_t(blockIdx.y) * M * r;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t row = m0 + 32 * warp + 8 * f + fr;
    if (row >= M) continue;
#pragma unroll
    for (int g = 0; g < NF; ++g) {
      const int c = 8 * g + 2 * fk;
      if (c < r) dst[row * r + c] = acc[f][g][0];
      if (c + 1 < r) dst[row * r + c + 1] = acc[f][g][1];
    }
  }
}

static bool dmma_k16() {  // BS_DMMA_K16=0 keeps the m8n8k4 instruction (A/B switch)
  static const bool on = [] {
    const char* e = getenv("BS_DMMA_K16");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int dmma_stages() {
  // BS_DMMA_STAGES=0 selects the register double-buffered kernel (A/B switch)
  static const int ns = [] {
    const char* s = getenv("BS_DMMA_STAGES");
    const int v = s ? atoi(s) : 2;
    return (v == 0 || v == 2 || v == 3 || v == 4) ? v : 2;
  }();
  return ns;
}

template <bool A_MN>
static bool launch_dmma(const double* X, const double* B, int64_t M, int64_t ldx, int r, int64_t K, int64_t kps,
                        dim3 grid, double* out, cudaStream_t st) {
  static const bool disabled = getenv("BS_DISABLE_DMMA") != nullptr;  // A/B switch for benchmarks
  if (disabled) return false;
  const int ns = dmma_stages();
  const bool async_ok = ns != 0 && (ldx % 2) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(B) & 7) == 0 && (A_MN || kps % 2 == 0);
  if (async_ok && dmma_k16() && r > 32 && r <= 64) {  // RP 48 / 64: the m16n8k16 form only
    const int rpw = r <= 48 ? 48 : 64;
    if (rpw == 48) {
      smem_attr(dmma_async_kernel<48, A_MN, 2, true>, DmmaAsyncCfg<48, A_MN, 2>::SMEM);
      dmma_async_kernel<48, A_MN, 2, true><<<grid, 128, DmmaAsyncCfg<48, A_MN, 2>::SMEM, st>>>(X, B, M, ldx, r, K, kps, out);
    } else {
      smem_attr(dmma_async_kernel<64, A_MN, 2, true>, DmmaAsyncCfg<64, A_MN, 2>::SMEM);
      dmma_async_kernel<64, A_MN, 2, true><<<grid, 128, DmmaAsyncCfg<64, A_MN, 2>::SMEM, st>>>(X, B, M, ldx, r, K, kps, out);
    }
    return true;
  }
  if (async_ok && r <= 32) {
    const int rpa = r <= 8 ? 8 : r <= 16 ? 16 : r <= 24 ? 24 : 32;
#define BS_DMMA_A(RPV, NSV)                                                                                    \
  {                                                                                                            \
    if (dmma_k16()) {                                                                                          \
      smem_attr(dmma_async_kernel<RPV, A_MN, NSV, true>, DmmaAsyncCfg<RPV, A_MN, NSV>::SMEM);                \
      dmma_async_kernel<RPV, A_MN, NSV, true>                                                                  \
          <<<grid, 128, DmmaAsyncCfg<RPV, A_MN, NSV>::SMEM, st>>>(X, B, M, ldx, r, K, kps, out);             \
      return true;                                                                                             \
    }                                                                                                          \
    smem_attr(dmma_async_kernel<RPV, A_MN, NSV>, DmmaAsyncCfg<RPV, A_MN, NSV>::SMEM);                        \
    dmma_async_kernel<RPV, A_MN, NSV>                                                                          \
        <<<grid, 128, DmmaAsyncCfg<RPV, A_MN, NSV>::SMEM, st>>>(X, B, M, ldx, r, K, kps, out);               \
    return true;                                                                                               \
  }
    if (ns == 2) {
      switch (rpa) {
        case 8: BS_DMMA_A(8, 2)
        case 16: BS_DMMA_A(16, 2)
        case 24: BS_DMMA_A(24, 2)
        default: BS_DMMA_A(32, 2)
      }
    }
    if (ns == 4) {
      switch (rpa) {
        case 8: BS_DMMA_A(8, 4)
        case 16: BS_DMMA_A(16, 4)
        case 24: BS_DMMA_A(24, 4)
        default: BS_DMMA_A(32, 4)
      }
    }
    switch (rpa) {
      case 8: BS_DMMA_A(8, 3)
      case 16: BS_DMMA_A(16, 3)
      case 24: BS_DMMA_A(24, 3)
      default: BS_DMMA_A(32, 3)
    }
#undef BS_DMMA_A
  }
  // N padded to the next multiple of 8 the DMMA fragments need (r = 20 -> 24, not 32)
  const int rp = r <= 8 ? 8 : r <= 16 ? 16 : r <= 24 ? 24 : r <= 32 ? 32 : r <= 48 ? 48 : r <= 64 ? 64 : 0;
#define BS_DMMA(RPV)                                                                                         \
  {                                                                                                          \
    smem_attr(dmma_gemm_kernel<RPV, A_MN>, DmmaCfg<RPV, A_MN>::SMEM);                                      \
    dmma_gemm_kernel<RPV, A_MN><<<grid, 128, DmmaCfg<RPV, A_MN>::SMEM, st>>>(X, B, M, ldx, r, K, kps, out); \
    return true;                                                                                             \
  }
  switch (rp) {
    case 8: BS_DMMA(8)
    case 16: BS_DMMA(16)
    case 24: BS_DMMA(24)
    case 32: BS_DMMA(32)
    case 48: BS_DMMA(48)
    case 64: BS_DMMA(64)
    default: return false;
  }
#undef BS_DMMA
}

// scn b through the register-tiled kernel (RP <= 64) or the legacy one (RP = 128).
template <typename T>
static void launch_wxt_core(const T* X, const T* W, int64_t m, int64_t n_loc, int r, int64_t cps,
                            int S, T* out, cudaStream_t st) {
  note_gemm_path(sizeof(T) == 8 ? 3 : 2);
  dim3 grid(unsigned(ceil_div(m, 128)), unsigned(S));
  if constexpr (sizeof(T) == 8) {
    if (launch_dmma<true>(X, W, m, m, r, n_loc, cps, grid, out, st)) return;
  }
  switch (pick_rp(r)) {
    case 16: cc_gemm_kernel<T, 16, true><<<grid, 128, 0, st>>>(X, W, m, m, r, n_loc, cps, out); return;
    case 32: cc_gemm_kernel<T, 32, true><<<grid, 128, 0, st>>>(X, W, m, m, r, n_loc, cps, out); return;
    case 64: cc_gemm_kernel<T, 64, true><<<grid, 128, 0, st>>>(X, W, m, m, r, n_loc, cps, out); return;
    default: break;
  }
  switch (pick_rp(r)) {
    case 16: gemm_wxt_kernel<T, 16><<<grid, 256, 0, st>>>(X, W, m, n_loc, r, cps, out); break;
    case 32: gemm_wxt_kernel<T, 32><<<grid, 256, 0, st>>>(X, W, m, n_loc, r, cps, out); break;
    case 64: gemm_wxt_kernel<T, 64><<<grid, 256, 0, st>>>(X, W, m, n_loc, r, cps, out); break;
    default: gemm_wxt_kernel<T, 128><<<grid, 256, 0, st>>>(X, W, m, n_loc, r, cps, out); break;
  }
}

template <typename T>
static void launch_vtx_core(const T* X, const T* Vt, int64_t m, int64_t n_loc, int r, int64_t rps,
                            int S, T* out, cudaStream_t st) {
  note_gemm_path(sizeof(T) == 8 ? 3 : 2);
  dim3 grid128(unsigned(ceil_div(n_loc, 128)), unsigned(S));
  if constexpr (sizeof(T) == 8) {
    if (launch_dmma<false>(X, Vt, n_loc, m, r, m, rps, grid128, out, st)) return;
  }
  switch (pick_rp(r)) {
    case 16: cc_gemm_kernel<T, 16, false><<<grid128, 128, 0, st>>>(X, Vt, n_loc, m, r, m, rps, out); return;
    case 32: cc_gemm_kernel<T, 32, false><<<grid128, 128, 0, st>>>(X, Vt, n_loc, m, r, m, rps, out); return;
    case 64: cc_gemm_kernel<T, 64, false><<<grid128, 128, 0, st>>>(X, Vt, n_loc, m, r, m, rps, out); return;
    default: break;
  }
  dim3 grid(unsigned(ceil_div(n_loc, 64)), unsigned(S));
  switch (pick_rp(r)) {
    case 16: gemm_vtx_kernel<T, 16><<<grid, 256, 0, st>>>(X, Vt, m, n_loc, r, rps, out); break;
    case 32: gemm_vtx_kernel<T, 32><<<grid, 256, 0, st>>>(X, Vt, m, n_loc, r, rps, out); break;
    case 64: gemm_vtx_kernel<T, 64><<<grid, 256, 0, st>>>(X, Vt, m, n_loc, r, rps, out); break;
    default: gemm_vtx_kernel<T, 128><<<grid, 256, 0, st>>>(X, Vt, m, n_loc, r, rps, out); break;
  }
}

static int wxt_splits(int64_t m, int64_t n_loc) { return pick_splits(ceil_div(m, 128), n_loc, 256); }
static int vtx_splits(int64_t m, int64_t n_loc) { return pick_splits(ceil_div(n_loc, 128), m, 512); }

// float64 split count <= s_max that fills whole waves of the DMMA kernel (3 CTAs per SM):
// C1 has 79 row tiles, where the default 8 splits give 632 CTAs = 1.42 waves of 444 and 5
// give 395 = 0.89 of one.  Ties go to the larger count.  BS_DMMA_SPLITS overrides (A/B).
static int dmma_stages();

static int f64_splits(int64_t tiles, int s_max) {
  static const int forced = [] { const char* e = getenv("BS_DMMA_SPLITS"); return e ? atoi(e) : 0; }();
  if (forced > 0) return std::min(forced, s_max);
  const int64_t slots = int64_t(num_sms()) * (dmma_stages() == 2 ? 4 : 3);  // resident CTAs per SM (smem)
  int best = s_max;
  double best_eff = 0.0;
  for (int s = s_max; s >= 1; --s) {
    const int64_t ctas = tiles * s;
    const double eff = double(ctas) / double(ceil_div(ctas, slots) * slots);
    if (eff > best_eff + 0.02) { best_eff = eff; best = s; }
  }
  return best;
}

static int dsize(int dtype) { return dtype == BS_F64 ? 8 : 4; }

extern "C" int64_t bs_nmf_wxt_workspace(int dtype, int64_t m, int64_t n_loc, int r) {
  int64_t core = ws_bytes<char>(int64_t(wxt_splits(m, n_loc)) * m * r * dsize(dtype));
  if (dtype == BS_F32) core = std::max(core, tc_wxt_workspace(m, n_loc, r) + i8_gemm_workspace(n_loc));
  return core;
}

static int nmf_wxt_impl(const void* X, const void* W, int dtype, int64_t m, int64_t n_loc, int r, void* P,
                        const void* xscale, double* stats, void* work, int64_t work_bytes, void* stream);

extern "C" int bs_nmf_wxt(const void* X, const void* W, int dtype, int64_t m, int64_t n_loc, int r,
                          void* P, const void* xscale, void* work, int64_t work_bytes, void* stream) {
  return nmf_wxt_impl(X, W, dtype, m, n_loc, r, P, xscale, nullptr, work, work_bytes, stream);
}

extern "C" int64_t bs_nmf_wxt_scan_workspace(int dtype, int64_t m, int64_t n_loc, int r) {
  return bs_nmf_wxt_workspace(dtype, m, n_loc, r) + ws_bytes<char>(64 * 1024) + 512;
}

extern "C" int bs_nmf_wxt_scan(const void* X, const void* W, int dtype, int64_t m, int64_t n_loc, int r, void* P,
                               double* stats_dev, void* work, int64_t work_bytes, void* stream) {
  return nmf_wxt_impl(X, W, dtype, m, n_loc, r, P, nullptr, stats_dev, work, work_bytes, stream);
}

static int nmf_wxt_impl(const void* X, const void* W, int dtype, int64_t m, int64_t n_loc, int r, void* P,
                        const void* xscale, double* stats, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  if (r < 1 || r > MAX_R || m < 0 || n_loc < 0) {
    set_error("bs_nmf_wxt: bad shape m=%lld n_loc=%lld r=%d", (long long)m, (long long)n_loc, r);
    return BS_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  Workspace all(work, work_bytes);
  Workspace sws(nullptr, 0);
  if (stats) sws = all.split(ws_bytes<char>(64 * 1024));  // the scan's slice (fixed counter offset)
  Workspace ws = all.rest();
  bool scanned = false;
  auto plain_scan = [&]() -> int {
    scanned = true;
    return bs_nmf_scan(X, dtype, m * n_loc, stats, sws.base, sws.size, stream);
  };
  if (stats && (m == 0 || n_loc == 0 || dtype != BS_F32)) {
    const int rc = plain_scan();
    if (rc != BS_OK) return rc;
  }
  if (m == 0) return BS_OK;
  if (n_loc == 0) {
    return cudaMemsetAsync(P, 0, size_t(m) * r * dsize(dtype), st) == cudaSuccess ? BS_OK : BS_ECUDA;
  }
  if (dtype == BS_F32 && xscale && !stats) {
    bool used = false;
    int rc = i8_wxt(static_cast<const float*>(X), static_cast<const float*>(W), m, n_loc, r,
                    static_cast<const int8_t*>(xscale), static_cast<float*>(P), ws, st, &used);
    if (rc != BS_OK) return rc;
    if (used) return BS_OK;
  }
  if (dtype == BS_F32) {
    bool used = false;
    int rc = tc_wxt(static_cast<const float*>(X), static_cast<const float*>(W), m, n_loc, r,
                    static_cast<float*>(P), ws, st, &used, scanned ? nullptr : stats);
    if (rc != BS_OK) return rc;
    if (used) return BS_OK;
    if (stats && !scanned) {  // tcgen05 path not taken: plain scan
      rc = plain_scan();
      if (rc != BS_OK) return rc;
    }
  }
  const int S = dtype == BS_F64 ? f64_splits(ceil_div(m, 128), wxt_splits(m, n_loc)) : wxt_splits(m, n_loc);
  const int64_t cps = ceil_div(ceil_div(n_loc, S), 32) * 32;
  const int Seff = int(ceil_div(n_loc, cps));
  if (dtype == BS_F64) {
    double* out = static_cast<double*>(P);
    double* parts = Seff > 1 ? ws.take<double>(int64_t(Seff) * m * r) : out;
    if (!parts) { set_error("bs_nmf_wxt: workspace too small"); return BS_EWORK; }
    launch_wxt_core<double>(static_cast<const double*>(X), static_cast<const double*>(W), m, n_loc, r,
                            cps, Seff, parts, st);
    if (Seff > 1)
      sum_slabs_kernel<double><<<int(std::min<int64_t>(ceil_div(m * r, 256), 4096)), 256, 0, st>>>(
          parts, Seff, m * r, out);
  } else if (dtype == BS_F32) {
    float* out = static_cast<float*>(P);
    float* parts = Seff > 1 ? ws.take<float>(int64_t(Seff) * m * r) : out;
    if (!parts) { set_error("bs_nmf_wxt: workspace too small"); return BS_EWORK; }
    launch_wxt_core<float>(static_cast<const float*>(X), static_cast<const float*>(W), m, n_loc, r,
                           cps, Seff, parts, st);
    if (Seff > 1)
      sum_slabs_kernel<float><<<int(std::min<int64_t>(ceil_div(m * r, 256), 4096)), 256, 0, st>>>(
          parts, Seff, m * r, out);
  } else {
    set_error("bs_nmf_wxt: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_nmf_wxt", Seff > 1 ? 2 : 1);
}

// ---------------------------------------------------------------------------
// Fused factor half-step (shared by the Vt and the W half-steps).
//   NUM = sum over S slabs of num (r x ncols, layout F), den = GRAM F
//   F <- MU:  F * NUM / (den + eps)      APG: max(0, F - step (den - NUM))
//   red[0..r*r) += F_new F_new^T,  red[r*r] += <NUM, F_new>
// One warp per column (lane k, k+32, ...), columns staged in smem for the Gram.
// ---------------------------------------------------------------------------

constexpr int UPD_THREADS = 256;
constexpr int UPD_COLS = 32;  // columns per smem stage (one per warp-iteration)

template <typename T, typename TN, int RP>
__global__ void __launch_bounds__(UPD_THREADS)
factor_update_kernel(int algo, T* __restrict__ F, const TN* __restrict__ num, int S,
                     int64_t num_slab, const double* __restrict__ gram, int r, int64_t ncols,
                     double eps, int64_t cols_per_block, T* __restrict__ Fcopy,
                     double* __restrict__ parts, unsigned int* counter, double* __restrict__ red) {
  extern __shared__ double smem[];
  double* gT = smem;                 // [r][r] gram transposed: gT[l*r + k] = gram[k][l]
  double* tile = smem + r * r;       // [UPD_COLS][r] updated columns
  __shared__ double sh_red[32];
  __shared__ double sh_step;
  const int rr = r * r;
  for (int e = threadIdx.x; e < rr; e += blockDim.x) {
    const int k = e / r, l = e % r;
    gT[l * r + k] = gram[e];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int e = 0; e < rr; ++e) s = fma(gram[e], gram[e], s);
    sh_step = 1.0 / (2.0 * s + eps);  // solvers.py:174 / 180
  }
  __syncthreads();
  const double step = sh_step;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int KPL = (RP + 31) / 32;  // rows k per lane
  const int npairs = r * (r + 1) / 2;
  constexpr int MAXP = (RP * (RP + 1) / 2 + UPD_THREADS - 1) / UPD_THREADS;
  double gacc[MAXP];
  int ia[MAXP], ib[MAXP];
#pragma unroll
  for (int t = 0; t < MAXP; ++t) {
    gacc[t] = 0.0;
    int a = 0, rem = threadIdx.x + t * UPD_THREADS;
    if (rem < npairs) {
      while (rem >= r - a) { rem -= r - a; ++a; }
    } else {
      rem = -1;
    }
    ia[t] = a;
    ib[t] = a + rem;
  }
  double cross = 0.0;
  const int64_t c_begin = int64_t(blockIdx.x) * cols_per_block;
  const int64_t c_end = min(ncols, c_begin + cols_per_block);
  for (int64_t cb = c_begin; cb < c_end; cb += UPD_COLS) {
    const int nc = int(c_end - cb < UPD_COLS ? c_end - cb : UPD_COLS);
    __syncthreads();  // tile reuse
    for (int cc = wid; cc < nc; cc += UPD_THREADS / 32) {
      const int64_t c = cb + cc;
      double f[KPL], nm[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        f[q] = 0.0;
        nm[q] = 0.0;
        if (k < r) {
          f[q] = double(F[c * r + k]);
          double s = double(num[c * r + k]);
          for (int p = 1; p < S; ++p) s += double(num[int64_t(p) * num_slab + c * r + k]);
          // NUM is rounded to the storage type like the reference's WXt / VtX
          nm[q] = double(T(s));
        }
      }
      // den[k] = sum_l gram[k][l] f[l]
      double den[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) den[q] = 0.0;
#pragma unroll
      for (int ql = 0; ql < KPL; ++ql) {
        const int lmax = min(32, r - 32 * ql);
        for (int ll = 0; ll < lmax; ++ll) {
          const int l = 32 * ql + ll;
          const double fl = __shfl_sync(0xffffffffu, f[ql], ll);
#pragma unroll
          for (int q = 0; q < KPL; ++q) {
            const int k = lane + 32 * q;
            if (k < r) den[q] = fma(gT[l * r + k], fl, den[q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k < r) {
          const T dd = T(den[q]);  // WWtVt / VtVW in the storage type
          T fn;
          if (algo == BS_NMF_MU) {
            fn = T(f[q]) * T(nm[q]) / (dd + T(eps));
          } else {
            const T v = T(f[q]) - T(step) * (dd - T(nm[q]));
            fn = v > T(0) ? v : T(0);
          }
          F[c * r + k] = fn;
          if (Fcopy) Fcopy[c * r + k] = fn;
          tile[cc * r + k] = double(fn);
          cross = fma(nm[q], double(fn), cross);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < MAXP; ++t) {
      const int p = threadIdx.x + t * UPD_THREADS;
      if (p < npairs) {
        double s = gacc[t];
        for (int cc = 0; cc < nc; ++cc) s = fma(tile[cc * r + ia[t]], tile[cc * r + ib[t]], s);
        gacc[t] = s;
      }
    }
  }
  // per-block partial: [r*r gram][cross]
  double* mine = parts + int64_t(blockIdx.x) * (rr + 1);
#pragma unroll
  for (int t = 0; t < MAXP; ++t) {
    const int p = threadIdx.x + t * UPD_THREADS;
    if (p < npairs) {
      mine[ia[t] * r + ib[t]] = gacc[t];
      mine[ib[t] * r + ia[t]] = gacc[t];
    }
  }
  const double csum = block_sum(cross, sh_red);
  if (threadIdx.x == 0) mine[rr] = csum;
  (void)counter;
  (void)red;  // folded by fold_rows_kernel
}

// out[e] = sum_p parts[p * len + e] (deterministic).  A CTA owns 32 consecutive outputs;
// its 8 warps each sum a contiguous run of p ascending (lane = output, so every load is a
// coalesced 256-byte row segment, eight in flight), then warp partials fold in warp order
// through shared memory.  C1's 157 x 401 partials took 15 us as one thread per output
// walking all p; this spreads them over 13 CTAs x 8 warps.
constexpr int FOLD_WARPS = 8;
__global__ void __launch_bounds__(32 * FOLD_WARPS) fold_rows_kernel(const double* __restrict__ parts, int np,
                                                                    int len, double* __restrict__ out) {
  __shared__ double part[FOLD_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int per = (np + FOLD_WARPS - 1) / FOLD_WARPS;
  const int p0 = w * per, p1 = min(np, p0 + per);
  double s = 0.0;
  if (e < len) {
    int p = p0;
    for (; p + 8 <= p1; p += 8) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = parts[int64_t(p + u) * len + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += t[u];
    }
    for (; p < p1; ++p) s += parts[int64_t(p) * len + e];
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < len) {
    double t = part[0][lane];
#pragma unroll
    for (int u = 1; u < FOLD_WARPS; ++u) t += part[u][lane];
    out[e] = t;
  }
}

// Register-blocked variant (RP <= 64): per stage of UPD_COLS columns the old factor
// columns and NUM (slabs summed, rounded to T) are staged in shared memory; each thread
// computes den = GRAM f for KB = RP/16 rows x 2 columns (l ascending: the same order as
// the shuffle kernel, so den is bitwise identical), applies the update, and later
// accumulates a GB x GB block (GB = RP/16) of the new factor's Gram over the stage.
// Writes of F (and the copy) go back coalesced from the staged tile.
template <typename T, typename TN, int RP>
__global__ void __launch_bounds__(UPD_THREADS)
factor_update_rb_kernel(int algo, T* __restrict__ F, const TN* __restrict__ num, int S,
                        int64_t num_slab, const double* __restrict__ gram, int r, int64_t ncols,
                        double eps, int64_t cols_per_block, T* __restrict__ Fcopy,
                        double* __restrict__ parts) {
  static_assert(RP % 16 == 0 && RP <= 64, "register-blocked update needs RP in {16, 32, 64}");
  constexpr int KB = RP / 16;   // den rows per thread (16 row groups x 16 column pairs)
  constexpr int GB = RP / 16;   // Gram block edge per thread (16 x 16 thread grid)
  constexpr int C = UPD_COLS;   // 32 columns per stage
  extern __shared__ double upd_smem[];
  auto gT = reinterpret_cast<double (*)[RP]>(upd_smem);                             // [RP][RP]: gram[k][l] at [l][k]
  auto fs = reinterpret_cast<double (*)[RP + 1]>(upd_smem + RP * RP);               // [C] old columns
  auto ns = reinterpret_cast<double (*)[RP + 1]>(upd_smem + RP * RP + C * (RP + 1));  // [C] NUM (rounded to T)
  auto tile = reinterpret_cast<double (*)[RP + 1]>(upd_smem + RP * RP + 2 * C * (RP + 1));  // [C] new columns
  __shared__ double sh_red[32];
  __shared__ double sh_step;
  const int tid = threadIdx.x;
  const int rr = r * r;
  for (int e = tid; e < RP * RP; e += UPD_THREADS) {
    const int l = e / RP, k = e % RP;
    gT[l][k] = (l < r && k < r) ? gram[k * r + l] : 0.0;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int e = 0; e < rr; ++e) s = fma(gram[e], gram[e], s);
    sh_step = 1.0 / (2.0 * s + eps);  // solvers.py:174 / 180
  }
  __syncthreads();
  const double step = sh_step;
  const int cp = tid & 15, kg = tid >> 4;  // den: columns 2cp, 2cp+1; rows KB*kg ..
  const int gi = tid & 15, gj = tid >> 4;  // Gram block rows GB*gi.., columns GB*gj..
  double gacc[GB][GB];
#pragma unroll
  for (int a = 0; a < GB; ++a)
#pragma unroll
    for (int b = 0; b < GB; ++b) gacc[a][b] = 0.0;
  double cross = 0.0;
  const int64_t c_begin = int64_t(blockIdx.x) * cols_per_block;
  const int64_t c_end = min(ncols, c_begin + cols_per_block);
  for (int64_t cb = c_begin; cb < c_end; cb += C) {
    const int nc = int(c_end - cb < C ? c_end - cb : C);
    __syncthreads();  // stage buffers free
    // stage old F and NUM (columns contiguous: nc * r elements each, coalesced)
    for (int e = tid; e < C * RP; e += UPD_THREADS) {
      const int cc = e / RP, k = e % RP;
      double f = 0.0, nm = 0.0;
      if (cc < nc && k < r) {
        const int64_t o = (cb + cc) * r + k;
        f = double(F[o]);
        double sn = double(num[o]);
        for (int p = 1; p < S; ++p) sn += double(num[int64_t(p) * num_slab + o]);
        nm = double(T(sn));  // NUM is rounded to the storage type like the reference's WXt / VtX
      }
      fs[cc][k] = f;
      ns[cc][k] = nm;
    }
    __syncthreads();
    // den = GRAM f, update, new column values into the tile
    {
      double den[KB][2];
#pragma unroll
      for (int a = 0; a < KB; ++a) den[a][0] = den[a][1] = 0.0;
      for (int l = 0; l < r; ++l) {
        const double f0 = fs[2 * cp][l], f1 = fs[2 * cp + 1][l];
#pragma unroll
        for (int a = 0; a < KB; ++a) {
          const double g = gT[l][KB * kg + a];
          den[a][0] = fma(g, f0, den[a][0]);
          den[a][1] = fma(g, f1, den[a][1]);
        }
      }
#pragma unroll
      for (int a = 0; a < KB; ++a)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = KB * kg + a, cc = 2 * cp + h;
          double out = 0.0;
          if (k < r && cc < nc) {
            const T dd = T(den[a][h]);  // WWtVt / VtVW in the storage type
            const T fo = T(fs[cc][k]), nmT = T(ns[cc][k]);
            T fn;
            if (algo == BS_NMF_MU) {
              fn = fo * nmT / (dd + T(eps));
            } else {
              const T vv = fo - T(step) * (dd - nmT);
              fn = vv > T(0) ? vv : T(0);
            }
            out = double(fn);
            cross = fma(ns[cc][k], out, cross);
          }
          tile[cc][k] = out;
        }
    }
    __syncthreads();
    // coalesced write-back of the new columns
    for (int e = tid; e < nc * r; e += UPD_THREADS) {
      const int cc = e / r, k = e - cc * r;
      const T v = T(tile[cc][k]);
      F[cb * r + e] = v;
      if (Fcopy) Fcopy[cb * r + e] = v;
    }
    // Gram of the new columns: GB x GB block per thread, columns in order
    for (int cc = 0; cc < nc; ++cc) {
      double av[GB], bv[GB];
#pragma unroll
      for (int a = 0; a < GB; ++a) {
        av[a] = tile[cc][GB * gi + a];
        bv[a] = tile[cc][GB * gj + a];
      }
#pragma unroll
      for (int a = 0; a < GB; ++a)
#pragma unroll
        for (int b = 0; b < GB; ++b) gacc[a][b] = fma(av[a], bv[b], gacc[a][b]);
    }
  }
  // per-block partial: [r*r gram][cross]
  double* mine = parts + int64_t(blockIdx.x) * (rr + 1);
#pragma unroll
  for (int a = 0; a < GB; ++a)
#pragma unroll
    for (int b = 0; b < GB; ++b) {
      const int k = GB * gi + a, l = GB * gj + b;
      if (k < r && l < r) mine[k * r + l] = gacc[a][b];
    }
  const double csum = block_sum(cross, sh_red);
  if (tid == 0) mine[rr] = csum;
}

// >= 32 columns (one stage) per block, at most 3 blocks per SM; fold_rows_kernel folds the
// grid x (r^2 + 1) partials.  C1 (10,000 columns): 313 one-stage blocks instead of 157
// two-stage ones, which halves each block's serial load -> den -> Gram chain.
static int upd_grid(int64_t ncols) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(ncols, 32), int64_t(num_sms()) * 3)));
}

static int64_t upd_workspace(int r, int64_t ncols) {
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(int64_t(upd_grid(ncols)) * (r * r + 1)) +
         ws_bytes<double>(r * r + 1);
}

template <typename T, typename TN>
static int launch_update(int algo, T* F, const TN* num, int S, int64_t slab, const double* gram, int r,
                         int64_t ncols, double eps, T* Fcopy, double* red, Workspace& ws,
                         cudaStream_t st) {
  const int grid = upd_grid(ncols);
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(int64_t(grid) * (r * r + 1));
  if (!counter || !parts) {
    set_error("factor update: workspace too small");
    return BS_EWORK;
  }
  const size_t smem = sizeof(double) * (r * r + UPD_COLS * r);
  {
    const int big = int(sizeof(double) * (MAX_R * MAX_R + UPD_COLS * MAX_R));
    smem_attr(factor_update_kernel<T, TN, 16>, big);
    smem_attr(factor_update_kernel<T, TN, 32>, big);
    smem_attr(factor_update_kernel<T, TN, 64>, big);
    smem_attr(factor_update_kernel<T, TN, 128>, big);
  }
  const int64_t cpb = ceil_div(ncols, grid);
#define BS_UPD(RPV)                                                                              \
  factor_update_kernel<T, TN, RPV><<<grid, UPD_THREADS, smem, st>>>(algo, F, num, S, slab, gram, r, \
                                                                     ncols, eps, cpb, Fcopy, parts,  \
                                                                     counter, red)
  static const bool legacy = getenv("BS_UPD_LEGACY") != nullptr;  // A/B switch
#define BS_UPD_RB(RPV)                                                                                      \
  {                                                                                                          \
    const int sm_rb = int(sizeof(double) * (RPV * RPV + 3 * UPD_COLS * (RPV + 1)));                          \
    smem_attr(factor_update_rb_kernel<T, TN, RPV>, sm_rb);                                                   \
    factor_update_rb_kernel<T, TN, RPV><<<grid, UPD_THREADS, sm_rb, st>>>(algo, F, num, S, slab, gram, r, ncols, \
                                                                          eps, cpb, Fcopy, parts);           \
  }
  if (!legacy && r <= 64) {
    switch (pick_rp(r)) {
      case 16: BS_UPD_RB(16); break;
      case 32: BS_UPD_RB(32); break;
      default: BS_UPD_RB(64); break;
    }
  } else {
    switch (pick_rp(r)) {
      case 16: BS_UPD(16); break;
      case 32: BS_UPD(32); break;
      case 64: BS_UPD(64); break;
      default: BS_UPD(128); break;
    }
  }
#undef BS_UPD_RB
#undef BS_UPD
  fold_rows_kernel<<<(r * r + 1 + 31) / 32, 32 * FOLD_WARPS, 0, st>>>(parts, grid, r * r + 1, red);
  return check_launch("factor update", 2);
}

extern "C" int64_t bs_nmf_vt_step_workspace(int r, int64_t m_loc) {
  return upd_workspace(r, m_loc) + ws_bytes<double>(r * r + 1) + 256;
}

extern "C" int bs_nmf_vt_step(int algo, void* Vt, const void* WXt, const double* WWt, int dtype,
                              int r, int64_t m_loc, double eps, double* VtV, void* Vt_copy, void* work,
                              int64_t work_bytes, void* stream) {
  clear_error();
  if (r < 1 || r > MAX_R || (algo != BS_NMF_MU && algo != BS_NMF_APG)) {
    set_error("bs_nmf_vt_step: bad r=%d / algo=%d", r, algo);
    return BS_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  Workspace all(work, work_bytes);
  Workspace ws = all.split(upd_workspace(r, m_loc));
  double* red = VtV;  // the kernel writes r*r+1 values; stage them and copy the gram out
  double* tmp = all.take<double>(r * r + 1);
  if (!tmp) { set_error("bs_nmf_vt_step: workspace too small"); return BS_EWORK; }
  int rc;
  if (m_loc == 0) {
    if (cudaMemsetAsync(tmp, 0, sizeof(double) * (r * r + 1), st) != cudaSuccess) return BS_ECUDA;
    rc = BS_OK;
  } else if (dtype == BS_F64) {
    rc = launch_update<double, double>(algo, static_cast<double*>(Vt), static_cast<const double*>(WXt), 1,
                                       0, WWt, r, m_loc, eps, static_cast<double*>(Vt_copy), tmp, ws, st);
  } else if (dtype == BS_F32) {
    rc = launch_update<float, float>(algo, static_cast<float*>(Vt), static_cast<const float*>(WXt), 1, 0,
                                     WWt, r, m_loc, eps, static_cast<float*>(Vt_copy), tmp, ws, st);
  } else {
    set_error("bs_nmf_vt_step: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  if (rc != BS_OK) return rc;
  if (cudaMemcpyAsync(red, tmp, sizeof(double) * r * r, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    set_error("bs_nmf_vt_step: copy failed");
    return BS_ECUDA;
  }
  return BS_OK;
}

extern "C" int64_t bs_nmf_w_step_workspace(int dtype, int64_t m, int64_t n_loc, int r) {
  const int slabs = dtype == BS_F32 ? std::max(vtx_splits(m, n_loc), TC_MAX_SPLITS) : vtx_splits(m, n_loc);
  int64_t g = ws_bytes<char>(int64_t(slabs) * n_loc * r * dsize(dtype));
  if (dtype == BS_F32) g += tc_vtx_workspace(m, n_loc, r) + i8_gemm_workspace(m);
  return g + upd_workspace(r, n_loc) + 512;
}

extern "C" int bs_nmf_w_step(int algo, const void* X, const void* Vt_full, void* W, const double* VtV,
                             int dtype, int64_t m, int64_t n_loc, int r, double eps, double* red,
                             const void* xscale, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  if (r < 1 || r > MAX_R || (algo != BS_NMF_MU && algo != BS_NMF_APG) || m < 0 || n_loc < 0) {
    set_error("bs_nmf_w_step: bad arguments");
    return BS_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  if (n_loc == 0) {
    return cudaMemsetAsync(red, 0, sizeof(double) * (r * r + 1), st) == cudaSuccess ? BS_OK : BS_ECUDA;
  }
  Workspace ws(work, work_bytes);
  Workspace upd = ws.split(upd_workspace(r, n_loc));
  const int S = dtype == BS_F64 ? f64_splits(ceil_div(n_loc, 128), vtx_splits(m, n_loc)) : vtx_splits(m, n_loc);
  const int64_t rps = std::max<int64_t>(1, ceil_div(ceil_div(std::max<int64_t>(m, 1), S), 32) * 32);
  const int Seff = int(std::max<int64_t>(1, ceil_div(m, rps)));
  if (dtype == BS_F64) {
    double* C = ws.take<double>(int64_t(Seff) * n_loc * r);
    if (!C) { set_error("bs_nmf_w_step: workspace too small"); return BS_EWORK; }
    if (m == 0) {
      if (cudaMemsetAsync(C, 0, sizeof(double) * n_loc * r, st) != cudaSuccess) return BS_ECUDA;
    } else {
      launch_vtx_core<double>(static_cast<const double*>(X), static_cast<const double*>(Vt_full), m, n_loc,
                              r, rps, Seff, C, st);
    }
    int rc = check_launch("bs_nmf_w_step gemm");
    if (rc != BS_OK) return rc;
    return launch_update<double, double>(algo, static_cast<double*>(W), C, Seff, n_loc * r, VtV, r, n_loc,
                                         eps, nullptr, red, upd, st);
  } else if (dtype == BS_F32) {
    // tcgen05 3xTF32 when available for this shape, CUDA cores otherwise
    int splits = 1;
    bool used = false;
    const int cap = std::max(Seff, TC_MAX_SPLITS);
    float* Cbuf = ws.take<float>(int64_t(cap) * n_loc * r);
    if (!Cbuf) { set_error("bs_nmf_w_step: workspace too small"); return BS_EWORK; }
    if (m > 0 && xscale) {
      const int8_t* xexp_a = static_cast<const int8_t*>(xscale) + xgroups(n_loc) * m;
      int rc = i8_vtx(static_cast<const float*>(X), static_cast<const float*>(Vt_full), m, n_loc, r, xexp_a, Cbuf,
                      cap, &splits, ws, st, &used);
      if (rc != BS_OK) return rc;
    }
    if (m > 0 && !used) {
      int rc = tc_vtx(static_cast<const float*>(X), static_cast<const float*>(Vt_full), m, n_loc, r, Cbuf,
                      cap, &splits, ws, st, &used);
      if (rc != BS_OK) return rc;
    }
    if (!used) {
      splits = Seff;
      if (m == 0) {
        if (cudaMemsetAsync(Cbuf, 0, sizeof(float) * n_loc * r, st) != cudaSuccess) return BS_ECUDA;
      } else {
        launch_vtx_core<float>(static_cast<const float*>(X), static_cast<const float*>(Vt_full), m, n_loc, r,
                               rps, Seff, Cbuf, st);
      }
      int rc = check_launch("bs_nmf_w_step gemm");
      if (rc != BS_OK) return rc;
    }
    return launch_update<float, float>(algo, static_cast<float*>(W), Cbuf, splits, n_loc * r, VtV, r, n_loc,
                                       eps, nullptr, red, upd, st);
  }
  set_error("bs_nmf_w_step: unsupported dtype %d", dtype);
  return BS_EINVAL;
}

// ---------------------------------------------------------------------------
// bs_nmf_prepare: the per-call X pass (solvers.py:139-141) — min, ||X||^2, and for
// float32 the per-block scales of the integer tensor-core GEMMs (nmf_i8.cu).
// ---------------------------------------------------------------------------

extern "C" int64_t bs_nmf_xscale_bytes(int64_t m, int64_t n_loc) { return i8_xscale_bytes(m, n_loc); }

extern "C" int64_t bs_nmf_prepare_workspace(int64_t m, int64_t n_loc) {
  return std::max<int64_t>(i8_prepare_workspace(m, n_loc), 64 * 1024) + 512;
}

// stats[2] (nonfinite) is produced by the integer path's pass; the plain scan does not look
// for nonfinite values, and without scales (ready = 0) the caller keeps the other GEMM paths.
__global__ void prep_stats_tail_kernel(double* stats, double ready) {
  if (ready == 0.0) stats[2] = 0.0;
  stats[3] = ready;
}

extern "C" int bs_nmf_prepare(const void* X, int dtype, int64_t m, int64_t n_loc, double* stats_dev, void* xscale,
                              void* work, int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (m < 0 || n_loc < 0) {
    set_error("bs_nmf_prepare: bad shape");
    return BS_EINVAL;
  }
  Workspace ws(work, work_bytes);
  const bool i8 = dtype == BS_F32 && xscale && m > 0 && n_loc > 0 && m % 4 == 0 &&
                  !(reinterpret_cast<uintptr_t>(X) & 15);
  if (i8) {
    int rc = i8_prepare(static_cast<const float*>(X), m, n_loc, stats_dev, static_cast<int8_t*>(xscale), ws, st);
    if (rc != BS_OK) return rc;
    prep_stats_tail_kernel<<<1, 1, 0, st>>>(stats_dev, 1.0);
    // keep the nonfinite flag the pass produced: rewrite only the ready flag
    return check_launch("bs_nmf_prepare tail");
  }
  int rc = bs_nmf_scan(X, dtype, m * n_loc, stats_dev, ws.base, ws.size, stream);
  if (rc != BS_OK) return rc;
  prep_stats_tail_kernel<<<1, 1, 0, st>>>(stats_dev, 0.0);
  return check_launch("bs_nmf_prepare tail");
}

// ---------------------------------------------------------------------------
// Objective via the Gram identity (after an update), with a cancellation guard:
// when ||X||^2 / obj exceeds kappa (or obj <= 0; kappa < 0: always) the value cannot be
// trusted to the parity tolerance and *direct_flag is raised — the caller then evaluates the
// reference's own direct residual (solvers.py:124-136) with bs_nmf_residual.
// ---------------------------------------------------------------------------

__global__ void nmf_objective_kernel(const double* xsq, const double* red, const double* VtV, int r,
                                     double* out, int* flag, double kappa) {
  __shared__ double sh[32];
  const int rr = r * r;
  double s = 0.0;
  for (int e = threadIdx.x; e < rr; e += blockDim.x) s = fma(VtV[e], red[e], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) {
    const double obj = (xsq[0] - 2.0 * red[rr]) + s;
    out[0] = obj;
    if (flag) *flag = (kappa < 0.0 || (kappa > 0.0 && (!(obj > 0.0) || obj * kappa < xsq[0]))) ? 1 : 0;
  }
}

extern "C" int bs_nmf_objective(const double* xsq, const double* red, const double* VtV, int r,
                                double* out_dev, int* direct_flag, double kappa, void* stream) {
  clear_error();
  nmf_objective_kernel<<<1, 256, 0, as_stream(stream)>>>(xsq, red, VtV, r, out_dev, direct_flag, kappa);
  return check_launch("bs_nmf_objective");
}

__global__ void objective_select_kernel(const int* flag, const double* direct, double* out) {
  if (*flag) out[0] = direct[0];
}

extern "C" int bs_nmf_objective_select(const int* direct_flag, const double* direct_dev, double* out_dev,
                                       void* stream) {
  clear_error();
  objective_select_kernel<<<1, 1, 0, as_stream(stream)>>>(direct_flag, direct_dev, out_dev);
  return check_launch("bs_nmf_objective_select");
}

// ---------------------------------------------------------------------------
// Direct residual sum((X - Vt^T W)^2) over the local block (solvers.py:124-136).
// A warp owns 32 consecutive rows (lane = row, its Vt column in registers) and a
// run of columns; the block stages those columns of W in shared memory and every
// lane reads them as broadcasts.  The reconstruction runs in the storage precision
// (float32 FMA chains for float32, like the reference's float32 matmul), the squares
// are summed in float64.  flag (nullable): when *flag == 0 the kernel only zeroes out.
// ---------------------------------------------------------------------------

template <typename T, int RP>
__global__ void __launch_bounds__(256)
residual_kernel(const T* __restrict__ X, const T* __restrict__ Vt, const T* __restrict__ W, int64_t m,
                int64_t n_loc, int r, int64_t col_chunk, double* __restrict__ parts, unsigned int* counter,
                double* out, const int* flag) {
  constexpr int RES_COLS = 16384 / (RP * int(sizeof(T))) < 64 ? 16384 / (RP * int(sizeof(T))) : 64;
  __shared__ T sw[RES_COLS * RP];
  __shared__ double sh[32];
  if (flag && *flag == 0) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) out[0] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t(blockIdx.x) * 8 + warp) * 32 + lane;
  const bool row_ok = i < m;
  T v[RP];
#pragma unroll
  for (int k = 0; k < RP; ++k) v[k] = (row_ok && k < r) ? Vt[i * r + k] : T(0);
  const int64_t j0 = int64_t(blockIdx.y) * col_chunk;
  const int64_t j1 = min(n_loc, j0 + col_chunk);
  double acc = 0.0;
  for (int64_t jb = j0; jb < j1; jb += RES_COLS) {
    const int nc = int(j1 - jb < int64_t(RES_COLS) ? j1 - jb : int64_t(RES_COLS));
    __syncthreads();
    for (int e = threadIdx.x; e < nc * RP; e += 256) {
      const int c = e / RP, k = e - c * RP;
      sw[e] = k < r ? W[(jb + c) * r + k] : T(0);
    }
    __syncthreads();
    if (row_ok) {
      for (int c = 0; c < nc; ++c) {
        const T* w = sw + c * RP;
        T rec0 = T(0), rec1 = T(0);
#pragma unroll
        for (int k = 0; k < RP; k += 2) {
          rec0 = fma(v[k], w[k], rec0);
          rec1 = fma(v[k + 1], w[k + 1], rec1);
        }
        const double d = double(X[(jb + c) * m + i] - (rec0 + rec1));
        acc = fma(d, d, acc);
      }
    }
  }
  acc = block_sum(acc, sh);
  const unsigned int nb = gridDim.x * gridDim.y;
  const unsigned int b = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) parts[b] = acc;
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == nb - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = parts[0];
    for (unsigned int q = 1; q < nb; ++q) s += parts[q];
    out[0] = s;
    *counter = 0u;
  }
}

static void residual_grid(int64_t m, int64_t n_loc, dim3* grid, int64_t* chunk) {
  if (m <= 0 || n_loc <= 0) {
    *grid = dim3(1, 1, 1);
    *chunk = 1;
    return;
  }
  const int64_t rows = ceil_div(std::max<int64_t>(m, 1), 256);
  const int64_t want = int64_t(num_sms()) * 8;
  int64_t cs = std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, rows), ceil_div(n_loc, 64)));
  cs = std::min<int64_t>(cs, 65535);
  *chunk = ceil_div(n_loc, cs);
  *grid = dim3(unsigned(rows), unsigned(ceil_div(n_loc, *chunk)));
}

extern "C" int64_t bs_nmf_residual_workspace(int64_t m, int64_t n_loc) {
  dim3 g;
  int64_t c;
  residual_grid(m, n_loc, &g, &c);
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(int64_t(g.x) * g.y);
}

extern "C" int bs_nmf_residual(const void* X, const void* Vt_full, const void* W, int dtype, int64_t m,
                               int64_t n_loc, int r, double* out_dev, const int* flag_dev, void* work,
                               int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (n_loc == 0 || m == 0)
    return cudaMemsetAsync(out_dev, 0, sizeof(double), st) == cudaSuccess ? BS_OK : BS_ECUDA;
  if (r < 1 || r > MAX_R) {
    set_error("bs_nmf_residual: bad rank %d", r);
    return BS_EINVAL;
  }
  Workspace ws(work, work_bytes);
  dim3 grid;
  int64_t chunk;
  residual_grid(m, n_loc, &grid, &chunk);
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(int64_t(grid.x) * grid.y);
  if (!counter || !parts) { set_error("bs_nmf_residual: workspace too small"); return BS_EWORK; }
#define BS_RES(T, RPV)                                                                                          \
  residual_kernel<T, RPV><<<grid, 256, 0, st>>>(static_cast<const T*>(X), static_cast<const T*>(Vt_full),      \
                                                static_cast<const T*>(W), m, n_loc, r, chunk, parts, counter,  \
                                                out_dev, flag_dev)
  const int rp = r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 128;
  if (dtype == BS_F64) {
    switch (rp) {
      case 16: BS_RES(double, 16); break;
      case 32: BS_RES(double, 32); break;
      case 64: BS_RES(double, 64); break;
      default: BS_RES(double, 128); break;
    }
  } else if (dtype == BS_F32) {
    switch (rp) {
      case 16: BS_RES(float, 16); break;
      case 32: BS_RES(float, 32); break;
      case 64: BS_RES(float, 64); break;
      default: BS_RES(float, 128); break;
    }
  } else {
    set_error("bs_nmf_residual: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
#undef BS_RES
  return check_launch("bs_nmf_residual");
}
