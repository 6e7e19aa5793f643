// l1-regularized Cox proportional hazards by proximal gradient
// (solvers.py:308-450) as memory-bound kernels.
//
//   scn m   xb   = X_loc beta_loc            one streamed pass over X  (distlinalg.py:334-337)
//   risk    w = exp(min(xb, clamp)), W = cumsum(w), loglik          (solvers.py:376-398)
//   pi_delta pd_i = w_i sum_{j: cuts_j >= i} delta_j / W[cuts_j]    (solvers.py:401-419)
//   scn p   grad = X_loc^T (delta - pd)      one streamed pass over X  (distlinalg.py:355-358)
//   prox    beta <- S_lam(beta + sigma grad)                         (solvers.py:448-449)
//
// X local block: m x n_loc column-major (X[j*m + i]) in float32, float64 or int8
// (genotypes, widened in-register).  The O(m) scans run in float64 regardless of
// the storage type (PAPER.md:864 records fp32 cumsum instability).
#include "bsb200.cuh"

#include <algorithm>
#include <mutex>
#include <type_traits>

using namespace bs;

// ---------------------------------------------------------------------------
// Vector load helpers: VEC consecutive elements of a column as doubles.
// ---------------------------------------------------------------------------

template <typename TX, int VEC> struct VecLoad;
template <> struct VecLoad<float, 4> {
  static __device__ __forceinline__ void widen(uint4 v, double* o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y); o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
  }
  static __device__ __forceinline__ void load(const float* p, double* o) {
    widen(ld_stream(reinterpret_cast<const uint4*>(p)), o);
  }
};
template <> struct VecLoad<double, 2> {
  static __device__ __forceinline__ void widen(uint4 v, double* o) {
    o[0] = __hiloint2double(int(v.y), int(v.x));
    o[1] = __hiloint2double(int(v.w), int(v.z));
  }
  static __device__ __forceinline__ void load(const double* p, double* o) {
    widen(ld_stream(reinterpret_cast<const uint4*>(p)), o);
  }
};
template <> struct VecLoad<int8_t, 16> {
  static __device__ __forceinline__ void widen(uint4 v, double* o) {
    const unsigned int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) o[4 * a + b] = double(int8_t((w[a] >> (8 * b)) & 0xff));
  }
  static __device__ __forceinline__ void load(const int8_t* p, double* o) {
    widen(ld_stream(reinterpret_cast<const uint4*>(p)), o);
  }
};
template <typename TX> struct VecLoad<TX, 1> {
  static __device__ __forceinline__ void widen(uint4, double*) {}
  static __device__ __forceinline__ void load(const TX* p, double* o) { o[0] = double(*p); }
};

template <typename TX> constexpr int vec_of() { return 16 / int(sizeof(TX)); }

// int8 byte k of w as an exact float: PRMT places (byte ^ 0x80) under the exponent of 2^23,
// the subtraction removes 2^23 + 128 (two full-rate instructions; no conversion unit).
__device__ __forceinline__ float i8_to_f32(unsigned int w_flipped, int k) {
  const unsigned int bits = __byte_perm(w_flipped, 0x4B000000u, unsigned(k) | (4u << 4) | (4u << 8) | (7u << 12));
  return __uint_as_float(bits) - 8388736.0f;
}

// ---------------------------------------------------------------------------
// scn m: partial xb over a column chunk, VEC rows per thread.
// grid = (row tiles, column splits); out slab s = parts + s*m.
// ---------------------------------------------------------------------------

constexpr int XB_THREADS = 256;
constexpr int XB_UNROLL = 4;

template <typename TX, typename TB, int VEC>
__global__ void __launch_bounds__(XB_THREADS)
xbeta_kernel(const TX* __restrict__ X, const TB* __restrict__ beta, int64_t m, int64_t n_loc,
             int64_t cols_per_split, double* __restrict__ parts) {
  const int64_t i0 = (int64_t(blockIdx.x) * XB_THREADS + threadIdx.x) * VEC;
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
  const bool full = i0 + VEC <= m;
  if (i0 < m) {
    int64_t j = j_begin;
    if (full) {
      for (; j + XB_UNROLL <= j_end; j += XB_UNROLL) {
        double x[XB_UNROLL][VEC];
        double b[XB_UNROLL];
#pragma unroll
        for (int u = 0; u < XB_UNROLL; ++u) {
          VecLoad<TX, VEC>::load(X + (j + u) * m + i0, x[u]);
          b[u] = double(__ldg(beta + j + u));
        }
#pragma unroll
        for (int u = 0; u < XB_UNROLL; ++u)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[v] = fma(x[u][v], b[u], acc[v]);
      }
      for (; j < j_end; ++j) {
        double x[VEC];
        VecLoad<TX, VEC>::load(X + j * m + i0, x);
        const double b = double(__ldg(beta + j));
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = fma(x[v], b, acc[v]);
      }
    } else {
      for (; j < j_end; ++j) {
        const double b = double(__ldg(beta + j));
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (i0 + v < m) acc[v] = fma(double(X[j * m + i0 + v]), b, acc[v]);
      }
    }
    double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      if (i0 + v < m) out[i0 + v] = acc[v];
  }
}

__global__ void sum_slabs_f64(const double* __restrict__ parts, int S, int64_t len, double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < len;
       e += int64_t(gridDim.x) * blockDim.x) {
    double acc = parts[e];
    for (int s = 1; s < S; ++s) acc += parts[int64_t(s) * len + e];
    dst[e] = acc;
  }
}

// packed genotypes (float32 or float64 arithmetic): the tensor-core gradient pass (genotype_tc.cu);
// BS_U2_TC=0 restores the CUDA-core ring kernel (A/B only)
static bool u2_tc() {
  static const bool on = [] {
    const char* e = getenv("BS_U2_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int xsize(int xdtype) { return xdtype == BS_F64 ? 8 : xdtype == BS_F32 ? 4 : 1; }  // BS_U2: 16 rows / word

namespace bs {
int launch_xbeta_u2(const void* P, const void* beta, bool f64, int64_t m, int64_t n_loc, int64_t splits,
                    int64_t cps, double* parts, int* splits_used, cudaStream_t st);
int64_t u2_grad_tc_workspace(int64_t m);
bool launch_grad_u2_tc(const void* P, const double* v, int64_t m, int64_t n_loc, double* out, const int* flags,
                       Workspace& ws, cudaStream_t st, int* rc, bool f64);
bool launch_xbeta_u2t_tc(const void* Q, const float* beta, int64_t m, int64_t n_loc, double* out, Workspace& ws,
                         cudaStream_t st, int* rc);
bool launch_xbeta_u2t_tc(const void* Q, const double* beta, int64_t m, int64_t n_loc, double* out, Workspace& ws,
                         cudaStream_t st, int* rc);
int launch_grad_u2(const void* P, bool f64, const double* v, int64_t m, int64_t n_loc, int groups, int segs,
                   int64_t cpg, double* parts, const int* flags, cudaStream_t st);
bool launch_xbeta_i8_ring(const int8_t* X, const float* beta, int64_t m, int64_t n_loc, int64_t splits,
                          double* parts, int* splits_used, cudaStream_t st);
bool launch_grad_i8_ring(const int8_t* X, const double* v, int64_t m, int64_t n_loc, int segs, double* parts,
                         const int* flags, cudaStream_t st);
}  // namespace bs

struct GrGrid {
  int groups, segs;
  int64_t cpg;
};
static GrGrid gr_grid(int64_t m, int64_t n_loc);

template <typename T>
__global__ void widen_f64_kernel(const T* __restrict__ x, int64_t n, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = double(x[i]);
}

struct XbGrid {
  int64_t tiles;
  int splits;
  int64_t cps;
  int vec;
};

static XbGrid xb_grid(int xdtype, int64_t m, int64_t n_loc, bool vec_ok) {
  XbGrid g;
  g.vec = vec_ok ? 16 / xsize(xdtype) : 1;
  g.tiles = std::max<int64_t>(1, ceil_div(m, int64_t(XB_THREADS) * g.vec));
  const int64_t want = int64_t(num_sms()) * 6;
  int64_t s = std::max<int64_t>(1, ceil_div(want, g.tiles));
  s = std::min<int64_t>(s, std::max<int64_t>(1, n_loc / 64));
  s = std::min<int64_t>(s, 128);
  g.cps = ceil_div(std::max<int64_t>(n_loc, 1), s);
  g.splits = int(ceil_div(std::max<int64_t>(n_loc, 1), g.cps));
  return g;
}

extern "C" int64_t bs_cox_xbeta_workspace(int xdtype, int64_t m, int64_t n_loc) {
  if (xdtype == BS_U2T) {  // the tensor-core pass, or the CUDA-core fallback (beta widened + slabs)
    const GrGrid g = gr_grid(n_loc, m);
    return std::max<int64_t>(u2_grad_tc_workspace(n_loc),
                             ws_bytes<double>(n_loc) + ws_bytes<double>(int64_t(g.segs) * std::max<int64_t>(m, 1)));
  }
  XbGrid g = xb_grid(xdtype, m, n_loc, false);  // vec=1 gives the most tiles, splits <= that case
  XbGrid h = xb_grid(xdtype, m, n_loc, true);
  return ws_bytes<double>(int64_t(std::max(g.splits, h.splits)) * m);
}

// scn m for int8 X with float32 arithmetic (the dtype of beta): 16 rows per thread (one
// 16-byte word per column), PRMT widening and packed f32x2 FMAs, float partial sums over
// 32-column blocks added into float64.
__global__ void __launch_bounds__(XB_THREADS)
xbeta_i8f_kernel(const int8_t* __restrict__ X, const float* __restrict__ beta, int64_t m, int64_t n_loc,
                 int64_t cols_per_split, double* __restrict__ parts) {
  typedef unsigned long long f2x;
  auto pack = [](float a, float b) {
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
  };
  auto fma2 = [](f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
  };
  auto add2 = [](f2x a, f2x b) {
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  };
  const int64_t i0 = (int64_t(blockIdx.x) * XB_THREADS + threadIdx.x) * 16;
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  if (i0 >= m) return;
  const f2x off = pack(-8388736.0f, -8388736.0f);
  double accd[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) accd[v] = 0.0;
  auto word = [&](uint4 w, float b, f2x* acc) {  // acc[8] pairs += x(16 rows) * b
    const unsigned int ww[4] = {w.x ^ 0x80808080u, w.y ^ 0x80808080u, w.z ^ 0x80808080u, w.w ^ 0x80808080u};
    const f2x bb = pack(b, b);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const unsigned int p0 = __byte_perm(ww[a], 0x4B000000u, 0x7440u), p1 = __byte_perm(ww[a], 0x4B000000u, 0x7441u);
      const unsigned int p2 = __byte_perm(ww[a], 0x4B000000u, 0x7442u), p3 = __byte_perm(ww[a], 0x4B000000u, 0x7443u);
      acc[2 * a] = fma2(add2(pack(__uint_as_float(p0), __uint_as_float(p1)), off), bb, acc[2 * a]);
      acc[2 * a + 1] = fma2(add2(pack(__uint_as_float(p2), __uint_as_float(p3)), off), bb, acc[2 * a + 1]);
    }
  };
  for (int64_t jb = j_begin; jb < j_end; jb += 32) {
    const int64_t je = min(j_end, jb + 32);
    f2x acc[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[v] = pack(0.f, 0.f);
    int64_t j = jb;
    for (; j + 4 <= je; j += 4) {
      uint4 w[4];
      float b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        w[u] = ld_stream(reinterpret_cast<const uint4*>(X + (j + u) * m + i0));
        b[u] = __ldg(beta + j + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) word(w[u], b[u], acc);
    }
    for (; j < je; ++j) word(ld_stream(reinterpret_cast<const uint4*>(X + j * m + i0)), __ldg(beta + j), acc);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[v]));
      accd[2 * v] += double(lo);
      accd[2 * v + 1] += double(hi);
    }
  }
  double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
  for (int v = 0; v < 16; ++v) out[i0 + v] = accd[v];
}

template <typename TX, typename TB>
static void launch_xbeta(const TX* X, const TB* beta, int64_t m, int64_t n_loc, const XbGrid& g, double* out,
                         cudaStream_t st) {
  dim3 grid(unsigned(g.tiles), unsigned(g.splits));
  constexpr int V = vec_of<TX>();
  if constexpr (sizeof(TX) == 1 && sizeof(TB) == 4) {
    if (g.vec == V) {  // int8 genotypes, float32 arithmetic: no per-element conversion unit work
      xbeta_i8f_kernel<<<grid, XB_THREADS, 0, st>>>(reinterpret_cast<const int8_t*>(X),
                                                    reinterpret_cast<const float*>(beta), m, n_loc, g.cps, out);
      return;
    }
  }
  if (g.vec == V)
    xbeta_kernel<TX, TB, V><<<grid, XB_THREADS, 0, st>>>(X, beta, m, n_loc, g.cps, out);
  else
    xbeta_kernel<TX, TB, 1><<<grid, XB_THREADS, 0, st>>>(X, beta, m, n_loc, g.cps, out);
}

extern "C" int bs_cox_xbeta(const void* X, int xdtype, const void* beta, int dtype, int64_t m, int64_t n_loc,
                            double* out, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (m < 0 || n_loc < 0) { set_error("bs_cox_xbeta: negative shape"); return BS_EINVAL; }
  if (m == 0) return BS_OK;
  if (n_loc == 0) return cudaMemsetAsync(out, 0, sizeof(double) * m, st) == cudaSuccess ? BS_OK : BS_ECUDA;
  if (xdtype == BS_U2T) {  // packed transpose: one tensor-core pass (genotype_tc.cu)
    if (dtype != BS_F32 && dtype != BS_F64) { set_error("bs_cox_xbeta: BS_U2T takes float32 or float64 beta"); return BS_EINVAL; }
    Workspace ws(work, work_bytes);
    int rc = BS_OK;
    const bool ok = dtype == BS_F32
                        ? launch_xbeta_u2t_tc(X, static_cast<const float*>(beta), m, n_loc, out, ws, st, &rc)
                        : launch_xbeta_u2t_tc(X, static_cast<const double*>(beta), m, n_loc, out, ws, st, &rc);
    if (ok) return rc;
    // no tcgen05 (BS_DISABLE_TCGEN05, another part) or a misaligned block: the CUDA-core packed
    // gradient kernel on the transpose computes the same sums, (X beta)_i = sum_j Q[j][i] beta_j
    Workspace wf(work, work_bytes);
    const GrGrid g = gr_grid(n_loc, m);
    double* bd = wf.take<double>(n_loc);
    double* slabs = wf.take<double>(int64_t(g.segs) * m);
    if (!bd || !slabs) { set_error("bs_cox_xbeta: workspace too small"); return BS_EWORK; }
    const int wg = int(std::min<int64_t>(ceil_div(n_loc, 256), 1024));
    if (dtype == BS_F32) widen_f64_kernel<float><<<wg, 256, 0, st>>>(static_cast<const float*>(beta), n_loc, bd);
    else widen_f64_kernel<double><<<wg, 256, 0, st>>>(static_cast<const double*>(beta), n_loc, bd);
    launch_grad_u2(X, dtype == BS_F64, bd, n_loc, m, g.groups, g.segs, g.cpg, slabs, nullptr, st);
    if (g.segs > 1)
      sum_slabs_f64<<<int(std::min<int64_t>(ceil_div(m, 256), 2048)), 256, 0, st>>>(slabs, g.segs, m, out);
    else
      cudaMemcpyAsync(out, slabs, sizeof(double) * m, cudaMemcpyDeviceToDevice, st);
    return check_launch("bs_cox_xbeta", 3);
  }
  const bool vec_ok = xdtype == BS_U2 ||
                      ((m % (16 / xsize(xdtype)) == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0));
  XbGrid g = xb_grid(xdtype, m, n_loc, vec_ok);
  Workspace ws(work, work_bytes);
  double* parts = g.splits > 1 ? ws.take<double>(int64_t(g.splits) * m) : out;
  if (!parts) { set_error("bs_cox_xbeta: workspace too small"); return BS_EWORK; }
  if (xdtype == BS_U2) {  // 2-bit packed genotypes (genotype_u2.cu)
    if (dtype != BS_F32 && dtype != BS_F64) { set_error("bs_cox_xbeta: unsupported dtype %d", dtype); return BS_EINVAL; }
    int used = 1;
    launch_xbeta_u2(X, beta, dtype == BS_F64, m, n_loc, g.splits, g.cps, parts, &used, st);
    if (used > 1)
      sum_slabs_f64<<<int(std::min<int64_t>(ceil_div(m, 256), 2048)), 256, 0, st>>>(parts, used, m, out);
    else if (parts != out)
      cudaMemcpyAsync(out, parts, sizeof(double) * m, cudaMemcpyDeviceToDevice, st);
    return check_launch("bs_cox_xbeta", used > 1 ? 2 : 1);
  }
  if (xdtype == BS_I8 && dtype == BS_F32 && vec_ok) {  // genotypes, float32 arithmetic: TMA ring
    int used = 1;
    if (launch_xbeta_i8_ring(static_cast<const int8_t*>(X), static_cast<const float*>(beta), m, n_loc, g.splits, parts,
                             &used, st)) {
      if (used > 1)
        sum_slabs_f64<<<int(std::min<int64_t>(ceil_div(m, 256), 2048)), 256, 0, st>>>(parts, used, m, out);
      else if (parts != out)
        cudaMemcpyAsync(out, parts, sizeof(double) * m, cudaMemcpyDeviceToDevice, st);
      return check_launch("bs_cox_xbeta", used > 1 ? 2 : 1);
    }
  }
#define BS_XB(TXT, TBT) launch_xbeta<TXT, TBT>(static_cast<const TXT*>(X), static_cast<const TBT*>(beta), m, n_loc, g, parts, st)
  if (dtype == BS_F64) {
    if (xdtype == BS_F64) BS_XB(double, double);
    else if (xdtype == BS_F32) BS_XB(float, double);
    else if (xdtype == BS_I8) BS_XB(int8_t, double);
    else { set_error("bs_cox_xbeta: unsupported X dtype %d", xdtype); return BS_EINVAL; }
  } else if (dtype == BS_F32) {
    if (xdtype == BS_F32) BS_XB(float, float);
    else if (xdtype == BS_I8) BS_XB(int8_t, float);
    else if (xdtype == BS_F64) BS_XB(double, float);
    else { set_error("bs_cox_xbeta: unsupported X dtype %d", xdtype); return BS_EINVAL; }
  } else {
    set_error("bs_cox_xbeta: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
#undef BS_XB
  if (g.splits > 1)
    sum_slabs_f64<<<int(std::min<int64_t>(ceil_div(m, 256), 2048)), 256, 0, st>>>(parts, g.splits, m, out);
  return check_launch("bs_cox_xbeta", g.splits > 1 ? 2 : 1);
}

// ---------------------------------------------------------------------------
// Single-CTA inclusive scan helpers (float64, deterministic order).
// ---------------------------------------------------------------------------

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER;

// Exclusive block scan of one value per thread; returns exclusive prefix and total.
__device__ __forceinline__ double block_exscan(double v, double* sh, double* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    double s = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  const double warp_prefix = wid > 0 ? sh[wid - 1] : 0.0;
  *total = sh[(blockDim.x >> 5) - 1];
  return warp_prefix + x - v;
}

// risk: Xbeta = T(xb), w = exp(min(Xbeta, clamp)), W = cumsum(w), loglik.
template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
risk_kernel(const double* __restrict__ xb, const T* __restrict__ delta, const int64_t* __restrict__ cuts, int64_t m,
            double clamp, T* __restrict__ Xbeta, T* __restrict__ w, T* __restrict__ W, double* loglik,
            int* flags) {
  __shared__ double sh[32];
  __shared__ int sflag;
  if (*flags & BS_FLAG_NONFINITE) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  int myflag = 0;
  double carry = 0.0;
  for (int64_t t0 = 0; t0 < m; t0 += SCAN_TILE) {
    const int64_t base = t0 + int64_t(threadIdx.x) * SCAN_PER;
    double wv[SCAN_PER];
    double loc = 0.0;
#pragma unroll
    for (int u = 0; u < SCAN_PER; ++u) {
      const int64_t i = base + u;
      wv[u] = 0.0;
      if (i < m) {
        const T xt = T(xb[i]);
        Xbeta[i] = xt;
        T arg = xt;
        if (xt > T(clamp)) {  // solvers.py:383-385
          myflag |= BS_FLAG_CLAMPED;
          arg = T(clamp);
        }
        const T e = exp(arg);
        if (!isfinite(double(e))) myflag |= BS_FLAG_NONFINITE;
        w[i] = e;
        wv[u] = double(e);
        loc += wv[u];
      }
    }
    double total;
    double run = carry + block_exscan(loc, sh, &total);
#pragma unroll
    for (int u = 0; u < SCAN_PER; ++u) {
      const int64_t i = base + u;
      run += wv[u];
      if (i < m) W[i] = T(run);
    }
    carry += total;
  }
  if (myflag) atomicOr(&sflag, myflag);
  __syncthreads();  // W visible block-wide
  // loglik = sum delta (Xbeta - log W[cuts])   (solvers.py:398)
  double ll = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double dl = double(delta[i]);
    if (dl != 0.0) {
      const int64_t c = cuts ? cuts[i] : i;
      ll += dl * (double(Xbeta[i]) - log(double(W[c])));
    }
  }
  ll = block_sum(ll, sh);
  if (threadIdx.x == 0) {
    loglik[0] = ll;
    if (sflag) atomicOr(flags, sflag);
  }
}

// ---------------------------------------------------------------------------
// Multi-CTA versions of the scans for long m (C5: m = 400,000 took ~1.2 ms per
// iteration in the single-CTA kernels, paid on every GPU).  Tile t of SCAN_TILE
// elements is scanned by CTA t with the same block_exscan tree as the single-CTA
// kernels, and the carries are the same sequential sums of tile totals, so W and S
// are bitwise identical to the single-CTA results.  Phase 1: per-tile totals (and
// Xbeta, w); phase 2: one thread sums the totals in tile order; phase 3: the tiles'
// scans in parallel.  loglik is a fixed-grid reduction folded in CTA order.
// ---------------------------------------------------------------------------
constexpr int64_t SCAN_MULTI_MIN = 8 * SCAN_TILE;  // shorter vectors keep the single-CTA kernels
constexpr int LL_GRID = 128;

__global__ void scan_carry_kernel(const double* __restrict__ totals, int64_t tiles, double* __restrict__ carries) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double c = 0.0;
    for (int64_t t = 0; t < tiles; ++t) {
      carries[t] = c;
      c += totals[t];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
risk_tile_kernel(const double* __restrict__ xb, int64_t m, double clamp, T* __restrict__ Xbeta, T* __restrict__ w,
                 double* __restrict__ totals, int* __restrict__ newflags, const int* flags) {
  __shared__ double sh[32];
  if (*flags & BS_FLAG_NONFINITE) return;
  const int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_PER;
  int myflag = 0;
  double loc = 0.0;
#pragma unroll
  for (int u = 0; u < SCAN_PER; ++u) {
    const int64_t i = base + u;
    if (i < m) {
      const T xt = T(xb[i]);
      Xbeta[i] = xt;
      T arg = xt;
      if (xt > T(clamp)) {  // solvers.py:383-385
        myflag |= BS_FLAG_CLAMPED;
        arg = T(clamp);
      }
      const T e = exp(arg);
      if (!isfinite(double(e))) myflag |= BS_FLAG_NONFINITE;
      w[i] = e;
      loc += double(e);
    }
  }
  double total;
  block_exscan(loc, sh, &total);
  if (threadIdx.x == 0) totals[blockIdx.x] = total;
  if (myflag) atomicOr(newflags, myflag);
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
risk_scan_kernel(const T* __restrict__ w, int64_t m, const double* __restrict__ carries, T* __restrict__ W,
                 const int* flags) {
  __shared__ double sh[32];
  if (*flags & BS_FLAG_NONFINITE) return;
  const int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_PER;
  double wv[SCAN_PER];
  double loc = 0.0;
#pragma unroll
  for (int u = 0; u < SCAN_PER; ++u) {
    const int64_t i = base + u;
    wv[u] = i < m ? double(w[i]) : 0.0;
    loc += wv[u];
  }
  double total;
  double run = carries[blockIdx.x] + block_exscan(loc, sh, &total);
#pragma unroll
  for (int u = 0; u < SCAN_PER; ++u) {
    const int64_t i = base + u;
    run += wv[u];
    if (i < m) W[i] = T(run);
  }
}

// loglik = sum delta (Xbeta - log W[cuts]) (solvers.py:398); the last CTA folds the
// partials in CTA order and publishes the flags the tile pass raised.
template <typename T>
__global__ void __launch_bounds__(256)
loglik_kernel(const T* __restrict__ Xbeta, const T* __restrict__ W, const T* __restrict__ delta,
              const int64_t* __restrict__ cuts, int64_t m, double* __restrict__ parts, unsigned int* counter,
              int* newflags, double* loglik, int* flags) {
  __shared__ double sh[32];
  if (*flags & BS_FLAG_NONFINITE) return;
  double ll = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const double dl = double(delta[i]);
    if (dl != 0.0) {
      const int64_t c = cuts ? cuts[i] : i;
      ll += dl * (double(Xbeta[i]) - log(double(W[c])));
    }
  }
  ll = block_sum(ll, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = ll;
  if (last_block_done(counter) && threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned int k = 0; k < gridDim.x; ++k) t += parts[k];
    loglik[0] = t;
    const int nf = *newflags;
    if (nf) atomicOr(flags, nf);
    *newflags = 0;
  }
}

static int64_t risk_multi_ws(int64_t m) {
  const int64_t tiles = ceil_div(m, int64_t(SCAN_TILE));
  return 2 * ws_bytes<double>(tiles) + ws_bytes<double>(LL_GRID) + ws_bytes<unsigned int>(1) + ws_bytes<int>(1);
}

extern "C" int64_t bs_cox_risk_workspace(int64_t m) { return m >= SCAN_MULTI_MIN ? risk_multi_ws(m) : 0; }

template <typename T>
static void launch_risk_multi(const double* xb, const T* delta, const int64_t* cuts, int64_t m, double clamp,
                              T* Xbeta, T* w, T* W, double* loglik, int* flags, double* totals, double* carries,
                              double* llp, unsigned int* counter, int* newflags, cudaStream_t st) {
  const int64_t tiles = ceil_div(m, int64_t(SCAN_TILE));
  risk_tile_kernel<T><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(xb, m, clamp, Xbeta, w, totals, newflags, flags);
  scan_carry_kernel<<<1, 32, 0, st>>>(totals, tiles, carries);
  risk_scan_kernel<T><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(w, m, carries, W, flags);
  loglik_kernel<T><<<LL_GRID, 256, 0, st>>>(Xbeta, W, delta, cuts, m, llp, counter, newflags, loglik, flags);
}

extern "C" int bs_cox_risk(const double* xb, const void* delta, const int64_t* cuts, int dtype, int64_t m,
                           double clamp, void* Xbeta, void* w, void* W, double* loglik_dev, int* flags, void* work,
                           int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (m >= SCAN_MULTI_MIN && work && work_bytes >= risk_multi_ws(m) && (dtype == BS_F64 || dtype == BS_F32)) {
    Workspace ws(work, work_bytes);
    const int64_t tiles = ceil_div(m, int64_t(SCAN_TILE));
    unsigned int* counter = ws.take<unsigned int>(1);  // zeroed by the caller once, re-armed by the last CTA
    int* newflags = ws.take<int>(1);                    // idem
    double* totals = ws.take<double>(tiles);
    double* carries = ws.take<double>(tiles);
    double* llp = ws.take<double>(LL_GRID);
    if (dtype == BS_F64)
      launch_risk_multi<double>(xb, static_cast<const double*>(delta), cuts, m, clamp, static_cast<double*>(Xbeta),
                                static_cast<double*>(w), static_cast<double*>(W), loglik_dev, flags, totals, carries,
                                llp, counter, newflags, st);
    else
      launch_risk_multi<float>(xb, static_cast<const float*>(delta), cuts, m, clamp, static_cast<float*>(Xbeta),
                               static_cast<float*>(w), static_cast<float*>(W), loglik_dev, flags, totals, carries, llp,
                               counter, newflags, st);
    return check_launch("bs_cox_risk", 4);
  }
  if (dtype == BS_F64)
    risk_kernel<double><<<1, SCAN_THREADS, 0, st>>>(xb, static_cast<const double*>(delta), cuts, m, clamp,
                                                    static_cast<double*>(Xbeta), static_cast<double*>(w),
                                                    static_cast<double*>(W), loglik_dev, flags);
  else if (dtype == BS_F32)
    risk_kernel<float><<<1, SCAN_THREADS, 0, st>>>(xb, static_cast<const float*>(delta), cuts, m, clamp,
                                                   static_cast<float*>(Xbeta), static_cast<float*>(w),
                                                   static_cast<float*>(W), loglik_dev, flags);
  else {
    set_error("bs_cox_risk: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_cox_risk");
}

// ---------------------------------------------------------------------------
// pi_delta: suffix sums of c_j = delta_j / W[cuts_j] over [lo, hi) (single CTA),
// then pd_i = w_i * S[first(i)] with first(i) = min{j in [lo,hi): cuts_j >= i}.
// ---------------------------------------------------------------------------

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
suffix_kernel(const T* __restrict__ W, const T* __restrict__ delta, const int64_t* __restrict__ cuts, int64_t lo,
              int64_t hi, double* __restrict__ S, const int* flags) {
  __shared__ double sh[32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int64_t len = hi - lo;
  double carry = 0.0;
  // walk tiles from the end; within a tile, reversed index r = len-1-k
  for (int64_t t0 = 0; t0 < len; t0 += SCAN_TILE) {
    const int64_t base = t0 + int64_t(threadIdx.x) * SCAN_PER;
    double cv[SCAN_PER];
    double loc = 0.0;
#pragma unroll
    for (int u = 0; u < SCAN_PER; ++u) {
      const int64_t rk = base + u;  // position in reversed order
      cv[u] = 0.0;
      if (rk < len) {
        const int64_t j = hi - 1 - rk;
        const int64_t c = cuts ? cuts[j] : j;
        // solvers.py:412 contrib = delta / W[seg] in the storage type
        cv[u] = double(T(delta[j]) / W[c]);
        loc += cv[u];
      }
    }
    double total;
    double run = carry + block_exscan(loc, sh, &total);
#pragma unroll
    for (int u = 0; u < SCAN_PER; ++u) {
      const int64_t rk = base + u;
      run += cv[u];
      if (rk < len) S[hi - 1 - rk - lo] = run;
    }
    carry += total;
  }
}

template <typename T>
__global__ void pd_kernel(const T* __restrict__ w, const T* __restrict__ delta, const int64_t* __restrict__ cuts,
                          const double* __restrict__ S, int64_t m, int64_t lo, int64_t hi, T* __restrict__ pd,
                          double* __restrict__ dmpd, const int* flags) {
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    // first j in [lo, hi) with cuts_j >= i  (searchsorted left, solvers.py:414)
    int64_t a = lo, b = hi;
    if (cuts) {
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (cuts[mid] < i) a = mid + 1; else b = mid;
      }
    } else {
      a = i < lo ? lo : i;
    }
    T v = T(0);
    if (a < hi) v = T(S[a - lo]) * w[i];  // solvers.py:416-417
    pd[i] = v;
    if (dmpd) dmpd[i] = double(T(delta[i]) - v);  // solvers.py:446
  }
}

// suffix sums, multi-CTA (see the risk scans above): tile t covers reversed positions
// [t SCAN_TILE, (t+1) SCAN_TILE); phase 1 totals, phase 2 carries, phase 3 scans.
template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
suffix_tile_kernel(const T* __restrict__ W, const T* __restrict__ delta, const int64_t* __restrict__ cuts,
                   int64_t lo, int64_t hi, const double* __restrict__ carries, double* __restrict__ totals,
                   double* __restrict__ S, const int* flags) {
  __shared__ double sh[32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int64_t len = hi - lo;
  const int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_PER;
  double cv[SCAN_PER];
  double loc = 0.0;
#pragma unroll
  for (int u = 0; u < SCAN_PER; ++u) {
    const int64_t rk = base + u;
    cv[u] = 0.0;
    if (rk < len) {
      const int64_t j = hi - 1 - rk;
      const int64_t c = cuts ? cuts[j] : j;
      cv[u] = double(T(delta[j]) / W[c]);  // solvers.py:412
      loc += cv[u];
    }
  }
  double total;
  const double ex = block_exscan(loc, sh, &total);
  if (carries == nullptr) {  // phase 1
    if (threadIdx.x == 0) totals[blockIdx.x] = total;
    return;
  }
  double run = carries[blockIdx.x] + ex;
#pragma unroll
  for (int u = 0; u < SCAN_PER; ++u) {
    const int64_t rk = base + u;
    run += cv[u];
    if (rk < len) S[hi - 1 - rk - lo] = run;
  }
}

extern "C" int64_t bs_cox_pi_delta_workspace(int64_t m) {
  const int64_t tiles = ceil_div(std::max<int64_t>(m, 1), int64_t(SCAN_TILE));
  return ws_bytes<double>(m) + 2 * ws_bytes<double>(tiles);
}

extern "C" int bs_cox_pi_delta(const void* w, const void* W, const void* delta, const int64_t* cuts, int dtype,
                               int64_t m, int64_t lo, int64_t hi, void* pd, double* dmpd, const int* flags,
                               void* work, int64_t work_bytes, void* stream) {
  clear_error();
  if (lo < 0 || hi < lo || hi > m) {
    set_error("bs_cox_pi_delta: bad range [%lld, %lld) for m=%lld", (long long)lo, (long long)hi, (long long)m);
    return BS_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  if (m == 0) return BS_OK;
  Workspace ws(work, work_bytes);
  double* S = ws.take<double>(std::max<int64_t>(hi - lo, 1));
  if (!S) { set_error("bs_cox_pi_delta: workspace too small"); return BS_EWORK; }
  const int grid = int(std::min<int64_t>(ceil_div(m, 256), int64_t(num_sms()) * 4));
  const int64_t tiles = ceil_div(std::max<int64_t>(hi - lo, 1), int64_t(SCAN_TILE));
  double* totals = ws.take<double>(tiles);
  double* carries = ws.take<double>(tiles);
  const bool multi = hi - lo >= SCAN_MULTI_MIN && totals && carries;
  if (multi && (dtype == BS_F64 || dtype == BS_F32)) {
    if (dtype == BS_F64) {
      suffix_tile_kernel<double><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(
          static_cast<const double*>(W), static_cast<const double*>(delta), cuts, lo, hi, nullptr, totals, S, flags);
      scan_carry_kernel<<<1, 32, 0, st>>>(totals, tiles, carries);
      suffix_tile_kernel<double><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(
          static_cast<const double*>(W), static_cast<const double*>(delta), cuts, lo, hi, carries, totals, S, flags);
      pd_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), static_cast<const double*>(delta), cuts,
                                              S, m, lo, hi, static_cast<double*>(pd), dmpd, flags);
    } else {
      suffix_tile_kernel<float><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(
          static_cast<const float*>(W), static_cast<const float*>(delta), cuts, lo, hi, nullptr, totals, S, flags);
      scan_carry_kernel<<<1, 32, 0, st>>>(totals, tiles, carries);
      suffix_tile_kernel<float><<<unsigned(tiles), SCAN_THREADS, 0, st>>>(
          static_cast<const float*>(W), static_cast<const float*>(delta), cuts, lo, hi, carries, totals, S, flags);
      pd_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), static_cast<const float*>(delta), cuts, S,
                                             m, lo, hi, static_cast<float*>(pd), dmpd, flags);
    }
    return check_launch("bs_cox_pi_delta", 4);
  }
  if (dtype == BS_F64) {
    if (hi > lo)
      suffix_kernel<double><<<1, SCAN_THREADS, 0, st>>>(static_cast<const double*>(W),
                                                        static_cast<const double*>(delta), cuts, lo, hi, S, flags);
    pd_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), static_cast<const double*>(delta), cuts,
                                            S, m, lo, hi, static_cast<double*>(pd), dmpd, flags);
  } else if (dtype == BS_F32) {
    if (hi > lo)
      suffix_kernel<float><<<1, SCAN_THREADS, 0, st>>>(static_cast<const float*>(W), static_cast<const float*>(delta),
                                                       cuts, lo, hi, S, flags);
    pd_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), static_cast<const float*>(delta), cuts, S,
                                           m, lo, hi, static_cast<float*>(pd), dmpd, flags);
  } else {
    set_error("bs_cox_pi_delta: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_cox_pi_delta", hi > lo ? 2 : 1);
}

// ---------------------------------------------------------------------------
// scn p: column dot products over row segments; v = dmpd segment staged in smem.
// grid = (column groups, row segments); warps take columns round-robin.
// ---------------------------------------------------------------------------

constexpr int GR_THREADS = 256;
constexpr int GR_SEG = 8192;  // rows per segment (64 KB of float64 v in smem)

template <typename TX, int VEC>
__global__ void __launch_bounds__(GR_THREADS)
grad_kernel(const TX* __restrict__ X, const double* __restrict__ v, int64_t m, int64_t n_loc,
            int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  extern __shared__ __align__(16) double vs[];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r0 = int64_t(blockIdx.y) * GR_SEG;
  const int len = int(m - r0 < GR_SEG ? m - r0 : GR_SEG);
  for (int e = threadIdx.x; e < len; e += blockDim.x) vs[e] = v[r0 + e];
  __syncthreads();
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  const int nvec = len / VEC;  // whole vectors; tail handled scalar
  for (int64_t j = c0 + wid; j < c1; j += GR_THREADS / 32) {
    const TX* col = X + j * m + r0;
    double acc0 = 0.0, acc1 = 0.0;
    int e = lane;
    // eight 16-byte loads in flight per lane (a warp streams one column); raw words are
    // held until all eight have been issued, then widened and accumulated in order
    if constexpr (VEC > 1)
    for (; e + 224 < nvec; e += 256) {
      uint4 w[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) w[t] = ld_stream(reinterpret_cast<const uint4*>(col + (e + 32 * t) * VEC));
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        double xv[VEC];
        VecLoad<TX, VEC>::widen(w[t], xv);
#pragma unroll
        for (int u = 0; u < VEC; ++u) {
          if (t & 1) acc1 = fma(xv[u], vs[(e + 32 * t) * VEC + u], acc1);
          else acc0 = fma(xv[u], vs[(e + 32 * t) * VEC + u], acc0);
        }
      }
    }
    for (; e + 32 < nvec; e += 64) {
      double x0[VEC], x1[VEC];
      VecLoad<TX, VEC>::load(col + e * VEC, x0);
      VecLoad<TX, VEC>::load(col + (e + 32) * VEC, x1);
#pragma unroll
      for (int u = 0; u < VEC; ++u) {
        acc0 = fma(x0[u], vs[e * VEC + u], acc0);
        acc1 = fma(x1[u], vs[(e + 32) * VEC + u], acc1);
      }
    }
    for (; e < nvec; e += 32) {
      double x0[VEC];
      VecLoad<TX, VEC>::load(col + e * VEC, x0);
#pragma unroll
      for (int u = 0; u < VEC; ++u) acc0 = fma(x0[u], vs[e * VEC + u], acc0);
    }
    for (int t = nvec * VEC + lane; t < len; t += 32) acc1 = fma(double(col[t]), vs[t], acc1);
    const double s = warp_sum(acc0 + acc1);
    if (lane == 0) parts[int64_t(blockIdx.y) * n_loc + j] = s;
  }
}

// prox: grad_j = sum_s parts[s][j]; beta_j <- S_lam(beta_j + sigma grad_j); l1 = sum |beta|.
template <typename T>
__global__ void __launch_bounds__(256)
prox_kernel(const double* __restrict__ parts, int segs, int64_t n_loc, T* __restrict__ grad, T* __restrict__ beta,
            double sigma, double lam, int do_step, double* __restrict__ bparts, unsigned int* counter,
            double* __restrict__ l1, const int* flags) {
  __shared__ double sh[32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  double acc = 0.0;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n_loc; j += int64_t(gridDim.x) * blockDim.x) {
    double g = parts[j];
    for (int s = 1; s < segs; ++s) g += parts[int64_t(s) * n_loc + j];
    const T gt = T(g);
    grad[j] = gt;
    T b = beta[j];
    if (do_step) {
      // soft_threshold(b + sigma g, lam) = sign(x) max(|x| - lam, 0)   (solvers.py:48-51)
      const T x = b + T(sigma) * gt;
      const T mag = fabs(x) - T(lam);
      b = mag > T(0) ? copysign(mag, x) : T(0);
      beta[j] = b;
    }
    acc += fabs(double(b));
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) bparts[blockIdx.x] = acc;
  if (last_block_done(counter) && threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned int k = 0; k < gridDim.x; ++k) s += bparts[k];
    l1[0] = s;
  }
}

static GrGrid gr_grid(int64_t m, int64_t n_loc) {
  GrGrid g;
  g.segs = int(std::max<int64_t>(1, ceil_div(m, GR_SEG)));
  const int64_t want = int64_t(num_sms()) * 3;
  int64_t groups = std::max<int64_t>(1, ceil_div(want, g.segs));
  groups = std::min<int64_t>(groups, std::max<int64_t>(1, ceil_div(n_loc, 8)));
  g.cpg = ceil_div(std::max<int64_t>(n_loc, 1), groups);
  g.groups = int(ceil_div(std::max<int64_t>(n_loc, 1), g.cpg));
  return g;
}

static int prox_grid(int64_t n_loc) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_loc, 256), int64_t(num_sms()))));
}

extern "C" int64_t bs_cox_grad_workspace(int xdtype, int64_t m, int64_t n_loc) {
  GrGrid g = gr_grid(m, n_loc);
  return ws_bytes<double>(int64_t(g.segs) * std::max<int64_t>(n_loc, 1)) + ws_bytes<unsigned int>(1) +
         ws_bytes<double>(prox_grid(n_loc)) + (xdtype == BS_U2 ? u2_grad_tc_workspace(m) : 0);
}

// scn p for int8 X with float32 arithmetic.  Warp w of a CTA owns rows
// [w*1024, (w+1)*1024) of the CTA's 8192-row segment; lane l the 16-row words at
// 16l and 512 + 16l, whose v values stay in registers (as float) for every column, so
// the only memory traffic is the X stream: four columns at a time, eight 16-byte words
// in flight per lane.  Per genotype: PRMT + packed FADD/FMA (f32x2).  Warp partials are
// reduced across the eight warps in a fixed order per 32-column batch.
typedef unsigned long long i8_f2;
__device__ __forceinline__ i8_f2 i8_pack(float a, float b) {
  i8_f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float i8_hsum(i8_f2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a + b;
}
__device__ __forceinline__ i8_f2 i8_fma2(i8_f2 a, i8_f2 b, i8_f2 c) {
  i8_f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ i8_f2 i8_add2(i8_f2 a, i8_f2 b) {
  i8_f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// sum_k x_k v_k over the 16 int8 of word w (flipped by 0x80) against v[0..16)
__device__ __forceinline__ float i8_word_dot(uint4 w, const float* v) {
  const unsigned int ww[4] = {w.x ^ 0x80808080u, w.y ^ 0x80808080u, w.z ^ 0x80808080u, w.w ^ 0x80808080u};
  const i8_f2 off = i8_pack(-8388736.0f, -8388736.0f);
  i8_f2 s0 = i8_pack(0.f, 0.f), s1 = i8_pack(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const unsigned int p0 = __byte_perm(ww[a], 0x4B000000u, 0x7440u), p1 = __byte_perm(ww[a], 0x4B000000u, 0x7441u);
    const unsigned int p2 = __byte_perm(ww[a], 0x4B000000u, 0x7442u), p3 = __byte_perm(ww[a], 0x4B000000u, 0x7443u);
    const i8_f2 x01 = i8_add2(i8_pack(__uint_as_float(p0), __uint_as_float(p1)), off);
    const i8_f2 x23 = i8_add2(i8_pack(__uint_as_float(p2), __uint_as_float(p3)), off);
    s0 = i8_fma2(x01, i8_pack(v[4 * a], v[4 * a + 1]), s0);
    s1 = i8_fma2(x23, i8_pack(v[4 * a + 2], v[4 * a + 3]), s1);
  }
  return i8_hsum(s0) + i8_hsum(s1);
}

__global__ void __launch_bounds__(GR_THREADS)
grad_i8f_kernel(const int8_t* __restrict__ X, const double* __restrict__ v, int64_t m, int64_t n_loc,
                int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  __shared__ double red[GR_THREADS / 32][32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r0 = int64_t(blockIdx.y) * GR_SEG;
  const int64_t ra = r0 + int64_t(wid) * 1024 + 16 * lane, rb = ra + 512;  // this lane's two words
  const bool ha = ra < m, hb = rb < m;  // m % 16 == 0: a word is either whole or absent
  float va[16], vb[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    va[k] = ha ? float(v[ra + k]) : 0.f;
    vb[k] = hb ? float(v[rb + k]) : 0.f;
  }
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  const uint4 zero = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);  // int8 zeros once flipped back
  for (int64_t cb = c0; cb < c1; cb += 32) {
    const int nb = int(c1 - cb < 32 ? c1 - cb : 32);
    for (int jj = 0; jj < nb; jj += 4) {  // four columns: eight 16-byte words in flight per lane
      uint4 wa[4], wb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = cb + jj + u;
        const bool live = jj + u < nb;
        const int8_t* col = X + j * m;
        wa[u] = (live && ha) ? ld_stream(reinterpret_cast<const uint4*>(col + ra)) : zero;
        wb[u] = (live && hb) ? ld_stream(reinterpret_cast<const uint4*>(col + rb)) : zero;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // 32 rows per lane, then the warp's 1024 rows, in float; float64 across warps / segments
        const float sf = warp_sum(i8_word_dot(wa[u], va) + i8_word_dot(wb[u], vb));
        if (lane == 0 && jj + u < nb) red[wid][jj + u] = double(sf);
      }
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      double t = 0.0;
      for (int w = 0; w < GR_THREADS / 32; ++w) t += red[w][threadIdx.x];
      parts[int64_t(blockIdx.y) * n_loc + cb + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

template <typename TX>
static void launch_grad(const TX* X, const double* v, int64_t m, int64_t n_loc, const GrGrid& g, bool vec_ok,
                        double* parts, const int* flags, cudaStream_t st) {
  dim3 grid(unsigned(g.groups), unsigned(g.segs));
  constexpr int V = vec_of<TX>();
  const int smem = int(sizeof(double) * GR_SEG);
  if (vec_ok) smem_attr(grad_kernel<TX, V>, smem);
  else smem_attr(grad_kernel<TX, 1>, smem);
  if (vec_ok)
    grad_kernel<TX, V><<<grid, GR_THREADS, smem, st>>>(X, v, m, n_loc, g.cpg, parts, flags);
  else
    grad_kernel<TX, 1><<<grid, GR_THREADS, smem, st>>>(X, v, m, n_loc, g.cpg, parts, flags);
}

extern "C" int bs_cox_grad_step(const void* X, int xdtype, const double* dmpd, int dtype, int64_t m, int64_t n_loc,
                                void* grad, void* beta, double sigma, double lam, int do_step, double* l1_dev,
                                const int* flags, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (dtype != BS_F32 && dtype != BS_F64) { set_error("bs_cox_grad_step: unsupported dtype %d", dtype); return BS_EINVAL; }
  if (n_loc == 0) return cudaMemsetAsync(l1_dev, 0, sizeof(double), st) == cudaSuccess ? BS_OK : BS_ECUDA;
  Workspace ws(work, work_bytes);
  GrGrid g = gr_grid(m, n_loc);
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(int64_t(g.segs) * n_loc);
  const int pg = prox_grid(n_loc);
  double* bparts = ws.take<double>(pg);
  if (!parts || !counter || !bparts) { set_error("bs_cox_grad_step: workspace too small"); return BS_EWORK; }
  int segs_used = g.segs;
  if (m == 0) {
    if (cudaMemsetAsync(parts, 0, sizeof(double) * n_loc, st) != cudaSuccess) return BS_ECUDA;
  } else {
    const bool vec_ok = (m % (16 / xsize(xdtype)) == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
    int tc_rc = BS_OK;
    if (xdtype == BS_U2 && (dtype == BS_F32 || dtype == BS_F64) && u2_tc() &&
        launch_grad_u2_tc(X, dmpd, m, n_loc, parts, flags, ws, st, &tc_rc, dtype == BS_F64)) {
      // integer tensor-core pass (genotype_tc.cu): one slab
      if (tc_rc != BS_OK) return tc_rc;
      segs_used = 1;
    } else if (xdtype == BS_U2) {
      launch_grad_u2(X, dtype == BS_F64, dmpd, m, n_loc, g.groups, g.segs, g.cpg, parts, flags, st);
    } else if (xdtype == BS_F64) launch_grad<double>(static_cast<const double*>(X), dmpd, m, n_loc, g, vec_ok, parts, flags, st);
    else if (xdtype == BS_F32) launch_grad<float>(static_cast<const float*>(X), dmpd, m, n_loc, g, vec_ok, parts, flags, st);
    else if (xdtype == BS_I8 && dtype == BS_F32 && vec_ok &&
             launch_grad_i8_ring(static_cast<const int8_t*>(X), dmpd, m, n_loc, g.segs, parts, flags, st)) {
    } else if (xdtype == BS_I8 && dtype == BS_F32 && vec_ok) {  // genotypes, float32 arithmetic
      dim3 grid(unsigned(g.groups), unsigned(g.segs));
      grad_i8f_kernel<<<grid, GR_THREADS, 0, st>>>(static_cast<const int8_t*>(X), dmpd, m, n_loc, g.cpg, parts, flags);
    } else if (xdtype == BS_I8) launch_grad<int8_t>(static_cast<const int8_t*>(X), dmpd, m, n_loc, g, vec_ok, parts, flags, st);
    else { set_error("bs_cox_grad_step: unsupported X dtype %d", xdtype); return BS_EINVAL; }
  }
  const int segs = m == 0 ? 1 : segs_used;
  if (dtype == BS_F64)
    prox_kernel<double><<<pg, 256, 0, st>>>(parts, segs, n_loc, static_cast<double*>(grad), static_cast<double*>(beta),
                                            sigma, lam, do_step, bparts, counter, l1_dev, flags);
  else if (dtype == BS_F32)
    prox_kernel<float><<<pg, 256, 0, st>>>(parts, segs, n_loc, static_cast<float*>(grad), static_cast<float*>(beta),
                                           sigma, lam, do_step, bparts, counter, l1_dev, flags);
  else {
    set_error("bs_cox_grad_step: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_cox_grad_step", m > 0 ? 2 : 1);
}

__global__ void cox_objective_kernel(const double* loglik, const double* l1, double lam, double* out) {
  out[0] = -loglik[0] + lam * l1[0];
}

extern "C" int bs_cox_objective(const double* loglik_dev, const double* l1_dev, double lam, double* out_dev,
                                void* stream) {
  clear_error();
  cox_objective_kernel<<<1, 1, 0, as_stream(stream)>>>(loglik_dev, l1_dev, lam, out_dev);
  return check_launch("bs_cox_objective");
}

// ---------------------------------------------------------------------------
// Fused iteration pass: scn p of iteration k and scn m of iteration k+1 with ONE
// stream of X from HBM (solvers.py:443-449 then :436 of the next iteration).
//
// grad_j needs every row before beta_j(k+1) is known, and X beta(k+1) needs
// beta(k+1); the reference therefore reads X twice per iteration.  Here the
// columns are processed in waves of W; CTA c (one per SM, all co-resident: a
// cooperative launch) owns the row segment [c*seg, (c+1)*seg):
//   A(w)  a producer warp streams the wave's columns (this CTA's rows) from HBM
//         through a shared-memory ring (bulk copies, L2 evict_last); eight
//         consumer warps form the partial dots with v = delta - pd ->
//         partials[w % R][c][.], then arrive on the wave's grid counter
//   B(w-L) L = 2 waves later (the counter is long complete, so no one waits):
//         fold the column partials in CTA order (every CTA, identical values),
//         beta_new = S_lam(beta + sigma g), and xb_seg += X[seg, wave] beta_new
//         with the wave re-read from L2 by the same producer into a second ring
//         (3 waves x 148 CTAs x seg x W bytes stay resident: 38 MB at C4).
// HBM is read once per iteration; every fold has a fixed order (rows in a CTA,
// CTAs by index, columns in wave order), so results are deterministic.  Needs
// m * sizeof(X) % 16 == 0; otherwise the caller's two-pass path runs.
//
// Status (r01): correct (tests/test_cox_gpu.py, NCCL parity at 4 GPUs) but slower
// than the two-pass path at C4 (58 ms vs 28 ms per iteration), so cox_fit uses it
// only with BS_COX_FUSION=1.  ncu (profiles/r01_ncu_cox_fused_summary.txt): 27
// instructions per X element against ~3 DFMA/F2F/LDS of real work -- loop and
// address overhead of the runtime-bounded row/column loops with 8 consumer warps
// per SM; issue slots 27% busy.  Next: compile-time stage loops, v in registers,
// more consumer warps.
// ---------------------------------------------------------------------------

constexpr int FU_THREADS = 288;     // warp 0 producer, warps 1..8 consumers
constexpr int FU_CONS = 256;
constexpr int FU_RING = 8;          // partial / counter slots (>= 2L + 2)
constexpr int FU_LAG = 2;           // waves between A(w) and B(w)
constexpr int FU_CW = 8;            // columns per ring stage (one per consumer warp)
constexpr int FU_STAGES = 3;        // A ring (HBM stream)
constexpr int FU_BSTAGES = 2;       // B ring (L2 re-read of wave w - LAG)

__device__ __forceinline__ void fu_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void fu_wait(uint32_t bar, uint32_t parity) {  // traps after ~10 s
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (!done && (spin & 1023) == 1023) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ULL) __trap();
    }
  }
}
constexpr int FU_F32_KB = 4;                     // float4 row groups per consumer thread
constexpr int64_t FU_F32_SEGMAX = 1024 * FU_F32_KB;  // largest segment of the float32 fast path
typedef unsigned long long u2f;
__device__ __forceinline__ u2f f2_pack(float a, float b) {
  u2f r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(u2f v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u2f f2_fma(u2f a, u2f b, u2f c) {
  u2f d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u2f f2_add(u2f a, u2f b) {
  u2f d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float f2_hsum(u2f v) {
  float a, b;
  f2_unpack(v, a, b);
  return a + b;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <typename TX, typename TB, int W>
__global__ void __launch_bounds__(FU_THREADS, 1)
cox_fused_kernel(const TX* __restrict__ X, int64_t m, int64_t n_loc, int64_t seg, const double* __restrict__ v,
                 TB* __restrict__ grad, TB* __restrict__ beta, double sigma, double lam, double* __restrict__ xb_out,
                 double* __restrict__ partials, unsigned int* __restrict__ counters, const int* flags) {
  static_assert(W % FU_CW == 0, "a wave is whole ring stages");
  constexpr int QPW = W / FU_CW;  // ring stages per wave
  extern __shared__ __align__(128) uint8_t fu_smem[];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;  // every CTA sees the same flag
  const int G = int(gridDim.x), c = int(blockIdx.x), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = int64_t(c) * seg;
  const int rows = int(r0 >= m ? 0 : (m - r0 < seg ? m - r0 : seg));
  const int64_t stage_elems = int64_t(FU_CW) * seg;
  TX* ring = reinterpret_cast<TX*>(fu_smem);                                               // [STAGES][CW][seg]
  TX* bring = ring + FU_STAGES * stage_elems;                                               // [BSTAGES][CW][seg]
  double* pbuf = reinterpret_cast<double*>(fu_smem + (FU_STAGES + FU_BSTAGES) * stage_elems * sizeof(TX));  // [2][G][W]
  double* vseg = pbuf + 2 * int64_t(G) * W;                                                 // [seg]
  double* xbseg = vseg + seg;                                                               // [seg]
  double* bold = xbseg + seg;                                                               // [LAG+1][W]
  double* bnew = bold + (FU_LAG + 1) * W;                                                   // [W]
  double* gsum = bnew + W;                                                                  // [FU_CONS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(gsum + FU_CONS);  // full[S], empty[S], bfull[BS], bempty[BS], pfull[2], pempty[2]
  constexpr int PB0 = 2 * FU_STAGES + 2 * FU_BSTAGES;
  // float32 X with float32 arithmetic (the C4 setting) runs float fast paths: v as float in
  // smem next to the barriers, xb for the CTA's rows in registers (seg <= FU_F32_SEGMAX)
  constexpr bool F32 = std::is_same<TX, float>::value && std::is_same<TB, float>::value;
  float* vsegf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(bars + PB0 + 4) + 15) & ~uintptr_t(15));  // [seg]
  __shared__ double l1_sh[FU_CONS / 32];
  auto bar_u32 = [&](int i) { return static_cast<uint32_t>(__cvta_generic_to_shared(bars + i)); };
  const int64_t nwaves = (n_loc + W - 1) / W;
  if (tid == 0) {
    for (int i = 0; i < FU_STAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_u32(i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_u32(FU_STAGES + i)), "r"(FU_CONS / 32));
    }
    for (int i = 0; i < FU_BSTAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_u32(2 * FU_STAGES + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_u32(2 * FU_STAGES + FU_BSTAGES + i)),
                   "r"(FU_CONS / 32));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_u32(PB0 + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_u32(PB0 + 2 + i)), "r"(FU_CONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < rows; i += FU_THREADS) {
    vseg[i] = v[r0 + i];
    xbseg[i] = 0.0;
    if constexpr (F32) vsegf[i] = float(v[r0 + i]);
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: every stage of every wave, in order ----------------
    if (lane == 0) {
      uint64_t keep, drop;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(drop));
      const uint32_t bytes = uint32_t(rows) * uint32_t(sizeof(TX));
      // one ring stage: columns j0 .. j0+CW of this CTA's rows into `dst`, completing on `full`
      auto stage = [&](TX* dst, int64_t j0, uint32_t full, uint64_t pol) {
        const int nc = int(n_loc - j0 <= 0 ? 0 : (n_loc - j0 < FU_CW ? n_loc - j0 : FU_CW));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(bytes * uint32_t(nc))
                     : "memory");
        if (bytes)
          for (int jj = 0; jj < nc; ++jj)
            fu_bulk_load(static_cast<uint32_t>(__cvta_generic_to_shared(dst + int64_t(jj) * seg)),
                         X + (j0 + jj) * m + r0, bytes, full, pol);
      };
      int64_t k = 0, kb = 0;  // A / B stage sequences
      for (int64_t w = 0; w < nwaves + FU_LAG; ++w) {
        if (w < nwaves)
          for (int q = 0; q < QPW; ++q, ++k) {  // A(w): from HBM, kept in L2 for B
            const int s = int(k % FU_STAGES);
            fu_wait(bar_u32(FU_STAGES + s), uint32_t((k / FU_STAGES) & 1) ^ 1u);
            stage(ring + s * stage_elems, w * W + q * FU_CW, bar_u32(s), keep);
          }
        if (w >= FU_LAG) {
          // wave u's grid counter (all CTAs' A(u) partials are out), then its partial block
          const int64_t u = w - FU_LAG;
          unsigned int* ctr = counters + (u % FU_RING);
          const unsigned int target = unsigned(G) * unsigned(u / FU_RING + 1);
          uint64_t t0 = 0;
          for (uint32_t spin = 0; ld_acquire_u32(ctr) < target; ++spin) {
            __nanosleep(32);
            if ((spin & 4095) == 4095) {
              uint64_t now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
              if (t0 == 0) t0 = now;
              else if (now - t0 > 10000000000ULL) __trap();
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const int pb = int(u & 1);
          fu_wait(bar_u32(PB0 + 2 + pb), uint32_t((u >> 1) & 1) ^ 1u);
          const uint32_t pbytes = uint32_t(G) * W * 8u;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_u32(PB0 + pb)), "r"(pbytes)
                       : "memory");
          fu_bulk_load(static_cast<uint32_t>(__cvta_generic_to_shared(pbuf + int64_t(pb) * G * W)),
                       partials + int64_t(u % FU_RING) * G * W, pbytes, bar_u32(PB0 + pb), drop);
        }
        if (w >= FU_LAG)
          for (int q = 0; q < QPW; ++q, ++kb) {  // B(w - LAG): the same columns again, from L2
            const int s = int(kb % FU_BSTAGES);
            fu_wait(bar_u32(2 * FU_STAGES + FU_BSTAGES + s), uint32_t((kb / FU_BSTAGES) & 1) ^ 1u);
            stage(bring + s * stage_elems, (w - FU_LAG) * W + q * FU_CW, bar_u32(2 * FU_STAGES + s), drop);
          }
      }
    }
    return;  // the consumers never sync with warp 0 again
  }

  // ---------------- consumers (warps 1..8) ----------------
  const int ct = tid - 32, cw = warp - 1;  // consumer thread / warp index
  double l1 = 0.0;
  double xbr[F32 ? 4 * FU_F32_KB : 1];  // F32: rows 4ct + 1024k + e of the CTA's segment
#pragma unroll
  for (int e = 0; e < (F32 ? 4 * FU_F32_KB : 1); ++e) xbr[e] = 0.0;
  int64_t k = 0, kb = 0;
  auto cons_sync = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
  for (int64_t w = 0; w < nwaves + FU_LAG; ++w) {
    if (w < nwaves) {
      // ---- A(w) ----
      const int slot = int(w % FU_RING);
      if (ct < W && w * W + ct < n_loc) bold[int(w % (FU_LAG + 1)) * W + ct] = double(beta[w * W + ct]);
      double* part = partials + (int64_t(slot) * G + c) * W;
      for (int q = 0; q < QPW; ++q, ++k) {
        const int s = int(k % FU_STAGES);
        fu_wait(bar_u32(s), uint32_t((k / FU_STAGES) & 1));
        const int64_t j = w * W + q * FU_CW + cw;
        double acc = 0.0;
        if constexpr (F32) {
          if (j < n_loc) {
            const float* col = reinterpret_cast<const float*>(ring + s * stage_elems + int64_t(cw) * seg);
            u2f a0 = f2_pack(0.f, 0.f), a1 = f2_pack(0.f, 0.f);
            for (int i = 4 * lane; i < rows; i += 128) {
              const float4 x = *reinterpret_cast<const float4*>(col + i);
              const float4 vv = *reinterpret_cast<const float4*>(vsegf + i);
              a0 = f2_fma(f2_pack(x.x, x.y), f2_pack(vv.x, vv.y), a0);
              a1 = f2_fma(f2_pack(x.z, x.w), f2_pack(vv.z, vv.w), a1);
            }
            acc = double(warp_sum(f2_hsum(f2_add(a0, a1))));
          }
        } else if (j < n_loc) {
          const TX* col = ring + s * stage_elems + int64_t(cw) * seg;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int i = lane;
          const int full = rows - 96;
#pragma unroll 2
          for (; i < full; i += 128) {
            a0 = fma(double(col[i]), vseg[i], a0);
            a1 = fma(double(col[i + 32]), vseg[i + 32], a1);
            a2 = fma(double(col[i + 64]), vseg[i + 64], a2);
            a3 = fma(double(col[i + 96]), vseg[i + 96], a3);
          }
          for (; i < rows; i += 32) a0 = fma(double(col[i]), vseg[i], a0);
          acc = (a0 + a1) + (a2 + a3);
        }
        if constexpr (!F32) acc = warp_sum(acc);
        if (lane == 0) {
          part[q * FU_CW + cw] = acc;
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_u32(FU_STAGES + s)) : "memory");
        }
      }
      cons_sync();
      if (ct == 0) {
        __threadfence();
        atomicAdd(counters + slot, 1u);
      }
    }
    const int64_t u = w - FU_LAG;
    if (u >= 0) {
      // ---- B(u): the producer fetched wave u's partial block once its counter completed ----
      const int pb = int(u & 1);
      fu_wait(bar_u32(PB0 + pb), uint32_t((u >> 1) & 1));
      const double* pbu = pbuf + int64_t(pb) * G * W;
      const int nc = int(n_loc - u * W < W ? n_loc - u * W : W);
      {
        constexpr int GROUPS = FU_CONS / W;
        const int col = ct % W, grp = ct / W;
        const int chunk = (G + GROUPS - 1) / GROUPS;
        const int k0 = grp * chunk, k1 = min(G, k0 + chunk);
        double sacc = 0.0;
        for (int kk = k0; kk < k1; ++kk) sacc += pbu[kk * W + col];
        gsum[grp * W + col] = sacc;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_u32(PB0 + 2 + pb)) : "memory");
      cons_sync();
      if (ct < nc) {
        constexpr int GROUPS = FU_CONS / W;
        double g = 0.0;
        for (int kk = 0; kk < GROUPS; ++kk) g += gsum[kk * W + ct];
        const TB gt = TB(g);
        // soft_threshold(b + sigma g, lam) = sign(x) max(|x| - lam, 0)   (solvers.py:48-51, 447-449)
        const TB x = TB(bold[int(u % (FU_LAG + 1)) * W + ct]) + TB(sigma) * gt;
        const TB mag = fabs(x) - TB(lam);
        const TB bn = mag > TB(0) ? copysign(mag, x) : TB(0);
        bnew[ct] = double(bn);
        l1 += fabs(double(bn));
        if (c == 0) {
          grad[u * W + ct] = gt;
          beta[u * W + ct] = bn;
        }
      }
      cons_sync();
      for (int q = 0; q < QPW; ++q, ++kb) {
        const int s = int(kb % FU_BSTAGES);
        fu_wait(bar_u32(2 * FU_STAGES + s), uint32_t((kb / FU_BSTAGES) & 1));
        const TX* tile = bring + s * stage_elems;
        const int ncq = min(FU_CW, nc - q * FU_CW);
        if constexpr (F32) {
          float bq[FU_CW];
#pragma unroll
          for (int jj = 0; jj < FU_CW; ++jj) bq[jj] = jj < ncq ? float(bnew[q * FU_CW + jj]) : 0.f;
          const float* tf = reinterpret_cast<const float*>(tile);
#pragma unroll
          for (int kq = 0; kq < FU_F32_KB; ++kq) {
            const int i = 4 * ct + 1024 * kq;
            if (i < rows) {
              u2f lo = f2_pack(0.f, 0.f), hi = f2_pack(0.f, 0.f);
#pragma unroll
              for (int jj = 0; jj < FU_CW; ++jj) {  // absent columns: stale smem times 0
                const float4 x = *reinterpret_cast<const float4*>(tf + int64_t(jj) * seg + i);
                const u2f bb = f2_pack(bq[jj], bq[jj]);
                lo = f2_fma(f2_pack(x.x, x.y), bb, lo);
                hi = f2_fma(f2_pack(x.z, x.w), bb, hi);
              }
              float l0, l1_, h0, h1;
              f2_unpack(lo, l0, l1_);
              f2_unpack(hi, h0, h1);
              xbr[4 * kq] += double(l0);
              xbr[4 * kq + 1] += double(l1_);
              xbr[4 * kq + 2] += double(h0);
              xbr[4 * kq + 3] += double(h1);
            }
          }
        } else if (ncq == FU_CW) {  // full stage: the 8 coefficients in registers, compile-time column loop
          double bq[FU_CW];
#pragma unroll
          for (int jj = 0; jj < FU_CW; ++jj) bq[jj] = bnew[q * FU_CW + jj];
          const int sg = int(seg);
          for (int i = ct; i < rows; i += FU_CONS) {
            double acc = xbseg[i];
#pragma unroll
            for (int jj = 0; jj < FU_CW; ++jj) acc = fma(double(tile[jj * sg + i]), bq[jj], acc);
            xbseg[i] = acc;
          }
        } else {
          for (int i = ct; i < rows; i += FU_CONS) {
            double acc = xbseg[i];
            for (int jj = 0; jj < ncq; ++jj) acc = fma(double(tile[int64_t(jj) * seg + i]), bnew[q * FU_CW + jj], acc);
            xbseg[i] = acc;
          }
        }
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_u32(2 * FU_STAGES + FU_BSTAGES + s)) : "memory");
      }
      cons_sync();  // bnew / gsum / pbuf reusable
    }
  }
  if constexpr (F32) {
#pragma unroll
    for (int kq = 0; kq < FU_F32_KB; ++kq)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * ct + 1024 * kq + e;
        if (i < rows) xb_out[r0 + i] = xbr[4 * kq + e];
      }
  } else {
    for (int i = ct; i < rows; i += FU_CONS) xb_out[r0 + i] = xbseg[i];
  }
  if (c == 0) {  // ||beta_new||_1 in a fixed order: consumer threads by column residue, warps in order
    const double sm = warp_sum(l1);
    if (lane == 0) l1_sh[cw] = sm;
    cons_sync();
    if (ct == 0) {
      double t = 0.0;
      for (int kk = 0; kk < FU_CONS / 32; ++kk) t += l1_sh[kk];
      xb_out[m] = t;
    }
  }
}

struct FuPlan {
  bool ok;
  int grid, W;
  int64_t seg;
  size_t smem;
};

static FuPlan fu_plan(int xdtype, int64_t m, int64_t n_loc) {
  FuPlan p{false, 0, 0, 0, 0};
  const int es = xsize(xdtype);
  if (m <= 0 || n_loc <= 0 || (m * es) % 16) return p;
  int dev = 0, coop = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (!coop) return p;
  const int G = num_sms();
  const int64_t align = 16 / es;
  const int64_t seg = ceil_div(ceil_div(m, G), align) * align;
  const int64_t budget = int64_t(maxsm) - 2048;
  const int W = 32;
  const int64_t need = int64_t(FU_STAGES + FU_BSTAGES) * FU_CW * seg * es + 2 * int64_t(G) * W * 8 + 2 * seg * 8 +
                       (FU_LAG + 2) * W * 8 + FU_CONS * 8 + (2 * (FU_STAGES + FU_BSTAGES) + 4) * 8 + seg * 4 + 80;
  if (need > budget) return p;
  p.ok = true;
  p.grid = int(std::min<int64_t>(G, ceil_div(m, seg)));
  p.W = W;
  p.seg = seg;
  p.smem = size_t(need);
  return p;
}

template <typename TX, typename TB, int W>
static int launch_fused(const void* X, int64_t m, int64_t n_loc, const FuPlan& p, const double* v, void* grad,
                        void* beta, double sigma, double lam, double* xb_out, double* partials, unsigned int* counters,
                        const int* flags, cudaStream_t st) {
  auto kern = cox_fused_kernel<TX, TB, W>;
  smem_attr(kern, int(p.smem));
  const TX* Xp = static_cast<const TX*>(X);
  int64_t seg = p.seg;
  TB* g = static_cast<TB*>(grad);
  TB* b = static_cast<TB*>(beta);
  void* args[] = {&Xp, &m, &n_loc, &seg, &v, &g, &b, &sigma, &lam, &xb_out, &partials, &counters, &flags};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(p.grid), dim3(FU_THREADS),
                                              args, p.smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("bs_cox_grad_xbeta: cooperative launch failed: %s", cudaGetErrorString(e));
    return BS_ECUDA;
  }
  return BS_OK;
}

template <typename TX, typename TB>
static int dispatch_fused(const void* X, int64_t m, int64_t n_loc, const FuPlan& p, const double* v, void* grad,
                          void* beta, double sigma, double lam, double* xb_out, double* partials,
                          unsigned int* counters, const int* flags, cudaStream_t st) {
  return launch_fused<TX, TB, 32>(X, m, n_loc, p, v, grad, beta, sigma, lam, xb_out, partials, counters, flags, st);
}

static int64_t fused_ws(const FuPlan& p) {
  return ws_bytes<unsigned int>(FU_RING) + ws_bytes<double>(int64_t(FU_RING) * p.grid * p.W);
}

namespace bs {  // cox_fused2.cu: 2-D grid one-stream pass, float32 X and arithmetic
struct F2Plan {
  bool ok;
  int S, Gc, cfg;
  int64_t R, cpg;
  size_t smem;
};
F2Plan f2_plan(int64_t m, int64_t n_loc);
int64_t f2_workspace(const F2Plan& p, int64_t m);
int f2_launch(const F2Plan& p, const float* X, int64_t m, int64_t n_loc, const double* v, float* grad, float* beta,
              double sigma, double lam, double* xb_out, const int* flags, Workspace& ws, cudaStream_t st);
}  // namespace bs

extern "C" int64_t bs_cox_grad_xbeta_workspace(int xdtype, int64_t m, int64_t n_loc) {
  const FuPlan p = fu_plan(xdtype, m, n_loc);
  const int64_t two = bs_cox_grad_workspace(xdtype, m, n_loc) + bs_cox_xbeta_workspace(xdtype, m, n_loc) + 512;
  int64_t need = std::max<int64_t>(p.ok ? fused_ws(p) : 0, two);
  if (xdtype == BS_F32) {
    const F2Plan q = f2_plan(m, n_loc);
    if (q.ok) need = std::max<int64_t>(need, f2_workspace(q, m) + 512);
  }
  return need;
}

extern "C" int bs_cox_grad_xbeta(const void* X, int xdtype, const double* dmpd, int dtype, int64_t m, int64_t n_loc,
                                 void* grad, void* beta, double sigma, double lam, double* xb_out, const int* flags,
                                 int allow_fused, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (m < 0 || n_loc < 0) { set_error("bs_cox_grad_xbeta: negative shape"); return BS_EINVAL; }
  if (allow_fused && xdtype == BS_F32 && dtype == BS_F32 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    const F2Plan q = f2_plan(m, n_loc);
    if (q.ok) {
      Workspace ws(work, work_bytes);
      const int rc = f2_launch(q, static_cast<const float*>(X), m, n_loc, dmpd, static_cast<float*>(grad),
                               static_cast<float*>(beta), sigma, lam, xb_out, flags, ws, st);
      if (rc != -1000) return rc;  // F2_REFUSED
      // the cooperative launch was refused (e.g. SMs taken by another context): two passes
      return bs_cox_grad_xbeta(X, xdtype, dmpd, dtype, m, n_loc, grad, beta, sigma, lam, xb_out, flags, 0, work,
                               work_bytes, stream);
    }
  }
  const FuPlan p = fu_plan(xdtype, m, n_loc);
  const bool fuse = allow_fused && p.ok && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                    (dtype == BS_F32 || dtype == BS_F64) &&
                    (xdtype == BS_F32 || xdtype == BS_F64 || xdtype == BS_I8) &&
                    !(xdtype == BS_F32 && dtype == BS_F32 && p.seg > FU_F32_SEGMAX);
  if (!fuse) {
    // two passes: scn p + prox (l1 -> xb_out[m]), then scn m with the new beta
    Workspace ws(work, work_bytes);
    Workspace wg = ws.split(bs_cox_grad_workspace(xdtype, m, n_loc));
    Workspace wx = ws.rest();
    int rc = bs_cox_grad_step(X, xdtype, dmpd, dtype, m, n_loc, grad, beta, sigma, lam, 1, xb_out + m, flags, wg.base,
                              wg.size, stream);
    if (rc != BS_OK) return rc;
    return bs_cox_xbeta(X, xdtype, beta, dtype, m, n_loc, xb_out, wx.base, wx.size, stream);
  }
  Workspace ws(work, work_bytes);
  unsigned int* counters = ws.take<unsigned int>(FU_RING);
  double* partials = ws.take<double>(int64_t(FU_RING) * p.grid * p.W);
  if (!counters || !partials) { set_error("bs_cox_grad_xbeta: workspace too small"); return BS_EWORK; }
  if (cudaMemsetAsync(counters, 0, FU_RING * sizeof(unsigned int), st) != cudaSuccess) {
    set_error("bs_cox_grad_xbeta: cudaMemsetAsync failed");
    return BS_ECUDA;
  }
  int rc;
#define BS_FU(TXT, TBT) \
  rc = dispatch_fused<TXT, TBT>(X, m, n_loc, p, dmpd, grad, beta, sigma, lam, xb_out, partials, counters, flags, st)
  if (dtype == BS_F64) {
    if (xdtype == BS_F64) BS_FU(double, double);
    else if (xdtype == BS_F32) BS_FU(float, double);
    else BS_FU(int8_t, double);
  } else {
    if (xdtype == BS_F32) BS_FU(float, float);
    else if (xdtype == BS_F64) BS_FU(double, float);
    else BS_FU(int8_t, float);
  }
#undef BS_FU
  if (rc != BS_OK) return rc;
  return check_launch("bs_cox_grad_xbeta", 1);
}
