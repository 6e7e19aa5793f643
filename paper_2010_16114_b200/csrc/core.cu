// Library plumbing plus the L1 primitives of distarray.py that the hot path
// needs on device: numpy-exact Philox draws (rand_fill), reduce_all folds, the
// in-process ascending-rank fold (comm.py:93-99), diag_get and the r x r Gram
// (scn d local part).
#include "bsb200.cuh"

#include <map>
#include <mutex>

#include <cfloat>
#include <cmath>
#include <atomic>
#include <mutex>
#include <string>

namespace bs {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
void clear_error() { g_err.clear(); }

static std::atomic<long long> g_launches{0};
void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

void smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  have = bytes;
}

}  // namespace bs

using namespace bs;

extern "C" const char* bs_last_error(void) { return g_err.c_str(); }
extern "C" int bs_abi_version(void) { return 1; }
extern "C" int bs_num_sms(void) { return num_sms(); }
extern "C" int64_t bs_launch_count(void) { return g_launches.load(); }

// A CUDA graph replay launches the kernels its capture recorded without calling back into the
// host code that counts them; the caller reports them here (solvers.py, NMF graphs).
extern "C" void bs_note_replayed_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// Philox4x64-10, numpy's counter layout (distarray.py:170-182 → numpy
// bit_generator philox.h): block b (0-based) is philox(counter = b + 1, key) and
// yields raw words 4b .. 4b+3.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c[0];
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c[0]);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c[2];
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0;
    const uint64_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// One thread per Philox block; elements [first, first+count) of the stream.
template <typename T>
__global__ void philox_uniform_kernel(T* __restrict__ out, int64_t count, int64_t first,
                                      uint64_t k0, uint64_t k1) {
  constexpr int PER = sizeof(T) == 8 ? 4 : 8;  // elements per 4-word block
  const int64_t b_first = first / PER;
  const int64_t b_last = (first + count - 1) / PER;
  for (int64_t b = b_first + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b <= b_last;
       b += int64_t(gridDim.x) * blockDim.x) {
    uint64_t c[4] = {uint64_t(b) + 1ULL, 0ULL, 0ULL, 0ULL};
    philox4x64_10(c, k0, k1);
    const int64_t e0 = b * PER;
#pragma unroll
    for (int l = 0; l < PER; ++l) {
      const int64_t e = e0 + l;
      if (e < first || e >= first + count) continue;
      T v;
      if constexpr (sizeof(T) == 8) {
        v = double(c[l] >> 11) * (1.0 / 9007199254740992.0);
      } else {
        const uint64_t wd = c[l >> 1];
        const uint32_t u = (l & 1) ? uint32_t(wd >> 32) : uint32_t(wd & 0xffffffffULL);
        v = float(u >> 8) * (1.0f / 16777216.0f);
      }
      out[e - first] = v;
    }
  }
}

extern "C" int bs_philox_uniform(void* out, int dtype, int64_t count, int64_t first,
                                 uint64_t key0, uint64_t key1, void* stream) {
  clear_error();
  if (count < 0 || first < 0) {
    set_error("bs_philox_uniform: negative count/first");
    return BS_EINVAL;
  }
  if (count == 0) return BS_OK;
  const int per = dtype == BS_F64 ? 4 : 8;
  const int64_t blocks = (first + count - 1) / per - first / per + 1;
  const int threads = 256;
  const int grid = int(std::min<int64_t>(ceil_div(blocks, threads), int64_t(num_sms()) * 16));
  if (dtype == BS_F64)
    philox_uniform_kernel<double><<<grid, threads, 0, as_stream(stream)>>>(
        static_cast<double*>(out), count, first, key0, key1);
  else if (dtype == BS_F32)
    philox_uniform_kernel<float><<<grid, threads, 0, as_stream(stream)>>>(
        static_cast<float*>(out), count, first, key0, key1);
  else {
    set_error("bs_philox_uniform: random fill requires a float dtype");
    return BS_EINVAL;
  }
  return check_launch("bs_philox_uniform");
}

// Counter-based standard normals (SURVEY §8(f)1 allows a documented GPU normal in place of
// numpy's ziggurat, whose data-dependent consumption defeats a counter-based restatement).
// Element e of the global stream takes Philox4x64-10 block (e / 2 + 1, 1, 0, 0) under the seed's
// key — counter word 1 set, so the words are disjoint from the uniform stream — and Box-Muller:
// u1 = ((w0 >> 11) + 0.5) 2^-53 in (0, 1), u2 = (w1 >> 11) 2^-53, r = sqrt(-2 ln u1),
// z = r cos(2 pi u2) for even e, r sin(2 pi u2) for odd e (float64 arithmetic, then rounded).
// Depends only on (key, e): a column split over any number of ranks draws the same matrix.
template <typename T>
__global__ void philox_normal_kernel(T* __restrict__ out, int64_t count, int64_t first, uint64_t k0, uint64_t k1) {
  const int64_t p_first = first / 2, p_last = (first + count - 1) / 2;
  for (int64_t p = p_first + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p <= p_last;
       p += int64_t(gridDim.x) * blockDim.x) {
    uint64_t c[4] = {uint64_t(p) + 1ULL, 1ULL, 0ULL, 0ULL};
    philox4x64_10(c, k0, k1);
    const double u1 = (double(c[0] >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = double(c[1] >> 11) * (1.0 / 9007199254740992.0);
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    const int64_t e0 = 2 * p;
    if (e0 >= first && e0 < first + count) out[e0 - first] = T(r * cs);
    if (e0 + 1 >= first && e0 + 1 < first + count) out[e0 + 1 - first] = T(r * sn);
  }
}

extern "C" int bs_philox_normal(void* out, int dtype, int64_t count, int64_t first, uint64_t key0, uint64_t key1,
                                void* stream) {
  clear_error();
  if (count < 0 || first < 0) {
    set_error("bs_philox_normal: negative count/first");
    return BS_EINVAL;
  }
  if (count == 0) return BS_OK;
  const int threads = 256;
  const int grid = int(std::min<int64_t>(ceil_div(count / 2 + 2, threads), int64_t(num_sms()) * 16));
  if (dtype == BS_F64)
    philox_normal_kernel<double><<<grid, threads, 0, as_stream(stream)>>>(static_cast<double*>(out), count, first,
                                                                         key0, key1);
  else if (dtype == BS_F32)
    philox_normal_kernel<float><<<grid, threads, 0, as_stream(stream)>>>(static_cast<float*>(out), count, first,
                                                                        key0, key1);
  else {
    set_error("bs_philox_normal: requires a float dtype");
    return BS_EINVAL;
  }
  return check_launch("bs_philox_normal");
}

// Counter-based genotypes: X[i, j] = [u1 < p_j] + [u2 < p_j] with u1, u2
// elements 2e, 2e+1 (e = j*m + i, j global) of Generator(Philox(key)).random(., float64) and
// p_j = maf[j_local].  Each element depends only on (key, i, j): any rank count / partition
// produces the same global matrix without a scatter.  One thread per Philox block = 2 elements.
__global__ void genotype_kernel(int8_t* __restrict__ X, const double* __restrict__ maf, int64_t m, int64_t lo,
                                int64_t n_loc, uint64_t k0, uint64_t k1) {
  const int64_t total = m * n_loc;  // local elements, column-major
  const int64_t e_first = lo * m;   // global index of local element 0
  const int64_t b_first = e_first / 2, b_last = (e_first + total - 1) / 2;
  for (int64_t b = b_first + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b <= b_last;
       b += int64_t(gridDim.x) * blockDim.x) {
    uint64_t c[4] = {uint64_t(b) + 1ULL, 0ULL, 0ULL, 0ULL};
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t e = 2 * b + h;  // global element; words 2e, 2e+1 = c[2h], c[2h+1]
      const int64_t el = e - e_first;
      if (el < 0 || el >= total) continue;
      const double p = maf[el / m];
      const double u1 = double(c[2 * h] >> 11) * (1.0 / 9007199254740992.0);
      const double u2 = double(c[2 * h + 1] >> 11) * (1.0 / 9007199254740992.0);
      X[el] = int8_t((u1 < p ? 1 : 0) + (u2 < p ? 1 : 0));
    }
  }
}

extern "C" int bs_genotype_fill(int8_t* X, const double* maf, int64_t m, int64_t lo, int64_t n_loc, uint64_t key0,
                                uint64_t key1, void* stream) {
  clear_error();
  if (m < 0 || lo < 0 || n_loc < 0) {
    set_error("bs_genotype_fill: negative shape");
    return BS_EINVAL;
  }
  if (m == 0 || n_loc == 0) return BS_OK;
  const int64_t blocks = (m * n_loc + 2) / 2 + 1;
  const int grid = int(std::min<int64_t>(ceil_div(blocks, 256), int64_t(num_sms()) * 16));
  genotype_kernel<<<grid, 256, 0, as_stream(stream)>>>(X, maf, m, lo, n_loc, key0, key1);
  return check_launch("bs_genotype_fill");
}

// ---------------------------------------------------------------------------
// reduce_all (distarray.py:335-348) — deterministic two-level fold in float64.
// ---------------------------------------------------------------------------

constexpr int RED_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(RED_THREADS)
reduce_kernel(const T* __restrict__ x, int64_t count, int op, int transform,
              double* __restrict__ parts, unsigned int* counter, double* out) {
  __shared__ double sh[32];
  double acc = rop_neutral(op);
  stream_elems(x, count, [&](double v) { acc = rop_apply(op, acc, rtransform(transform, v)); });
  // block tree in fixed order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = rop_apply(op, acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (lane == 0) sh[wid] = acc;
  __syncthreads();
  if (wid == 0) {
    double v = lane < (blockDim.x >> 5) ? sh[lane] : rop_neutral(op);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = rop_apply(op, v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) parts[blockIdx.x] = v;
  }
  if (last_block_done(counter)) {
    if (threadIdx.x == 0) {
      double r = parts[0];
      for (unsigned int b = 1; b < gridDim.x; ++b) r = rop_apply(op, r, parts[b]);
      out[0] = r;
    }
  }
}

static int reduce_grid(int64_t count) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, RED_THREADS * 8),
                                                     int64_t(num_sms()) * 4)));
}

extern "C" int64_t bs_reduce_workspace(int64_t count) {
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(reduce_grid(count));
}

namespace bs {
// Shared by NMF's scan: launches reduce over x with the given op/transform.
int launch_reduce(const void* x, int dtype, int64_t count, int op, int transform, double* out,
                  void* work, int64_t work_bytes, cudaStream_t st) {
  Workspace ws(work, work_bytes);
  const int grid = reduce_grid(count);
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(grid);
  if (!counter || !parts) {
    set_error("reduce: workspace too small (%lld bytes)", (long long)work_bytes);
    return BS_EWORK;
  }
  switch (dtype) {
    case BS_F32:
      reduce_kernel<float><<<grid, RED_THREADS, 0, st>>>(static_cast<const float*>(x), count, op,
                                                         transform, parts, counter, out);
      break;
    case BS_F64:
      reduce_kernel<double><<<grid, RED_THREADS, 0, st>>>(static_cast<const double*>(x), count, op,
                                                          transform, parts, counter, out);
      break;
    case BS_I64:
      reduce_kernel<long long><<<grid, RED_THREADS, 0, st>>>(static_cast<const long long*>(x),
                                                             count, op, transform, parts, counter, out);
      break;
    case BS_I8:
      reduce_kernel<int8_t><<<grid, RED_THREADS, 0, st>>>(static_cast<const int8_t*>(x), count, op,
                                                          transform, parts, counter, out);
      break;
    default:
      set_error("reduce: unsupported dtype %d", dtype);
      return BS_EINVAL;
  }
  return check_launch("reduce");
}
}  // namespace bs

extern "C" int bs_reduce(const void* x, int dtype, int64_t count, int op, int transform,
                         double* out_dev, void* work, int64_t work_bytes, void* stream) {
  clear_error();
  if (op < 0 || op > 3 || transform < 0 || transform > 2 || count < 0) {
    set_error("bs_reduce: bad op/transform/count");
    return BS_EINVAL;
  }
  return launch_reduce(x, dtype, count, op, transform, out_dev, work, work_bytes,
                       as_stream(stream));
}

// ---------------------------------------------------------------------------
// Ascending-rank fold (comm.py:93-99) for the in-process backend.
// ---------------------------------------------------------------------------

constexpr int MAX_FOLD = 64;
struct FoldSrcs {
  const void* p[MAX_FOLD];
};

template <typename T>
__device__ __forceinline__ T fold_op(int op, T a, T b) {
  switch (op) {
    case BS_SUM: return a + b;
    case BS_PROD: return a * b;
    case BS_MAX:
      if constexpr (sizeof(T) == 8 && T(0.5) != T(0)) {
        return (a != a || b != b) ? T(a + b) : (a > b ? a : b);
      } else {
        return (a != a || b != b) ? T(a + b) : (a > b ? a : b);
      }
    default: return (a != a || b != b) ? T(a + b) : (a < b ? a : b);
  }
}

template <typename T>
__global__ void fold_kernel(T* __restrict__ dst, FoldSrcs srcs, int nsrc, int64_t count, int op) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(srcs.p[0])[i];
    for (int r = 1; r < nsrc; ++r) acc = fold_op(op, acc, static_cast<const T*>(srcs.p[r])[i]);
    dst[i] = acc;
  }
}

extern "C" int bs_fold(void* dst, const void* const* srcs, int nsrc, int64_t count, int dtype,
                       int op, void* stream) {
  clear_error();
  if (nsrc < 1 || nsrc > MAX_FOLD || count < 0 || op < 0 || op > 3) {
    set_error("bs_fold: bad nsrc/count/op");
    return BS_EINVAL;
  }
  if (count == 0) return BS_OK;
  FoldSrcs s{};
  for (int r = 0; r < nsrc; ++r) s.p[r] = srcs[r];
  const int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(num_sms()) * 8));
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case BS_F32: fold_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(dst), s, nsrc, count, op); break;
    case BS_F64: fold_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(dst), s, nsrc, count, op); break;
    case BS_I64: fold_kernel<long long><<<grid, 256, 0, st>>>(static_cast<long long*>(dst), s, nsrc, count, op); break;
    default: set_error("bs_fold: unsupported dtype %d", dtype); return BS_EINVAL;
  }
  return check_launch("bs_fold");
}

// ---------------------------------------------------------------------------
// diag_get (distlinalg.py:97-99)
// ---------------------------------------------------------------------------

template <typename T>
__global__ void diag_get_kernel(const T* __restrict__ M, int64_t rows, int64_t lo, int64_t n_loc,
                                T* __restrict__ out) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n_loc;
       k += int64_t(gridDim.x) * blockDim.x)
    out[k] = M[k * rows + lo + k];
}

extern "C" int bs_diag_get(const void* M, int dtype, int64_t rows, int64_t lo, int64_t n_loc,
                           void* out, void* stream) {
  clear_error();
  if (n_loc == 0) return BS_OK;
  if (lo < 0 || lo + n_loc > rows) {
    set_error("bs_diag_get: owned range [%lld, %lld) outside %lld rows", (long long)lo,
              (long long)(lo + n_loc), (long long)rows);
    return BS_EINVAL;
  }
  const int grid = int(std::min<int64_t>(ceil_div(n_loc, 256), 1024));
  if (dtype == BS_F64)
    diag_get_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const double*>(M), rows,
                                                                 lo, n_loc, static_cast<double*>(out));
  else if (dtype == BS_F32)
    diag_get_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const float*>(M), rows,
                                                                lo, n_loc, static_cast<float*>(out));
  else {
    set_error("bs_diag_get: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("bs_diag_get");
}

// ---------------------------------------------------------------------------
// r x r Gram of a column-split r x ncols block (scn d local part), float64.
// Each block folds a contiguous column range into a private r x r partial;
// the last block sums the partials in block order (deterministic).
// ---------------------------------------------------------------------------

constexpr int GRAM_COLS = 64;  // columns staged per smem tile
constexpr int GRAM_MAXR = 128;

template <typename T>
__global__ void __launch_bounds__(256)
gram_kernel(const T* __restrict__ A, int r, int64_t ncols, int64_t cols_per_block,
            double* __restrict__ parts, unsigned int* counter, double* __restrict__ G) {
  extern __shared__ double tile[];  // [GRAM_COLS][r]
  const int rr = r * r;
  const int64_t c0 = blockIdx.x * cols_per_block;
  const int64_t c1 = min(ncols, c0 + cols_per_block);
  // each thread owns pairs p = tid, tid + 256, ... of the upper triangle (a<=b)
  constexpr int MAXP = (GRAM_MAXR * (GRAM_MAXR + 1) / 2 + 255) / 256;
  double acc[MAXP];
#pragma unroll
  for (int t = 0; t < MAXP; ++t) acc[t] = 0.0;
  const int npairs = r * (r + 1) / 2;
  int ia[MAXP], ib[MAXP];
#pragma unroll
  for (int t = 0; t < MAXP; ++t) {
    int a = 0, rem = threadIdx.x + t * 256;
    if (rem < npairs) {
      while (rem >= r - a) { rem -= r - a; ++a; }
    } else {
      a = 0; rem = -1;
    }
    ia[t] = a;
    ib[t] = a + rem;
  }
  for (int64_t cb = c0; cb < c1; cb += GRAM_COLS) {
    const int nc = int(c1 - cb < GRAM_COLS ? c1 - cb : GRAM_COLS);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * r; e += blockDim.x) tile[e] = double(A[cb * r + e]);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < MAXP; ++t) {
      const int p = threadIdx.x + t * 256;
      if (p < npairs) {
        const int a = ia[t], b = ib[t];
        double s = acc[t];
        for (int c = 0; c < nc; ++c) s = fma(tile[c * r + a], tile[c * r + b], s);
        acc[t] = s;
      }
    }
  }
  double* mine = parts + int64_t(blockIdx.x) * rr;
#pragma unroll
  for (int t = 0; t < MAXP; ++t) {
    const int p = threadIdx.x + t * 256;
    if (p < npairs) {
      const int a = ia[t], b = ib[t];
      mine[a * r + b] = acc[t];
      mine[b * r + a] = acc[t];
    }
  }
  if (last_block_done(counter)) fold_parts_block(parts, gridDim.x, rr, BS_SUM, G);
}

static int gram_grid(int r, int64_t ncols) {
  (void)r;
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(ncols, 512), int64_t(num_sms()) * 2)));
}

extern "C" int64_t bs_gram_workspace(int r, int64_t ncols) {
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(int64_t(gram_grid(r, ncols)) * r * r);
}

namespace bs {
int launch_gram(const void* A, int dtype, int r, int64_t ncols, double* G, Workspace& ws,
                cudaStream_t st) {
  if (r < 1 || r > GRAM_MAXR) {
    set_error("gram: rank %d outside [1, %d]", r, GRAM_MAXR);
    return BS_EINVAL;
  }
  if (ncols == 0) return cudaMemsetAsync(G, 0, sizeof(double) * r * r, st) == cudaSuccess ? BS_OK : BS_ECUDA;
  const int grid = gram_grid(r, ncols);
  unsigned int* counter = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(int64_t(grid) * r * r);
  if (!counter || !parts) {
    set_error("gram: workspace too small");
    return BS_EWORK;
  }
  const int64_t cpb = ceil_div(ncols, grid);
  const size_t smem = sizeof(double) * GRAM_COLS * r;
  smem_attr(gram_kernel<double>, int(sizeof(double) * GRAM_COLS * GRAM_MAXR));
  smem_attr(gram_kernel<float>, int(sizeof(double) * GRAM_COLS * GRAM_MAXR));
  if (dtype == BS_F64)
    gram_kernel<double><<<grid, 256, smem, st>>>(static_cast<const double*>(A), r, ncols, cpb, parts,
                                                  counter, G);
  else if (dtype == BS_F32)
    gram_kernel<float><<<grid, 256, smem, st>>>(static_cast<const float*>(A), r, ncols, cpb, parts,
                                                 counter, G);
  else {
    set_error("gram: unsupported dtype %d", dtype);
    return BS_EINVAL;
  }
  return check_launch("gram");
}
}  // namespace bs

extern "C" int bs_gram(const void* A, int dtype, int r, int64_t ncols, double* G, void* work,
                       int64_t work_bytes, void* stream) {
  clear_error();
  Workspace ws(work, work_bytes);
  return launch_gram(A, dtype, r, ncols, G, ws, as_stream(stream));
}
