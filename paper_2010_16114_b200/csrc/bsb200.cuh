// Common device/host utilities for the B200 blockstat hot path.
//
// Every exported entry point (see include/bsb200.h) returns an int status and
// records a thread-local message retrievable with bs_last_error().  Nothing in
// this library allocates device memory: the caller (the Python host layer,
// which owns every buffer through torch) passes device pointers, sizes, a
// workspace and the cudaStream_t to launch on.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>
#include <math_constants.h>

#include "../../include/bsb200.h"

namespace bs {

void set_error(const char* fmt, ...);
void clear_error();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// One SM count per process (148 on B200); queried lazily.
int num_sms();

// Process-wide count of kernels this library launched (bs_launch_count).
void note_launches(int n);

// Launch-error check used right after every entry point's <<<>>> sequence;
// `n` is the number of kernels the entry point launched.
inline int check_launch(const char* what, int n = 1) {
  note_launches(n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return BS_ECUDA;
  }
  return BS_OK;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Raises a kernel's dynamic shared-memory limit to `bytes` on the CURRENT device
// (function attributes are per device: a process driving several GPUs -- the
// in-process backend -- needs it once per device).  Cached per (kernel, device).
void smem_attr(const void* kernel, int bytes);
template <typename K>
inline void smem_attr(K* kernel, int bytes) { smem_attr(reinterpret_cast<const void*>(kernel), bytes); }

// Most split-K slabs the tcgen05 GEMMs write (nmf_tc.cu).
constexpr int TC_MAX_SPLITS = 16;

// out = {min, sum} folded in order from np (min, sum) partial pairs (nmf.cu).
void launch_fold_minsq(const double* parts, int np, double* out, cudaStream_t st);

// dst[e] = sum_s parts[s*len + e], slabs folded in order (nmf.cu).
void launch_sum_slabs_f32(const float* parts, int S, int64_t len, float* dst, cudaStream_t st);

// Workspace bump allocator over a caller-provided buffer (256-B aligned).
struct Workspace {
  char* base;
  int64_t size;
  int64_t used = 0;
  Workspace(void* b, int64_t s) : base(static_cast<char*>(b)), size(s) {}
  // Carves a sub-workspace of `bytes` (so its counters sit at a fixed offset).
  Workspace split(int64_t bytes) {
    int64_t off = (used + 255) & ~int64_t(255);
    if (base == nullptr || off + bytes > size) return Workspace(nullptr, 0);
    used = off + bytes;
    return Workspace(base + off, bytes);
  }
  // Everything not yet handed out, as its own workspace.
  Workspace rest() {
    int64_t off = (used + 255) & ~int64_t(255);
    if (base == nullptr || off >= size) return Workspace(nullptr, 0);
    used = size;
    return Workspace(base + off, size - off);
  }
  template <typename T>
  T* take(int64_t count) {
    int64_t off = (used + 255) & ~int64_t(255);
    int64_t bytes = count * int64_t(sizeof(T));
    if (base == nullptr || off + bytes > size) return nullptr;
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
};

// Bytes needed for `count` items of T under the Workspace alignment rule.
template <typename T>
inline int64_t ws_bytes(int64_t count) {
  return ((count * int64_t(sizeof(T)) + 255) & ~int64_t(255)) + 256;
}

}  // namespace bs

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of one value per thread (blockDim.x multiple of 32, <= 1024).
// Result valid in every thread.  `sh` must hold 32 elements.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = (lane < nw) ? sh[lane] : T(0);
  r = warp_sum(r);
  return r;
}

// Streaming (evict-first) 16-byte loads for data read exactly once per pass.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Grid-stride walk over x[0..count) calling f(double) per element: 16-byte
// streaming loads, eight in flight per thread, scalar head/tail.  Every element is
// visited exactly once by exactly one thread; the per-thread order is fixed for
// a fixed grid, so folds built on it are deterministic.
template <typename T, typename F>
__device__ __forceinline__ void stream_elems(const T* __restrict__ x, int64_t count, F&& f) {
  constexpr int V = 16 / int(sizeof(T));
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  // scalar head up to 16-byte alignment
  const int64_t mis = (reinterpret_cast<uintptr_t>(x) & 15) / sizeof(T);
  const int64_t head = mis ? (count < V - mis ? count : V - mis) : 0;
  for (int64_t i = tid; i < head; i += nth) f(double(x[i]));
  const T* xa = x + head;
  const int64_t nvec = (count - head) / V;
  const uint4* xv = reinterpret_cast<const uint4*>(xa);
  int64_t v = tid;
  for (; v + 7 * nth < nvec; v += 8 * nth) {
    uint4 w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = ld_stream(xv + v + u * nth);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const T* e = reinterpret_cast<const T*>(&w[u]);
#pragma unroll
      for (int k = 0; k < V; ++k) f(double(e[k]));
    }
  }
  for (; v < nvec; v += nth) {
    const uint4 w = ld_stream(xv + v);
    const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int k = 0; k < V; ++k) f(double(e[k]));
  }
  for (int64_t i = head + nvec * V + tid; i < count; i += nth) f(double(x[i]));
}

// ReduceOp semantics in float64 (comm.py:60-65 ufuncs; NaN-propagating like np.min/np.max).
__device__ __forceinline__ double rop_neutral(int op) {
  switch (op) {
    case BS_SUM: return 0.0;
    case BS_PROD: return 1.0;
    case BS_MAX: return -CUDART_INF;
    default: return CUDART_INF;
  }
}
// NaN-propagating like numpy's np.min/np.max.
__device__ __forceinline__ double rop_apply(int op, double a, double b) {
  switch (op) {
    case BS_SUM: return a + b;
    case BS_PROD: return a * b;
    case BS_MAX: return (a != a || b != b) ? (a + b) : fmax(a, b);
    default: return (a != a || b != b) ? (a + b) : fmin(a, b);
  }
}
__device__ __forceinline__ double rtransform(int t, double v) {
  return t == BS_T_ABS ? fabs(v) : (t == BS_T_SQUARE ? v * v : v);
}


// Folds rows of `parts` [nparts][len] in order into out[len] (single block).
__device__ inline void fold_parts_block(const double* parts, int nparts, int len, int op, double* out) {
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    double acc = parts[i];
    for (int p = 1; p < nparts; ++p) acc = rop_apply(op, acc, parts[int64_t(p) * len + i]);
    out[i] = acc;
  }
}

// Last-block-done: returns true in every thread of the last block to finish.
__device__ __forceinline__ bool last_block_done(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;  // re-arm for the next launch
  }
  return am_last;
}

