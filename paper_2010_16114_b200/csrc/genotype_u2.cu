// 2-bit packed genotypes ("so C5 fits on 1 GPU"): X in {0,1,2} stored
// four per byte, PLINK-style dense packing, so the C5 matrix (400,000 x 500,000) takes
// 50 GB instead of 200 GB as int8.
//
// Layout (BS_U2): column j of the local block occupies ld = ceil(m / 64) * 16 bytes at
// byte offset j * ld; genotype i sits in byte i / 4, bits 2 (i % 4) .. +1 (row 0 in the
// low bits).  Pad bits are 0 (genotype 0, contributes nothing).  Each 32-bit word holds
// 16 consecutive rows.
//
// Arithmetic is float32 (the dtype of beta; int8 with float32 arithmetic is the C5
// setting).  A genotype field is widened without a conversion instruction: for the 16-bit
// half h (rows 8h .. 8h+7 of a word) field j sits under the exponent of 2^23, which gives
// 2^23 + g * 4^j exactly; one FADD removes 2^23 and the multiplier carries the 4^-j
// (exact powers of two).  Partial sums are float per word /
// 32-column block and float64 beyond, as in the int8 kernels (cox.cu).
#include "bsb200.cuh"
#include "tc_common.cuh"

#include <algorithm>

using namespace bs;
using namespace tc;

namespace {

constexpr int U2_THREADS = 256;

__device__ __forceinline__ int64_t u2_ld(int64_t m) { return ((m + 63) / 64) * 16; }  // bytes per column

// Fields are widened in pairs (rows 2p, 2p+1 of a 16-bit half) into one 64-bit register
// pair, then one packed FADD removes 2^23 from both and one packed FMA accumulates: per
// genotype one LOP3 + half an FADD2 + half an FFMA2 (+ one PRMT per 8 genotypes).
typedef unsigned long long u2_f2;
__device__ __forceinline__ u2_f2 u2_pack(float a, float b) {
  u2_f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void u2_unpack(u2_f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u2_f2 u2_fma2(u2_f2 a, u2_f2 b, u2_f2 c) {
  u2_f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u2_f2 u2_add2(u2_f2 a, u2_f2 b) {
  u2_f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// The 16-bit halves are first placed under the exponent of 2^23 with one PRMT each
// (bytes {w.b0, w.b1, 0x00, 0x4B} / {w.b2, w.b3, 0x00, 0x4B}); a field is then a single
// AND that keeps the exponent: (H & (0x4B000000 | 3 << 2q)) = 2^23 + g * 4^q as a float.
__device__ __forceinline__ unsigned int u2_half(uint32_t w, int h) {
  return __byte_perm(w, 0x4B000000u, h ? 0x7632u : 0x7610u);
}
__device__ __forceinline__ u2_f2 u2_pair(unsigned int H, int q) {  // (g_q 4^q, g_{q+1} 4^{q+1})
  const float a = __uint_as_float(H & (0x4B000000u | (3u << (2 * q))));
  const float b = __uint_as_float(H & (0x4B000000u | (3u << (2 * q + 2))));
  return u2_add2(u2_pack(a, b), u2_pack(-8388608.0f, -8388608.0f));
}
__device__ __forceinline__ float u2_scale(int q) { return __uint_as_float(uint32_t(127 - 2 * q) << 23); }  // 4^-q

// Subnormal widening (grad ring kernel): the field bits alone, g * 4^q at bit 2q of a float
// with a zero exponent, are the subnormal g * 4^q * 2^-149; an FMA with vs = v * 4^-q * 2^S
// gives g * v * 2^(S - 149) exactly rounded (FMA keeps subnormal inputs; no FTZ in this
// build), so no FADD is needed.  S is chosen per lane from its largest |v| so every nonzero
// product stays normal unless |v| is 2^103 below that maximum; the lane's sums are scaled
// back by 2^(149 - S) before the warp reduction (a power of two: exact).
__device__ __forceinline__ u2_f2 u2_word_dot_den(uint32_t w, const float* vs, u2_f2 acc) {
  const unsigned int hw[2] = {w, w >> 16};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < 8; q += 2)
      acc = u2_fma2(u2_pack(__uint_as_float(hw[h] & (3u << (2 * q))), __uint_as_float(hw[h] & (3u << (2 * q + 2)))),
                    u2_pack(vs[8 * h + q], vs[8 * h + q + 1]), acc);
  return acc;
}

// acc += sum over the 16 genotypes of word w times vs[0..16) (vs[8h + q] pre-scaled by 4^-q)
__device__ __forceinline__ u2_f2 u2_word_dot(uint32_t w, const float* vs, u2_f2 acc) {
  const unsigned int hw[2] = {u2_half(w, 0), u2_half(w, 1)};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < 8; q += 2) acc = u2_fma2(u2_pair(hw[h], q), u2_pack(vs[8 * h + q], vs[8 * h + q + 1]), acc);
  return acc;
}

// pack: one thread per 32-bit output word (16 rows of one column)
__global__ void pack_kernel(const int8_t* __restrict__ X, int64_t m, int64_t n_loc, uint32_t* __restrict__ P) {
  const int64_t wpc = u2_ld(m) / 4;  // words per column
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < wpc * n_loc;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / wpc, wi = e - j * wpc;
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t i = wi * 16 + k;
      const uint32_t g = i < m ? uint32_t(X[j * m + i]) & 3u : 0u;
      w |= g << (2 * k);
    }
    P[e] = w;
  }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ P, int64_t m, int64_t n_loc, int8_t* __restrict__ X) {
  const int64_t wpc = u2_ld(m) / 4;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * n_loc;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    X[e] = int8_t((P[j * wpc + i / 16] >> (2 * (i % 16))) & 3u);
  }
}

// Philox4x64-10 (numpy's counter layout), as in core.cu.
__device__ __forceinline__ void philox4x64_10u(uint64_t c[4], uint64_t k0, uint64_t k1) {
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

// Counter-based genotypes written packed (same values as bs_genotype_fill): one thread per
// output word = 16 rows = 8 Philox blocks (two uniforms per genotype, element e = j*m + i).
__global__ void fill_packed_kernel(uint32_t* __restrict__ P, const double* __restrict__ maf, int64_t m, int64_t lo,
                                   int64_t n_loc, uint64_t k0, uint64_t k1) {
  const int64_t wpc = u2_ld(m) / 4;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < wpc * n_loc;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t jl = e / wpc, wi = e - jl * wpc;
    const double p = maf[jl];
    uint32_t w = 0;
    for (int k = 0; k < 16; k += 2) {
      const int64_t i = wi * 16 + k;
      if (i >= m) break;
      const int64_t g0 = (lo + jl) * m + i;  // global element; rows i, i+1 are elements g0, g0+1
      // element g uses words 2g, 2g+1 = Philox block g/2, lanes 2(g%2), 2(g%2)+1
      const int64_t b0 = g0 / 2;
      uint64_t c[4] = {uint64_t(b0) + 1ULL, 0ULL, 0ULL, 0ULL};
      philox4x64_10u(c, k0, k1);
      uint64_t d[4] = {uint64_t(b0) + 2ULL, 0ULL, 0ULL, 0ULL};
      if (g0 & 1) philox4x64_10u(d, k0, k1);  // element g0+1 lies in the next block
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t g = g0 + h;
        if (i + h >= m) break;
        const uint64_t* blk = ((g / 2) == b0) ? c : d;
        const int l = int(g & 1);
        const double u1 = double(blk[2 * l] >> 11) * (1.0 / 9007199254740992.0);
        const double u2 = double(blk[2 * l + 1] >> 11) * (1.0 / 9007199254740992.0);
        const uint32_t gt = (u1 < p ? 1u : 0u) + (u2 < p ? 1u : 0u);
        w |= gt << (2 * (k + h));
      }
    }
    P[e] = w;
  }
}

// scn m: xb partial over a column chunk.  A thread owns the 16 rows of one word per column;
// columns go in batches of 8 with the next batch's words already in flight (register double
// buffer).  The accumulator of row 8h + q collects g * 4^q * b (the raw field times beta) and
// is scaled by 4^-q once at the end: powers of two, so the sum is the one of g * b.
constexpr int XU_CF = 8;  // columns per batch
__global__ void __launch_bounds__(U2_THREADS)
xbeta_u2_kernel(const uint32_t* __restrict__ P, const float* __restrict__ beta, int64_t m, int64_t n_loc,
                int64_t cols_per_split, double* __restrict__ parts) {
  const int64_t wpc = u2_ld(m) / 4;
  const int64_t wi = int64_t(blockIdx.x) * U2_THREADS + threadIdx.x;  // word within the column
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  if (wi * 16 >= m) return;
  const uint32_t* col = P + wi;
  auto load = [&](int64_t j, uint32_t* w, float* b) {
#pragma unroll
    for (int u = 0; u < XU_CF; ++u) {
      const bool live = j + u < j_end;
      w[u] = live ? __ldcs(col + (j + u) * wpc) : 0u;
      b[u] = live ? __ldg(beta + j + u) : 0.f;
    }
  };
  double accd[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) accd[v] = 0.0;
  uint32_t w[2][XU_CF];
  float b[2][XU_CF];
  load(j_begin, w[0], b[0]);
  for (int64_t jb = j_begin; jb < j_end; jb += 32) {
    u2_f2 acc[8];  // row pairs (2p, 2p+1), raw-field scale
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[v] = u2_pack(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 32 / XU_CF; ++k) {  // four batches; batch k sits in buffer k & 1
      load(jb + XU_CF * (k + 1), w[(k + 1) & 1], b[(k + 1) & 1]);  // next batch (or the next block's first)
#pragma unroll
      for (int u = 0; u < XU_CF; ++u) {
        const unsigned int hw[2] = {u2_half(w[k & 1][u], 0), u2_half(w[k & 1][u], 1)};
        const u2_f2 bb = u2_pack(b[k & 1][u], b[k & 1][u]);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          acc[q / 2] = u2_fma2(u2_pair(hw[0], q), bb, acc[q / 2]);
          acc[4 + q / 2] = u2_fma2(u2_pair(hw[1], q), bb, acc[4 + q / 2]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      float lo, hi;
      u2_unpack(acc[v], lo, hi);
      const int q = (2 * v) & 7;
      accd[2 * v] += double(lo * u2_scale(q));
      accd[2 * v + 1] += double(hi * u2_scale(q + 1));
    }
  }
  double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
  for (int v = 0; v < 16; ++v)
    if (wi * 16 + v < m) out[wi * 16 + v] = accd[v];
}

// After a lane holds one partial per column c = 0..31 in a[c], leave the warp total of
// column `lane` in a[0]: 31 shuffles for 32 columns (halve the live columns at each step).
__device__ __forceinline__ float transpose_reduce32(float (&a)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const float send = up ? a[k] : a[k + o];
      const float keep = up ? a[k + o] : a[k];
      a[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return a[0];
}

// scn p: warp w of a CTA owns rows [w*1024, (w+1)*1024) of the CTA's 8192-row segment, lane l
// the 32 rows (two words) at 32l; v for them stays in registers (float, pre-scaled by 4^-j)
// across all columns.  Columns go in batches of 8 (eight 8-byte loads per lane) with the next
// batch in flight; a lane keeps one float per column of a 32-column block and the warp
// folds them with one transpose-reduction.
constexpr int U2_SEG = 8192;
constexpr int GU_CF = 8;
__global__ void __launch_bounds__(U2_THREADS)
grad_u2_kernel(const uint32_t* __restrict__ P, const double* __restrict__ v, int64_t m, int64_t n_loc,
               int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  __shared__ float red[U2_THREADS / 32][32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t wpc = u2_ld(m) / 4;
  const int64_t r0 = int64_t(blockIdx.y) * U2_SEG;
  const int64_t rl = r0 + int64_t(wid) * 1024 + 32 * lane;  // this lane's first row
  const bool has = rl < m;
  float vs[32];  // v[rl + 16a + 8h + q] / 4^q  at index 16a + 8h + q
#pragma unroll
  for (int k = 0; k < 32; ++k) vs[k] = (rl + k < m) ? float(v[rl + k]) * u2_scale(k & 7) : 0.f;
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  const uint2* base = reinterpret_cast<const uint2*>(P + rl / 16);
  const int64_t stride = wpc / 2;  // uint2 per column
  auto load = [&](int64_t j, uint2* w) {
#pragma unroll
    for (int u = 0; u < GU_CF; ++u)
      w[u] = (has && j + u < c1) ? __ldcs(base + (j + u) * stride) : make_uint2(0u, 0u);
  };
  uint2 w[2][GU_CF];
  load(c0, w[0]);
  for (int64_t cb = c0; cb < c1; cb += 32) {
    float cs[32];
#pragma unroll
    for (int k = 0; k < 32 / GU_CF; ++k) {
      load(cb + GU_CF * (k + 1), w[(k + 1) & 1]);
#pragma unroll
      for (int u = 0; u < GU_CF; ++u) {
        float s0, s1;
        u2_unpack(u2_word_dot(w[k & 1][u].y, vs + 16, u2_word_dot(w[k & 1][u].x, vs, u2_pack(0.f, 0.f))), s0, s1);
        cs[GU_CF * k + u] = s0 + s1;
      }
    }
    red[wid][lane] = transpose_reduce32(cs, lane);  // column cb + lane, this warp's 1024 rows
    __syncthreads();
    const int nb = int(c1 - cb < 32 ? c1 - cb : 32);
    if (threadIdx.x < nb) {
      double t = 0.0;
      for (int w2 = 0; w2 < U2_THREADS / 32; ++w2) t += double(red[w2][threadIdx.x]);
      parts[int64_t(blockIdx.y) * n_loc + cb + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Ring variants (default): a producer warp streams the CTA's slice of each column into a
// shared-memory ring with cp.async.bulk (TMA 1-D, L2 evict-first) and mbarriers, so the
// X stream stays in flight while the eight consumer warps compute; the consumers read
// their words back with one LDS per column.  Same arithmetic and partial layouts as the
// register kernels above (BS_U2_RING=0 selects those).
// ---------------------------------------------------------------------------
constexpr int UR_THREADS = 288;  // warp 0 producer, warps 1..8 consumers
constexpr int UR_STAGES = 4;
constexpr int UR_STAGE_BYTES = 16384;
constexpr int UR_SMEM = UR_STAGES * UR_STAGE_BYTES + 2 * UR_STAGES * 8 + 2 * 8 * 32 * 4 + 64;

__device__ __forceinline__ void ur_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t ur_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void ur_consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Producer: batches of CF columns (CF * chunk <= UR_STAGE_BYTES) of `chunk` bytes starting at
// byte `off` of each column, columns [c0, c1).
template <int CF>
__device__ __forceinline__ void ur_produce(const uint8_t* P, int64_t ld, int64_t off, uint32_t chunk, int64_t c0,
                                           int64_t c1, uint32_t ring, uint32_t full, uint32_t empty) {
  const uint64_t pol = ur_evict_first();
  int k = 0;
  for (int64_t c = c0; c < c1; c += CF, ++k) {
    const int s = k % UR_STAGES;
    mbar_wait_sleep(empty + 8 * s, uint32_t((k / UR_STAGES) & 1) ^ 1u);
    const int nc = int(c1 - c < CF ? c1 - c : CF);
    mbar_expect_tx(full + 8 * s, uint32_t(nc) * chunk);
    for (int u = 0; u < nc; ++u)
      ur_bulk(ring + s * UR_STAGE_BYTES + u * (UR_STAGE_BYTES / CF), P + (c + u) * ld + off, chunk, full + 8 * s, pol);
  }
}

template <bool DEN>
__global__ void __launch_bounds__(UR_THREADS, 2)
grad_u2_ring_kernel(const uint32_t* __restrict__ P, const double* __restrict__ v, int64_t m, int64_t n_loc,
                    int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CF = 8;  // columns per stage, 2 KB each
  const uint32_t ring = smem_u32(smem);
  const uint32_t full = ring + UR_STAGES * UR_STAGE_BYTES, empty = full + 8 * UR_STAGES;
  float(*red)[32] = reinterpret_cast<float(*)[32]>(smem + UR_STAGES * UR_STAGE_BYTES + 16 * UR_STAGES);
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = u2_ld(m);
  const int64_t r0 = int64_t(blockIdx.y) * U2_SEG;
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  if (threadIdx.x == 0) {
    for (int s = 0; s < UR_STAGES; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const int64_t off = r0 / 4;
      ur_produce<CF>(reinterpret_cast<const uint8_t*>(P), ld, off, uint32_t(ld - off < U2_SEG / 4 ? ld - off : U2_SEG / 4), c0,
                     c1, ring, full, empty);
    }
    return;
  }
  const int wid = warp - 1;
  const int64_t rl = r0 + int64_t(wid) * 1024 + 32 * lane;
  float vs[32];
  float unscale = 1.f;
  if constexpr (DEN) {
    float vmax = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      vs[k] = (rl + k < m) ? float(v[rl + k]) : 0.f;
      vmax = fmaxf(vmax, fabsf(vs[k]));
    }
    int e = vmax > 0.f ? ilogbf(vmax) + 1 : -100;  // 2^e > max |v|
    e = max(-100, min(e, 104));
#pragma unroll
    for (int k = 0; k < 32; ++k) vs[k] = ldexpf(vs[k], 126 - e - 2 * (k & 7));
    unscale = ldexpf(1.f, 23 + e);  // 2^(149 - S), S = 126 - e
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) vs[k] = (rl + k < m) ? float(v[rl + k]) * u2_scale(k & 7) : 0.f;
  }
  const uint32_t my = ring + uint32_t(wid * 256 + lane * 8);  // this lane's 8 bytes of a 2 KB column slice
  int k = 0;  // stage counter
  for (int64_t cb = c0; cb < c1; cb += 32) {
    float cs[32];
#pragma unroll
    for (int b = 0; b < 32 / CF; ++b) {
      if (cb + CF * b < c1) {
        const int s = k % UR_STAGES;
        mbar_wait(full + 8 * s, uint32_t((k / UR_STAGES) & 1));
        uint2 w[CF];
#pragma unroll
        for (int u = 0; u < CF; ++u) {
          const uint32_t addr = my + s * UR_STAGE_BYTES + u * (UR_STAGE_BYTES / CF);
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[u].x), "=r"(w[u].y) : "r"(addr));
        }
        ++k;
#pragma unroll
        for (int u = 0; u < CF; ++u) {
          float s0, s1;
          if constexpr (DEN) {
            u2_unpack(u2_word_dot_den(w[u].y, vs + 16, u2_word_dot_den(w[u].x, vs, u2_pack(0.f, 0.f))), s0, s1);
            cs[CF * b + u] = (s0 + s1) * unscale;
          } else {
            u2_unpack(u2_word_dot(w[u].y, vs + 16, u2_word_dot(w[u].x, vs, u2_pack(0.f, 0.f))), s0, s1);
            cs[CF * b + u] = s0 + s1;
          }
        }
        // the stage is released only behind the math that consumed every word read from it
        // (an arrive right behind the loads does not wait for them to return)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * s);
      } else {
#pragma unroll
        for (int u = 0; u < CF; ++u) cs[CF * b + u] = 0.f;
      }
    }
    // red is double-buffered by 32-column block: the next block's writes go to the other
    // half, and the one after that follows this block's barrier, so one barrier suffices
    float(*rb)[32] = red + ((cb - c0) / 32 & 1) * 8;
    rb[wid][lane] = transpose_reduce32(cs, lane);
    ur_consumer_sync();
    const int nb = int(c1 - cb < 32 ? c1 - cb : 32);
    const int t = threadIdx.x - 32;
    if (t < nb) {
      double acc = 0.0;
      for (int w2 = 0; w2 < 8; ++w2) acc += double(rb[w2][t]);
      parts[int64_t(blockIdx.y) * n_loc + cb + t] = acc;
    }
  }
}

// scn m, ring variant: the CTA owns 4096 rows (256 words, 1 KB of each column); stages of
// 16 columns; consumer thread t keeps word t.
template <bool DEN>
__global__ void __launch_bounds__(UR_THREADS, 2)
xbeta_u2_ring_kernel(const uint32_t* __restrict__ P, const float* __restrict__ beta, int64_t m, int64_t n_loc,
                     int64_t cols_per_split, double* __restrict__ parts) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CF = 16;  // columns per stage, 1 KB each
  const uint32_t ring = smem_u32(smem);
  const uint32_t full = ring + UR_STAGES * UR_STAGE_BYTES, empty = full + 8 * UR_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = u2_ld(m);
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  const int64_t off = int64_t(blockIdx.x) * 1024;  // byte offset of the tile in a column
  if (threadIdx.x == 0) {
    for (int s = 0; s < UR_STAGES; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0)
      ur_produce<CF>(reinterpret_cast<const uint8_t*>(P), ld, off, uint32_t(ld - off < 1024 ? ld - off : 1024), j_begin,
                     j_end, ring, full, empty);
    return;
  }
  const int t = threadIdx.x - 32;
  const int64_t wi = int64_t(blockIdx.x) * 256 + t;
  const bool has = wi * 16 < m;
  // subnormal widening (see u2_word_dot_den): beta scaled by 2^S, S = 126 - e from the largest
  // |beta| of this CTA's columns; accumulator of row 8h + q scaled back by 2^(23 + e - 2q)
  float bscale = 1.f, fq[8];
  if constexpr (DEN) {
    float bmax = 0.f;
    for (int64_t j = j_begin + t; j < j_end; j += 256) bmax = fmaxf(bmax, fabsf(__ldg(beta + j)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    float* red = reinterpret_cast<float*>(smem + UR_STAGES * UR_STAGE_BYTES + 16 * UR_STAGES);
    if (lane == 0) red[warp - 1] = bmax;
    ur_consumer_sync();
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) bmax = fmaxf(bmax, red[w2]);
    // e >= -1 keeps 2^S a float; |beta| < 2^-104 then meets subnormal products (absolute
    // error below 2^-149 per product)
    int e = bmax > 0.f ? ilogbf(bmax) + 1 : -1;
    e = max(-1, min(e, 104));
    bscale = ldexpf(1.f, 126 - e);
#pragma unroll
    for (int q = 0; q < 8; ++q) fq[q] = ldexpf(1.f, 23 + e - 2 * q);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) fq[q] = u2_scale(q);
  }
  double accd[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) accd[q] = 0.0;
  int k = 0;
  for (int64_t jb = j_begin; jb < j_end; jb += 32) {
    u2_f2 acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = u2_pack(0.f, 0.f);
#pragma unroll
    for (int b = 0; b < 32 / CF; ++b) {
      const int64_t j = jb + CF * b;
      if (j < j_end) {
        const int s = k % UR_STAGES;
        mbar_wait(full + 8 * s, uint32_t((k / UR_STAGES) & 1));
        uint32_t w[CF];
#pragma unroll
        for (int u = 0; u < CF; ++u)
          w[u] = ld_shared_u32(ring + s * UR_STAGE_BYTES + u * (UR_STAGE_BYTES / CF) + 4 * t);
        ++k;
        const int nc = int(j_end - j < CF ? j_end - j : CF);
#pragma unroll
        for (int u = 0; u < CF; ++u) {
          const float bj = u < nc ? __ldg(beta + j + u) * bscale : 0.f;  // stale smem of absent columns times 0
          const u2_f2 bb = u2_pack(bj, bj);
          if constexpr (DEN) {
            const unsigned int hw[2] = {w[u], w[u] >> 16};
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
              acc[q / 2] = u2_fma2(u2_pack(__uint_as_float(hw[0] & (3u << (2 * q))),
                                           __uint_as_float(hw[0] & (3u << (2 * q + 2)))), bb, acc[q / 2]);
              acc[4 + q / 2] = u2_fma2(u2_pack(__uint_as_float(hw[1] & (3u << (2 * q))),
                                               __uint_as_float(hw[1] & (3u << (2 * q + 2)))), bb, acc[4 + q / 2]);
            }
          } else {
            const unsigned int hw[2] = {u2_half(w[u], 0), u2_half(w[u], 1)};
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
              acc[q / 2] = u2_fma2(u2_pair(hw[0], q), bb, acc[q / 2]);
              acc[4 + q / 2] = u2_fma2(u2_pair(hw[1], q), bb, acc[4 + q / 2]);
            }
          }
        }
        // the stage is released only behind the math that consumed every word read from it
        // (an arrive right behind the loads does not wait for them to return)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * s);
      }
    }
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) {
      float lo, hi;
      u2_unpack(acc[q2], lo, hi);
      const int q = (2 * q2) & 7;
      accd[2 * q2] += double(lo * fq[q]);
      accd[2 * q2 + 1] += double(hi * fq[q + 1]);
    }
  }
  if (!has) return;
  double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (wi * 16 + q < m) out[wi * 16 + q] = accd[q];
}

// ---------------------------------------------------------------------------
// int8 X with float32 arithmetic through the same TMA ring (cox.cu's register kernels
// xbeta_i8f / grad_i8f keep too little in flight: 4.0 / 5.4 TB/s).  Widening as there:
// one PRMT puts byte ^ 0x80 under the exponent of 2^23, a packed FADD removes 2^23 + 128
// (exact for every int8), a packed FMA accumulates.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u2_f2 i8r_pair(uint32_t ww, int k) {  // bytes k, k+1 of ww (already ^ 0x80808080)
  const float a = __uint_as_float(__byte_perm(ww, 0x4B000000u, 0x7440u + k));
  const float b = __uint_as_float(__byte_perm(ww, 0x4B000000u, 0x7440u + k + 1));
  return u2_add2(u2_pack(a, b), u2_pack(-8388736.0f, -8388736.0f));
}

// scn p: as grad_u2_ring_kernel; lane owns 32 consecutive rows (two 16-byte words per column)
__global__ void __launch_bounds__(UR_THREADS, 2)
grad_i8_ring_kernel(const int8_t* __restrict__ X, const double* __restrict__ v, int64_t m, int64_t n_loc,
                    int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CF = 2;  // columns per stage, 8 KB each
  const uint32_t ring = smem_u32(smem);
  const uint32_t full = ring + UR_STAGES * UR_STAGE_BYTES, empty = full + 8 * UR_STAGES;
  float(*red)[32] = reinterpret_cast<float(*)[32]>(smem + UR_STAGES * UR_STAGE_BYTES + 16 * UR_STAGES);
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = int64_t(blockIdx.y) * U2_SEG;
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  if (threadIdx.x == 0) {
    for (int s = 0; s < UR_STAGES; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0)
      ur_produce<CF>(reinterpret_cast<const uint8_t*>(X), m, r0, uint32_t(m - r0 < U2_SEG ? m - r0 : U2_SEG), c0, c1,
                     ring, full, empty);
    return;
  }
  const int wid = warp - 1;
  // lane owns the 16-row words at 16 lane and 512 + 16 lane of the warp's 1024 rows
  // (consecutive lanes, consecutive 16-byte words: conflict-free LDS.128)
  float vs[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int64_t r = r0 + int64_t(wid) * 1024 + 512 * (k >> 4) + 16 * lane + (k & 15);
    vs[k] = r < m ? float(v[r]) : 0.f;
  }
  const uint32_t my = ring + uint32_t(wid * 1024 + lane * 16);
  int k = 0;
  for (int64_t cb = c0; cb < c1; cb += 32) {
    float cs[32];
#pragma unroll
    for (int b = 0; b < 32 / CF; ++b) {
      if (cb + CF * b < c1) {
        const int s = k % UR_STAGES;
        mbar_wait(full + 8 * s, uint32_t((k / UR_STAGES) & 1));
        uint4 w[CF][2];
#pragma unroll
        for (int u = 0; u < CF; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) w[u][h] = ld_shared_v4(my + s * UR_STAGE_BYTES + u * (UR_STAGE_BYTES / CF) + 512 * h);
        ++k;
#pragma unroll
        for (int u = 0; u < CF; ++u) {
          u2_f2 acc = u2_pack(0.f, 0.f);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t q4[4] = {w[u][h].x ^ 0x80808080u, w[u][h].y ^ 0x80808080u, w[u][h].z ^ 0x80808080u,
                                    w[u][h].w ^ 0x80808080u};
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              acc = u2_fma2(i8r_pair(q4[a], 0), u2_pack(vs[16 * h + 4 * a], vs[16 * h + 4 * a + 1]), acc);
              acc = u2_fma2(i8r_pair(q4[a], 2), u2_pack(vs[16 * h + 4 * a + 2], vs[16 * h + 4 * a + 3]), acc);
            }
          }
          float s0, s1;
          u2_unpack(acc, s0, s1);
          cs[CF * b + u] = s0 + s1;
        }
        // the stage is released only behind the math that consumed every word read from it
        // (an arrive right behind the loads does not wait for them to return)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * s);
      } else {
#pragma unroll
        for (int u = 0; u < CF; ++u) cs[CF * b + u] = 0.f;
      }
    }
    red[wid][lane] = transpose_reduce32(cs, lane);
    ur_consumer_sync();
    const int nb = int(c1 - cb < 32 ? c1 - cb : 32);
    const int t = threadIdx.x - 32;
    if (t < nb) {
      double acc = 0.0;
      for (int w2 = 0; w2 < 8; ++w2) acc += double(red[w2][t]);
      parts[int64_t(blockIdx.y) * n_loc + cb + t] = acc;
    }
    ur_consumer_sync();
  }
}

// scn m: the CTA owns 4096 rows (one 16-byte word of 16 rows per consumer thread), stages of
// 4 columns x 4 KB
__global__ void __launch_bounds__(UR_THREADS, 2)
xbeta_i8_ring_kernel(const int8_t* __restrict__ X, const float* __restrict__ beta, int64_t m, int64_t n_loc,
                     int64_t cols_per_split, double* __restrict__ parts) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CF = 4;
  const uint32_t ring = smem_u32(smem);
  const uint32_t full = ring + UR_STAGES * UR_STAGE_BYTES, empty = full + 8 * UR_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  const int64_t off = int64_t(blockIdx.x) * 4096;
  if (threadIdx.x == 0) {
    for (int s = 0; s < UR_STAGES; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0)
      ur_produce<CF>(reinterpret_cast<const uint8_t*>(X), m, off, uint32_t(m - off < 4096 ? m - off : 4096), j_begin,
                     j_end, ring, full, empty);
    return;
  }
  const int t = threadIdx.x - 32;
  const int64_t i0 = off + 16 * int64_t(t);
  double accd[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) accd[q] = 0.0;
  int k = 0;
  for (int64_t jb = j_begin; jb < j_end; jb += 32) {
    u2_f2 acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = u2_pack(0.f, 0.f);
#pragma unroll
    for (int b = 0; b < 32 / CF; ++b) {
      const int64_t j = jb + CF * b;
      if (j < j_end) {
        const int s = k % UR_STAGES;
        mbar_wait(full + 8 * s, uint32_t((k / UR_STAGES) & 1));
        uint4 w[CF];
#pragma unroll
        for (int u = 0; u < CF; ++u) w[u] = ld_shared_v4(ring + s * UR_STAGE_BYTES + u * (UR_STAGE_BYTES / CF) + 16 * t);
        ++k;
        const int nc = int(j_end - j < CF ? j_end - j : CF);
#pragma unroll
        for (int u = 0; u < CF; ++u) {
          const float bj = u < nc ? __ldg(beta + j + u) : 0.f;
          const u2_f2 bb = u2_pack(bj, bj);
          const uint32_t q4[4] = {w[u].x ^ 0x80808080u, w[u].y ^ 0x80808080u, w[u].z ^ 0x80808080u,
                                  w[u].w ^ 0x80808080u};
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            acc[2 * a] = u2_fma2(i8r_pair(q4[a], 0), bb, acc[2 * a]);
            acc[2 * a + 1] = u2_fma2(i8r_pair(q4[a], 2), bb, acc[2 * a + 1]);
          }
        }
        // the stage is released only behind the math that consumed every word read from it
        // (an arrive right behind the loads does not wait for them to return)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * s);
      }
    }
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) {
      float lo, hi;
      u2_unpack(acc[q2], lo, hi);
      accd[2 * q2] += double(lo);
      accd[2 * q2 + 1] += double(hi);
    }
  }
  if (i0 >= m) return;
  double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (i0 + q < m) out[i0 + q] = accd[q];
}

static bool i8_ring() {
  static const bool on = [] {
    const char* e = getenv("BS_I8_RING");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool u2_den() {
  static const bool on = [] {
    const char* e = getenv("BS_U2_SUBNORMAL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool u2_ring() {
  static const bool on = [] {
    const char* e = getenv("BS_U2_RING");
    return !(e && e[0] == '0');
  }();
  return on;
}

// float64 arithmetic (the power iteration of opnorm, distlinalg.py:375-423, and Cox
// fits run in float64): plain shifts and conversions, same grids and partial layouts.
__global__ void __launch_bounds__(U2_THREADS)
xbeta_u2_f64_kernel(const uint32_t* __restrict__ P, const double* __restrict__ beta, int64_t m, int64_t n_loc,
                    int64_t cols_per_split, double* __restrict__ parts) {
  const int64_t wpc = u2_ld(m) / 4;
  const int64_t wi = int64_t(blockIdx.x) * U2_THREADS + threadIdx.x;
  const int64_t j_begin = int64_t(blockIdx.y) * cols_per_split;
  const int64_t j_end = min(n_loc, j_begin + cols_per_split);
  if (wi * 16 >= m) return;
  double acc[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) acc[v] = 0.0;
  for (int64_t j = j_begin; j < j_end; ++j) {
    const uint32_t w = __ldcs(P + j * wpc + wi);
    const double b = __ldg(beta + j);
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = fma(double((w >> (2 * k)) & 3u), b, acc[k]);
  }
  double* out = parts + int64_t(blockIdx.y) * m;
#pragma unroll
  for (int v = 0; v < 16; ++v)
    if (wi * 16 + v < m) out[wi * 16 + v] = acc[v];
}

__global__ void __launch_bounds__(U2_THREADS)
grad_u2_f64_kernel(const uint32_t* __restrict__ P, const double* __restrict__ v, int64_t m, int64_t n_loc,
                   int64_t cols_per_group, double* __restrict__ parts, const int* flags) {
  __shared__ double red[U2_THREADS / 32][32];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t wpc = u2_ld(m) / 4;
  const int64_t rl = int64_t(blockIdx.y) * U2_SEG + int64_t(wid) * 1024 + 32 * lane;
  const bool has = rl < m;
  double vr[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) vr[k] = (rl + k < m) ? v[rl + k] : 0.0;
  const int64_t c0 = int64_t(blockIdx.x) * cols_per_group;
  const int64_t c1 = min(n_loc, c0 + cols_per_group);
  for (int64_t cb = c0; cb < c1; cb += 32) {
    const int nb = int(c1 - cb < 32 ? c1 - cb : 32);
    for (int u = 0; u < nb; ++u) {
      const uint2 w = has ? __ldcs(reinterpret_cast<const uint2*>(P + (cb + u) * wpc + rl / 16)) : make_uint2(0u, 0u);
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) s = fma(double((w.x >> (2 * k)) & 3u), vr[k], s);
#pragma unroll
      for (int k = 0; k < 16; ++k) s = fma(double((w.y >> (2 * k)) & 3u), vr[16 + k], s);
      s = warp_sum(s);
      if (lane == 0) red[wid][u] = s;
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      double t = 0.0;
      for (int w2 = 0; w2 < U2_THREADS / 32; ++w2) t += red[w2][threadIdx.x];
      parts[int64_t(blockIdx.y) * n_loc + cb + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

}  // namespace

namespace bs {

int64_t u2_bytes_per_column(int64_t m) { return ((m + 63) / 64) * 16; }

// xb partial slabs for packed X (float32 arithmetic); grid (tiles, splits) chosen by caller.
int launch_xbeta_u2(const void* P, const void* beta, bool f64, int64_t m, int64_t n_loc, int64_t splits,
                    int64_t cps, double* parts, int* splits_used, cudaStream_t st) {
  const int64_t words = (m + 15) / 16;
  const int64_t tiles = ceil_div(words, U2_THREADS);
  if (!f64 && u2_ring()) {  // fewer splits: two ring CTAs per SM in one wave
    int64_t sp = std::max<int64_t>(1, (2 * int64_t(num_sms())) / tiles);
    sp = std::min<int64_t>({sp, splits, std::max<int64_t>(1, n_loc / 64)});
    const int64_t c = ceil_div(std::max<int64_t>(n_loc, 1), sp);
    sp = ceil_div(std::max<int64_t>(n_loc, 1), c);
    *splits_used = int(sp);
    const dim3 grid{unsigned(tiles), unsigned(sp)};
    if (u2_den()) {
      smem_attr(xbeta_u2_ring_kernel<true>, UR_SMEM);
      xbeta_u2_ring_kernel<true><<<grid, UR_THREADS, UR_SMEM, st>>>(static_cast<const uint32_t*>(P),
                                                                    static_cast<const float*>(beta), m, n_loc, c, parts);
    } else {
      smem_attr(xbeta_u2_ring_kernel<false>, UR_SMEM);
      xbeta_u2_ring_kernel<false><<<grid, UR_THREADS, UR_SMEM, st>>>(static_cast<const uint32_t*>(P),
                                                                     static_cast<const float*>(beta), m, n_loc, c,
                                                                     parts);
    }
    return BS_OK;
  }
  *splits_used = int(splits);
  const dim3 grid{unsigned(tiles), unsigned(splits)};
  if (f64)
    xbeta_u2_f64_kernel<<<grid, U2_THREADS, 0, st>>>(static_cast<const uint32_t*>(P),
                                                     static_cast<const double*>(beta), m, n_loc, cps, parts);
  else
    xbeta_u2_kernel<<<grid, U2_THREADS, 0, st>>>(static_cast<const uint32_t*>(P), static_cast<const float*>(beta),
                                                 m, n_loc, cps, parts);
  return BS_OK;
}

int launch_grad_u2(const void* P, bool f64, const double* v, int64_t m, int64_t n_loc, int groups, int segs,
                   int64_t cpg, double* parts, const int* flags, cudaStream_t st) {
  if (!f64 && u2_ring()) {  // two ring CTAs per SM, one wave
    int64_t gr = std::max<int64_t>(1, (2 * int64_t(num_sms())) / segs);
    gr = std::min<int64_t>(gr, std::max<int64_t>(1, ceil_div(n_loc, 8)));
    const int64_t c = ceil_div(std::max<int64_t>(n_loc, 1), gr);
    gr = ceil_div(std::max<int64_t>(n_loc, 1), c);
    const dim3 grid{unsigned(gr), unsigned(segs)};
    if (u2_den()) {
      smem_attr(grad_u2_ring_kernel<true>, UR_SMEM);
      grad_u2_ring_kernel<true><<<grid, UR_THREADS, UR_SMEM, st>>>(static_cast<const uint32_t*>(P), v, m, n_loc, c,
                                                                   parts, flags);
    } else {
      smem_attr(grad_u2_ring_kernel<false>, UR_SMEM);
      grad_u2_ring_kernel<false><<<grid, UR_THREADS, UR_SMEM, st>>>(static_cast<const uint32_t*>(P), v, m, n_loc, c,
                                                                    parts, flags);
    }
    return BS_OK;
  }
  const dim3 grid{unsigned(groups), unsigned(segs)};
  if (f64)
    grad_u2_f64_kernel<<<grid, U2_THREADS, 0, st>>>(static_cast<const uint32_t*>(P), v, m, n_loc, cpg, parts, flags);
  else
    grad_u2_kernel<<<grid, U2_THREADS, 0, st>>>(static_cast<const uint32_t*>(P), v, m, n_loc, cpg, parts, flags);
  return BS_OK;
}

// int8 X, float32 arithmetic, m % 16 == 0 and X 16-byte aligned: ring kernels; returns
// false (nothing launched) when disabled (BS_I8_RING=0) so the caller uses cox.cu's kernels.
bool launch_xbeta_i8_ring(const int8_t* X, const float* beta, int64_t m, int64_t n_loc, int64_t splits,
                          double* parts, int* splits_used, cudaStream_t st) {
  if (!i8_ring()) return false;
  const int64_t tiles = ceil_div(m, int64_t(4096));
  int64_t sp = std::max<int64_t>(1, (2 * int64_t(num_sms())) / tiles);
  sp = std::min<int64_t>({sp, splits, std::max<int64_t>(1, n_loc / 64)});
  const int64_t c = ceil_div(std::max<int64_t>(n_loc, 1), sp);
  sp = ceil_div(std::max<int64_t>(n_loc, 1), c);
  *splits_used = int(sp);
  smem_attr(xbeta_i8_ring_kernel, UR_SMEM);
  const dim3 grid{unsigned(tiles), unsigned(sp)};
  xbeta_i8_ring_kernel<<<grid, UR_THREADS, UR_SMEM, st>>>(X, beta, m, n_loc, c, parts);
  return true;
}

bool launch_grad_i8_ring(const int8_t* X, const double* v, int64_t m, int64_t n_loc, int segs, double* parts,
                         const int* flags, cudaStream_t st) {
  if (!i8_ring()) return false;
  int64_t gr = std::max<int64_t>(1, (2 * int64_t(num_sms())) / segs);
  gr = std::min<int64_t>(gr, std::max<int64_t>(1, ceil_div(n_loc, 8)));
  const int64_t c = ceil_div(std::max<int64_t>(n_loc, 1), gr);
  gr = ceil_div(std::max<int64_t>(n_loc, 1), c);
  smem_attr(grad_i8_ring_kernel, UR_SMEM);
  const dim3 grid{unsigned(gr), unsigned(segs)};
  grad_i8_ring_kernel<<<grid, UR_THREADS, UR_SMEM, st>>>(X, v, m, n_loc, c, parts, flags);
  return true;
}

}  // namespace bs

extern "C" int64_t bs_genotype_packed_bytes(int64_t m) { return bs::u2_bytes_per_column(m); }

extern "C" int bs_genotype_pack(const int8_t* X, int64_t m, int64_t n_loc, void* P, void* stream) {
  clear_error();
  if (m < 0 || n_loc < 0) { set_error("bs_genotype_pack: negative shape"); return BS_EINVAL; }
  if (m == 0 || n_loc == 0) return BS_OK;
  const int64_t words = u2_bytes_per_column(m) / 4 * n_loc;
  pack_kernel<<<int(std::min<int64_t>(ceil_div(words, 256), int64_t(num_sms()) * 16)), 256, 0, as_stream(stream)>>>(
      X, m, n_loc, static_cast<uint32_t*>(P));
  return check_launch("bs_genotype_pack");
}

namespace bs {
int launch_u2_transpose(const void* P, int64_t m, int64_t n, void* Q, cudaStream_t st);
}

extern "C" int bs_genotype_transpose_packed(const void* P, int64_t m, int64_t n_loc, void* Q, void* stream) {
  clear_error();
  if (m < 0 || n_loc < 0) { set_error("bs_genotype_transpose_packed: negative shape"); return BS_EINVAL; }
  if (m == 0 || n_loc == 0) return BS_OK;
  if ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15) {
    set_error("bs_genotype_transpose_packed: P and Q must be 16-byte aligned");
    return BS_EINVAL;
  }
  return bs::launch_u2_transpose(P, m, n_loc, Q, as_stream(stream));
}

extern "C" int bs_genotype_unpack(const void* P, int64_t m, int64_t n_loc, int8_t* X, void* stream) {
  clear_error();
  if (m < 0 || n_loc < 0) { set_error("bs_genotype_unpack: negative shape"); return BS_EINVAL; }
  if (m == 0 || n_loc == 0) return BS_OK;
  unpack_kernel<<<int(std::min<int64_t>(ceil_div(m * n_loc, 256), int64_t(num_sms()) * 16)), 256, 0,
                  as_stream(stream)>>>(static_cast<const uint32_t*>(P), m, n_loc, X);
  return check_launch("bs_genotype_unpack");
}

extern "C" int bs_genotype_fill_packed(void* P, const double* maf, int64_t m, int64_t lo, int64_t n_loc,
                                       uint64_t key0, uint64_t key1, void* stream) {
  clear_error();
  if (m < 0 || lo < 0 || n_loc < 0) { set_error("bs_genotype_fill_packed: negative shape"); return BS_EINVAL; }
  if (m == 0 || n_loc == 0) return BS_OK;
  const int64_t words = u2_bytes_per_column(m) / 4 * n_loc;
  fill_packed_kernel<<<int(std::min<int64_t>(ceil_div(words, 256), int64_t(num_sms()) * 16)), 256, 0,
                       as_stream(stream)>>>(static_cast<uint32_t*>(P), maf, m, lo, n_loc, key0, key1);
  return check_launch("bs_genotype_fill_packed");
}
