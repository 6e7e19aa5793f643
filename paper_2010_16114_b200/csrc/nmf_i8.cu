// Integer digit-slice tensor-core GEMMs for float32 NMF (scenarios b and a).
//
//   scn b  P[i][k] = sum_j X[j][i] W[j][k]    A = X MN-major (i contiguous), K = j   (distlinalg.py:246-252)
//   scn a  C[j][k] = sum_i X[j][i] Vt[i][k]   A = X K-major  (i contiguous), K = i   (distlinalg.py:239-243)
//
// Precision scheme (float32-emulating, exact accumulation).  NMF operands are
// nonnegative (X is checked every call, solvers.py:139-141; MU and APG keep the
// factors >= 0).  Every operand block of 512 consecutive K values of one row
// (the "scale group") gets a power-of-two scale 2^t chosen so the block maximum
// lands in [2^21, 2^22); each value becomes the integer N = RN(x 2^t) <= 2^22.  With
// M = N + 0x8080 — exactly the low 24 bits of the float fma(x, 2^t, 2^23 + 0x8080) —
// N = d0 2^16 + d1 2^8 + d2 with signed digits d0 = byte2(M) in [0, 64] and
// d1, d2 = byte(M) - 128 in [-128, 127].  The products
//   acc0 = a0 b0,  acc1 = a0 b1 + a1 b0,  acc2 = a0 b2 + a1 b1 + a2 b0
// are formed by tcgen05 kind::i8 MMAs (s8 x s8 -> s32) and accumulate EXACTLY in int32
// over the group.  The dropped terms (a1 b2 + a2 b1 at 2^-24, a2 b2 at 2^-32) are
// products of zero-mean signed digits, so every rounding in the scheme is symmetric:
// RN to 22 bits per value (<= 2^-22 of the block maximum) and the float32 fold of the
// group partials.  No truncation bias (the tf32 accumulator of nmf_tc.cu truncates).
//
// Tensor work per 32-wide k-block (M = 128, r padded to NP = 64), A from TMEM:
//   A0 x [B0|B1|B2] (N = 3 NP) -> acc0..2,  A1 x [B0|B1] -> acc1..2,  A2 x B0 -> acc2
//   = 192 tensor cycles (floor N/2 per MMA) against ~640 cycles of HBM time per 16 KB tile.
// The digits of A live in TMEM (TS-form MMA): shared memory then carries only the TMA
// tiles, the converters' reads and the B operand (~50 KB per k-block instead of ~78 KB
// with A in shared memory, which made the SS form shared-memory-bandwidth bound).
//
// Data flow (one CTA per SM, persistent over (tile, k-split) units):
//   warp 0      producer: raw X tile (16 KB TMA) into a deep ring
//   warp 14     producer: the factor's pre-sliced digit image (3 x NP x 32 B, cp.async.bulk)
//   warps 6-13  two converter sets (alternate k-blocks): one X row per thread ->
//               3 digit planes (1 packed FMA per 2 values + byte permutes) -> TMEM
//   warp 1      MMA issuer (one elected lane)
//   warps 2-5   epilogue: every group drains the 3 int32 accumulators, scales by
//               2^-(t_row + t_k) and folds into float32 registers (round to nearest)
// The X scales come from bs_nmf_prepare (one pass over X per solver call, fused with
// the reference's _nmf_check scan); the factor is sliced once per GEMM.
#include "tc_common.cuh"

#include <algorithm>
#include <atomic>

using namespace bs;

namespace bs {
static std::atomic<int64_t> g_gemm_path[8];
void note_gemm_path(int path) { g_gemm_path[path & 7].fetch_add(1, std::memory_order_relaxed); }
}  // namespace bs

// Graph replays (solvers.py) run captured GEMMs without the host code that counts them.
extern "C" void bs_add_gemm_path_counts(const int64_t* delta8) {
  for (int i = 0; i < 8; ++i) g_gemm_path[i].fetch_add(delta8[i], std::memory_order_relaxed);
}

extern "C" int bs_gemm_path_counts(int64_t* out8, int reset) {
  for (int i = 0; i < 8; ++i) {
    out8[i] = reset ? g_gemm_path[i].exchange(0) : g_gemm_path[i].load();
  }
  return BS_OK;
}

namespace {

using namespace tc;

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int G = 16;               // k-blocks per scale group = accumulation run
constexpr int GROUP = G * BK;       // 512 K values
constexpr int THREADS = 480;        // X producer, MMA, 4 epilogue warps, 2 x 4 converter warps, B producer
constexpr int RAW_BYTES = BM * BK * 4;   // 16 KB fp32 tile
#ifndef I8_RS
#define I8_RS 10
#endif
#ifndef I8_BS
#define I8_BS 8
#endif
constexpr int RS = I8_RS, BS = I8_BS, CS = 4;  // raw X stages, B image stages, TMEM A stages
constexpr float DIGIT_BIAS = 8388608.0f + 32896.0f;  // 2^23 + 0x8080: bytes of M = N + 0x8080

// scale exponent for a block whose largest |value| has float bits `bits`:
// t = 148 - E puts the maximum in [2^21, 2^22) (N <= 2^22 after rounding).
__host__ __device__ __forceinline__ int exp_code(uint32_t bits) {
  const int e = int(bits >> 23);
  return min(148 - e, 126);
}
__device__ __forceinline__ float pow2f(int t) { return __int_as_float((127 + t) << 23); }

// (x0, x1) * m + DIGIT_BIAS for two values at once (packed f32x2 FMA)
__device__ __forceinline__ void fma2_digits(uint32_t& a, uint32_t& b, float m) {
  uint64_t v = (uint64_t(b) << 32) | a, r;
  const uint64_t mm = (uint64_t(__float_as_uint(m)) << 32) | __float_as_uint(m);
  const uint64_t cc = (uint64_t(__float_as_uint(DIGIT_BIAS)) << 32) | __float_as_uint(DIGIT_BIAS);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(v), "l"(mm), "l"(cc));
  a = uint32_t(r);
  b = uint32_t(r >> 32);
}

// B operand (factor digits, shared memory): canonical K-major SWIZZLE_NONE, core matrix =
// 8 rows x 16 B, K-chunk stride 128 B, 8-row-group stride 256 B (probed: scripts/i8_probe.cu)
__device__ __forceinline__ uint64_t i8_desc(uint32_t addr) { return sdesc(addr, 128, 256, 0); }

// kind::i8, s8 x s8 -> s32, both K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

// One k-block of digit products, issued by one elected lane with warp-uniform operands:
//   acc0..2 (+)= A0 [B0|B1|B2];  acc1..2 += A1 [B0|B1];  acc2 += A2 B0
// a: TMEM column of plane 0 (planes 8 columns apart); b: B0 descriptor; first: restart acc.
template <int NP>
__device__ __forceinline__ void mma_i8_kblock(uint32_t d, uint32_t a, uint64_t b, uint32_t first) {
  constexpr uint32_t id3 = idesc_i8(3 * NP), id2 = idesc_i8(2 * NP), id1 = idesc_i8(NP);
  asm volatile(
      "{\n\t.reg .pred p, acc;\n\t.reg .b32 a1, a2, d1, d2;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.eq.b32 acc, %3, 0;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\t"
      "add.u32 d1, %0, %4;\n\tadd.u32 d2, %0, %5;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %6, acc;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [d1], [a1], %2, %7, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [d2], [a2], %2, %8, 1;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(first), "n"(NP), "n"(2 * NP), "n"(id3), "n"(id2), "n"(id1)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// ---------------------------------------------------------------------------
// bs_nmf_prepare: one pass over X (m x n_loc, column-major float32).
//   * min, sum x^2 and a nonfinite count (the reference's _nmf_check, solvers.py:139-141,
//     and ||X||^2 for the Gram-identity objective)
//   * exp_b[g][i]: scale of row i over columns [512 g, 512 g + 512)    (scn b, K = columns)
//   * exp_a[g][j]: scale of column j over rows [512 g, 512 g + 512)    (scn a, K = rows)
// CTA = 512 rows x 512 columns; thread t owns 4 consecutive rows (float4 loads).
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(128) prep_kernel(const float* __restrict__ X, int64_t m, int64_t n_loc,
                                                   int8_t* __restrict__ exp_b, int8_t* __restrict__ exp_a,
                                                   double* __restrict__ parts) {
  __shared__ uint32_t cmax[4][GROUP];
  __shared__ float smin[4];
  __shared__ double ssq[4];
  __shared__ uint32_t sbad[4];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t i0 = int64_t(blockIdx.x) * GROUP, j0 = int64_t(blockIdx.y) * GROUP;
  const int64_t i = i0 + 4 * t;
  const bool valid = i < m;  // m % 4 == 0: a thread's four rows are all in range or none is
  const int jn = int(n_loc - j0 < GROUP ? n_loc - j0 : int64_t(GROUP));
  uint32_t rmax[4] = {0u, 0u, 0u, 0u};
  float mn = CUDART_INF_F;
  double sq = 0.0;
  uint32_t bad = 0u;
  const float4* col = reinterpret_cast<const float4*>(X + j0 * m + (valid ? i : 0));
  const int64_t cstride = m / 4;
  for (int jj = 0; jj < jn; jj += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (valid && jj + u < jn) v[u] = __ldcs(col + int64_t(jj + u) * cstride);
      else v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float c[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      const bool in = valid && jj + u < jn;
      uint32_t cm = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t b = __float_as_uint(c[q]) & 0x7FFFFFFFu;
        rmax[q] = max(rmax[q], b);
        cm = max(cm, b);
        bad |= (b >= 0x7F800000u) ? 1u : 0u;
        mn = fminf(mn, in ? c[q] : CUDART_INF_F);
      }
      s0 = fmaf(c[0], c[0], s0);
      s1 = fmaf(c[1], c[1], s1);
      s0 = fmaf(c[2], c[2], s0);
      s1 = fmaf(c[3], c[3], s1);
      cm = __reduce_max_sync(0xffffffffu, cm);
      if (lane == 0 && jj + u < jn) cmax[warp][jj + u] = cm;
    }
    sq += double(s0) + double(s1);
  }
  // row scales (scn b)
  if (valid) {
    char4 e;
    e.x = char(exp_code(rmax[0]));
    e.y = char(exp_code(rmax[1]));
    e.z = char(exp_code(rmax[2]));
    e.w = char(exp_code(rmax[3]));
    *reinterpret_cast<char4*>(exp_b + int64_t(blockIdx.y) * m + i) = e;
  }
  // block stats
  mn = warp_min(mn);
  sq = warp_sum(sq);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0) { smin[warp] = mn; ssq[warp] = sq; sbad[warp] = bad; }
  __syncthreads();
  // column scales (scn a)
  for (int j = t; j < jn; j += 128) {
    const uint32_t cm = max(max(cmax[0][j], cmax[1][j]), max(cmax[2][j], cmax[3][j]));
    exp_a[int64_t(blockIdx.x) * n_loc + j0 + j] = int8_t(exp_code(cm));
  }
  if (t == 0) {
    const int64_t b = int64_t(blockIdx.y) * gridDim.x + blockIdx.x;
    parts[3 * b] = double(fminf(fminf(smin[0], smin[1]), fminf(smin[2], smin[3])));
    parts[3 * b + 1] = ((ssq[0] + ssq[1]) + ssq[2]) + ssq[3];
    parts[3 * b + 2] = double(sbad[0] | sbad[1] | sbad[2] | sbad[3]);
  }
}

// stats[0] = min, stats[1] = sum x^2, stats[2] = 1 if X holds a nonfinite value; fixed order.
__global__ void __launch_bounds__(1024) prep_fold_kernel(const double* __restrict__ parts, int64_t np,
                                                         double* __restrict__ stats) {
  __shared__ double smin[32], ssq[32], sbad[32];
  double mn = CUDART_INF, sq = 0.0, bad = 0.0;
  for (int64_t b = threadIdx.x; b < np; b += blockDim.x) {
    mn = fmin(mn, parts[3 * b]);
    sq += parts[3 * b + 1];
    bad = fmax(bad, parts[3 * b + 2]);
  }
  mn = warp_min(mn);
  sq = warp_sum(sq);
  bad = warp_max(bad);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { smin[w] = mn; ssq[w] = sq; sbad[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x >> 5); ++k) {
      mn = fmin(mn, smin[k]);
      bad = fmax(bad, sbad[k]);
    }
    double s = ssq[0];
    for (int k = 1; k < int(blockDim.x >> 5); ++k) s += ssq[k];
    stats[0] = fmin(mn, smin[0]);
    stats[1] = s;
    stats[2] = fmax(bad, sbad[0]);
  }
}

// ---------------------------------------------------------------------------
// Factor slicing: F (r x K, column-major: F[k + r i]) -> per 32-wide k-block a
// digit image [plane][NP rows][32 B] in the canonical K-major layout (what the MMA
// reads as B = [B0|B1|B2]) and per (group, k) unscaling factors 2^(16 - t) (NaN when
// the group holds a nonfinite or negative value).  CTA = one 512-wide group.
// ---------------------------------------------------------------------------

template <int NP>
__global__ void __launch_bounds__(256) fslice_kernel(const float* __restrict__ F, int r, int64_t K,
                                                     uint8_t* __restrict__ img, float* __restrict__ fmul) {
  extern __shared__ __align__(16) uint8_t simg[];  // G k-blocks x 3 NP x 32 B
  constexpr int KB_BYTES = 3 * NP * BK;
  __shared__ uint32_t kmax[NP], kbad[NP];
  __shared__ float kmul[NP];
  const int t = threadIdx.x, lane = t & 31;
  const int64_t i0 = int64_t(blockIdx.x) * GROUP;
  for (int k = t; k < NP; k += 256) { kmax[k] = 0u; kbad[k] = 0u; }
  __syncthreads();
  // pass 1: per-k maxima over the group (warp-reduced, then one smem atomic per warp)
  for (int c = 0; c < 2; ++c) {
    const int64_t i = i0 + t + 256 * c;
    const bool in = i < K;
    const float* col = F + (in ? i : 0) * int64_t(r);
    for (int k = 0; k < r; ++k) {
      const uint32_t b = in ? __float_as_uint(col[k]) : 0u;
      const uint32_t a = b & 0x7FFFFFFFu;
      const uint32_t m_ = __reduce_max_sync(0xffffffffu, a);
      const uint32_t bad = __reduce_or_sync(0xffffffffu, (a >= 0x7F800000u || (b >> 31)) ? 1u : 0u);
      if (lane == 0) {
        atomicMax(&kmax[k], m_);
        if (bad) atomicOr(&kbad[k], 1u);
      }
    }
  }
  __syncthreads();
  const int64_t g = blockIdx.x;
  for (int k = t; k < NP; k += 256) {
    int code = k < r ? exp_code(kmax[k]) : 0;
    const bool bad = k < r && kbad[k];
    fmul[g * NP + k] = bad ? CUDART_NAN_F : pow2f(16 - code);  // the epilogue's unscaling factor
    kmul[k] = bad ? 0.f : pow2f(code);
  }
  __syncthreads();
  // pass 2: digits into the smem image (warp = one k-block, lane = byte position)
  for (int c = 0; c < 2; ++c) {
    const int li = t + 256 * c;  // 0..511 within the group
    const int64_t i = i0 + li;
    const bool in = i < K;
    const float* col = F + (in ? i : 0) * int64_t(r);
    uint8_t* kbimg = simg + (li >> 5) * KB_BYTES;
    const int kk = li & 31;
    const uint32_t inner = uint32_t(kk >> 4) * 128u + uint32_t(kk & 15);
    for (int k = 0; k < NP; ++k) {
      const float x = (in && k < r) ? col[k < r ? k : 0] : 0.f;
      const uint32_t nb = __float_as_uint(fmaf(x, kmul[k], DIGIT_BIAS));
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const int row = p * NP + k;
        const uint32_t d = (nb >> (8 * (2 - p))) & 0xFFu;
        kbimg[uint32_t(row >> 3) * 256u + uint32_t(row & 7) * 16u + inner] = uint8_t(p == 0 ? d : d ^ 0x80u);
      }
    }
  }
  __syncthreads();
  // copy the group's valid k-blocks out (16-B chunks)
  const int64_t kb0 = i0 / BK;
  const int64_t kb_total = (K + BK - 1) / BK;
  const int nkb = int(kb_total - kb0 < G ? kb_total - kb0 : int64_t(G));
  const int chunks = nkb * KB_BYTES / 16;
  uint4* dst = reinterpret_cast<uint4*>(img + kb0 * KB_BYTES);
  const uint4* src = reinterpret_cast<const uint4*>(simg);
  for (int e = t; e < chunks; e += 256) dst[e] = src[e];
}

// ---------------------------------------------------------------------------
// the GEMM kernel
// ---------------------------------------------------------------------------

template <int NP>
struct I8Cfg {
  static constexpr int B_BYTES = 3 * NP * BK;  // factor digit image per k-block
  static constexpr int SMEM = RS * RAW_BYTES + BS * B_BYTES + 1024 + 512;
  static constexpr int ACC = 3 * NP;           // int32 columns per accumulator buffer
  static constexpr int A_COL0 = 2 * ACC;       // TMEM A stages: 3 planes x 8 columns each (32 reserved)
  static constexpr int TMEM_COLS = 2 * ACC + CS * 32 <= 256 ? 256 : 512;
  static_assert(2 * ACC + CS * 32 <= 512 && 3 * NP <= 256, "i8 tile");
};

template <bool A_MN, int NP>
__global__ void __launch_bounds__(THREADS, 1)
i8_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const uint8_t* __restrict__ bimg,
               const int8_t* __restrict__ xexp, int64_t ldx, const float* __restrict__ fmul, int M, int K, int r,
               int tiles, int kb_per_split, int units, float* __restrict__ out, int64_t slab, int mode) {
  using C = I8Cfg<NP>;
#ifndef BS_DEBUG_MODES
  mode = 0;  // work-skipping modes exist only in debug builds (scripts/i8_modes.py)
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* b_base = smem + RS * RAW_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + BS * C::B_BYTES);
  // raw_full[RS] raw_empty[RS] b_full[BS] b_empty[BS] a_full[CS] a_empty[CS] acc_full[2] acc_empty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * RS + 2 * BS + 2 * CS + 4);
  auto raw_full = [&](int s) { return smem_u32(bars + s); };
  auto raw_empty = [&](int s) { return smem_u32(bars + RS + s); };
  auto b_full = [&](int s) { return smem_u32(bars + 2 * RS + s); };
  auto b_empty = [&](int s) { return smem_u32(bars + 2 * RS + BS + s); };
  auto a_full = [&](int s) { return smem_u32(bars + 2 * RS + 2 * BS + s); };
  auto a_empty = [&](int s) { return smem_u32(bars + 2 * RS + 2 * BS + CS + s); };
  auto acc_full = [&](int b) { return smem_u32(bars + 2 * RS + 2 * BS + 2 * CS + b); };
  auto acc_empty = [&](int b) { return smem_u32(bars + 2 * RS + 2 * BS + 2 * CS + 2 + b); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_total = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) { mbar_init(raw_full(s), 1); mbar_init(raw_empty(s), 128); }
    for (int s = 0; s < BS; ++s) { mbar_init(b_full(s), 1); mbar_init(b_empty(s), 1); }
    for (int s = 0; s < CS; ++s) { mbar_init(a_full(s), 128); mbar_init(a_empty(s), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(acc_full(b), 1); mbar_init(acc_empty(b), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 14) {
    // ---------------- producers: X tiles (warp 0) and factor digit images (warp 14) ----------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const bool xprod = warp == 0;
      const int S = xprod ? RS : BS;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int split = u / tiles, tile = u - split * tiles;
        const int kb0 = split * kb_per_split, kb1 = min(kb_total, kb0 + kb_per_split);
        const int m0 = tile * BM;
        for (int kb = kb0; kb < kb1; ++kb) {
          if (xprod && (mode & 8)) {
            mbar_wait_sleep(raw_empty(st), ph ^ 1);
            mbar_arrive(raw_full(st));
          } else if (!xprod && (mode & 4)) {
            mbar_wait_sleep(b_empty(st), ph ^ 1);
            mbar_arrive(b_full(st));
          } else if (xprod) {
            mbar_wait_sleep(raw_empty(st), ph ^ 1);
            mbar_expect_tx(raw_full(st), RAW_BYTES);
            const uint32_t dst = smem_u32(smem + st * RAW_BYTES);
            if constexpr (A_MN) {
#pragma unroll
              for (int a = 0; a < BM / 32; ++a) tma_load_2d(dst + a * 4096, &tmA, m0 + 32 * a, kb * BK, raw_full(st));
            } else {
              tma_load_2d(dst, &tmA, kb * BK, m0, raw_full(st));
            }
          } else {
            mbar_wait_sleep(b_empty(st), ph ^ 1);
            mbar_expect_tx(b_full(st), C::B_BYTES);
            bulk_g2s(smem_u32(b_base + st * C::B_BYTES), bimg + int64_t(kb) * C::B_BYTES, C::B_BYTES, b_full(st));
          }
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int cs = 0, bs = 0;
    uint32_t cph = 0, bph = 0, gi = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles;
      const int kb0 = split * kb_per_split, kb1 = min(kb_total, kb0 + kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int in_group = (kb - kb0) % G;
        const uint32_t buf = gi & 1;
        if (in_group == 0) {
          mbar_wait(acc_empty(buf), ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(a_full(cs), cph);
        mbar_wait(b_full(bs), bph);
        tc_fence_after();
        const bool last = (in_group == G - 1) || (kb == kb1 - 1);
        const uint32_t d = __shfl_sync(0xffffffffu, tmem + buf * C::ACC, 0);
        const uint32_t aa = __shfl_sync(0xffffffffu, tmem + C::A_COL0 + cs * 32, 0);
        const uint32_t bb = __shfl_sync(0xffffffffu, smem_u32(b_base + bs * C::B_BYTES), 0);
        if (!(mode & 2)) mma_i8_kblock<NP>(d, aa, i8_desc(bb), in_group == 0 ? 1u : 0u);
        __syncwarp();
        mma_commit_elect(a_empty(cs));
        mma_commit_elect(b_empty(bs));
        if (last) {
          mma_commit_elect(acc_full(buf));
          ++gi;
        }
        if (++cs == CS) { cs = 0; cph ^= 1; }
        if (++bs == BS) { bs = 0; bph ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ---------------- epilogue: int32 groups -> scaled float32 partials ----------------
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t gi = 0;
    float acc[NP];
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles, tile = u - split * tiles;
      const int kb0 = split * kb_per_split, kb1 = min(kb_total, kb0 + kb_per_split);
      const int groups = (kb1 - kb0 + G - 1) / G;
      const int row = tile * BM + row_in_tile;
#pragma unroll
      for (int i = 0; i < NP; ++i) acc[i] = 0.f;
      for (int g = 0; g < groups; ++g, ++gi) {
        const int gg = kb0 / G + g;  // global scale group
        const int tx = row < M ? int(xexp[int64_t(gg) * ldx + row]) : 0;
        const float sx = pow2f(16 - tx);
        const float* fm = fmul + int64_t(gg) * NP;
        const uint32_t buf = gi & 1;
        mbar_wait(acc_full(buf), (gi >> 1) & 1);
        tc_fence_after();
        const uint32_t base = tmem + lane_addr + buf * C::ACC;
#pragma unroll
        for (int c0 = 0; c0 < NP; c0 += 8) {
          uint32_t v[3][8];
#pragma unroll
          for (int w = 0; w < 3; ++w) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[w][0]), "=r"(v[w][1]), "=r"(v[w][2]), "=r"(v[w][3]), "=r"(v[w][4]),
                           "=r"(v[w][5]), "=r"(v[w][6]), "=r"(v[w][7])
                         : "r"(base + uint32_t(w * NP + c0)));
          }
          tmem_wait_ld();
          const float4 f0 = *reinterpret_cast<const float4*>(fm + c0);
          const float4 f1 = *reinterpret_cast<const float4*>(fm + c0 + 4);
          const float sf[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float s = fmaf(__int2float_rn(int(v[2][i])), 0.00390625f, __int2float_rn(int(v[1][i])));
            s = fmaf(s, 0.00390625f, __int2float_rn(int(v[0][i])));
            acc[c0 + i] = fmaf(s * sx, sf[i], acc[c0 + i]);
          }
        }
        tc_fence_before();
        mbar_arrive(acc_empty(buf));
      }
      if (row < M) {
        float* dst = out + int64_t(split) * slab + int64_t(row) * r;
#pragma unroll
        for (int i = 0; i < NP; ++i)
          if (i < r) dst[i] = acc[i];
      }
    }
  } else {
    // ---------------- converters: X row -> three digit planes in TMEM ----------------
    const int set = (warp - 6) >> 2;
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t j0 = 0;  // CTA-local sequence number of the unit's first k-block
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles, tile = u - split * tiles;
      const int kb0 = split * kb_per_split, kb1 = min(kb_total, kb0 + kb_per_split);
      const int row = tile * BM + row_in_tile;
      const int nk = kb1 - kb0;
      const int g0 = kb0 / G, ng = (nk + G - 1) / G;
      // row scales of this unit's first two groups; later ones are fetched a group ahead
      const int8_t e_cur = row < M ? xexp[int64_t(g0) * ldx + row] : int8_t(0);
      int8_t e_nxt = (row < M && ng > 1) ? xexp[int64_t(g0 + 1) * ldx + row] : int8_t(0);
      int cur_g = 0;
      float mul = row < M ? pow2f(int(e_cur)) : 0.f;
      for (int t = int((uint32_t(set) - j0) & 1u); t < nk; t += 2) {
        const uint32_t j = j0 + uint32_t(t);
        if (t / G != cur_g) {
          cur_g = t / G;
          mul = row < M ? pow2f(int(e_nxt)) : 0.f;
          e_nxt = (row < M && cur_g + 1 < ng) ? xexp[int64_t(g0 + cur_g + 1) * ldx + row] : int8_t(0);
        }
        const int rst = int(j % RS), cst = int(j % CS);
        mbar_wait(raw_full(rst), (j / RS) & 1);
        mbar_wait(a_empty(cst), ((j / CS) & 1) ^ 1);
        tc_fence_after();
        if (mode & 1) {
          tc_fence_before();
          mbar_arrive(raw_empty(rst));
          mbar_arrive(a_full(cst));
          continue;
        }
        uint32_t x[32];
        const uint32_t raw = smem_u32(smem + rst * RAW_BYTES);
        if constexpr (A_MN) {
          const uint32_t atom = raw + uint32_t(row_in_tile >> 5) * 4096u;
          const uint32_t mb = uint32_t(row_in_tile & 31) * 4u;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t off = uint32_t(k) * 128u + mb;
            x[k] = ld_shared_u32(atom + (off ^ (((off >> 7) & 3u) << 5)));
          }
        } else {
          const uint32_t rowb = raw + uint32_t(row_in_tile) * 128u;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = ld_shared_v4(rowb + (uint32_t(c ^ (row_in_tile & 7)) << 4));
            x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
          }
        }
        // M = RN(x 2^t) + 0x8080 sits in the low 24 bits of fma(x, 2^t, 2^23 + 0x8080):
        // digit 0 = byte 2, digits 1 and 2 = bytes 1 and 0 minus 128 (xor 0x80 as s8)
#pragma unroll
        for (int k = 0; k < 32; k += 2) fma2_digits(x[k], x[k + 1], mul);
        uint32_t pl[24];  // plane 0 (8 words), plane 1, plane 2: TMEM columns in this order
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const uint32_t a = x[4 * w], b = x[4 * w + 1], c = x[4 * w + 2], d = x[4 * w + 3];
          const uint32_t ab = __byte_perm(a, b, 0x5140);  // a.b0 b.b0 a.b1 b.b1
          const uint32_t cd = __byte_perm(c, d, 0x5140);
          pl[16 + w] = __byte_perm(ab, cd, 0x5410) ^ 0x80808080u;  // byte 0 of a b c d
          pl[8 + w] = __byte_perm(ab, cd, 0x7632) ^ 0x80808080u;   // byte 1
          const uint32_t ab2 = __byte_perm(a, b, 0x0062);          // a.b2 b.b2
          const uint32_t cd2 = __byte_perm(c, d, 0x0062);
          pl[w] = __byte_perm(ab2, cd2, 0x5410);                   // byte 2
        }
        const uint32_t ta = tmem + lane_addr + uint32_t(C::A_COL0 + cst * 32);
        tmem_st16(ta, pl);
        tmem_st8(ta + 16, pl + 16);
        tmem_wait_st();
        tc_fence_before();
        // The raw stage is released only here, behind stores that depend on every value read
        // from it: an arrive issued right behind the LDS does not wait for them to return
        // (seen on B200: refilled stages read back stale when it did).
        mbar_arrive(raw_empty(rst));
        mbar_arrive(a_full(cst));
      }
      j0 += uint32_t(nk);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

int pick_np(int r) { return r <= 32 ? 32 : r <= 64 ? 64 : 0; }

int64_t groups_of(int64_t k) { return ceil_div(k, GROUP); }

// Split count over K: units of whole scale groups, enough units for a balanced grid.
int i8_splits(int64_t tiles, int64_t K) {
  const int64_t kb = ceil_div(K, BK);
  const int64_t sms = num_sms();
  int best = 1;
  double best_eff = -1.0;
  for (int s = 1; s <= TC_MAX_SPLITS; ++s) {
    const int64_t per = ceil_div(ceil_div(kb, s), G) * G;
    const int64_t real = ceil_div(kb, per);
    if (real < s) break;
    const double waves = double(tiles * real) / double(sms);
    const double score = waves / std::ceil(waves) - 0.004 * s;
    if (score > best_eff + 1e-9) { best_eff = score; best = s; }
  }
  return best;
}

template <int NP>
int launch_fslice(const float* F, int r, int64_t K, uint8_t* img, float* fmul, cudaStream_t st) {
  constexpr int SM = G * 3 * NP * BK;
  smem_attr(fslice_kernel<NP>, SM);
  fslice_kernel<NP><<<int(groups_of(K)), 256, SM, st>>>(F, r, K, img, fmul);
  return check_launch("i8 factor slice");
}

template <bool A_MN, int NP>
int launch_i8(const CUtensorMap& ta, const uint8_t* img, const int8_t* xexp, int64_t ldx, const float* fexp, int M,
              int K, int r, int splits, float* out, int64_t slab, cudaStream_t st) {
  using C = I8Cfg<NP>;
  smem_attr(i8_gemm_kernel<A_MN, NP>, C::SMEM);
  const int tiles = int(ceil_div(M, BM));
  const int kb_total = int(ceil_div(K, BK));
  const int kb_per = int(ceil_div(ceil_div(kb_total, splits), G) * G);
  const int real = int(ceil_div(kb_total, kb_per));
  const int units = tiles * real;
  const int grid = std::min(units, num_sms());
  static const int mode = [] {
#ifdef BS_DEBUG_MODES
    const char* e = getenv("BS_I8_MODE");
    return e ? atoi(e) : 0;
#else
    return 0;
#endif
  }();
  i8_gemm_kernel<A_MN, NP><<<grid, THREADS, C::SMEM, st>>>(ta, img, xexp, ldx, fexp, M, K, r, tiles, kb_per, units,
                                                            out, slab, mode);
  return real;
}

bool i8_shape_ok(const float* X, const float* F, int64_t m, int64_t n_loc, int r) {
  return tc_enabled() && pick_np(r) != 0 && m % 4 == 0 && m <= INT32_MAX && n_loc <= INT32_MAX &&
         !(reinterpret_cast<uintptr_t>(X) & 15) && !(reinterpret_cast<uintptr_t>(F) & 15);
}

}  // namespace

namespace bs {

int64_t i8_xscale_bytes(int64_t m, int64_t n_loc) { return groups_of(n_loc) * m + groups_of(m) * n_loc; }

int64_t i8_prepare_workspace(int64_t m, int64_t n_loc) {
  return ws_bytes<double>(3 * groups_of(m) * groups_of(n_loc));
}

int i8_prepare(const float* X, int64_t m, int64_t n_loc, double* stats, int8_t* xscale, Workspace& ws,
               cudaStream_t st) {
  const int64_t gm = groups_of(m), gn = groups_of(n_loc);
  double* parts = ws.take<double>(3 * gm * gn);
  if (!parts) { set_error("bs_nmf_prepare: workspace too small"); return BS_EWORK; }
  if (gm > 65535 * 4096LL || gn > 65535) { set_error("bs_nmf_prepare: shape too large"); return BS_EINVAL; }
  const dim3 grid{unsigned(gm), unsigned(gn), 1u};
  prep_kernel<<<grid, 128, 0, st>>>(X, m, n_loc, xscale, xscale + gn * m, parts);
  prep_fold_kernel<<<1, 1024, 0, st>>>(parts, gm * gn, stats);
  return check_launch("bs_nmf_prepare", 2);
}

int64_t i8_gemm_workspace(int64_t K) {
  return ws_bytes<uint8_t>(ceil_div(K, BK) * 3 * 64 * BK) + ws_bytes<float>(groups_of(K) * 64);
}

// scn b: P (r x m) = W X^T; S slabs folded into P.  xexp_b: [groups(n_loc)][m].
int i8_wxt(const float* X, const float* W, int64_t m, int64_t n_loc, int r, const int8_t* xexp_b, float* P,
           Workspace& ws, cudaStream_t st, bool* used) {
  *used = false;
  const int np = pick_np(r);
  if (!xexp_b || !i8_shape_ok(X, W, m, n_loc, r) || m < 128 || n_loc < 32) return BS_OK;
  CUtensorMap ta;
  if (!make_map_f32(&ta, X, uint64_t(m), uint64_t(n_loc), 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return BS_OK;
  uint8_t* img = ws.take<uint8_t>(ceil_div(n_loc, BK) * 3 * np * BK);
  float* fexp = ws.take<float>(groups_of(n_loc) * np);
  if (!img || !fexp) { set_error("i8_wxt: workspace too small"); return BS_EWORK; }
  int rc = np == 32 ? launch_fslice<32>(W, r, n_loc, img, fexp, st) : launch_fslice<64>(W, r, n_loc, img, fexp, st);
  if (rc != BS_OK) return rc;
  const int64_t tiles = ceil_div(m, BM);
  const int splits = i8_splits(tiles, n_loc);
  float* out = P;
  float* slabs = nullptr;
  if (splits > 1) {
    slabs = ws.take<float>(int64_t(TC_MAX_SPLITS) * m * r);
    if (!slabs) { set_error("i8_wxt: workspace too small"); return BS_EWORK; }
    out = slabs;
  }
  const int S = np == 32 ? launch_i8<true, 32>(ta, img, xexp_b, m, fexp, int(m), int(n_loc), r, splits, out, m * r, st)
                         : launch_i8<true, 64>(ta, img, xexp_b, m, fexp, int(m), int(n_loc), r, splits, out, m * r, st);
  rc = check_launch("i8_wxt");
  if (rc != BS_OK) return rc;
  if (S > 1) {
    launch_sum_slabs_f32(slabs, S, m * r, P, st);
    rc = check_launch("i8_wxt fold");
    if (rc != BS_OK) return rc;
  }
  note_gemm_path(0);
  *used = true;
  return BS_OK;
}

// scn a: up to cap_slabs partial slabs of C (r x n_loc); *splits = slabs written.  xexp_a: [groups(m)][n_loc].
int i8_vtx(const float* X, const float* Vt, int64_t m, int64_t n_loc, int r, const int8_t* xexp_a, float* Cout,
           int cap_slabs, int* splits, Workspace& ws, cudaStream_t st, bool* used) {
  *used = false;
  const int np = pick_np(r);
  if (!xexp_a || !i8_shape_ok(X, Vt, m, n_loc, r) || n_loc < 128 || m < 32) return BS_OK;
  CUtensorMap ta;
  if (!make_map_f32(&ta, X, uint64_t(m), uint64_t(n_loc), 32, 128, CU_TENSOR_MAP_SWIZZLE_128B)) return BS_OK;
  uint8_t* img = ws.take<uint8_t>(ceil_div(m, BK) * 3 * np * BK);
  float* fexp = ws.take<float>(groups_of(m) * np);
  if (!img || !fexp) { set_error("i8_vtx: workspace too small"); return BS_EWORK; }
  int rc = np == 32 ? launch_fslice<32>(Vt, r, m, img, fexp, st) : launch_fslice<64>(Vt, r, m, img, fexp, st);
  if (rc != BS_OK) return rc;
  const int64_t tiles = ceil_div(n_loc, BM);
  const int want = std::min(i8_splits(tiles, m), cap_slabs);
  const int S = np == 32 ? launch_i8<false, 32>(ta, img, xexp_a, n_loc, fexp, int(n_loc), int(m), r, want, Cout,
                                                 n_loc * r, st)
                         : launch_i8<false, 64>(ta, img, xexp_a, n_loc, fexp, int(n_loc), int(m), r, want, Cout,
                                                 n_loc * r, st);
  rc = check_launch("i8_vtx");
  if (rc != BS_OK) return rc;
  note_gemm_path(0);
  *splits = S;
  *used = true;
  return BS_OK;
}

}  // namespace bs
