// tcgen05 3xTF32 skinny GEMMs for float32 NMF (scenarios b and a).
//
//   scn b  P[i][k] = sum_j X[j][i] W[j][k]    A = X MN-major (i contiguous), K = j   (distlinalg.py:246-252)
//   scn a  C[j][k] = sum_i X[j][i] Vt[i][k]   A = X K-major  (i contiguous), K = i   (distlinalg.py:239-243)
//
// M = 128 rows per tile on the tensor cores, N = r padded to a multiple of 32,
// K in blocks of 32.  Precision: float32 via 3xTF32 — every operand x is split
// into hi = tf32(x) (mantissa truncated: an exact tf32 value) and lo = x - hi
// (exact in fp32); the products hi*hi + hi*lo + lo*hi are accumulated and the
// dropped lo*lo term is ~2^-22 relative.
//
// Data flow per k-block (one CTA per SM, persistent over (tile, k-split) units):
//   warp 0       TMA producer: raw X tile (16 KB) + raw B tile (r x 32) into a
//                6-deep smem ring (SWIZZLE_128B for K-major X, SWIZZLE_128B_ATOM_32B
//                for MN-major operands — the only MN-major layout tf32 accepts)
//   warps 6-13   two converter sets (alternate k-blocks): each thread takes one
//                X row, splits it, tcgen05.st's hi|lo into TMEM (A operand, K-major),
//                splits the B tile into hi|lo smem buffers, then frees the raw stage
//   warp 1       tcgen05.mma issuer, one elected lane for the whole warp: per 8-wide
//                k step D[:,0:2N] += A_hi [Bh|Bl] and D[:,0:N] += A_lo Bh (N <= 64)
//   warps 2-5    epilogue: tcgen05.ld each finished accumulator group and fold it
//                into fp32 registers (round-to-nearest), store the unit's rows
// X is read exactly once per GEMM; split-K slabs are folded in order by the
// consumer.  The TMEM accumulator is double-buffered and restarted every G
// k-blocks because the tensor core's fp32 accumulation truncates (see below).
#include "tc_common.cuh"

#include <algorithm>
#include <mutex>

using namespace bs;

namespace bs {
void note_gemm_path(int path);
}

namespace {

using namespace tc;

constexpr int TC_THREADS = 448;  // producer, MMA, 4 epilogue warps, 2 x 4 converter warps
constexpr int BM = 128;
constexpr int BK = 32;
constexpr int A_STAGE_BYTES = BM * BK * 4;  // 16 KB
#ifndef BS_TC_CSTAGES
#define BS_TC_CSTAGES 3
#endif
constexpr int SMEM_BUDGET = 220 * 1024;

// MN-major operand slab (32 MN x 32 K of a stage): k step s covers rows 8s..8s+7 = two 512 B atoms.
__device__ __forceinline__ uint64_t mn_desc(uint32_t base, int s) {
  return sdesc(base + uint32_t(s) * 1024u, 4096, 512, LAYOUT_SW128_32B);
}

// Non-concatenated variant (NP > 64): three MMAs per k step, Bl slab at bdesc_lo.
__device__ __forceinline__ void mma_kblock_3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                             uint32_t id, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b64 h1, h2, h3, l1, l2, l3;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "add.s64 h1, %3, 64;\n\tadd.s64 h2, %3, 128;\n\tadd.s64 h3, %3, 192;\n\t"
      "add.s64 l1, %4, 64;\n\tadd.s64 l2, %4, 128;\n\tadd.s64 l3, %4, 192;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, q;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2+8], h1, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+8], l1, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+8], h1, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2+16], h2, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+16], l2, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+16], h2, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2+24], h3, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+24], l3, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+24], h3, %5, 1;\n\t}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(id), "r"(acc0)
      : "memory");
}

// Stage layout.  Raw ring (TMA targets): A raw (16 KB) + B raw (NP x 32 fp32).  Converted
// ring: B hi | B lo in smem (MN-major, same swizzled layout as the raw tile) and the A
// tile's tf32 hi | lo halves in TMEM (128 lanes x 64 columns, K-major: lane = row).
// With NP <= 64 the MMA uses [B hi | B lo] as one N = 2*NP operand: per 8-wide k step
// D[:, 0:2NP] += A_hi [Bh|Bl]  and  D[:, 0:NP] += A_lo Bh — two instructions instead of
// three (an M=128 MMA costs ~45 cycles up to N = 64, measured).
template <int NP>
struct TcCfg {
  static constexpr bool CONCAT = NP <= 64;
  static constexpr int ACC_COLS = CONCAT ? 2 * NP : NP;     // per accumulator buffer
  static constexpr int B_BYTES = NP * BK * 4;                 // one of B raw / B hi / B lo
  static constexpr int RAW = A_STAGE_BYTES + B_BYTES;
  static constexpr int CONV = 2 * B_BYTES;
  static constexpr int CSTAGES = BS_TC_CSTAGES;               // converted stages (TMEM A + smem B)
  static constexpr int RSTAGES_FIT = (SMEM_BUDGET - 2048 - CSTAGES * CONV) / RAW;
  static constexpr int RSTAGES = RSTAGES_FIT > 8 ? 8 : RSTAGES_FIT;
  static constexpr int SMEM = RSTAGES * RAW + CSTAGES * CONV + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int TMEM_COLS = 512;                       // 2 accumulators + CSTAGES x 64 A columns
  static constexpr int A_COL0 = 2 * ACC_COLS;                 // first TMEM column of the A stages
  static_assert(2 * ACC_COLS + CSTAGES * 64 <= 512, "TMEM budget");
};

// ---------------------------------------------------------------------------
// the kernel
//
// Accumulation precision: the tensor core adds each MMA into the fp32 TMEM
// accumulator with truncation, so a long K run drifts by ~6e-8 per MMA (measured:
// 7e-6 relative after K = 320).  The K range of a unit is therefore cut into
// groups of G k-blocks; each group accumulates into a fresh TMEM buffer (two
// buffers alternate) and the epilogue warps fold the group partial into fp32
// registers with round-to-nearest adds.  The error is then bounded by one group.
// ---------------------------------------------------------------------------

template <bool A_MN, int NP>
__global__ void __launch_bounds__(TC_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int K, int r,
               int tiles, int kb_per_split, int units, int G, float* __restrict__ out, int64_t slab, int mode,
               double* __restrict__ stats_part) {
  using C = TcCfg<NP>;
  constexpr int RS = C::RSTAGES, CS = C::CSTAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* conv_base = smem + RS * C::RAW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(conv_base + CS * C::CONV);
  // bars: raw_full[RS], raw_empty[RS], conv_full[CS], conv_empty[CS], acc_full[2], acc_empty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * RS + 2 * CS + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_total = (K + BK - 1) / BK;

  auto raw_a = [&](int s) { return smem + s * C::RAW; };
  auto raw_b = [&](int s) { return smem + s * C::RAW + A_STAGE_BYTES; };
  auto conv_bh = [&](int c) { return conv_base + c * C::CONV; };
  auto conv_bl = [&](int c) { return conv_base + c * C::CONV + C::B_BYTES; };
  auto raw_full = [&](int s) { return smem_u32(bars + s); };
  auto raw_empty = [&](int s) { return smem_u32(bars + RS + s); };
  auto conv_full = [&](int c) { return smem_u32(bars + 2 * RS + c); };
  auto conv_empty = [&](int c) { return smem_u32(bars + 2 * RS + CS + c); };
  auto acc_full = [&](int b) { return smem_u32(bars + 2 * RS + 2 * CS + b); };
  auto acc_empty = [&](int b) { return smem_u32(bars + 2 * RS + 2 * CS + 2 + b); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(raw_full(s), 1);
      mbar_init(raw_empty(s), 128);
    }
    for (int c = 0; c < CS; ++c) {
      mbar_init(conv_full(c), 128);
      mbar_init(conv_empty(c), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
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

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int split = u / tiles, tile = u - split * tiles;
        const int kb0 = split * kb_per_split;
        const int kb1 = min(kb_total, kb0 + kb_per_split);
        const int m0 = tile * BM;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(raw_empty(stage), phase ^ 1);
          const uint32_t fb = raw_full(stage);
          mbar_expect_tx(fb, A_STAGE_BYTES + C::B_BYTES);
          const int k0 = kb * BK;
          if constexpr (A_MN) {
#pragma unroll
            for (int a = 0; a < BM / 32; ++a) tma_load_2d(smem_u32(raw_a(stage) + a * 4096), &tmA, m0 + 32 * a, k0, fb);
          } else {
            tma_load_2d(smem_u32(raw_a(stage)), &tmA, k0, m0, fb);
          }
#pragma unroll
          for (int b = 0; b < NP / 32; ++b) tma_load_2d(smem_u32(raw_b(stage) + b * 4096), &tmB, 32 * b, k0, fb);
          if (++stage == RS) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // idesc: D f32, A/B tf32, A K-major (TMEM), B MN-major; N per instruction set below, M = 128
    const uint32_t idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(BM >> 4) << 24);
    const uint32_t idesc_wide = idesc_base | (uint32_t(C::ACC_COLS >> 3) << 17);
    const uint32_t idesc_narrow = idesc_base | (uint32_t(NP >> 3) << 17);
    int cst = 0;
    uint32_t cphase = 0;
    uint32_t gi = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles;
      const int kb0 = split * kb_per_split;
      const int kb1 = min(kb_total, kb0 + kb_per_split);
      int in_group = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        const uint32_t buf = gi & 1;
        if (in_group == 0) {
          mbar_wait(acc_empty(buf), ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(conv_full(cst), cphase);
        tc_fence_after();
        const bool last = (in_group == G - 1) || (kb == kb1 - 1);
        {
          // warp-uniform operands (broadcast so ptxas can use uniform registers)
          const uint32_t d = __shfl_sync(0xffffffffu, tmem + buf * C::ACC_COLS, 0);
          const uint32_t a_hi = __shfl_sync(0xffffffffu, tmem + C::A_COL0 + cst * 64, 0);
          const uint32_t bh = __shfl_sync(0xffffffffu, smem_u32(conv_bh(cst)), 0);
          const uint32_t acc0 = in_group > 0 ? 1u : 0u;
          if (!(mode & 2)) {
            if constexpr (C::CONCAT) {
              mma_kblock_concat(d, a_hi, a_hi + 32, mn_desc(bh, 0), idesc_wide, idesc_narrow, acc0);
            } else {
              const uint32_t bl = __shfl_sync(0xffffffffu, smem_u32(conv_bl(cst)), 0);
              mma_kblock_3(d, a_hi, a_hi + 32, mn_desc(bh, 0), mn_desc(bl, 0), idesc_narrow, acc0);
            }
          }
          mma_commit_elect(conv_empty(cst));
          if (last) mma_commit_elect(acc_full(buf));
        }
        __syncwarp();
        if (last) {
          ++gi;
          in_group = 0;
        } else {
          ++in_group;
        }
        if (++cst == CS) { cst = 0; cphase ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ---------------- epilogue (warps 2..5): fold TMEM group partials in fp32 RN ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t gi = 0;
    float acc[NP];
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles, tile = u - split * tiles;
      const int kb0 = split * kb_per_split;
      const int kb1 = min(kb_total, kb0 + kb_per_split);
      const int groups = (kb1 - kb0 + G - 1) / G;
#pragma unroll
      for (int i = 0; i < NP; ++i) acc[i] = 0.f;
      for (int g = 0; g < groups; ++g, ++gi) {
        const uint32_t buf = gi & 1;
        mbar_wait(acc_full(buf), (gi >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < NP; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + lane_addr + buf * C::ACC_COLS + uint32_t(c0), v);
          if constexpr (C::CONCAT) {
            float w[16];
            tmem_ld16(tmem + lane_addr + buf * C::ACC_COLS + uint32_t(NP + c0), w);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c0 + i] = __fadd_rn(acc[c0 + i], __fadd_rn(v[i], w[i]));
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c0 + i] = __fadd_rn(acc[c0 + i], v[i]);
          }
        }
        tc_fence_before();
        mbar_arrive(acc_empty(buf));
      }
      if (tile * BM + row_in_tile < M) {
        float* dst = out + int64_t(split) * slab + int64_t(tile * BM + row_in_tile) * r;
#pragma unroll
        for (int i = 0; i < NP; ++i)
          if (i < r) dst[i] = acc[i];
      }
    }
  } else {
    // ---------------- converters (warps 6..13): two sets alternate k-blocks ----------------
    const int set = (warp - 6) >> 2;
    const int ct = threadIdx.x - 192 - set * 128;  // 0..127 within the set
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t j = 0;  // CTA-local block sequence number
    float xmin = CUDART_INF_F;
    double xsq = 0.0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles;
      const int kb0 = split * kb_per_split;
      const int kb1 = min(kb_total, kb0 + kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++j) {
        if (int(j & 1) != set) continue;
        const int rst = int(j % RS), cst = int(j % CS);
        const uint32_t rphase = (j / RS) & 1, cphase = (j / CS) & 1;
        mbar_wait(raw_full(rst), rphase);
        mbar_wait(conv_empty(cst), cphase ^ 1);
        tc_fence_after();
        // ---- A: this thread's row (32 K values) -> hi/lo -> TMEM ----
        uint32_t hi[32], lo[32];
        const uint32_t a_base = smem_u32(raw_a(rst));
        if (!(mode & 1)) {
          if constexpr (A_MN) {
            // MN-major, Swizzle<2,5,2> atoms of 32 rows x 128 B (one atom per 32 M rows)
            const uint32_t atom = a_base + uint32_t(row_in_tile >> 5) * 4096u;
            const uint32_t mb = uint32_t(row_in_tile & 31) * 4u;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const uint32_t off = uint32_t(k) * 128u + mb;
              hi[k] = ld_shared_u32(atom + (off ^ (((off >> 7) & 3u) << 5)));
            }
          } else {
            // K-major SW128: row at row*128 B, 16 B chunk c stored at c ^ (row & 7)
            const uint32_t rowb = a_base + uint32_t(row_in_tile) * 128u;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint4 v = ld_shared_v4(rowb + (uint32_t(c ^ (row_in_tile & 7)) << 4));
              hi[4 * c] = v.x; hi[4 * c + 1] = v.y; hi[4 * c + 2] = v.z; hi[4 * c + 3] = v.w;
            }
          }
          if (stats_part) {  // _nmf_check + ||X||^2 ride on this pass (solvers.py:139-141)
            // squares summed in fp32 over the row's 32 values (two chains), then into float64
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              const float x0 = __uint_as_float(hi[k]), x1 = __uint_as_float(hi[k + 1]);
              xmin = fminf(xmin, fminf(x0, x1));
              s0 = fmaf(x0, x0, s0);
              s1 = fmaf(x1, x1, s1);
            }
            xsq += double(s0) + double(s1);
          }
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t h = hi[k] & 0xFFFFE000u;
            lo[k] = __float_as_uint(__uint_as_float(hi[k]) - __uint_as_float(h));
            hi[k] = h;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) hi[k] = lo[k] = 0u;
        }
        const uint32_t a_col = tmem + lane_addr + uint32_t(C::A_COL0 + cst * 64);
        tmem_st32(a_col, hi);
        tmem_st32(a_col + 32, lo);
        // ---- B: elementwise split into the converted buffers (same swizzled layout) ----
        {
          const uint32_t bsrc = smem_u32(raw_b(rst));
          const uint32_t bh = smem_u32(conv_bh(cst)), bl = smem_u32(conv_bl(cst));
#pragma unroll
          for (int e = ct; e < C::B_BYTES / 16; e += 128) {
            const uint4 v = ld_shared_v4(bsrc + 16u * e);
            uint4 h, l;
            h.x = v.x & 0xFFFFE000u; h.y = v.y & 0xFFFFE000u; h.z = v.z & 0xFFFFE000u; h.w = v.w & 0xFFFFE000u;
            l.x = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(h.x));
            l.y = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(h.y));
            l.z = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(h.z));
            l.w = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(h.w));
            st_shared_v4(bh + 16u * e, h);
            st_shared_v4(bl + 16u * e, l);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(raw_empty(rst));  // the raw stage is free again: TMA can refill it
        mbar_arrive(conv_full(cst));
      }
    }
    if (stats_part) {
      // deterministic CTA fold of the converters' (min, sum x^2): warps in order
      __shared__ float smin[8];
      __shared__ double ssq[8];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        xmin = fminf(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
        xsq += __shfl_xor_sync(0xffffffffu, xsq, o);
      }
      const int cw = warp - 6;
      if (lane == 0) { smin[cw] = xmin; ssq[cw] = xsq; }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (cw == 0 && lane == 0) {
        float a = smin[0];
        double b = ssq[0];
        for (int w2 = 1; w2 < 8; ++w2) { a = fminf(a, smin[w2]); b += ssq[w2]; }
        stats_part[2 * blockIdx.x] = double(a);
        stats_part[2 * blockIdx.x + 1] = b;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launch
// ---------------------------------------------------------------------------

bool make_map(CUtensorMap* map, const float* base, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1, bool mn_major) {
  return make_map_f32(map, base, d0, d1, b0, b1,
                      mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
}

int pick_np(int r) { return r <= 32 ? 32 : r <= 64 ? 64 : r <= 96 ? 96 : r <= 128 ? 128 : 0; }

template <bool A_MN, int NP>
int launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, int M, int K, int r, int splits, float* out, int64_t slab,
              cudaStream_t st, double* stats_part = nullptr, int* grid_out = nullptr) {
  using C = TcCfg<NP>;
  smem_attr(tc_gemm_kernel<A_MN, NP>, C::SMEM);
  const int tiles = int(ceil_div(M, BM));
  const int kb_total = int(ceil_div(K, BK));
  const int kb_per = int(ceil_div(kb_total, splits));
  const int real_splits = int(ceil_div(kb_total, kb_per));
  const int units = tiles * real_splits;
  const int grid = std::min(units, num_sms());
  static int group = -1;
  static std::once_flag g_once;
  std::call_once(g_once, [] {
    const char* e = getenv("BS_TC_GROUP");
    group = (e && atoi(e) > 0) ? atoi(e) : 4;
  });
  // Work-skipping modes (bit 1: skip the A split, bit 2: skip the MMAs) exist only in
  // debug builds (-DBS_DEBUG_MODES, used by scripts/nmf_modes.sh); the shipped library
  // always runs the full kernel.
  static int mode = 0;
#ifdef BS_DEBUG_MODES
  static std::once_flag m_once;
  std::call_once(m_once, [] {
    const char* e = getenv("BS_TC_MODE");
    mode = e ? atoi(e) : 0;
  });
#endif
  if (grid_out) *grid_out = grid;
  tc_gemm_kernel<A_MN, NP><<<grid, TC_THREADS, C::SMEM, st>>>(ta, tb, M, K, r, tiles, kb_per, units, group, out, slab, mode,
                                                               stats_part);
  return real_splits;
}

// Split count: enough units for a balanced persistent grid, each unit >= 8 k-blocks.
int tc_splits(int64_t M, int64_t K) {
  const int64_t tiles = ceil_div(M, BM), kb = ceil_div(K, BK);
  const int64_t sms = num_sms();
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 16; ++s) {
    if (s > 1 && kb / s < 8) break;
    const int64_t units = tiles * s;
    const double waves = double(units) / double(sms);
    const double eff = waves / std::ceil(waves);
    const double score = eff - 0.004 * s;  // small penalty per extra slab
    if (score > best_eff + 1e-9) { best_eff = score; best = s; }
  }
  return best;
}

}  // namespace

namespace bs {

int64_t tc_wxt_workspace(int64_t m, int64_t n_loc, int r) {
  (void)n_loc;
  return ws_bytes<float>(int64_t(TC_MAX_SPLITS) * m * r) + ws_bytes<double>(2 * int64_t(num_sms()));
}
int64_t tc_vtx_workspace(int64_t m, int64_t n_loc, int r) {
  (void)m; (void)n_loc; (void)r;
  return 0;
}

#define BS_TC_DISPATCH(AMN)                                                                            \
  switch (np) {                                                                                        \
    case 32: S = launch_tc<AMN, 32>(ta, tb, M, K, r, nsplit, out, slab, st, sp, &gsz); break;          \
    case 64: S = launch_tc<AMN, 64>(ta, tb, M, K, r, nsplit, out, slab, st, sp, &gsz); break;          \
    case 96: S = launch_tc<AMN, 96>(ta, tb, M, K, r, nsplit, out, slab, st, sp, &gsz); break;          \
    default: S = launch_tc<AMN, 128>(ta, tb, M, K, r, nsplit, out, slab, st, sp, &gsz); break;         \
  }

// scn b: writes S partial slabs of P (r x m) into the workspace and folds them into P.
// stats (nullable): {min, sum x^2} of X gathered during the same pass (float64, device).
int tc_wxt(const float* X, const float* W, int64_t m, int64_t n_loc, int r, float* P, Workspace& ws, cudaStream_t st,
           bool* used, double* stats) {
  *used = false;
  const int np = pick_np(r);
  if (!tc_enabled() || np == 0 || m % 4 || r % 4 || m > INT32_MAX || n_loc > INT32_MAX || m < 128 || n_loc < 32 ||
      (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(W) & 15))
    return BS_OK;
  CUtensorMap ta, tb;
  if (!make_map(&ta, X, uint64_t(m), uint64_t(n_loc), 32, 32, true)) return BS_OK;
  if (!make_map(&tb, W, uint64_t(r), uint64_t(n_loc), 32, 32, true)) return BS_OK;
  const int M = int(m), K = int(n_loc);
  const int nsplit = tc_splits(M, K);
  double* sp = nullptr;
  int gsz = 0;
  if (stats) {
    sp = ws.take<double>(2 * int64_t(num_sms()));
    if (!sp) { set_error("tc_wxt: workspace too small"); return BS_EWORK; }
  }
  float* out = P;
  float* slabs = nullptr;
  if (nsplit > 1) {
    slabs = ws.take<float>(int64_t(TC_MAX_SPLITS) * m * r);
    if (!slabs) { set_error("tc_wxt: workspace too small"); return BS_EWORK; }
    out = slabs;
  }
  const int64_t slab = m * r;
  int S = 1;
  BS_TC_DISPATCH(true)
  int rc = check_launch("tc_wxt");
  if (rc != BS_OK) return rc;
  if (stats) {
    launch_fold_minsq(sp, gsz, stats, st);
    rc = check_launch("tc_wxt stats");
    if (rc != BS_OK) return rc;
  }
  if (S > 1) {
    launch_sum_slabs_f32(slabs, S, m * r, P, st);
    rc = check_launch("tc_wxt fold");
    if (rc != BS_OK) return rc;
  }
  note_gemm_path(1);
  *used = true;
  return BS_OK;
}

// scn a: writes up to cap_slabs partial slabs of C (r x n_loc) into C; *splits = slabs written.
int tc_vtx(const float* X, const float* Vt, int64_t m, int64_t n_loc, int r, float* Cout, int cap_slabs, int* splits,
           Workspace& ws, cudaStream_t st, bool* used) {
  (void)ws;
  *used = false;
  const int np = pick_np(r);
  if (!tc_enabled() || np == 0 || m % 4 || r % 4 || m > INT32_MAX || n_loc > INT32_MAX || n_loc < 128 || m < 32 ||
      (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Vt) & 15))
    return BS_OK;
  CUtensorMap ta, tb;
  if (!make_map(&ta, X, uint64_t(m), uint64_t(n_loc), 32, 128, false)) return BS_OK;
  if (!make_map(&tb, Vt, uint64_t(r), uint64_t(m), 32, 32, true)) return BS_OK;
  const int M = int(n_loc), K = int(m);
  const int want = std::min(tc_splits(M, K), cap_slabs);
  float* out = Cout;
  const int64_t slab = n_loc * r;
  int S = 1;
  const int nsplit = want;
  double* sp = nullptr;
  int gsz = 0;
  BS_TC_DISPATCH(false)
  int rc = check_launch("tc_vtx");
  if (rc != BS_OK) return rc;
  *splits = S;
  note_gemm_path(1);
  *used = true;
  return BS_OK;
}

}  // namespace bs
