// Tensor-core passes over 2-bit packed genotypes (C5), float32 arithmetic:
//   scn p   grad_j = sum_i X_ij v_i   (distlinalg.py:355-358, solvers.py:446-447), and
//   scn m   (X beta)_i = sum_j X_ij beta_j from the packed transpose (same pass, K = columns)
// as tcgen05 kind::mxf4 MMAs (e2m1 x e2m1 -> f32, K = 64 per instruction, block scales 1).
//
// Why mxf4: below N = 128 every tcgen05 MMA costs a fixed ~64 cycles (scripts/ts_rate.cu,
// profiles/r02_tcgen05_i8_rate.txt), so the genotypes one instruction consumes set the speed:
// kind::i8 (K = 32 bytes) capped the previous version at 16 packed bytes per cycle per SM
// (4.8 TB/s); e2m1 takes 64 per instruction, twice that, above the HBM rate.
//
// A = X^T (M = 128 columns j, K = rows i, K-major in shared memory): genotype g in {0, 1, 2}
// is exactly the e2m1 code g (0, 0.5, 1.0).  A packed word w holds 16 genotypes at bits 2r;
// w & 0x33333333 leaves the 8 even-row genotypes as nibbles, (w >> 2) & 0x33333333 the 8
// odd-row ones, so each converter thread turns 16 genotypes into 8 bytes of A with three
// integer instructions.  K order inside every 16-row group is therefore
//   position s < 8: row 2s,   position s >= 8: row 2(s - 8) + 1,
// and the B image uses the same order.
//
// B = the v digits (N = NB): v is scaled per group of 2048 rows by 2^t so |v| < 2^(3 NB - 2),
// rounded to an integer V, and split into NB balanced base-8 digits in [-4, 4] (exact e2m1
// values), digit n in row n of the image.  D[j][n] = sum_i (g_ij / 2) d_n(v_i) is a sum of
// multiples of 1/2 below 2^14 per 2048-row group, exact in the f32 accumulator; the epilogue
// forms 2 sum_n 8^n D[j][n] 2^-t in float64.  The only rounding is v to 3 NB - 2 bits of its
// group maximum: NB = 16 (46 bits) for float32 arithmetic, NB = 32 (94 bits: float64 values
// 2^41 below their group's largest still keep all 53 bits) for float64 arithmetic — the MMA
// costs the same for any N <= 128.
//
// Shared memory carries, per k-block: the packed tile (TMA write, converter read, 16 KB
// each way), the e2m1 A operand (converter write, tensor-core read, 32 KB each way) and the
// digit image (4 KB): ~100 KB, which at 128 B per cycle is the pass's bound (~0.75 of HBM;
// loading X straight into converter registers instead was slower, 17.8 ms at C5, for lack
// of loads in flight).  The precision gain over kind::i8 (v to 46 bits instead of 27) is the
// main reason for this form.
//
// CTA (one per SM, persistent over 128-column tiles; each tile runs the whole K):
//   warp 0      TMA: packed tile (128 B x 128 columns = 512 rows x 128 columns) per k-block
//   warp 14     bulk copy of the v-digit image (16 rows x 256 B) per k-block
//   warps 6-13  two converter sets (alternate k-blocks): packed -> e2m1, into shared memory
//   warp 1      MMA issuer: 8 MMAs (M = 128, N = 16, K = 64) per k-block
//   warps 2-5   epilogue: every group drains D (16 f32 per column) into a float64 sum
#include "tc_common.cuh"

#include <algorithm>

using namespace bs;
using namespace tc;

namespace bs {
void note_gemm_path(int path);
}

namespace {

constexpr int BM = 128;            // columns j per tile (MMA M)
constexpr int BKR = 512;           // rows i per k-block
constexpr int BKB = BKR / 4;       // packed bytes per column per k-block (128)
constexpr int KSTEPS = BKR / 64;   // MMAs per k-block (K = 64)
static_assert(KSTEPS == 8, "mma_kblock8 issues eight K = 64 steps");
constexpr int G = 4;               // k-blocks per scale group (2048 rows)
constexpr int GROWS = G * BKR;
constexpr int ROWB = BKR / 2;      // e2m1 bytes per operand row per k-block (256)
constexpr int SBO = (ROWB / 16) * 128;  // 8-row-group stride: 16 K chunks x (8 rows x 16 B)
constexpr int A_BYTES = BM * ROWB;  // 32 KB per k-block
constexpr int NB_MAX = 32;          // B rows (base-8 digits): 16 (float32) or 32 (float64)
template <int NB>
constexpr int b_bytes() { return NB * ROWB; }  // 4 / 8 KB per k-block
constexpr int X_BYTES = BM * BKB;   // 16 KB per k-block
constexpr int THREADS = 480;
// Ring depths.  The pass is bound by bytes in flight and by shared memory: 6 packed-tile stages
// and three A stages (the converters run a k-block further ahead of the MMAs), with the B-image
// ring shrunk to 3 stages for the 8 KB float64 image so both fit the 227 KB (C5 gradient pass,
// measured: RS/CS 6/2 10.2 ms, 5/3 9.0, 6/3 8.6, 4/3 10.1; float64 RS 5 -> 6 with 3 B stages -3%).
template <int NB>
constexpr int rs_of() { return 6; }
// B-image stages: 6 of 4 KB (float32) or 3 of 8 KB (float64, so the packed ring keeps 6 stages)
template <int NB>
constexpr int bs_of() { return NB <= 16 ? 6 : 3; }
constexpr int CS = 3;
constexpr int ACC = 32;             // TMEM columns per accumulator buffer (>= NB)
constexpr uint32_t T_SFA = 64, T_SFB = 96;  // scale-factor columns (all 2^0)
constexpr int TMEM_COLS = 512;
template <int NB>
constexpr int off_a() { return rs_of<NB>() * X_BYTES; }
template <int NB>
constexpr int off_b() { return off_a<NB>() + CS * A_BYTES; }
template <int NB>
constexpr int smem_bytes() { return off_b<NB>() + bs_of<NB>() * b_bytes<NB>() + 1024 + 512; }
static_assert(smem_bytes<16>() <= 232448 && smem_bytes<32>() <= 232448, "227 KB of shared memory per CTA");
// kind::mxf4 block-scaled descriptor: A, B e2m1 (1), scales ue8m0, N = NB, M = 128
template <int NB>
constexpr uint32_t idesc_f4() {
  return (1u << 7) | (1u << 10) | (uint32_t(NB >> 3) << 17) | (1u << 23) | (uint32_t(BM >> 4) << 24);
}

// One k-block (8 k steps of 64 rows) from the whole warp: one elected lane issues
// D (+)= A(smem) x B(smem) with unit block scales.  Both operands advance two 128-byte K
// chunks per step (+16 in the low word of each descriptor; no carry into the high word).
__device__ __forceinline__ void mma_kblock8(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                            uint32_t idesc, uint32_t first) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "mov.b64 a, {%1, %5};\n\tmov.b64 b, {%2, %6};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%7], [%8], q;\n\t"
#define BS_F4_STEP(OFF)                                                                  \
      "add.u32 t, %1, " #OFF ";\n\tmov.b64 a, {t, %5};\n\t"                            \
      "add.u32 t, %2, " #OFF ";\n\tmov.b64 b, {t, %6};\n\t"                            \
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%7], [%8], 1;\n\t"
      BS_F4_STEP(16) BS_F4_STEP(32) BS_F4_STEP(48) BS_F4_STEP(64) BS_F4_STEP(80) BS_F4_STEP(96) BS_F4_STEP(112)
#undef BS_F4_STEP
      "}" ::"r"(d),
      "r"(alo), "r"(blo), "r"(idesc), "r"(first), "r"(ahi), "r"(bhi), "r"(T_SFA), "r"(T_SFB)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// ---------------------------------------------------------------------------
// v digits: one CTA per 2048-row group, thread t owns rows [16 t, 16 t + 16) of the group,
// i.e. one 16-position K group of one k-block, and writes its 8 bytes of every image row.
// Image of a k-block: canonical K-major SWIZZLE_NONE, 8 rows x 16 B core matrices, K-chunk
// stride 128 B, 8-row-group stride SBO.
// ---------------------------------------------------------------------------
template <typename T, int NB>
__global__ void __launch_bounds__(128) vdigits_kernel(const T* __restrict__ v, int64_t m,
                                                      uint8_t* __restrict__ img, double* __restrict__ gscale,
                                                      const int* flags) {
  __shared__ double smax[4];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t i0 = int64_t(blockIdx.x) * GROWS + 16 * t;
  double vv[16];
  double mx = 0.0;
  int nonfinite = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    vv[e] = (i0 + e < m) ? double(v[i0 + e]) : 0.0;
    nonfinite |= !isfinite(vv[e]);
    mx = fmax(mx, fabs(vv[e]));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) smax[warp] = mx;
  // a NaN / inf in the group makes its scale NaN, so the sums come out NaN as float
  // arithmetic would give them (the digits are then zeros, not digits of a non-finite)
  nonfinite = __syncthreads_or(nonfinite);
  mx = fmax(fmax(smax[0], smax[1]), fmax(smax[2], smax[3]));
  // scale 2^s with mx 2^s in [2^(3 NB - 3), 2^(3 NB - 2)); an all-zero group keeps s = 0
  int ex = 0;
  frexp(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
  const int s = (mx > 0.0 && !nonfinite) ? 3 * NB - 2 - ex : 0;
  if (t == 0) gscale[blockIdx.x] = nonfinite ? __longlong_as_double(0x7ff8000000000000ll) : ldexp(1.0, -s);
  unsigned long long word[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) word[n] = 0ull;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    // r = rint(v 2^s) is an integer below 2^(3 NB - 2) in magnitude (exact in float64: above
    // 2^53 the scaled value is already integral); balanced base-8 digits from the top, each
    // step exact: q = floor(r / 8^k + 1/2) in [-4, 4], r -= q 8^k
    double r = nonfinite ? 0.0 : rint(ldexp(vv[e], s));
    const int pos = (e & 1) ? 8 + (e >> 1) : (e >> 1);  // K position of row e in its 16-group
#pragma unroll
    for (int n = NB - 1; n >= 0; --n) {
      const double q = floor(fma(r, ldexp(1.0, -3 * n), 0.5));
      r = fma(-q, ldexp(1.0, 3 * n), r);
      const unsigned long long code = (0x65420ACDEull >> (4 * (int(q) + 4))) & 0xFull;  // e2m1 of -4..4
      word[n] |= code << (4 * pos);
    }
  }
  // write: k-block kb = t / (BKR / 16), 8-byte half h of 16-byte K chunk c
  const int64_t kb = (int64_t(blockIdx.x) * GROWS) / BKR + t / (BKR / 16);
  const int tt = t % (BKR / 16);
  uint8_t* kimg = img + kb * b_bytes<NB>() + (tt >> 1) * 128 + (tt & 1) * 8;
#pragma unroll
  for (int n = 0; n < NB; ++n) *reinterpret_cast<unsigned long long*>(kimg + (n >> 3) * SBO + (n & 7) * 16) = word[n];
}

// ---------------------------------------------------------------------------
// the pass
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(THREADS, 1)
gradtc_kernel(const __grid_constant__ CUtensorMap tmX, const uint8_t* __restrict__ bimg,
              const double* __restrict__ gscale, int64_t m, int64_t n_loc, int tiles, double* __restrict__ out,
              const int* flags) {
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int RS = rs_of<NB>(), BS = bs_of<NB>();
  uint8_t* a_base = smem + off_a<NB>();
  uint8_t* b_base = smem + off_b<NB>();
  constexpr int B_BYTES = b_bytes<NB>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + BS * B_BYTES);
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
  const int nkb = int((m + BKR - 1) / BKR);

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) { mbar_init(raw_full(s), 1); mbar_init(raw_empty(s), 128); }
    for (int s = 0; s < BS; ++s) { mbar_init(b_full(s), 1); mbar_init(b_empty(s), 1); }
    for (int s = 0; s < CS; ++s) { mbar_init(a_full(s), 128); mbar_init(a_empty(s), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(acc_full(b), 1); mbar_init(acc_empty(b), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmX);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 2 && warp < 6) {  // unit block scales (ue8m0 127 = 2^0) in every lane of the SF columns
    uint32_t ones[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) ones[c] = 0x7F7F7F7Fu;
    const uint32_t la = uint32_t((warp & 3) * 32) << 16;
    tmem_st16(tmem + la + T_SFA, ones);
    tmem_st16(tmem + la + T_SFB, ones);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0 || warp == 14) {
    // ---------------- producers: packed X tiles (warp 0), v-digit images (warp 14) ----------------
    if (lane == 0) {
      const bool xprod = warp == 0;
      const int S = xprod ? RS : BS;
      int st = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          if (xprod) {
            mbar_wait_sleep(raw_empty(st), ph ^ 1);
            mbar_expect_tx(raw_full(st), X_BYTES);
            tma_load_2d(smem_u32(smem + st * X_BYTES), &tmX, kb * BKB, tile * BM, raw_full(st));
          } else {
            mbar_wait_sleep(b_empty(st), ph ^ 1);
            mbar_expect_tx(b_full(st), B_BYTES);
            bulk_g2s(smem_u32(b_base + st * B_BYTES), bimg + int64_t(kb) * B_BYTES, B_BYTES, b_full(st));
          }
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The k-blocks of this CTA run as one sequence g = 0, 1, ... (tile-major); g's A stage is
    // g % CS and its B stage g % BS.  Unrolling six k-blocks at a time makes both stages
    // compile-time constants: every MMA operand is then a loop-invariant base plus an
    // immediate, so the single issuing warp spends a few instructions per MMA.
    constexpr int UNR = BS;  // issue-loop unroll covering whole B and A rings
    static_assert(UNR % BS == 0 && UNR % CS == 0, "the unrolled issue loop covers whole B and A rings");
    static_assert(TMEM_COLS == 512, "a whole-TMEM allocation starts at address 0");
    if (tmem != 0u) __trap();
    const uint32_t my_tiles = uint32_t((tiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x));
    const uint32_t total = my_tiles * uint32_t(nkb);
    const uint64_t a_desc0 = sdesc(smem_u32(a_base), 128, SBO, 0);
    const uint64_t b_desc0 = sdesc(smem_u32(b_base), 128, SBO, 0);
    const uint32_t alo0 = uint32_t(a_desc0), ahi = uint32_t(a_desc0 >> 32);
    const uint32_t blo0 = uint32_t(b_desc0), bhi = uint32_t(b_desc0 >> 32);
    int kb = 0;
    uint32_t gi = 0;
    for (uint32_t g0 = 0; g0 < total; g0 += UNR) {
      const uint32_t bph = (g0 / UNR) & 1u;
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (g0 + uint32_t(u) >= total) break;
        const int cs = u % CS;
        const uint32_t cph = (g0 / CS + uint32_t(u / CS)) & 1u;
        const int in_group = kb % G;
        const uint32_t buf = gi & 1u;
        if (in_group == 0) {
          mbar_wait(acc_empty(buf), ((gi >> 1) & 1u) ^ 1u);
          tc_fence_after();
        }
        mbar_wait(a_full(cs), cph);
        mbar_wait(b_full(u), bph);
        tc_fence_after();
        const bool last = (in_group == G - 1) || (kb == nkb - 1);
        mma_kblock8(buf * ACC, alo0 + uint32_t((cs * A_BYTES) >> 4), ahi, blo0 + uint32_t((u * B_BYTES) >> 4), bhi,
                    idesc_f4<NB>(), in_group == 0 ? 0u : 1u);
        mma_commit_elect(a_empty(cs));
        mma_commit_elect(b_empty(u));
        if (last) {
          mma_commit_elect(acc_full(buf));
          ++gi;
        }
        if (++kb == nkb) kb = 0;
      }
    }
  } else if (warp < 6) {
    // ---------------- epilogue: float64 sum per column ----------------
    const int q = warp & 3;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const int ngroups = (nkb + G - 1) / G;
    uint32_t gi = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int64_t j = int64_t(tile) * BM + q * 32 + lane;
      double acc = 0.0;
      for (int g = 0; g < ngroups; ++g, ++gi) {
        const uint32_t buf = gi & 1;
        mbar_wait(acc_full(buf), (gi >> 1) & 1);
        tc_fence_after();
        uint32_t r[NB];
#pragma unroll
        for (int c = 0; c < NB; c += 8)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                         "=r"(r[c + 6]), "=r"(r[c + 7])
                       : "r"(tmem + lane_addr + buf * ACC + uint32_t(c)));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(acc_empty(buf));
        double sd = 0.0;
#pragma unroll
        for (int n = NB - 1; n >= 0; --n) sd = fma(sd, 8.0, double(__uint_as_float(r[n])));  // sum_n 8^n D[n]
        acc = fma(sd, 2.0 * __ldg(gscale + g), acc);  // genotype codes are g / 2
      }
      if (j < n_loc) out[j] = acc;
    }
  } else {
    // ---------------- converters: packed bytes -> e2m1 nibbles in shared memory ----------------
    const int set = (warp - 6) >> 2;
    const int q = warp & 3;
    const int col = q * 32 + lane;  // row of A = column of the tile
    const uint32_t dst0 = uint32_t((col >> 3) * SBO + (col & 7) * 16);
    uint32_t j0 = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      for (int t = int((uint32_t(set) - j0) & 1u); t < nkb; t += 2) {
        const uint32_t jj = j0 + uint32_t(t);
        const int rst = int(jj % RS), cst = int(jj % CS);
        mbar_wait(raw_full(rst), (jj / RS) & 1);
        mbar_wait(a_empty(cst), ((jj / CS) & 1) ^ 1);
        // the tile row (128 B) sits in SWIZZLE_128B: 16-byte chunk c of row r at chunk c ^ (r % 8),
        // so the 32 lanes' reads of one chunk spread over the banks
        const uint32_t src = smem_u32(smem + rst * X_BYTES) + uint32_t(col) * BKB;
        const uint32_t sw = uint32_t(col & 7);
        const uint32_t dst = smem_u32(a_base + cst * A_BYTES) + dst0;
#pragma unroll
        for (int c = 0; c < BKB / 16; ++c) {  // 64 genotypes -> two 16-byte K chunks of e2m1
          const uint4 p = ld_shared_v4(src + ((uint32_t(c) ^ sw) << 4));
          const uint32_t w[4] = {p.x, p.y, p.z, p.w};
          uint32_t e[4], o[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            e[k] = w[k] & 0x33333333u;         // even rows 2s -> nibble s
            o[k] = (w[k] >> 2) & 0x33333333u;  // odd rows 2s + 1 -> nibble s
          }
          st_shared_v4(dst + uint32_t(2 * c) * 128u, make_uint4(e[0], o[0], e[1], o[1]));
          st_shared_v4(dst + uint32_t(2 * c + 1) * 128u, make_uint4(e[2], o[2], e[3], o[3]));
        }
        fence_proxy_async_smem();  // the generic-proxy stores become visible to the tensor core
        mbar_arrive(raw_empty(rst));  // behind the stores, which depend on every loaded word
        mbar_arrive(a_full(cst));
      }
      j0 += uint32_t(nkb);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------------------
// packed transpose: Q = the packed (n x m) transpose of the packed (m x n) block P, so that
// X beta = Q^T beta runs through the same pass (K = the n columns, M = the m rows).
// CTA tile: 128 rows (32 bytes of each column) x 128 columns (32 bytes of each output row).
// Thread (a4 = word, jb = column byte) takes the 4 x 4 genotypes of one byte in each of four
// columns, gathers them into one word (byte c = column c) and transposes the 2-bit fields in
// place with two delta swaps (byte r = row r).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) u2_transpose_kernel(const uint8_t* __restrict__ P, int64_t m, int64_t n,
                                                           int64_t ld, uint8_t* __restrict__ Q, int64_t ldT) {
  __shared__ uint32_t s_in[128][9];                // column c: 8 words (128 rows), one word of padding
  __shared__ __align__(16) uint8_t s_out[128][32];  // output row r: 32 bytes (128 columns)
  const int t = threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * 128;
  const int64_t ntj = (n + 127) / 128;
  for (int64_t tj = blockIdx.y; tj < ntj; tj += gridDim.y) {
    const int64_t j0 = tj * 128;
    {
      const int c = t >> 1, h = t & 1;
      const int64_t b = i0 / 4 + 16 * h;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (j0 + c < n && b < ld) v = *reinterpret_cast<const uint4*>(P + (j0 + c) * ld + b);
      s_in[c][4 * h] = v.x;
      s_in[c][4 * h + 1] = v.y;
      s_in[c][4 * h + 2] = v.z;
      s_in[c][4 * h + 3] = v.w;
    }
    __syncthreads();
    {
      const int jb = t & 31, a4 = t >> 5;
      const uint32_t w0 = s_in[4 * jb][a4], w1 = s_in[4 * jb + 1][a4];
      const uint32_t w2 = s_in[4 * jb + 2][a4], w3 = s_in[4 * jb + 3][a4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t sel = uint32_t(e) | (uint32_t(e + 4) << 4);
        uint32_t w = __byte_perm(__byte_perm(w0, w1, sel), __byte_perm(w2, w3, sel), 0x5410u);
        uint32_t x = ((w >> 6) ^ w) & 0x00CC00CCu;
        w ^= x ^ (x << 6);
        x = ((w >> 12) ^ w) & 0x0000F0F0u;
        w ^= x ^ (x << 12);
        const int row = 4 * (4 * a4 + e);
#pragma unroll
        for (int r = 0; r < 4; ++r) s_out[row + r][jb] = uint8_t(w >> (8 * r));
      }
    }
    __syncthreads();
    {
      const int r = t >> 1, h = t & 1;
      const int64_t b = j0 / 4 + 16 * h;
      if (i0 + r < m && b < ldT)
        *reinterpret_cast<uint4*>(Q + (i0 + r) * ldT + b) = *reinterpret_cast<const uint4*>(&s_out[r][16 * h]);
    }
    __syncthreads();
  }
}

bool make_map_u8(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {d0};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace bs {

int64_t u2_grad_tc_workspace(int64_t m) {
  const int64_t nkb = (m + BKR - 1) / BKR, ng = (nkb + G - 1) / G;
  return ws_bytes<uint8_t>(ng * G * b_bytes<NB_MAX>()) + ws_bytes<double>(ng);
}

// One tensor-core pass: out[j] = sum_k P[k, j] v[k] for the packed (K x M) block P (ld =
// ceil(K / 64) * 16 bytes per column), one slab, with NB digits of v.  Returns false when the
// path does not apply (no tcgen05, misaligned P, or the tensor map is refused).
template <typename T, int NB>
static bool u2_tc_pass(const void* P, const T* v, int64_t K, int64_t M, double* out, const int* flags, Workspace& ws,
                       cudaStream_t st, int* rc, const char* what) {
  *rc = BS_OK;
  if (!tc_enabled() || K <= 0 || M <= 0 || (reinterpret_cast<uintptr_t>(P) & 15)) return false;
  const int64_t ld = ((K + 63) / 64) * 16;
  const int64_t nkb = (K + BKR - 1) / BKR, ng = (nkb + G - 1) / G;
  uint8_t* img = ws.take<uint8_t>(ng * G * b_bytes<NB>());
  double* gscale = ws.take<double>(ng);
  if (!img || !gscale) {
    set_error("%s: workspace too small", what);
    *rc = BS_EWORK;
    return true;
  }
  CUtensorMap tm;
  if (!make_map_u8(&tm, P, uint64_t(ld), uint64_t(M), BKB, BM)) return false;
  vdigits_kernel<T, NB><<<int(ng), 128, 0, st>>>(v, K, img, gscale, flags);
  const int tiles = int((M + BM - 1) / BM);
  const int grid = std::min(tiles, num_sms());
  smem_attr(gradtc_kernel<NB>, smem_bytes<NB>());
  gradtc_kernel<NB><<<grid, THREADS, smem_bytes<NB>(), st>>>(tm, img, gscale, K, M, tiles, out, flags);
  *rc = check_launch(what, 2);
  note_gemm_path(6);
  return true;
}

// grad partials (one slab: out[j], j < n_loc) of packed X against v on the tensor cores, with
// 16 digits of v for float32 arithmetic and 32 for float64.
bool launch_grad_u2_tc(const void* P, const double* v, int64_t m, int64_t n_loc, double* out, const int* flags,
                       Workspace& ws, cudaStream_t st, int* rc, bool f64) {
  return f64 ? u2_tc_pass<double, 32>(P, v, m, n_loc, out, flags, ws, st, rc, "u2 tensor-core grad")
             : u2_tc_pass<double, 16>(P, v, m, n_loc, out, flags, ws, st, rc, "u2 tensor-core grad");
}

// X beta (out[i], i < m) from the packed transpose Q of the local block (bs_genotype_transpose_packed):
// the same pass with K = n_loc and M = m.
bool launch_xbeta_u2t_tc(const void* Q, const float* beta, int64_t m, int64_t n_loc, double* out, Workspace& ws,
                         cudaStream_t st, int* rc) {
  return u2_tc_pass<float, 16>(Q, beta, n_loc, m, out, nullptr, ws, st, rc, "u2 tensor-core xbeta");
}
bool launch_xbeta_u2t_tc(const void* Q, const double* beta, int64_t m, int64_t n_loc, double* out, Workspace& ws,
                         cudaStream_t st, int* rc) {
  return u2_tc_pass<double, 32>(Q, beta, n_loc, m, out, nullptr, ws, st, rc, "u2 tensor-core xbeta");
}

int launch_u2_transpose(const void* P, int64_t m, int64_t n, void* Q, cudaStream_t st) {
  const int64_t ld = ((m + 63) / 64) * 16, ldT = ((n + 63) / 64) * 16;
  const int64_t nti = (m + 127) / 128, ntj = (n + 127) / 128;
  if (nti > 0x7fffffffLL) return BS_EINVAL;
  dim3 grid(unsigned(nti), unsigned(std::min<int64_t>(ntj, 65535)));
  u2_transpose_kernel<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(P), m, n, ld, static_cast<uint8_t*>(Q), ldT);
  return check_launch("bs_genotype_transpose_packed", 1);
}

}  // namespace bs
