// Tensor-core scn p for 2-bit packed genotypes (C5): grad_j = sum_i X_ij v_i
// (distlinalg.py:355-358, solvers.py:446-447) as tcgen05 kind::i8 MMAs with exact int32 sums.
//
// A = X^T (M = 128 columns j of the local block, K = rows i): a packed column is already
// K-major, four genotypes per byte.  One PRMT replicates a packed byte b into all four lanes
// of a word and one AND with 0xC0300C03 keeps field q in byte q, i.e. byte q = g_{4t+q} 4^q
// (0..128, u8) — no shifts; the 4^q is undone on the B side.  Each converter thread unpacks
// its column's 32 bytes of a 128-row k-block into 32 words and tcgen05.st's them into TMEM
// (A operand, K-major, lane = column).
//
// B = the v digits (K = i, N = 16): v is scaled per group of 2048 rows by 2^t so |v| < 2^27,
// rounded to an integer, and split into four balanced signed 7-bit digits
// (V = d0 2^21 + d1 2^14 + d2 2^7 + d3, d in [-64, 64]); row n = 4 d + q of the image holds
// digit d of v_i when i % 4 == q and 0 otherwise, so
//   D[j][4d + q] = 4^q sum_{i % 4 = q} X_ij d_d(v_i)
// and the epilogue forms sum_d 2^(7(3 - d)) sum_q 4^-q D[j][4d + q] 2^-t in float64.
// Products and sums are exact integers; the only rounding is v to 27 bits of its group
// maximum (symmetric) — tighter than the float32 arithmetic of the CUDA-core kernels.
//
// CTA (one per SM, persistent over 128-column tiles; each tile runs the whole m):
//   warp 0      TMA: packed tile (32 B x 128 columns = 128 rows x 128 columns) per k-block
//   warp 14     bulk copy of the v-digit image (16 x 128 B) per k-block
//   warps 6-13  two converter sets (alternate k-blocks): unpack -> TMEM
//   warp 1      MMA issuer: 4 MMAs (M = 128, N = 16, K = 32) per k-block
//   warps 2-5   epilogue: every group drains D (16 int32 per column) into a float64 sum
#include "tc_common.cuh"

#include <algorithm>

using namespace bs;
using namespace tc;

namespace bs {
void note_gemm_path(int path);
}

namespace {

constexpr int BM = 128;            // columns j per tile (MMA M)
constexpr int BKR = 512;           // rows i per k-block (MMA K, 16 x 32)
constexpr int BKB = BKR / 4;       // packed bytes per column per k-block (128)
constexpr int KSTEPS = BKR / 32;
constexpr int G = 4;               // k-blocks per scale group (2048 rows)
constexpr int GROWS = G * BKR;
constexpr int NB = 16;             // B rows: 4 digits x 4 phases
constexpr int B_BYTES = NB * BKR;  // 8 KB per k-block
constexpr int B_SBO = 8 * BKR;     // 8-row-group stride of the B image: BKR/16 chunks x 128 B
constexpr int X_BYTES = BM * BKB;  // 16 KB per k-block
constexpr int THREADS = 480;
constexpr int RS = 8, BS = 6, CS = 3;
constexpr int ACC = NB;            // TMEM columns per accumulator buffer
constexpr int A_COLS = BKR / 4;    // TMEM columns per A stage: BKR unpacked bytes (128)
constexpr int A_COL0 = 2 * ACC;
constexpr int TMEM_COLS = 512;
constexpr int SMEM = RS * X_BYTES + BS * B_BYTES + 1024 + 512;

__host__ __device__ constexpr uint32_t idesc_u8s8(int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

// One k-block (16 k steps of 32 rows) from the whole warp: one elected lane issues
// D (+)= A(TMEM) x B(smem), u8 x s8 -> s32, M = 128, N = NB, K = 32 per step.  A advances 8
// TMEM columns per step (immediate offsets), B two 128-byte K chunks (+16 in the low word
// of the descriptor; the 14-bit address field never carries into the high word here).
__device__ __forceinline__ void mma_kblock16(uint32_t d, uint32_t blo, uint32_t bhi, uint32_t a, uint32_t first) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b32 lo;\n\t.reg .b64 b;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "mov.b64 b, {%1, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3], b, %5, q;\n\t"
      "add.u32 lo, %1, 16;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+8], b, %5, 1;\n\t"
      "add.u32 lo, %1, 32;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+16], b, %5, 1;\n\t"
      "add.u32 lo, %1, 48;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+24], b, %5, 1;\n\t"
      "add.u32 lo, %1, 64;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+32], b, %5, 1;\n\t"
      "add.u32 lo, %1, 80;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+40], b, %5, 1;\n\t"
      "add.u32 lo, %1, 96;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+48], b, %5, 1;\n\t"
      "add.u32 lo, %1, 112;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+56], b, %5, 1;\n\t"
      "add.u32 lo, %1, 128;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+64], b, %5, 1;\n\t"
      "add.u32 lo, %1, 144;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+72], b, %5, 1;\n\t"
      "add.u32 lo, %1, 160;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+80], b, %5, 1;\n\t"
      "add.u32 lo, %1, 176;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+88], b, %5, 1;\n\t"
      "add.u32 lo, %1, 192;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+96], b, %5, 1;\n\t"
      "add.u32 lo, %1, 208;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+104], b, %5, 1;\n\t"
      "add.u32 lo, %1, 224;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+112], b, %5, 1;\n\t"
      "add.u32 lo, %1, 240;\n\tmov.b64 b, {lo, %2};\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%3+120], b, %5, 1;\n\t"
      "}" ::"r"(d), "r"(blo), "r"(bhi), "r"(a), "r"(first), "n"(idesc_u8s8(NB))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// ---------------------------------------------------------------------------
// v digits: one CTA per 2048-row group, thread t owns rows [16 t, 16 t + 16) of the group
// (one 16-byte K chunk of one k-block) and writes that chunk for all 16 image rows.
// image row n, k-block kb: canonical K-major SWIZZLE_NONE, 8 rows x 16 B core matrices,
// K-chunk stride 128 B, 8-row-group stride B_SBO.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) vdigits_kernel(const T* __restrict__ v, int64_t m,
                                                      uint8_t* __restrict__ img, double* __restrict__ gscale,
                                                      const int* flags) {
  __shared__ double smax[4];
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t i0 = int64_t(blockIdx.x) * GROWS + 16 * t;
  double vv[16];
  double mx = 0.0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    vv[e] = (i0 + e < m) ? double(v[i0 + e]) : 0.0;
    mx = fmax(mx, fabs(vv[e]));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) smax[warp] = mx;
  __syncthreads();
  mx = fmax(fmax(smax[0], smax[1]), fmax(smax[2], smax[3]));
  // scale 2^s with mx 2^s in [2^26, 2^27); an all-zero group keeps s = 0
  int ex = 0;
  frexp(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
  const int s = mx > 0.0 ? 27 - ex : 0;
  if (t == 0) gscale[blockIdx.x] = ldexp(1.0, -s);
  uint8_t dg[4][16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    double y = ldexp(vv[e], s);              // exact
    double r = y;
    const double w[4] = {2097152.0, 16384.0, 128.0, 1.0};  // 2^21, 2^14, 2^7, 1
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const double q = d < 3 ? floor(r / w[d] + 0.5) : rint(r);  // last digit: round to nearest
      r -= q * w[d];                          // exact
      dg[d][e] = uint8_t(int8_t(q));
    }
  }
  // write: k-block kb = t / (BKR / 16), chunk c = t % (BKR / 16)
  const int64_t kb = (int64_t(blockIdx.x) * GROWS) / BKR + t / (BKR / 16);
  const int c = t % (BKR / 16);
  uint8_t* kimg = img + kb * B_BYTES;
#pragma unroll
  for (int n = 0; n < NB; ++n) {
    const int d = n >> 2, q = n & 3;
    uint32_t wd[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      uint32_t x = 0;
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        const int e = 4 * b + e4;  // row 16 t + e: phase e % 4
        const uint32_t byte = (e % 4 == q) ? uint32_t(dg[d][e]) : 0u;
        x |= byte << (8 * e4);
      }
      wd[b] = x;
    }
    *reinterpret_cast<uint4*>(kimg + (n >> 3) * B_SBO + c * 128 + (n & 7) * 16) =
        make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
}

// ---------------------------------------------------------------------------
// the pass
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS, 1)
gradtc_kernel(const __grid_constant__ CUtensorMap tmX, const uint8_t* __restrict__ bimg,
              const double* __restrict__ gscale, int64_t m, int64_t n_loc, int tiles, double* __restrict__ out,
              const int* flags) {
  if (flags && (*flags & BS_FLAG_NONFINITE)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* b_base = smem + RS * X_BYTES;
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
    static_assert(BS == 6 && CS == 3, "the unrolled issue loop assumes 6 B stages and 3 A stages");
    static_assert(TMEM_COLS == 512, "a whole-TMEM allocation starts at address 0");
    if (tmem != 0u) __trap();
    const uint32_t my_tiles = uint32_t((tiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x));
    const uint32_t total = my_tiles * uint32_t(nkb);
    const uint64_t b_desc0 = sdesc(smem_u32(b_base), 128, B_SBO, 0);
    const uint32_t blo0 = uint32_t(b_desc0), bhi = uint32_t(b_desc0 >> 32);
    int kb = 0;
    uint32_t gi = 0;
    for (uint32_t g0 = 0; g0 < total; g0 += 6) {
      const uint32_t bph = (g0 / 6) & 1u;
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        if (g0 + uint32_t(u) >= total) break;
        const int cs = u % 3;
        const uint32_t cph = uint32_t(u / 3);  // (g / CS) & 1 with g0 a multiple of 6
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
        // the CTA owns all 512 TMEM columns, so its TMEM base is address 0 (checked above):
        // constant operand addresses keep the issue loop free of register-to-uniform moves
        mma_kblock16(buf * ACC, blo0 + uint32_t((u * B_BYTES) >> 4), bhi, uint32_t(A_COL0 + cs * A_COLS),
                     in_group == 0 ? 0u : 1u);
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
        uint32_t r[16];
        tmem_ld16_u(tmem + lane_addr + buf * ACC, r);
        tc_fence_before();
        mbar_arrive(acc_empty(buf));
        double s = 0.0;
#pragma unroll
        for (int dd = 0; dd < 4; ++dd) {
          double sd = 0.0;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) sd = fma(double(int(r[4 * dd + qq])), ldexp(1.0, -2 * qq), sd);
          s = fma(sd, ldexp(1.0, 7 * (3 - dd)), s);
        }
        acc = fma(s, __ldg(gscale + g), acc);
      }
      if (j < n_loc) out[j] = acc;
    }
  } else {
    // ---------------- converters: packed bytes -> u8 genotypes (x 4^q) in TMEM ----------------
    const int set = (warp - 6) >> 2;
    const int q = warp & 3;
    const int col = q * 32 + lane;  // row of A = column of the tile
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t j0 = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      for (int t = int((uint32_t(set) - j0) & 1u); t < nkb; t += 2) {
        const uint32_t jj = j0 + uint32_t(t);
        const int rst = int(jj % RS), cst = int(jj % CS);
        mbar_wait(raw_full(rst), (jj / RS) & 1);
        mbar_wait(a_empty(cst), ((jj / CS) & 1) ^ 1);
        tc_fence_after();
        // the tile row (128 B) sits in SWIZZLE_128B: 16-byte chunk c of row r at chunk c ^ (r % 8),
        // so the 32 lanes' reads of one chunk spread over the banks
        const uint32_t src = smem_u32(smem + rst * X_BYTES) + uint32_t(col) * BKB;
        const uint32_t sw = uint32_t(col & 7);
#pragma unroll
        for (int h = 0; h < BKB / 32; ++h) {  // 32 packed bytes -> 32 words -> one TMEM store
          const uint4 p0 = ld_shared_v4(src + ((uint32_t(2 * h) ^ sw) << 4));
          const uint4 p1 = ld_shared_v4(src + ((uint32_t(2 * h + 1) ^ sw) << 4));
          const uint32_t pw[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
          uint32_t u[32];
#pragma unroll
          for (int w = 0; w < 8; ++w)
#pragma unroll
            for (int b = 0; b < 4; ++b) u[4 * w + b] = __byte_perm(pw[w], 0u, 0x1111u * uint32_t(b)) & 0xC0300C03u;
          tmem_st32(tmem + lane_addr + uint32_t(A_COL0 + cst * A_COLS + 32 * h), u);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(raw_empty(rst));  // behind the TMEM store, which depends on every loaded word
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
  return ws_bytes<uint8_t>(ng * G * B_BYTES) + ws_bytes<double>(ng);
}

// One tensor-core pass: out[j] = sum_k P[k, j] v[k] for the packed (K x M) block P (ld =
// ceil(K / 64) * 16 bytes per column), one slab.  Returns false when the path does not apply
// (no tcgen05, misaligned P, or the tensor map is refused).
template <typename T>
static bool u2_tc_pass(const void* P, const T* v, int64_t K, int64_t M, double* out, const int* flags, Workspace& ws,
                       cudaStream_t st, int* rc, const char* what) {
  *rc = BS_OK;
  if (!tc_enabled() || K <= 0 || M <= 0 || (reinterpret_cast<uintptr_t>(P) & 15)) return false;
  const int64_t ld = ((K + 63) / 64) * 16;
  const int64_t nkb = (K + BKR - 1) / BKR, ng = (nkb + G - 1) / G;
  uint8_t* img = ws.take<uint8_t>(ng * G * B_BYTES);
  double* gscale = ws.take<double>(ng);
  if (!img || !gscale) {
    set_error("%s: workspace too small", what);
    *rc = BS_EWORK;
    return true;
  }
  CUtensorMap tm;
  if (!make_map_u8(&tm, P, uint64_t(ld), uint64_t(M), BKB, BM)) return false;
  vdigits_kernel<T><<<int(ng), 128, 0, st>>>(v, K, img, gscale, flags);
  const int tiles = int((M + BM - 1) / BM);
  const int grid = std::min(tiles, num_sms());
  smem_attr(gradtc_kernel, SMEM);
  gradtc_kernel<<<grid, THREADS, SMEM, st>>>(tm, img, gscale, K, M, tiles, out, flags);
  *rc = check_launch(what, 2);
  note_gemm_path(6);
  return true;
}

// grad partials (one slab: out[j], j < n_loc) of packed X against v on the tensor cores.
bool launch_grad_u2_tc(const void* P, const double* v, int64_t m, int64_t n_loc, double* out, const int* flags,
                       Workspace& ws, cudaStream_t st, int* rc) {
  return u2_tc_pass<double>(P, v, m, n_loc, out, flags, ws, st, rc, "u2 tensor-core grad");
}

// X beta (out[i], i < m) from the packed transpose Q of the local block (bs_genotype_transpose_packed):
// the same pass with K = n_loc and M = m.
bool launch_xbeta_u2t_tc(const void* Q, const float* beta, int64_t m, int64_t n_loc, double* out, Workspace& ws,
                         cudaStream_t st, int* rc) {
  return u2_tc_pass<float>(Q, beta, n_loc, m, out, nullptr, ws, st, rc, "u2 tensor-core xbeta");
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
