// tcgen05 MDS pass for float32 (solvers.py:269-305, mode 0 of bs_mds_pass).
//
// Per pair (i, j) of the rank's column block of Y the MM step needs
//   d2_ij = |theta_i|^2 + |theta_j|^2 - 2 theta_i . theta_j,  d = sqrt(d2)   (solvers.py:237-247)
//   stress += (y - d)^2,  zsum_j += y / d,  T_j += theta_i (1 - y / d)       (solvers.py:289-300)
// Both reductions over the q coordinates are GEMM-shaped.  With augmented rows
//   I-side  u_i = [theta_i, 1, |theta_i|^2]      J-side  v_j = [-2 theta_j, |theta_j|^2, 1]
// the Gram identity is one product, d2_ij = v_j . u_i, and with w_ij = 1 - z_ij
//   T_aug[j] = sum_i w_ij u_i   gives T_j (first q entries) and sum_i w_ij (entry q),
// so zsum_j = (#i) - T_aug[j][q].  For a tile of 128 columns j x 64 rows i:
//   MMA1  D1[j][i]  = sum_k V[j][k] U[i][k]       M = 128, N = 64, K = 8 * ceil((q + 2) / 8)
//   MMA2  D2[j][k] += sum_i W[j][i] U[i][k]       M = 128, N = 32, K = 64
// both in 3xTF32 (hi*hi + hi*lo + lo*hi: fp32-level error).  When 1 <= max_i |theta_i|^2 < 2^14
// MMA1 runs on an f16 hi/lo split instead (kind::f16, K = 16 per instruction: 6 MMAs per chunk
// instead of 9 at q = 20; same three products, error ~2^-23 of the operands; see f16_range).  Per pair the CUDA cores only
// do rsqrt, d, z, (y - d)^2, 1 - z and the tf32 split (about 9 instructions).  Y is read
// once, by TMA, like the CUDA-core pass (mds.cu).
//
// CTA (one per SM, persistent over (128-column block, row segment) units), 576 threads:
//   warp 0      TMA producer
//   warp 1      MMA issuer (one elected lane): MMA1 runs ahead of MMA2 (bounded by D1 buffers)
//   warps 2-17  epilogue: warp w owns TMEM lane quarter w % 4 (lane = column j) and one
//               16-row slice of the chunk: tcgen05.ld d2, elementwise chain, tcgen05.st
//               the hi/lo split of w as MMA2's A operand (TMEM, K-major)
// Shared-memory rings, each released as soon as its consumer is done:
//   Y  (2 boxes of 32 i x 128 j, SWIZZLE_128B)              freed by the epilogue once loaded
//   B1 (U hi | lo, 64 i x 32 k, K-major SWIZZLE_128B)        freed by MMA1's commit
//   B2 (U hi | lo, 2 x (32 i x 32 k) MN-major SW128_BASE32B) freed by MMA2's commit
// TMEM (512 columns): D1 x2 [0,128), D2 [128,192), A1 = V_J hi|lo [192,256), A2 x2 [256,512).
// D2 is restarted every G chunks and folded into fp32 registers (the tensor core's
// accumulator add truncates, see nmf_tc.cu).
//
// Cancellation guard: where d2 <= 2^-12 (|theta_j|^2 + max_i |theta_i|^2) the pair is
// recomputed from the coordinates, sum_k (theta_ik - theta_jk)^2, so exactly coincident
// points give d = 0 exactly, as the reference's Gram identity does on its own input
// (solvers.py:246, 290-296).
#include "tc_common.cuh"

#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <vector>

using namespace bs;
using namespace tc;

namespace {

constexpr int MT_THREADS = 576;  // TMA warp, MMA warp, 16 epilogue warps
constexpr int NEPI = 512;        // epilogue threads
constexpr int CHI = 64;          // rows i per chunk
constexpr int BJ = 128;          // columns j per unit (MMA M)
constexpr int KP = 32;           // augmented q padded (one 128-byte row of fp32)
constexpr int Y_BOX = 32 * 4 * BJ;   // 16 KB
constexpr int Y_STAGE = 2 * Y_BOX;
constexpr int B_STAGE = 16384;       // hi at 0, lo at 8192
constexpr int NY = 4, NB1 = 2, NB2 = 3;  // Y is held until its pairs are done
constexpr int OFF_B1 = NY * Y_STAGE;
constexpr int OFF_B2 = OFF_B1 + NB1 * B_STAGE;
constexpr int RINGS = OFF_B2 + NB2 * B_STAGE;
constexpr int SMEM = RINGS + 1024 /*align*/ + 512 /*barriers*/ + 16 * 2 * 8 /*stress fold*/ + 512;
constexpr uint32_t T_D1 = 0, T_D2 = 128, T_A1 = 192, T_A2 = 256;
constexpr int B1_F16 = CHI * 128;    // f16 B1 stage: one 128-byte row [hi k0..31 | lo k0..31] per i
// f16 range of MMA1's operands: |theta| < 128 and |theta|^2 < 2^14 keep every hi part finite;
// below max |theta|^2 = 1 the subnormal lo parts of small coordinates would cost more than the
// tf32 split's error, so that case stays on 3xTF32.
__host__ __device__ inline bool f16_range(float nmax) { return nmax >= 1.0f && nmax < 16384.0f; }
constexpr float CANCEL = 1.0f / 4096.0f;

// One 8-wide k step of MMA1: D += A_hi Bh + A_hi Bl + A_lo Bh (K-major smem B).
__device__ __forceinline__ void mma3_kstep(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                           uint32_t id, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, q;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, 1;\n\t}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(id), "r"(acc0)
      : "memory");
}

// The same k step on the f16 split (K = 16): D += A_hi Bh + A_hi Bl + A_lo Bh.
__device__ __forceinline__ void mma3_kstep_f16(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                               uint32_t id, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, q;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, 1;\n\t}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(id), "r"(acc0)
      : "memory");
}

// kind::f16 (f16 x f16 -> f32), both operands K-major.
constexpr uint32_t idesc_f16(int M, int N) { return (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24); }

__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)), "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // max rel. error 2^-22.9
  return r;
}

// sum_k (theta_ik - theta_jk)^2 from the coordinates (cancellation path only).
__device__ __noinline__ float direct_d2(const float* ti, const float* tj, int q) {
  float acc = 0.f;
  for (int k = 0; k < q; ++k) {
    const float df = ti[k] - tj[k];
    acc = fmaf(df, df, acc);
  }
  return acc;
}

// The 16 pairs of one (column, row slice) with every special case of the MM step:
// buf[0..16) = y, buf[16..32) = d2 from the tensor core; writes w = (W - Z)_ij to
// buf[32..48) and returns the slice's stress.
__device__ __noinline__ float careful_block(float* buf, int ib, int i_end, int jg, bool live, float thr,
                                           const float* theta, int q, int perturb, double& zeros) {
  float st = 0.f;
  for (int e = 0; e < 16; ++e) {
    const int i = ib + e;
    const float y = buf[e];
    float w = 0.f;
    if (live && i < i_end) {
      if (i == jg) {  // d_jj = 0 exactly, (W - Z)_jj = 0 (solvers.py:240-241, 299-300)
        st = fmaf(y, y, st);
      } else {
        float d2 = buf[16 + e];
        if (!(d2 > thr)) d2 = direct_d2(theta + int64_t(i) * q, theta + int64_t(jg) * q, q);
        float d, z;
        if (d2 > 0.f) {
          const float r = rsqrt_approx(d2);
          d = d2 * r;
          z = y * r;  // solvers.py:297
        } else {
          d = 0.f;
          zeros += 1.0;
          z = perturb ? y * 1e10f : __fdiv_rn(y, 0.f);  // solvers.py:296
        }
        const float er = y - d;
        st = fmaf(er, er, st);
        w = 1.f - z;  // solvers.py:299
      }
    }
    buf[32 + e] = w;
  }
  return st;
}

constexpr int TR_CHUNKS = 4096;  // trace: first chunks of CTA 0
__device__ __forceinline__ void tr_mark(unsigned long long* tr, int ev, uint32_t chunk) {
#ifndef BS_DEBUG_MODES
  return;  // the event trace (BS_MDS_TC_TRACE) exists only in debug builds
#endif
  if (tr && blockIdx.x == 0 && chunk < TR_CHUNKS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[ev * TR_CHUNKS + chunk] = t;
  }
}

struct MdsTcArgs {
  const float* theta;   // q x n (theta_full, column-major)
  const float* vj_hi;   // n x 32: [-2 theta_j, |theta_j|^2, 1, 0...] tf32 hi
  const float* vj_lo;   //         ... lo
  const uint32_t* vj16; // n x 32 words: the same row as f16 [hi k0..31 | lo k0..31]
  int f16_ok;           // 0: MMA1 always in 3xTF32 (BS_MDS_TC_F16=0)
  const float* norms;   // n
  const float* nmax;    // max_i |theta_i|^2 (1 float)
  int64_t n, lo, n_loc;
  int q, perturb, G;
  int mode;             // debug (BS_MDS_TC_MODE): 1 skips the pair math, 2 the MMAs
  unsigned long long* trace;  // debug (BS_MDS_TC_TRACE): CTA 0 event times, [event][chunk]
  int jblocks, segs;
  int64_t rows_per_seg;
  double* zsum_part;    // [segs][n_loc]
  double* T_part;       // [segs][n_loc][q]
  double* parts;        // [grid][2]
  unsigned int* counter;
  double* red;
};

template <int KS>
__global__ void __launch_bounds__(MT_THREADS, 1)
mds_tc_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmKh,
              const __grid_constant__ CUtensorMap tmKl, const __grid_constant__ CUtensorMap tmMh,
              const __grid_constant__ CUtensorMap tmMl, const __grid_constant__ CUtensorMap tmK16,
              const MdsTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RINGS);
  // d1_full[2], d1_empty[2], a2_full[2], a2_empty[2], d2_full, d2_empty, a1_full, a1_empty,
  // y_full[NY], y_empty[NY], b1_full[NB1], b1_empty[NB1], b2_full[NB2], b2_empty[NB2]
  constexpr int NBAR = 12 + 2 * (NY + NB1 + NB2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);
  double* red_sh = reinterpret_cast<double*>(smem + RINGS + 512);  // [16][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto d1_full = [&](int b) { return smem_u32(bars + b); };
  auto d1_empty = [&](int b) { return smem_u32(bars + 2 + b); };
  auto a2_full = [&](int b) { return smem_u32(bars + 4 + b); };
  auto a2_empty = [&](int b) { return smem_u32(bars + 6 + b); };
  const uint32_t d2_full = smem_u32(bars + 8), d2_empty = smem_u32(bars + 9);
  const uint32_t a1_full = smem_u32(bars + 10), a1_empty = smem_u32(bars + 11);
  auto y_full = [&](int s) { return smem_u32(bars + 12 + s); };
  auto y_empty = [&](int s) { return smem_u32(bars + 12 + NY + s); };
  auto b1_full = [&](int s) { return smem_u32(bars + 12 + 2 * NY + s); };
  auto b1_empty = [&](int s) { return smem_u32(bars + 12 + 2 * NY + NB1 + s); };
  auto b2_full = [&](int s) { return smem_u32(bars + 12 + 2 * NY + 2 * NB1 + s); };
  auto b2_empty = [&](int s) { return smem_u32(bars + 12 + 2 * NY + 2 * NB1 + NB2 + s); };
  auto y_at = [&](uint32_t c) { return smem + (c % NY) * Y_STAGE; };
  auto b1_at = [&](uint32_t c) { return smem + OFF_B1 + (c % NB1) * B_STAGE; };
  auto b2_at = [&](uint32_t c) { return smem + OFF_B2 + (c % NB2) * B_STAGE; };

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(d1_full(b), 1);
      mbar_init(d1_empty(b), NEPI);
      mbar_init(a2_full(b), NEPI);
      mbar_init(a2_empty(b), 1);
    }
    mbar_init(d2_full, 1);
    mbar_init(d2_empty, NEPI);
    mbar_init(a1_full, NEPI);
    mbar_init(a1_empty, 1);
    for (int s = 0; s < NY; ++s) {
      mbar_init(y_full(s), 1);
      mbar_init(y_empty(s), NEPI);
    }
    for (int s = 0; s < NB1; ++s) {
      mbar_init(b1_full(s), 1);
      mbar_init(b1_empty(s), 1);
    }
    for (int s = 0; s < NB2; ++s) {
      mbar_init(b2_full(s), 1);
      mbar_init(b2_empty(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmY);
    prefetch_tmap(&tmKh);
    prefetch_tmap(&tmK16);
    prefetch_tmap(&tmKl);
    prefetch_tmap(&tmMh);
    prefetch_tmap(&tmMl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int units = a.jblocks * a.segs;
  const bool f16 = a.f16_ok && f16_range(__ldg(a.nmax));  // uniform over the grid
  auto unit_range = [&](int u, int64_t& j0, int64_t& i0, int& nch, int& seg) {
    seg = u / a.jblocks;
    j0 = int64_t(u - seg * a.jblocks) * BJ;
    i0 = int64_t(seg) * a.rows_per_seg;
    const int64_t i1 = min(a.n, i0 + a.rows_per_seg);
    nch = int((i1 - i0 + CHI - 1) / CHI);
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      uint32_t cc = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t j0, i0;
        int nch, seg;
        unit_range(u, j0, i0, nch, seg);
        for (int t = 0; t < nch; ++t, ++cc) {
          const int ic = int(i0 + int64_t(t) * CHI);
          {  // MMA1's B first: it gates the chunk's first MMA
            const int s = int(cc % NB1);
            mbar_wait_sleep(b1_empty(s), ((cc / NB1) & 1) ^ 1);
            const uint32_t fb = b1_full(s), base = smem_u32(b1_at(cc));
            if (f16) {
              mbar_expect_tx(fb, B1_F16);
              tma_load_2d(base, &tmK16, 0, ic, fb);
            } else {
              mbar_expect_tx(fb, B_STAGE);
              tma_load_2d(base, &tmKh, 0, ic, fb);
              tma_load_2d(base + 8192, &tmKl, 0, ic, fb);
            }
          }
          {
            const int s = int(cc % NY);
            mbar_wait_sleep(y_empty(s), ((cc / NY) & 1) ^ 1);
            const uint32_t fb = y_full(s), base = smem_u32(y_at(cc));
            mbar_expect_tx(fb, Y_STAGE);
            tma_load_2d(base, &tmY, ic, int(j0), fb);
            tma_load_2d(base + Y_BOX, &tmY, ic + 32, int(j0), fb);
          }
          {
            const int s = int(cc % NB2);
            mbar_wait_sleep(b2_empty(s), ((cc / NB2) & 1) ^ 1);
            const uint32_t fb = b2_full(s), base = smem_u32(b2_at(cc));
            mbar_expect_tx(fb, B_STAGE);
            tma_load_2d(base, &tmMh, 0, ic, fb);
            tma_load_2d(base + 4096, &tmMh, 0, ic + 32, fb);
            tma_load_2d(base + 8192, &tmMl, 0, ic, fb);
            tma_load_2d(base + 8192 + 4096, &tmMl, 0, ic + 32, fb);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // Event loop: MMA1 of the next chunk is issued as soon as its B1 stage has landed and
    // its D1 buffer is free (the epilogue has loaded D1 of chunk t1 - 2, early in its
    // work on that chunk), so it overtakes MMA2 of the chunk the epilogue is finishing;
    // MMA2 of the oldest chunk goes as soon as its A2 is written.  The tensor pipe
    // executes in issue order.
    constexpr uint32_t id1 = idesc_tf32(128, CHI, false, false);
    constexpr uint32_t id1h = idesc_f16(128, CHI);
    constexpr int KS16 = (KS + 1) / 2;
    constexpr uint32_t id2w = idesc_tf32(128, 2 * KP, false, true);
    constexpr uint32_t id2n = idesc_tf32(128, KP, false, true);
    uint32_t cbase = 0, gi = 0, ut = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ut) {
      int64_t j0, i0;
      int nch, seg;
      unit_range(u, j0, i0, nch, seg);
      mbar_wait_sleep(a1_full, ut & 1);
      tc_fence_after();
      int t1 = 0, t2 = 0, g2 = 0;  // g2 = t2 mod G (no division in the loop)
      while (t2 < nch) {
        bool issued = false;
        if (t1 < nch) {  // bounded by d1_empty: at most two chunks ahead of the epilogue's D1 reads
          const uint32_t c = cbase + uint32_t(t1);
          const int s = int(c % NB1);
          const uint32_t b = c & 1;
          // lanes could see a phase complete at different instants: decide on lane 0 only,
          // or part of the warp would issue the MMA now and the rest again later
          int probe = 0;
          if (lane == 0) probe = mbar_test(b1_full(s), (c / NB1) & 1) && mbar_test(d1_empty(b), ((c >> 1) & 1) ^ 1);
          const bool go = __shfl_sync(0xffffffffu, probe, 0) != 0;
          if (go) {
            tc_fence_after();
            const uint32_t d = __shfl_sync(0xffffffffu, tmem + T_D1 + b * CHI, 0);
            const uint32_t ah = __shfl_sync(0xffffffffu, tmem + T_A1, 0);
            const uint32_t bh = __shfl_sync(0xffffffffu, smem_u32(b1_at(c)), 0);
            const uint64_t dh = sdesc(bh, 16, 1024, LAYOUT_SW128), dl = sdesc(bh + 8192, 16, 1024, LAYOUT_SW128);
            if (f16) {
              // A1: hi in columns 0-15, lo in 16-31 (two f16 per column); B1 row: hi at +0, lo at +64 B
#pragma unroll
              for (int k = 0; k < KS16; ++k)
                if (!(a.mode & 2)) mma3_kstep_f16(d, ah + 8 * k, ah + 16 + 8 * k, dh + 2 * k, dh + 4 + 2 * k, id1h, k > 0);
            } else {
#pragma unroll
              for (int k = 0; k < KS; ++k)
                if (!(a.mode & 2)) mma3_kstep(d, ah + 8 * k, ah + 32 + 8 * k, dh + 2 * k, dl + 2 * k, id1, k > 0);
            }
            mma_commit_elect(d1_full(b));
            if (lane == 0) tr_mark(a.trace, 0, c);  // MMA1 issued
            mma_commit_elect(b1_empty(s));
            if (t1 == nch - 1) mma_commit_elect(a1_empty);
            __syncwarp();
            ++t1;
            issued = true;
          }
        }
        if (t2 < t1) {
          const uint32_t c = cbase + uint32_t(t2);
          const uint32_t b = c & 1;
          const int s = int(c % NB2);
          const bool first = g2 == 0;
          const bool last = (g2 == a.G - 1) || (t2 == nch - 1);
          int probe = 0;
          if (lane == 0)
            probe = mbar_test(a2_full(b), (c >> 1) & 1) && (!first || mbar_test(d2_empty, (gi & 1) ^ 1)) &&
                    mbar_test(b2_full(s), (c / NB2) & 1);
          const bool go = __shfl_sync(0xffffffffu, probe, 0) != 0;
          if (go) {
            tc_fence_after();
            const uint32_t d = __shfl_sync(0xffffffffu, tmem + T_D2, 0);
            const uint32_t ah = __shfl_sync(0xffffffffu, tmem + T_A2 + b * 128, 0);
            const uint32_t b2 = __shfl_sync(0xffffffffu, smem_u32(b2_at(c)), 0);
            const uint64_t bd = sdesc(b2, 8192, 512, LAYOUT_SW128_32B);
            if (!(a.mode & 2)) {
              mma_kblock_concat(d, ah, ah + 64, bd, id2w, id2n, first ? 0u : 1u);
              mma_kblock_concat(d, ah + 32, ah + 96, bd + 256, id2w, id2n, 1u);
            }
            mma_commit_elect(a2_empty(b));
            if (lane == 0) tr_mark(a.trace, 1, c);  // MMA2 issued
            mma_commit_elect(b2_empty(s));
            if (last) {
              mma_commit_elect(d2_full);
              ++gi;
            }
            __syncwarp();
            ++t2;
            g2 = g2 == a.G - 1 ? 0 : g2 + 1;
            issued = true;
          }
        }
        if (!issued) __nanosleep(64);
      }
      cbase += uint32_t(nch);
    }
  } else {
    // ---------------- epilogue (warps 2..17) ----------------
    // warp w may touch TMEM lanes 32 (w % 4)..+31 (its column quarter); the four warps of a
    // quarter split the chunk's 64 rows into 16-row slices (sub).
    const int qd = warp & 3, sub = (warp - 2) >> 2, ew = warp - 2;
    const int jrow = qd * 32 + lane;
    const uint32_t lane_addr = uint32_t(qd * 32) << 16;
    const int q = a.q;
    const float nmax = __ldg(a.nmax);
    uint32_t cc = 0, gi = 0, ut = 0;
    double stress = 0.0, zeros = 0.0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ut) {
      int64_t j0, i0;
      int nch, seg;
      unit_range(u, j0, i0, nch, seg);
      // 32-bit row / column indices (n <= INT32_MAX is part of mds_tc_eligible): 64-bit ones
      // cost four registers the 96-register budget does not have (they were spilled)
      const int jl = int(j0) + jrow;
      const bool live = jl < a.n_loc;
      const int jg = int(a.lo) + (live ? jl : 0);
      const int i0i = int(i0);
      const int i_end = int(min(a.n, i0 + a.rows_per_seg));
      // A1: v_j into TMEM (K-major): sub 0/1 write hi k 0-15/16-31, sub 2/3 the lo half
      mbar_wait(a1_empty, (ut & 1) ^ 1);
      tc_fence_after();
      if (f16) {  // sub 0 / 1 write the hi / lo half (16 columns each)
        if (sub < 2) {
          uint32_t v[16];
          const uint4* src = reinterpret_cast<const uint4*>(a.vj16 + int64_t(jg) * KP + 16 * sub);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 w = live ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
            v[4 * c] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
          }
          tmem_st16(tmem + lane_addr + T_A1 + 16 * sub, v);
          tmem_wait_st();
        }
      } else {
        uint32_t v[16];
        const float4* src = reinterpret_cast<const float4*>((sub >= 2 ? a.vj_lo : a.vj_hi) + jg * KP + 16 * (sub & 1));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 w = live ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * c] = __float_as_uint(w.x); v[4 * c + 1] = __float_as_uint(w.y);
          v[4 * c + 2] = __float_as_uint(w.z); v[4 * c + 3] = __float_as_uint(w.w);
        }
        tmem_st16(tmem + lane_addr + T_A1 + 16 * sub, v);
        tmem_wait_st();
      }
      tc_fence_before();
      mbar_arrive(a1_full);
      const float nj = live ? __ldg(a.norms + jg) : 0.f;
      const float thr = CANCEL * (nj + nmax);
      float Tacc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) Tacc[k] = 0.f;
      bool fold_pending = false;
      int gpos = 0;  // t mod G
      auto fold = [&]() {
        mbar_wait(d2_full, gi & 1);
        tc_fence_after();
        float v[8], w[8];
        tmem_ld8(tmem + lane_addr + T_D2 + 8 * sub, v);
        tmem_ld8(tmem + lane_addr + T_D2 + KP + 8 * sub, w);
#pragma unroll
        for (int k = 0; k < 8; ++k) Tacc[k] = __fadd_rn(Tacc[k], __fadd_rn(v[k], w[k]));
        tc_fence_before();
        mbar_arrive(d2_empty);
        ++gi;
        fold_pending = false;
      };
      // D1 of the next chunk is waited for and its TMEM load started at the end of the previous
      // chunk; the load's completion is awaited only after the Y loads of the chunk are issued
      uint32_t g[16];
      auto d1_issue = [&](uint32_t c) {
        mbar_wait(d1_full(c & 1), (c >> 1) & 1);
        tc_fence_after();
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]), "=r"(g[7]),
              "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]), "=r"(g[12]), "=r"(g[13]), "=r"(g[14]), "=r"(g[15])
            : "r"(tmem + lane_addr + T_D1 + (c & 1) * CHI + 16 * sub));
      };
      if (nch > 0) d1_issue(cc);
      for (int t = 0; t < nch; ++t, ++cc) {
        const int s = int(cc % NY);
        const uint32_t b = cc & 1;
        const int ib = i0i + t * CHI + 16 * sub;  // first row of this warp's 16
        // Y tile: box sub/2 holds rows 32 (sub/2) .. +31; row jrow is 128 B of 16 B chunks
        // stored at chunk ^ (jrow & 7) (SWIZZLE_128B)
        uint4 yv[4];
        {
          mbar_wait(y_full(s), (cc / NY) & 1);
          if (warp == 2 && lane == 0) tr_mark(a.trace, 2, cc);  // Y landed
          const uint32_t ybase = smem_u32(y_at(cc) + (sub >> 1) * Y_BOX) + uint32_t(jrow) * 128u;
          const uint32_t c0 = uint32_t(sub & 1) * 4u;
#pragma unroll
          for (int c = 0; c < 4; ++c) yv[c] = ld_shared_v4(ybase + (((c0 + uint32_t(c)) ^ uint32_t(jrow & 7)) << 4));
          // y_empty is signalled only after the pair math has used every loaded value: an arrive
          // right behind the LDS does not wait for them to return (the TMA then refilled the stage
          // under the load — seen as run-to-run differences once the math was rescheduled)
        }
        float y[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          y[4 * c] = __uint_as_float(yv[c].x); y[4 * c + 1] = __uint_as_float(yv[c].y);
          y[4 * c + 2] = __uint_as_float(yv[c].z); y[4 * c + 3] = __uint_as_float(yv[c].w);
        }
        if (warp == 2 && lane == 0) tr_mark(a.trace, 3, cc);  // D1 ready
        asm volatile("tcgen05.wait::ld.sync.aligned;"  // tied to g: no use of g moves above it
                     : "+r"(g[0]), "+r"(g[1]), "+r"(g[2]), "+r"(g[3]), "+r"(g[4]), "+r"(g[5]), "+r"(g[6]), "+r"(g[7]),
                       "+r"(g[8]), "+r"(g[9]), "+r"(g[10]), "+r"(g[11]), "+r"(g[12]), "+r"(g[13]), "+r"(g[14]), "+r"(g[15])
                     :
                     : "memory");
        tc_fence_before();
        mbar_arrive(d1_empty(b));
        uint32_t wz[16], wl[16];
        float st_blk = 0.f, dmin = 1e30f;
        if (a.mode & 1) {
#pragma unroll
          for (int e = 0; e < 16; ++e) wz[e] = wl[e] = g[e] ^ __float_as_uint(y[e]);
        } else {
        // two pairs per packed f32x2 instruction (same per-element roundings as the scalar chain;
        // the slice's stress is summed in two interleaved chains)
        float2 st2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float2 d2 = make_float2(__uint_as_float(g[e]), __uint_as_float(g[e + 1]));  // solvers.py:246
          dmin = fminf(dmin, fminf(d2.x, d2.y));
          const float2 r = make_float2(rsqrt_approx(d2.x), rsqrt_approx(d2.y));
          const float2 yy = make_float2(y[e], y[e + 1]);
          const float2 d = mul2(d2, r);
          const float2 z = mul2(yy, r);        // solvers.py:297
          const float2 er = sub2(yy, d);
          st2 = fma2(er, er, st2);
          const float2 w = sub2(make_float2(1.f, 1.f), z);  // solvers.py:299
          const uint32_t h0 = tf32_hi(__float_as_uint(w.x)), h1 = tf32_hi(__float_as_uint(w.y));
          const float2 lo = sub2(w, make_float2(__uint_as_float(h0), __uint_as_float(h1)));
          wz[e] = h0;
          wz[e + 1] = h1;
          wl[e] = __float_as_uint(lo.x);
          wl[e + 1] = __float_as_uint(lo.y);
        }
        st_blk = st2.x + st2.y;
        }
        const bool bad = !(a.mode & 1) && (!(dmin > thr) || !live || (ib + 16 > i_end) || (jg >= ib && jg < ib + 16));
        if (bad) {
          // careful path (tails, the diagonal, padding columns, cancellation): out of line,
          // through a local buffer so the fast path keeps everything in registers
          float buf[48];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            buf[e] = y[e];
            buf[16 + e] = __uint_as_float(g[e]);
          }
          st_blk = careful_block(buf, ib, i_end, jg, live, thr, a.theta, q, a.perturb, zeros);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float w = buf[32 + e];
            const uint32_t hw = tf32_hi(__float_as_uint(w));
            wz[e] = hw;
            wl[e] = __float_as_uint(w - __uint_as_float(hw));
          }
        }
        mbar_arrive(y_empty(s));  // behind the math that consumed every y value
        stress += double(st_blk);
        // A2 <- hi | lo of W for this chunk
        mbar_wait(a2_empty(b), ((cc >> 1) & 1) ^ 1);
        tc_fence_after();
        {
          const uint32_t a2 = tmem + lane_addr + T_A2 + b * 128 + 16 * sub;
          tmem_st16(a2, wz);
          tmem_st16(a2 + 64, wl);
          tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(a2_full(b));
        if (warp == 2 && lane == 0) tr_mark(a.trace, 4, cc);  // A2 written (warp 2)
        if (t + 1 < nch) d1_issue(cc + 1);
        if (fold_pending) fold();
        if (gpos == a.G - 1 || t == nch - 1) fold_pending = true;
        gpos = gpos == a.G - 1 ? 0 : gpos + 1;
      }
      if (fold_pending) fold();
      // ---- unit outputs: T (each slice owns 8 of the augmented k) and zsum = #i - sum_i w ----
      if (live) {
        double* tp = a.T_part + (int64_t(seg) * a.n_loc + jl) * q;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int kk = 8 * sub + k;
          if (kk < q) tp[kk] = double(Tacc[k]);
          if (kk == q) {
            const int cnt = (i_end - i0i) - ((jg >= i0i && jg < i_end) ? 1 : 0);
            a.zsum_part[int64_t(seg) * a.n_loc + jl] = double(cnt) - double(Tacc[k]);
          }
        }
      }
    }
    // ---- CTA stress / zero-count partial: warps in order ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      stress += __shfl_xor_sync(0xffffffffu, stress, o);
      zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
    }
    if (lane == 0) {
      red_sh[2 * ew] = stress;
      red_sh[2 * ew + 1] = zeros;
    }
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (ew == 0 && lane == 0) {
      double s0 = 0.0, z0 = 0.0;
      for (int w = 0; w < 16; ++w) {
        s0 += red_sh[2 * w];
        z0 += red_sh[2 * w + 1];
      }
      a.parts[2 * blockIdx.x] = s0;
      a.parts[2 * blockIdx.x + 1] = z0;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (last_block_done(a.counter) && threadIdx.x == 0) {
    double s0 = 0.0, z0 = 0.0;
    for (unsigned int k = 0; k < gridDim.x; ++k) {
      s0 += a.parts[2 * k];
      z0 += a.parts[2 * k + 1];
    }
    a.red[0] = s0;
    a.red[1] = z0;
  }
}

// theta (q x n) -> augmented rows (tf32 hi / lo, padded to 32):
//   U_i = [theta_i, 1, |theta_i|^2]   V_i = [-2 theta_i, |theta_i|^2, 1]
// plus |theta_i|^2 and max_i |theta_i|^2 (nmax zeroed by the caller; norms are >= 0, so
// their float bits order like integers).
__global__ void mds_tc_prep_kernel(const float* __restrict__ theta, int64_t n, int q, float* __restrict__ uh,
                                   float* __restrict__ ul, float* __restrict__ vh, float* __restrict__ vl,
                                   __half* __restrict__ u16, __half* __restrict__ v16, float* __restrict__ norms,
                                   float* __restrict__ nmax) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float* t = theta + i * q;
    float s = 0.f;
    for (int k = 0; k < q; ++k) s = fmaf(t[k], t[k], s);
    norms[i] = s;
    atomicMax(reinterpret_cast<unsigned int*>(nmax), __float_as_uint(s));
    float* uhr = uh + i * KP;
    float* ulr = ul + i * KP;
    float* vhr = vh + i * KP;
    float* vlr = vl + i * KP;
    __half* u16r = u16 + i * 2 * KP;
    __half* v16r = v16 + i * 2 * KP;
    for (int k = 0; k < KP; ++k) {
      const float u = k < q ? t[k] : k == q ? 1.f : k == q + 1 ? s : 0.f;
      const float v = k < q ? -2.f * t[k] : k == q ? s : k == q + 1 ? 1.f : 0.f;
      const uint32_t hu = tf32_hi(__float_as_uint(u)), hv = tf32_hi(__float_as_uint(v));
      uhr[k] = __uint_as_float(hu);
      ulr[k] = u - __uint_as_float(hu);
      vhr[k] = __uint_as_float(hv);
      vlr[k] = v - __uint_as_float(hv);
      // f16 split (used only when f16_range holds: no overflow then)
      const __half u1 = __float2half_rn(u), v1 = __float2half_rn(v);
      u16r[k] = u1;
      u16r[KP + k] = __float2half_rn(u - __half2float(u1));
      v16r[k] = v1;
      v16r[KP + k] = __float2half_rn(v - __half2float(v1));
    }
  }
}

struct TcGrid {
  int jblocks, segs, grid;
  int64_t rows_per_seg;
};

TcGrid tc_grid(int64_t n, int64_t n_loc) {
  TcGrid g;
  g.jblocks = int(ceil_div(n_loc, BJ));
  const int64_t chunks = ceil_div(n, CHI);
  const int sms = num_sms();
  // Units differ in duration (diagonal / tail units take the careful path), so the
  // schedule needs enough of them: prefer >= 7.5 waves, then the best wave rounding
  // (measured at n = 100,000: n_loc = 25,000 takes 3.76 ms with 3 segments, 3.45 ms
  // with 6; n_loc = 12,500: 1.98 -> 1.78 ms).
  int best = 1;
  double best_score = -1e9;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && chunks / s < 16) break;
    const double units = double(g.jblocks) * s;
    const double waves = units / sms;
    const double score = waves / std::ceil(waves) - 0.002 * s - (waves < 7.5 ? 1.0 : 0.0);
    if (score > best_score + 1e-9) { best_score = score; best = s; }
  }
  static const int force = [] {
    const char* e = getenv("BS_MDS_TC_SEGS");  // experiments: fixed segment count
    return e ? atoi(e) : 0;
  }();
  if (force > 0) best = force;
  g.rows_per_seg = ceil_div(ceil_div(n, best), CHI) * CHI;
  g.segs = int(ceil_div(n, g.rows_per_seg));
  g.grid = int(std::min<int64_t>(int64_t(g.jblocks) * g.segs, sms));
  return g;
}

}  // namespace

namespace bs {

bool mds_tc_eligible(int dtype, int64_t n, int64_t n_loc, int q, int mode, const void* Y, const void* theta) {
  return dtype == BS_F32 && mode == 0 && q >= 1 && q + 2 <= KP && n % 4 == 0 && n >= CHI && n_loc >= 1 &&
         n <= INT32_MAX && n_loc <= INT32_MAX && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(theta) & 15) == 0 && tc::tc_enabled();
}

int64_t mds_tc_workspace(int64_t n, int64_t n_loc, int q) {
  TcGrid g = tc_grid(n, n_loc);
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(2 * int64_t(g.grid)) + ws_bytes<double>(int64_t(g.segs) * n_loc) +
         ws_bytes<double>(int64_t(g.segs) * n_loc * q) + ws_bytes<float>(n) + ws_bytes<float>(1) +
         6 * ws_bytes<float>(n * KP);
}

// Returns BS_OK with *segs_out / the partial pointers set for mds_fold_kernel.
int mds_tc_pass(const float* Y, const float* theta, int64_t n, int64_t lo, int64_t n_loc, int q, int perturb,
                double* red, Workspace& ws, cudaStream_t st, double** zp_out, double** tp_out, int* segs_out) {
  TcGrid g = tc_grid(n, n_loc);
  unsigned int* ctr = ws.take<unsigned int>(1);
  double* parts = ws.take<double>(2 * int64_t(g.grid));
  double* zp = ws.take<double>(int64_t(g.segs) * n_loc);
  double* tp = ws.take<double>(int64_t(g.segs) * n_loc * q);
  float* norms = ws.take<float>(n);
  float* nmax = ws.take<float>(1);
  float* uh = ws.take<float>(n * KP);
  float* ul = ws.take<float>(n * KP);
  float* vh = ws.take<float>(n * KP);
  float* vl = ws.take<float>(n * KP);
  float* u16 = ws.take<float>(n * KP);  // n rows of 64 halves
  float* v16 = ws.take<float>(n * KP);
  if (!ctr || !parts || !zp || !tp || !norms || !nmax || !uh || !ul || !vh || !vl || !u16 || !v16) {
    set_error("bs_mds_pass: workspace too small");
    return BS_EWORK;
  }
  CUtensorMap mY, mKh, mKl, mMh, mMl, mK16;
  bool ok = make_map_f32(&mY, Y, uint64_t(n), uint64_t(n_loc), 32, BJ, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mKh, uh, KP, uint64_t(n), KP, CHI, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mKl, ul, KP, uint64_t(n), KP, CHI, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mK16, u16, KP, uint64_t(n), KP, CHI, CU_TENSOR_MAP_SWIZZLE_128B) &&  // 128-byte f16 rows
            make_map_f32(&mMh, uh, KP, uint64_t(n), KP, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
            make_map_f32(&mMl, ul, KP, uint64_t(n), KP, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) {
    set_error("bs_mds_pass: cuTensorMapEncodeTiled failed");
    return BS_ECUDA;
  }
  static int group = -1, mode = 0, f16_ok = 1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("BS_MDS_TC_GROUP");
    group = (e && atoi(e) > 0) ? atoi(e) : 2;
    const char* h = getenv("BS_MDS_TC_F16");  // A/B switch: 0 keeps MMA1 in 3xTF32
    f16_ok = (h && atoi(h) == 0) ? 0 : 1;
#ifdef BS_DEBUG_MODES  // work-skipping switches only in debug builds (scripts/mds_modes.sh)
    const char* m = getenv("BS_MDS_TC_MODE");
    mode = m ? atoi(m) : 0;
#endif
  });
  smem_attr(mds_tc_kernel<1>, SMEM);
  smem_attr(mds_tc_kernel<2>, SMEM);
  smem_attr(mds_tc_kernel<3>, SMEM);
  smem_attr(mds_tc_kernel<4>, SMEM);
  if (cudaMemsetAsync(nmax, 0, sizeof(float), st) != cudaSuccess) {
    set_error("bs_mds_pass: cudaMemsetAsync failed");
    return BS_ECUDA;
  }
  mds_tc_prep_kernel<<<int(std::min<int64_t>(ceil_div(n, 256), 2048)), 256, 0, st>>>(theta, n, q, uh, ul, vh, vl,
      reinterpret_cast<__half*>(u16), reinterpret_cast<__half*>(v16), norms, nmax);
  static unsigned long long* trace = nullptr;
#ifdef BS_DEBUG_MODES  // the event trace exists only in debug builds (tr_mark)
  static const bool tracing = getenv("BS_MDS_TC_TRACE") != nullptr;
#else
  constexpr bool tracing = false;
#endif
  if (tracing && !trace) cudaMalloc(&trace, sizeof(unsigned long long) * 5 * TR_CHUNKS);
  MdsTcArgs args{theta, vh, vl, reinterpret_cast<const uint32_t*>(v16), f16_ok, norms, nmax, n, lo, n_loc, q, perturb, group, mode, trace, g.jblocks, g.segs, g.rows_per_seg,
                 zp, tp, parts, ctr, red};
  switch ((q + 2 + 7) / 8) {
    case 1: mds_tc_kernel<1><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mK16, args); break;
    case 2: mds_tc_kernel<2><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mK16, args); break;
    case 3: mds_tc_kernel<3><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mK16, args); break;
    default: mds_tc_kernel<4><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mK16, args); break;
  }
  if (tracing && trace) {  // debug: CTA 0 event intervals (ns), averaged over chunks 100..1100
    std::vector<unsigned long long> h(5 * TR_CHUNKS);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    const char* names[5] = {"MMA1 issued", "MMA2 issued", "Y landed", "D1 ready", "A2 written"};
    double per[5] = {0};
    for (int e = 0; e < 5; ++e) per[e] = double(h[e * TR_CHUNKS + 1100] - h[e * TR_CHUNKS + 100]) / 1000.0;
    fprintf(stderr, "[mds_tc trace] ns per chunk:");
    for (int e = 0; e < 5; ++e) fprintf(stderr, " %s %.0f;", names[e], per[e]);
    fprintf(stderr, "\n[mds_tc trace] chunk 500 offsets vs D1 ready (ns):");
    for (int e = 0; e < 5; ++e) fprintf(stderr, " %s %+lld;", names[e], (long long)(h[e * TR_CHUNKS + 500] - h[3 * TR_CHUNKS + 500]));
    fprintf(stderr, "\n");
  }
  *zp_out = zp;
  *tp_out = tp;
  *segs_out = g.segs;
  return BS_OK;
}

}  // namespace bs
