// tcgen05 MDS pass for float32 (solvers.py:269-305, mode 0 of bs_mds_pass).
//
// Per pair (i, j) of the rank's column block of Y the MM step needs
//   g_ij = theta_i . theta_j,  d_ij = sqrt(|theta_i|^2 + |theta_j|^2 - 2 g_ij)   (solvers.py:237-247)
//   stress += (y_ij - d_ij)^2,  zsum_j += y_ij / d_ij,  T_j += theta_i (1 - y_ij / d_ij)
// (solvers.py:289-300).  Both q-long dot products are GEMM-shaped: for a tile of
// 128 columns j x 64 rows i,
//   MMA1  D1[j][i] = sum_k ThJ[j][k] ThI[i][k]       M = 128, N = 64, K = 32 (q padded)
//   MMA2  D2[j][k] += sum_i WZ[j][i] ThI[i][k]       M = 128, N = 32, K = 64
// and run on the tensor cores in 3xTF32 (hi*hi + hi*lo + lo*hi, fp32-level error);
// the CUDA cores only do the per-pair elementwise chain between them.  Y is read
// once, by TMA, exactly as in the CUDA-core pass (mds.cu).
//
// CTA (one per SM, persistent over (128-column block, row segment) units), 320 threads:
//   warp 0     TMA producer: per 64-row chunk, Y tile (2 boxes of 32 i x 128 j, SWIZZLE_128B),
//              theta_i hi/lo K-major (B of MMA1), theta_i hi/lo MN-major (B of MMA2), norms
//   warp 1     MMA issuer (one elected lane): MMA1(c+1) is issued before MMA2(c)
//   warps 2-9  epilogue, two warps per TMEM lane quarter (lane = column j), each owning
//              32 of the chunk's 64 rows: tcgen05.ld g, elementwise chain, tcgen05.st
//              the hi/lo split of (1 - z) as MMA2's A operand (TMEM, K-major)
// TMEM (512 columns): D1 x2 [0,128), D2 [128,192), A1 = theta_J hi|lo [192,256),
//                     A2 x2 = WZ hi|lo [256,512).
// D2 is restarted every G chunks and folded into fp32 registers (the tensor core's
// accumulator add truncates, see nmf_tc.cu).
//
// Cancellation guard: where |theta_i|^2 + |theta_j|^2 - 2g loses more than 12 bits
// (near-coincident points) the pair is recomputed from the coordinates,
// sum_k (theta_ik - theta_jk)^2, so exactly coincident points give d = 0 exactly as
// the reference's Gram identity does on its own input (solvers.py:246, 290-296).
#include "tc_common.cuh"

#include <algorithm>
#include <mutex>

using namespace bs;
using namespace tc;

namespace {

constexpr int MT_THREADS = 320;
constexpr int CHI = 64;   // rows i per chunk
constexpr int BJ = 128;   // columns j per unit (MMA M)
constexpr int KP = 32;    // q padded (one 128-byte row of fp32)
constexpr int Y_BOX = 32 * 4 * BJ;              // 16 KB: 32 i x 128 j
constexpr int OFF_Y = 0;                        // 2 boxes
constexpr int OFF_B1H = 2 * Y_BOX;              // 64 i x 32 k, K-major SW128: 8 KB
constexpr int OFF_B1L = OFF_B1H + 8192;
constexpr int OFF_B2H = OFF_B1L + 8192;         // 2 boxes of 32 i x 32 k, MN-major SW128_32B: 8 KB
constexpr int OFF_B2L = OFF_B2H + 8192;
constexpr int OFF_NRM = OFF_B2L + 8192;         // 64 norms
constexpr int STAGE = OFF_NRM + 1024;
constexpr int NST = 3;
constexpr uint32_t TX_BYTES = 2 * Y_BOX + 4 * 8192 + CHI * 4;
constexpr int SMEM = NST * STAGE + 1024 /*align*/ + 256 /*barriers*/ + 2 * 2 * BJ * 8 /*zsum halves*/ + 512;
constexpr uint32_t T_D1 = 0, T_D2 = 128, T_A1 = 192, T_A2 = 256;
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

__device__ __forceinline__ float rsqrt_nr(float d2) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d2));
  return r * fmaf(-0.5f * d2 * r, r, 1.5f);
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

struct MdsTcArgs {
  const float* theta;   // q x n (theta_full, column-major)
  const float* th_hi;   // n x 32 tf32 hi (rows padded with zeros)
  const float* th_lo;   // n x 32 lo
  const float* norms;   // n
  int64_t n, lo, n_loc;
  int q, perturb, G;
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
              const __grid_constant__ CUtensorMap tmMl, const __grid_constant__ CUtensorMap tmN, const MdsTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  // st_full[NST], st_empty[NST], d1_full[2], d1_empty[2], a2_full[2], a2_empty[2], d2_full, d2_empty,
  // a1_full, a1_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 12);
  double* zsh = reinterpret_cast<double*>(smem + NST * STAGE + 256);       // [2][BJ]
  double* red_sh = zsh + 2 * BJ;                                             // [8][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto st_full = [&](int s) { return smem_u32(bars + s); };
  auto st_empty = [&](int s) { return smem_u32(bars + NST + s); };
  auto d1_full = [&](int b) { return smem_u32(bars + 2 * NST + b); };
  auto d1_empty = [&](int b) { return smem_u32(bars + 2 * NST + 2 + b); };
  auto a2_full = [&](int b) { return smem_u32(bars + 2 * NST + 4 + b); };
  auto a2_empty = [&](int b) { return smem_u32(bars + 2 * NST + 6 + b); };
  const uint32_t d2_full = smem_u32(bars + 2 * NST + 8), d2_empty = smem_u32(bars + 2 * NST + 9);
  const uint32_t a1_full = smem_u32(bars + 2 * NST + 10), a1_empty = smem_u32(bars + 2 * NST + 11);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(st_full(s), 1);
      mbar_init(st_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(d1_full(b), 1);
      mbar_init(d1_empty(b), 256);
      mbar_init(a2_full(b), 256);
      mbar_init(a2_empty(b), 1);
    }
    mbar_init(d2_full, 1);
    mbar_init(d2_empty, 256);
    mbar_init(a1_full, 256);
    mbar_init(a1_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmY);
    prefetch_tmap(&tmKh);
    prefetch_tmap(&tmKl);
    prefetch_tmap(&tmMh);
    prefetch_tmap(&tmMl);
    prefetch_tmap(&tmN);
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
          const int s = int(cc % NST);
          mbar_wait(st_empty(s), ((cc / NST) & 1) ^ 1);
          const uint32_t fb = st_full(s);
          mbar_expect_tx(fb, TX_BYTES);
          const uint32_t base = smem_u32(smem + s * STAGE);
          const int ic = int(i0 + int64_t(t) * CHI);
          tma_load_2d(base + OFF_Y, &tmY, ic, int(j0), fb);
          tma_load_2d(base + OFF_Y + Y_BOX, &tmY, ic + 32, int(j0), fb);
          tma_load_2d(base + OFF_B1H, &tmKh, 0, ic, fb);
          tma_load_2d(base + OFF_B1L, &tmKl, 0, ic, fb);
          tma_load_2d(base + OFF_B2H, &tmMh, 0, ic, fb);
          tma_load_2d(base + OFF_B2H + 4096, &tmMh, 0, ic + 32, fb);
          tma_load_2d(base + OFF_B2L, &tmMl, 0, ic, fb);
          tma_load_2d(base + OFF_B2L + 4096, &tmMl, 0, ic + 32, fb);
          tma_load_1d(base + OFF_NRM, &tmN, ic, fb);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t id1 = idesc_tf32(128, CHI, false, false);
    constexpr uint32_t id2w = idesc_tf32(128, 2 * KP, false, true);
    constexpr uint32_t id2n = idesc_tf32(128, KP, false, true);
    uint32_t cc = 0, gi = 0, ut = 0;
    auto issue_mma2 = [&](uint32_t c, int t, int nch) {
      const uint32_t b = c & 1;
      mbar_wait(a2_full(b), (c >> 1) & 1);
      const bool first = (t % a.G) == 0;
      const bool last = ((t % a.G) == a.G - 1) || (t == nch - 1);
      if (first) mbar_wait(d2_empty, (gi & 1) ^ 1);
      tc_fence_after();
      const int s = int(c % NST);
      const uint32_t d = __shfl_sync(0xffffffffu, tmem + T_D2, 0);
      const uint32_t ah = __shfl_sync(0xffffffffu, tmem + T_A2 + b * 128, 0);
      const uint32_t b2 = __shfl_sync(0xffffffffu, smem_u32(smem + s * STAGE + OFF_B2H), 0);
      const uint64_t bd = sdesc(b2, 8192, 512, LAYOUT_SW128_32B);
      mma_kblock_concat(d, ah, ah + 64, bd, id2w, id2n, first ? 0u : 1u);
      mma_kblock_concat(d, ah + 32, ah + 96, bd + 256, id2w, id2n, 1u);
      mma_commit_elect(a2_empty(b));
      mma_commit_elect(st_empty(s));
      if (last) {
        mma_commit_elect(d2_full);
        ++gi;
      }
      __syncwarp();
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ut) {
      int64_t j0, i0;
      int nch, seg;
      unit_range(u, j0, i0, nch, seg);
      mbar_wait(a1_full, ut & 1);
      tc_fence_after();
      for (int t = 0; t < nch; ++t, ++cc) {
        const int s = int(cc % NST);
        const uint32_t b = cc & 1;
        mbar_wait(st_full(s), (cc / NST) & 1);
        mbar_wait(d1_empty(b), ((cc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = __shfl_sync(0xffffffffu, tmem + T_D1 + b * CHI, 0);
        const uint32_t ah = __shfl_sync(0xffffffffu, tmem + T_A1, 0);
        const uint32_t bh = __shfl_sync(0xffffffffu, smem_u32(smem + s * STAGE + OFF_B1H), 0);
        const uint64_t dh = sdesc(bh, 16, 1024, LAYOUT_SW128), dl = sdesc(bh + 8192, 16, 1024, LAYOUT_SW128);
#pragma unroll
        for (int k = 0; k < KS; ++k) mma3_kstep(d, ah + 8 * k, ah + 32 + 8 * k, dh + 2 * k, dl + 2 * k, id1, k > 0);
        mma_commit_elect(d1_full(b));
        if (t == nch - 1) mma_commit_elect(a1_empty);
        __syncwarp();
        if (t > 0) issue_mma2(cc - 1, t - 1, nch);
      }
      issue_mma2(cc - 1, nch - 1, nch);
    }
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    const int qd = warp & 3, h = (warp - 2) >> 2;
    const int jrow = qd * 32 + lane;
    const uint32_t lane_addr = uint32_t(qd * 32) << 16;
    const int q = a.q;
    uint32_t cc = 0, gi = 0, ut = 0;
    double stress = 0.0, zeros = 0.0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ut) {
      int64_t j0, i0;
      int nch, seg;
      unit_range(u, j0, i0, nch, seg);
      const int64_t jl = j0 + jrow;
      const bool live = jl < a.n_loc;
      const int64_t jg = a.lo + (live ? jl : 0);
      const int64_t i_end = min(a.n, i0 + a.rows_per_seg);
      // A1: this column's theta_j (hi for h = 0, lo for h = 1) into TMEM, K-major
      mbar_wait(a1_empty, (ut & 1) ^ 1);
      tc_fence_after();
      {
        uint32_t v[32];
        const float4* src = reinterpret_cast<const float4*>((h ? a.th_lo : a.th_hi) + jg * KP);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 w = live ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * c] = __float_as_uint(w.x); v[4 * c + 1] = __float_as_uint(w.y);
          v[4 * c + 2] = __float_as_uint(w.z); v[4 * c + 3] = __float_as_uint(w.w);
        }
        tmem_st32(tmem + lane_addr + T_A1 + 32 * h, v);
        tmem_wait_st();
      }
      tc_fence_before();
      mbar_arrive(a1_full);
      const float nj = live ? __ldg(a.norms + jg) : 0.f;
      float Tacc[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) Tacc[k] = 0.f;
      double zsum = 0.0;
      bool fold_pending = false;
      auto fold = [&]() {
        mbar_wait(d2_full, gi & 1);
        tc_fence_after();
        float v[16], w[16];
        tmem_ld16(tmem + lane_addr + T_D2 + 16 * h, v);
        tmem_ld16(tmem + lane_addr + T_D2 + KP + 16 * h, w);
#pragma unroll
        for (int k = 0; k < 16; ++k) Tacc[k] = __fadd_rn(Tacc[k], __fadd_rn(v[k], w[k]));
        tc_fence_before();
        mbar_arrive(d2_empty);
        ++gi;
        fold_pending = false;
      };
      for (int t = 0; t < nch; ++t, ++cc) {
        const int s = int(cc % NST);
        const uint32_t b = cc & 1;
        const int64_t ib = i0 + int64_t(t) * CHI + 32 * h;  // first row of this thread's 32
        mbar_wait(st_full(s), (cc / NST) & 1);
        mbar_wait(d1_full(b), (cc >> 1) & 1);
        tc_fence_after();
        uint32_t g[32];
        tmem_ld32_nowait(tmem + lane_addr + T_D1 + b * CHI + 32 * h, g);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(d1_empty(b));
        const uint32_t ybase = smem_u32(smem + s * STAGE + OFF_Y + h * Y_BOX) + uint32_t(jrow) * 128u;
        const uint32_t nbase = smem_u32(smem + s * STAGE + OFF_NRM) + uint32_t(h) * 128u;
        uint32_t wz[32];
        float st_blk = 0.f, zs_blk = 0.f;
        const float sn = nj;
        bool bad = !live || (ib + 32 > i_end) || (jg >= ib && jg < ib + 32);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 yv = ld_shared_v4(ybase + (uint32_t(c ^ (jrow & 7)) << 4));
          const uint4 nv = ld_shared_v4(nbase + 16u * c);
          const uint32_t ya[4] = {yv.x, yv.y, yv.z, yv.w};
          const uint32_t na[4] = {nv.x, nv.y, nv.z, nv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t4 = 4 * c + e;
            const float y = __uint_as_float(ya[e]);
            const float sum = __uint_as_float(na[e]) + sn;
            const float d2 = fmaf(-2.f, __uint_as_float(g[t4]), sum);
            bad |= !(fmaf(-CANCEL, sum, d2) > 0.f);
            const float rs = rsqrt_nr(d2);
            const float d = d2 * rs;
            const float z = y * rs;
            const float er = y - d;
            st_blk = fmaf(er, er, st_blk);
            zs_blk += z;
            wz[t4] = __float_as_uint(1.f - z);
          }
        }
        if (bad) {
          // careful path: tails, the diagonal, padding columns and cancellation
          st_blk = 0.f;
          zs_blk = 0.f;
#pragma unroll
          for (int t4 = 0; t4 < 32; ++t4) {
            const int64_t i = ib + t4;
            const uint32_t c = uint32_t(t4 >> 2), e = uint32_t(t4 & 3);
            const float y = __uint_as_float(ld_shared_u32(ybase + ((c ^ uint32_t(jrow & 7)) << 4) + 4u * e));
            const float ni = __uint_as_float(ld_shared_u32(nbase + 4u * uint32_t(t4)));
            float w = 0.f;
            if (live && i < i_end) {
              if (i == jg) {  // d_jj = 0 exactly, (W - Z)_jj = 0 (solvers.py:240-241, 299-300)
                st_blk = fmaf(y, y, st_blk);
              } else {
                const float sum = ni + sn;
                float d2 = fmaf(-2.f, __uint_as_float(g[t4]), sum);
                if (!(fmaf(-CANCEL, sum, d2) > 0.f)) d2 = direct_d2(a.theta + i * q, a.theta + jg * q, q);
                float d, z;
                if (d2 > 0.f) {
                  const float rs = rsqrt_nr(d2);
                  d = d2 * rs;
                  z = y * rs;  // solvers.py:297
                } else {
                  d = 0.f;
                  zeros += 1.0;
                  z = a.perturb ? y * 1e10f : __fdiv_rn(y, 0.f);  // solvers.py:296
                }
                const float er = y - d;
                st_blk = fmaf(er, er, st_blk);
                zs_blk += z;
                w = 1.f - z;  // solvers.py:299
              }
            }
            wz[t4] = __float_as_uint(w);
          }
        }
        stress += double(st_blk);
        zsum += double(zs_blk);
        // A2 <- hi | lo of (W - Z) for this chunk
        mbar_wait(a2_empty(b), ((cc >> 1) & 1) ^ 1);
        tc_fence_after();
        {
          uint32_t lo[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t hi = tf32_hi(wz[k]);
            lo[k] = __float_as_uint(__uint_as_float(wz[k]) - __uint_as_float(hi));
            wz[k] = hi;
          }
          const uint32_t a2 = tmem + lane_addr + T_A2 + b * 128 + 32 * h;
          tmem_st32(a2, wz);
          tmem_st32(a2 + 64, lo);
          tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(a2_full(b));
        if (fold_pending) fold();
        if ((t % a.G) == a.G - 1 || t == nch - 1) fold_pending = true;
      }
      if (fold_pending) fold();
      // ---- unit outputs: zsum (two halves combined in order), T (each half owns 16 k) ----
      double* zs_sh = zsh;  // reuse is ordered by the two named barriers
      zs_sh[h * BJ + jrow] = zsum;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (live) {
        if (h == 0) a.zsum_part[int64_t(seg) * a.n_loc + jl] = zs_sh[jrow] + zs_sh[BJ + jrow];
        double* tp = a.T_part + (int64_t(seg) * a.n_loc + jl) * q;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (16 * h + k < q) tp[16 * h + k] = double(Tacc[k]);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    // ---- CTA stress / zero-count partial: warps in order ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      stress += __shfl_xor_sync(0xffffffffu, stress, o);
      zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
    }
    if (lane == 0) {
      red_sh[2 * (warp - 2)] = stress;
      red_sh[2 * (warp - 2) + 1] = zeros;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (warp == 2 && lane == 0) {
      double s0 = 0.0, z0 = 0.0;
      for (int w = 0; w < 8; ++w) {
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

// theta (q x n) -> tf32 hi / lo rows padded to 32, and |theta_i|^2.
__global__ void mds_tc_prep_kernel(const float* __restrict__ theta, int64_t n, int q, float* __restrict__ hi,
                                   float* __restrict__ lo, float* __restrict__ norms) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * KP; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / KP;
    const int k = int(e - i * KP);
    const float x = k < q ? theta[i * q + k] : 0.f;
    const uint32_t h = tf32_hi(__float_as_uint(x));
    hi[e] = __uint_as_float(h);
    lo[e] = x - __uint_as_float(h);
    if (k == 0) {
      float s = 0.f;
      for (int kk = 0; kk < q; ++kk) s = fmaf(theta[i * q + kk], theta[i * q + kk], s);
      norms[i] = s;
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
  int best = 1;
  double best_score = -1.0;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && chunks / s < 16) break;
    const double units = double(g.jblocks) * s;
    const double waves = units / sms;
    const double score = waves / std::ceil(waves) - 0.002 * s;
    if (score > best_score + 1e-9) { best_score = score; best = s; }
  }
  g.rows_per_seg = ceil_div(ceil_div(n, best), CHI) * CHI;
  g.segs = int(ceil_div(n, g.rows_per_seg));
  g.grid = int(std::min<int64_t>(int64_t(g.jblocks) * g.segs, sms));
  return g;
}

}  // namespace

namespace bs {

bool mds_tc_eligible(int dtype, int64_t n, int64_t n_loc, int q, int mode, const void* Y, const void* theta) {
  return dtype == BS_F32 && mode == 0 && q >= 1 && q <= KP && n % 4 == 0 && n >= CHI && n_loc >= 1 &&
         n <= INT32_MAX && n_loc <= INT32_MAX && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(theta) & 15) == 0 && tc::tc_enabled();
}

int64_t mds_tc_workspace(int64_t n, int64_t n_loc, int q) {
  TcGrid g = tc_grid(n, n_loc);
  return ws_bytes<unsigned int>(1) + ws_bytes<double>(2 * int64_t(g.grid)) + ws_bytes<double>(int64_t(g.segs) * n_loc) +
         ws_bytes<double>(int64_t(g.segs) * n_loc * q) + ws_bytes<float>(n) + 2 * ws_bytes<float>(n * KP);
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
  float* hi = ws.take<float>(n * KP);
  float* lo_ = ws.take<float>(n * KP);
  if (!ctr || !parts || !zp || !tp || !norms || !hi || !lo_) {
    set_error("bs_mds_pass: workspace too small");
    return BS_EWORK;
  }
  CUtensorMap mY, mKh, mKl, mMh, mMl, mN;
  bool ok = make_map_f32(&mY, Y, uint64_t(n), uint64_t(n_loc), 32, BJ, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mKh, hi, KP, uint64_t(n), KP, CHI, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mKl, lo_, KP, uint64_t(n), KP, CHI, CU_TENSOR_MAP_SWIZZLE_128B) &&
            make_map_f32(&mMh, hi, KP, uint64_t(n), KP, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
            make_map_f32(&mMl, lo_, KP, uint64_t(n), KP, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
            make_map_f32(&mN, norms, uint64_t(n), 0, CHI, 0, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) {
    set_error("bs_mds_pass: cuTensorMapEncodeTiled failed");
    return BS_ECUDA;
  }
  static int group = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("BS_MDS_TC_GROUP");
    group = (e && atoi(e) > 0) ? atoi(e) : 2;
    cudaFuncSetAttribute(mds_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(mds_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(mds_tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(mds_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  });
  mds_tc_prep_kernel<<<int(std::min<int64_t>(ceil_div(n * KP, 256), 4096)), 256, 0, st>>>(theta, n, q, hi, lo_, norms);
  MdsTcArgs args{theta, hi, lo_, norms, n, lo, n_loc, q, perturb, group, g.jblocks, g.segs, g.rows_per_seg,
                 zp, tp, parts, ctr, red};
  switch ((q + 7) / 8) {
    case 1: mds_tc_kernel<1><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mN, args); break;
    case 2: mds_tc_kernel<2><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mN, args); break;
    case 3: mds_tc_kernel<3><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mN, args); break;
    default: mds_tc_kernel<4><<<g.grid, MT_THREADS, SMEM, st>>>(mY, mKh, mKl, mMh, mMl, mN, args); break;
  }
  *zp_out = zp;
  *tp_out = tp;
  *segs_out = g.segs;
  return BS_OK;
}

}  // namespace bs
