// One-stream Cox pass for float32 X with float32 arithmetic (the C4 setting):
// bs_cox_grad_xbeta's fused path computes grad = X^T (delta - pd), the proximal step
// beta_new = S_lambda(beta + sigma grad) (solvers.py:447-449) and X beta_new (the next
// iteration's scn m, distlinalg.py:334-337) with ONE read of X from HBM instead of two.
//
// Grid: Gc column groups x S row segments (cooperative launch, one CTA per SM).  CTA
// (g, s) owns rows [s R, (s+1) R) and the columns of group g, processed in waves of W
// columns:
//   A(w)  a producer warp streams the wave's columns (this CTA's rows) from HBM into an
//         smem ring (cp.async.bulk, L2 evict_last); the consumers form the CTA's gradient
//         partial of each column (v = delta - pd in registers), write it to the group's
//         partial slot and bump the group's wave counter;
//   B(u)  (u = w - LAG) a second producer warp waits for wave u's counter to reach S, pulls
//         the S x W partial block, then re-streams wave u's columns from L2 (evict_first);
//         the consumers fold the S partials in segment order (deterministic, identical in
//         every CTA of the group), apply S_lambda and accumulate X[:, u] beta_new into the
//         rows' xb (float per 4-column stage, float64 across).
// Synchronisation is per group (S CTAs), not grid-wide, and the partial exchange is
// S * 8 bytes per column against R * 4 bytes of X.  The per-group xb partials are folded
// in group order by cox_fused2_finish.
#include "bsb200.cuh"
#include "tc_common.cuh"

#include <algorithm>

using namespace bs;
using namespace tc;

namespace {

constexpr int F2_THREADS = 320;  // warp 0: A producer, warp 1: B producer, warps 2..9 consumers
constexpr int F2_WMAX = 32;      // largest wave (columns); the wave is a template parameter
constexpr int F2_RING = 12;      // partial slots / counters per group (> 2 LAG)
constexpr int64_t F2_STAGE_MAX = 48 * 1024;  // bytes of one stage (F2_CW columns x R rows)

typedef unsigned long long f2r;
__device__ __forceinline__ f2r p2(float a, float b) {
  f2r r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void u2(f2r v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2r fma2(f2r a, f2r b, f2r c) {
  f2r d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ unsigned int ld_acq(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

struct F2Args {
  const float* X;
  int64_t m, n_loc, R, cpg;
  int S, Gc, pf;  // pf: stages of X prefetched into L2 ahead of the A ring (0 = off)
  const double* v;
  float* grad;
  float* beta;
  double sigma, lam;
  double* xb_parts;   // [Gc][m]
  double* l1_parts;   // [Gc]
  double* partials;   // [Gc][RING][S][W]
  unsigned int* counters;  // [Gc][RING]
  const int* flags;
};

// F2_AS A stages (HBM), F2_BS B stages (L2), F2_LAG waves between A(w) and B(w)
// F2_CW columns per ring stage, F2_KB float4 row groups per consumer thread (R <= 1024 KB)
template <int F2_AS, int F2_BS, int F2_LAG, int F2_W, int F2_CW, int F2_KB>
__global__ void __launch_bounds__(F2_THREADS, 1) cox_fused2_kernel(const F2Args a) {
  static_assert(F2_RING > 2 * F2_LAG, "partial slots must outlive the lag");
  static_assert(F2_W == 16 || F2_W == 32, "waves of 16 or 32 columns");
  constexpr int F2_QPW = F2_W / F2_CW;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (a.flags && (*a.flags & BS_FLAG_NONFINITE)) return;  // every CTA sees the same flag
  const int S = a.S, g = int(blockIdx.x) / S, sg = int(blockIdx.x) % S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t R = a.R, m = a.m;
  const int64_t r0 = int64_t(sg) * R;
  const int rows = int(r0 >= m ? 0 : (m - r0 < R ? m - r0 : R));
  const int64_t c0 = int64_t(g) * a.cpg;
  const int64_t c1 = min(a.n_loc, c0 + a.cpg);
  const int64_t ncols = c1 > c0 ? c1 - c0 : 0;
  const int nw = int((ncols + F2_W - 1) / F2_W);
  const int64_t stage_f = int64_t(F2_CW) * R;  // floats per stage
  float* aring = reinterpret_cast<float*>(smem);
  float* bring = aring + F2_AS * stage_f;
  double* pbuf = reinterpret_cast<double*>(bring + F2_BS * stage_f);  // [2][S][W]
  double* bold = pbuf + 2 * S * F2_W;                                  // [LAG+1][W]
  float* bnew = reinterpret_cast<float*>(bold + (F2_LAG + 1) * F2_W);  // [2][W]
  float* red = bnew + 2 * F2_W;                                        // [2][8][W]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * 8 * F2_W);
  // barriers: afull[AS], aempty[AS], bfull[BS], bempty[BS], pfull[2], pempty[2], bnfull[2], bnempty[2]
  auto bar = [&](int i) { return smem_u32(bars + i); };
  constexpr int AF = 0, AE = F2_AS, BF = 2 * F2_AS, BE = 2 * F2_AS + F2_BS, PF = 2 * F2_AS + 2 * F2_BS, PE = PF + 2;
  constexpr int NF = PE + 2, NE = NF + 2;
  if (tid == 0) {
    for (int i = 0; i < F2_AS; ++i) {
      mbar_init(bar(AF + i), 1);
      mbar_init(bar(AE + i), 8);
    }
    for (int i = 0; i < F2_BS; ++i) {
      mbar_init(bar(BF + i), 1);
      mbar_init(bar(BE + i), 8);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(PF + i), 1);
      mbar_init(bar(PE + i), 1);
      mbar_init(bar(NF + i), 1);
      mbar_init(bar(NE + i), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // absent columns / rows read stale ring data times 0: start from zeros, not garbage
  for (int64_t i = tid; i < (F2_AS + F2_BS) * stage_f; i += F2_THREADS) aring[i] = 0.f;
  fence_proxy_async_smem();
  __syncthreads();
  const uint32_t bytes_col = uint32_t(rows) * 4u;

  if (warp == 0) {  // ---------------- A producer: HBM -> ring, kept in L2 ----------------
    if (lane == 0 && rows > 0) {
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      const int nst = nw * F2_QPW;
      for (int k = 0; k < min(a.pf, nst); ++k)  // L2 prefetch of the first pf stages
        for (int jj = 0; jj < F2_CW; ++jj) {
          const int64_t j = c0 + int64_t(k) * F2_CW + jj;
          if (j < c1)
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a.X + j * m + r0),
                         "r"(bytes_col), "l"(keep) : "memory");
        }
      for (int w = 0; w < nw; ++w)
        for (int q = 0; q < F2_QPW; ++q) {
          const int k = w * F2_QPW + q, s = k % F2_AS;
          if (a.pf > 0 && k + a.pf < nst)
            for (int jj = 0; jj < F2_CW; ++jj) {
              const int64_t j = c0 + int64_t(k + a.pf) * F2_CW + jj;
              if (j < c1)
                asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a.X + j * m + r0),
                             "r"(bytes_col), "l"(keep) : "memory");
            }
          mbar_wait_sleep(bar(AE + s), uint32_t((k / F2_AS) & 1) ^ 1u);
          const int64_t j0 = c0 + int64_t(w) * F2_W + q * F2_CW;
          const int nc = int(c1 - j0 <= 0 ? 0 : (c1 - j0 < F2_CW ? c1 - j0 : F2_CW));
          mbar_expect_tx(bar(AF + s), bytes_col * uint32_t(nc));
          for (int jj = 0; jj < nc; ++jj)
            bulk(smem_u32(aring + s * stage_f + jj * R), a.X + (j0 + jj) * m + r0, bytes_col, bar(AF + s), keep);
        }
    }
    return;
  }
  if (warp == 1) {  // ---------------- B producer: partial block, L2 -> ring, and the fold ----------------
    // The warp also folds each wave's group partials into beta_new as soon as they land (lanes
    // 0..W-1, segment order: identical in every CTA of the group), so the consumers find
    // beta_new ready when they reach B(u) instead of waiting for one of them to fold.
    uint64_t drop = 0;
    if (lane == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(drop));
    // B stages do not depend on the partials: the first F2_BS stages of wave u are issued
    // before waiting for the group's counter, so they land while the fold is pending
    auto bstage = [&](int u, int q) {
      const int k = u * F2_QPW + q, s = k % F2_BS;
      mbar_wait_sleep(bar(BE + s), uint32_t((k / F2_BS) & 1) ^ 1u);
      const int64_t j0 = c0 + int64_t(u) * F2_W + q * F2_CW;
      const int nc = int(c1 - j0 <= 0 ? 0 : (c1 - j0 < F2_CW ? c1 - j0 : F2_CW));
      mbar_expect_tx(bar(BF + s), bytes_col * uint32_t(nc));
      for (int jj = 0; jj < nc; ++jj)
        bulk(smem_u32(bring + s * stage_f + jj * R), a.X + (j0 + jj) * m + r0, bytes_col, bar(BF + s), drop);
    };
    constexpr int EARLY = F2_BS < F2_QPW ? F2_BS : F2_QPW;
    double l1 = 0.0;
    for (int u = 0; u < nw; ++u) {
      const int pb = u & 1;
      if (lane == 0) {
        if (rows > 0)
          for (int q = 0; q < EARLY; ++q) bstage(u, q);
        const int slot = u % F2_RING;
        const unsigned int* ctr = a.counters + g * F2_RING + slot;
        const unsigned int target = unsigned(S) * unsigned(u / F2_RING + 1);
        uint64_t t0 = 0;
        for (uint32_t spin = 0; ld_acq(ctr) < target; ++spin) {
          __nanosleep(64);
          if ((spin & 4095) == 4095) {
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (t0 == 0) t0 = now;
            else if (now - t0 > 10000000000ULL) __trap();
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_wait_sleep(bar(PE + pb), uint32_t((u >> 1) & 1) ^ 1u);
        const uint32_t pbytes = uint32_t(S) * F2_W * 8u;
        mbar_expect_tx(bar(PF + pb), pbytes);
        bulk(smem_u32(pbuf + pb * S * F2_W), a.partials + (int64_t(g) * F2_RING + slot) * S * F2_W, pbytes, bar(PF + pb),
             drop);
      }
      __syncwarp();
      // ---- fold wave u: S_lambda(beta + sigma grad) (solvers.py:48-51, 447-449) ----
      mbar_wait(bar(PF + pb), uint32_t((u >> 1) & 1));
      mbar_wait(bar(NE + pb), uint32_t((u >> 1) & 1) ^ 1u);  // the consumers are done with bnew[pb] of wave u - 2
      const int64_t ju = c0 + int64_t(u) * F2_W;
      if (lane < F2_W) {
        const double* pp = pbuf + pb * S * F2_W;
        double gs = 0.0;
        for (int k = 0; k < S; ++k) gs += pp[k * F2_W + lane];  // segment order: same in every CTA
        const float gt = float(gs);
        const float x = float(bold[(u % (F2_LAG + 1)) * F2_W + lane]) + float(a.sigma) * gt;
        const float mag = fabsf(x) - float(a.lam);
        const bool live = ju + lane < c1;
        const float bn = live && mag > 0.f ? copysignf(mag, x) : 0.f;
        bnew[pb * F2_W + lane] = bn;
        if (sg == 0 && live) {
          a.grad[ju + lane] = gt;
          a.beta[ju + lane] = bn;
          l1 += fabs(double(bn));
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(PE + pb));
        mbar_arrive(bar(NF + pb));
        // the wave's later B stages reuse stages that only B(u) itself frees, so they go after
        // beta_new is published (issuing them first would wait on the consumers' B(u) forever)
        if (rows > 0)
          for (int q = EARLY; q < F2_QPW; ++q) bstage(u, q);
      }
      __syncwarp();
    }
    if (sg == 0) {  // ||beta_new||_1 of the group's columns, fixed order
      const double t = warp_sum(l1);
      if (lane == 0) a.l1_parts[g] = t;
    }
    return;
  }

  // ---------------- consumers: thread ct owns rows 4 ct + 1024 k + e ----------------
  const int ct = tid - 64, cw = warp - 2;
  float vr[4 * F2_KB];
  double xbr[4 * F2_KB];
#pragma unroll
  for (int k = 0; k < F2_KB; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * ct + 1024 * k + e;
      vr[4 * k + e] = i < rows ? float(a.v[r0 + i]) : 0.f;
      xbr[4 * k + e] = 0.0;
    }
  float bpre = (ct < F2_W && c0 + ct < c1) ? a.beta[c0 + ct] : 0.f;  // beta of the next wave, loaded a wave early
  for (int w = 0; w < nw + F2_LAG; ++w) {
    if (w < nw) {
      // ---- A(w): per-thread partial of each of the wave's 16 columns ----
      if (ct < F2_W) {
        bold[(w % (F2_LAG + 1)) * F2_W + ct] = double(bpre);
        const int64_t jn = c0 + int64_t(w + 1) * F2_W + ct;
        bpre = jn < c1 ? a.beta[jn] : 0.f;
      }
      float cs[F2_W];
#pragma unroll
      for (int q = 0; q < F2_QPW; ++q) {
        const int k = w * F2_QPW + q, s = k % F2_AS;
        if (rows > 0) mbar_wait(bar(AF + s), uint32_t((k / F2_AS) & 1));
        const float* tile = aring + s * stage_f;
#pragma unroll
        for (int jj = 0; jj < F2_CW; ++jj) {
          f2r acc = p2(0.f, 0.f);
#pragma unroll
          for (int kb = 0; kb < F2_KB; ++kb) {
            const int i = 4 * ct + 1024 * kb;
            if (i < R) {
              const float4 x = *reinterpret_cast<const float4*>(tile + jj * R + i);
              acc = fma2(p2(x.x, x.y), p2(vr[4 * kb], vr[4 * kb + 1]), acc);
              acc = fma2(p2(x.z, x.w), p2(vr[4 * kb + 2], vr[4 * kb + 3]), acc);
            }
          }
          float lo, hi;
          u2(acc, lo, hi);
          cs[q * F2_CW + jj] = lo + hi;
        }
        __syncwarp();
        if (lane == 0 && rows > 0) mbar_arrive(bar(AE + s));
      }
      // fold the wave's columns over the warp: lane l ends with column l % W
      if constexpr (F2_W == 16) {
#pragma unroll
        for (int j = 0; j < F2_W; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 16);
      }
#pragma unroll
      for (int o = F2_W / 2; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const float send = up ? cs[k] : cs[k + o];
          const float keep = up ? cs[k + o] : cs[k];
          cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      float* rw = red + (w & 1) * 8 * F2_W;
      if (lane < F2_W) rw[cw * F2_W + lane] = cs[0];
      cons_sync();
      if (ct < F2_W) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += double(rw[k * F2_W + ct]);
        a.partials[((int64_t(g) * F2_RING + (w % F2_RING)) * S + sg) * F2_W + ct] = t;
        __threadfence();
      }
      if (cw == 0) {
        __syncwarp();
        if (lane == 0) atomicAdd(a.counters + g * F2_RING + (w % F2_RING), 1u);
      }
    }
    const int u = w - F2_LAG;
    if (u >= 0) {
      // ---- B(u): fold the group's partials, S_lambda, then xb += X[:, wave u] beta_new ----
      const int pb = u & 1;
      mbar_wait(bar(NF + pb), uint32_t((u >> 1) & 1));  // beta_new of wave u, folded by warp 1
      float bq[F2_W];
#pragma unroll
      for (int j = 0; j < F2_W; ++j) bq[j] = bnew[pb * F2_W + j];
#pragma unroll
      for (int q = 0; q < F2_QPW; ++q) {
        const int k = u * F2_QPW + q, s = k % F2_BS;
        if (rows > 0) mbar_wait(bar(BF + s), uint32_t((k / F2_BS) & 1));
        const float* tile = bring + s * stage_f;
#pragma unroll
        for (int kb = 0; kb < F2_KB; ++kb) {
          const int i = 4 * ct + 1024 * kb;
          if (i < R) {
            f2r lo = p2(0.f, 0.f), hi = p2(0.f, 0.f);
#pragma unroll
            for (int jj = 0; jj < F2_CW; ++jj) {
              const float4 x = *reinterpret_cast<const float4*>(tile + jj * R + i);
              const f2r bb = p2(bq[q * F2_CW + jj], bq[q * F2_CW + jj]);
              lo = fma2(p2(x.x, x.y), bb, lo);
              hi = fma2(p2(x.z, x.w), bb, hi);
            }
            float l0, l1f, h0, h1;
            u2(lo, l0, l1f);
            u2(hi, h0, h1);
            xbr[4 * kb] += double(l0);
            xbr[4 * kb + 1] += double(l1f);
            xbr[4 * kb + 2] += double(h0);
            xbr[4 * kb + 3] += double(h1);
          }
        }
        __syncwarp();
        if (lane == 0 && rows > 0) mbar_arrive(bar(BE + s));
      }
      __syncwarp();  // bq is consumed: bnew[pb] may be rewritten (wave u + 2)
      if (lane == 0) mbar_arrive(bar(NE + pb));
    }
  }
#pragma unroll
  for (int k = 0; k < F2_KB; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * ct + 1024 * k + e;
      if (i < rows) a.xb_parts[int64_t(g) * m + r0 + i] = xbr[4 * k + e];
    }
}

// xb_out[i] = sum over groups of xb_parts[g][i] (group order); xb_out[m] = sum of l1_parts
__global__ void cox_fused2_finish(const double* __restrict__ xb_parts, const double* __restrict__ l1_parts, int Gc,
                                  int64_t m, double* __restrict__ xb_out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= m; i += int64_t(gridDim.x) * blockDim.x) {
    double t = 0.0;
    if (i < m)
      for (int k = 0; k < Gc; ++k) t += xb_parts[int64_t(k) * m + i];
    else
      for (int k = 0; k < Gc; ++k) t += l1_parts[k];
    xb_out[i] = t;
  }
}

}  // namespace

namespace bs {

constexpr int F2_REFUSED = -1000;  // internal: cooperative launch refused

struct F2Plan {
  bool ok;
  int S, Gc, cfg;
  int64_t R, cpg;
  size_t smem;
};

F2Plan f2_plan(int64_t m, int64_t n_loc) {
  F2Plan p{};
  p.ok = false;
  if (m < 4096 || n_loc < 4 * F2_WMAX || m % 4) return p;
  const char* e = getenv("BS_COX_FUSED2");
  if (e && e[0] == '0') return p;
  int dev = 0, coop = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (!coop) return p;
  const int G = num_sms();
  static const int cfg = [] {
    const char* c = getenv("BS_F2_CFG");
    return c ? atoi(c) : 0;
  }();
  static const int as_[17] = {2, 3, 2, 3, 2, 3, 3, 2, 4, 2, 2, 2, 4, 3, 4, 2, 3},
                   bs_[17] = {2, 1, 2, 1, 2, 2, 2, 3, 2, 2, 2, 3, 4, 3, 3, 2, 2},
                   lag_[17] = {1, 2, 3, 3, 4, 3, 2, 2, 2, 1, 2, 1, 2, 2, 2, 2, 1},
                   w_[17] = {16, 16, 16, 16, 16, 16, 16, 16, 16, 32, 32, 32, 16, 16, 16, 16, 16},
                   cw_[17] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 2, 2, 2, 4, 4},
                   kb_[17] = {3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 4, 4, 4, 3, 3};
  const int ci = cfg >= 0 && cfg < 17 ? cfg : 0;
  const int W = w_[ci], CW = cw_[ci];
  p.cfg = ci;
  const int nst = as_[ci] + bs_[ci];
  const int64_t rmax = std::min<int64_t>(1024 * kb_[ci], (4 * F2_STAGE_MAX / nst) / (4 * CW));
  int best_s = 0, best_u = 0;
  const int s_min = int(ceil_div(m, rmax));
  for (int S = s_min; S <= G; ++S) {  // a segment count that fills every SM, if one is near
    if (G % S == 0 && S * 4 <= s_min * 5) { best_s = S; best_u = G; break; }
  }
  for (int S = s_min; S <= G && best_u < G; ++S) {
    const int u = S * (G / S);
    if (u > best_u) { best_u = u; best_s = S; }
    if (u * 100 >= G * 96) { best_s = S; best_u = u; break; }
  }
  static const int force_s = [] {
    const char* c = getenv("BS_F2_S");  // experiments: fixed segment count
    return c ? atoi(c) : 0;
  }();
  if (force_s >= int(ceil_div(m, rmax)) && force_s <= G) best_s = force_s;
  if (best_s == 0) return p;
  p.S = best_s;
  p.Gc = G / best_s;
  p.R = ceil_div(ceil_div(m, p.S), int64_t(4)) * 4;
  if (p.R > rmax) return p;
  p.cpg = ceil_div(n_loc, int64_t(p.Gc));
  p.smem = size_t(nst * CW * p.R * 4 + 2 * int64_t(p.S) * W * 8 + (lag_[ci] + 1) * W * 8 + 2 * W * 4 +
                  2 * 8 * W * 4 + (2 * nst + 8) * 8 + 64);
  if (int64_t(p.smem) > int64_t(maxsm) - 1024) return p;
  p.ok = true;
  return p;
}

int64_t f2_workspace(const F2Plan& p, int64_t m) {
  return ws_bytes<unsigned int>(int64_t(p.Gc) * F2_RING) + ws_bytes<double>(int64_t(p.Gc) * F2_RING * p.S * F2_WMAX) +
         ws_bytes<double>(int64_t(p.Gc) * m) + ws_bytes<double>(p.Gc);
}

int f2_launch(const F2Plan& p, const float* X, int64_t m, int64_t n_loc, const double* v, float* grad, float* beta,
              double sigma, double lam, double* xb_out, const int* flags, Workspace& ws, cudaStream_t st) {
  unsigned int* counters = ws.take<unsigned int>(int64_t(p.Gc) * F2_RING);
  double* partials = ws.take<double>(int64_t(p.Gc) * F2_RING * p.S * F2_WMAX);
  double* xb_parts = ws.take<double>(int64_t(p.Gc) * m);
  double* l1_parts = ws.take<double>(p.Gc);
  if (!counters || !partials || !xb_parts || !l1_parts) {
    set_error("bs_cox_grad_xbeta: workspace too small");
    return BS_EWORK;
  }
  if (cudaMemsetAsync(counters, 0, sizeof(unsigned int) * p.Gc * F2_RING, st) != cudaSuccess) {
    set_error("bs_cox_grad_xbeta: cudaMemsetAsync failed");
    return BS_ECUDA;
  }
  static const int pf = [] {
    const char* c = getenv("BS_F2_PF");
    return c ? atoi(c) : 0;
  }();
  F2Args a{X, m, n_loc, p.R, p.cpg, p.S, p.Gc, pf, v, grad, beta, sigma, lam, xb_parts, l1_parts, partials, counters, flags};
  const void* k = nullptr;
#define F2K(A, B, L, W, CW, KB)                                                 \
  k = reinterpret_cast<const void*>(cox_fused2_kernel<A, B, L, W, CW, KB>);   \
  smem_attr(cox_fused2_kernel<A, B, L, W, CW, KB>, int(p.smem));
  switch (p.cfg) {
    case 1: F2K(3, 1, 2, 16, 4, 3) break;
    case 2: F2K(2, 2, 3, 16, 4, 3) break;
    case 3: F2K(3, 1, 3, 16, 4, 3) break;
    case 4: F2K(2, 2, 4, 16, 4, 3) break;
    case 5: F2K(3, 2, 3, 16, 4, 3) break;
    case 6: F2K(3, 2, 2, 16, 4, 3) break;
    case 7: F2K(2, 3, 2, 16, 4, 3) break;
    case 8: F2K(4, 2, 2, 16, 4, 3) break;
    case 9: F2K(2, 2, 1, 32, 4, 3) break;
    case 10: F2K(2, 2, 2, 32, 4, 3) break;
    case 11: F2K(2, 3, 1, 32, 4, 3) break;
    case 12: F2K(4, 4, 2, 16, 2, 4) break;
    case 13: F2K(3, 3, 2, 16, 2, 4) break;
    case 14: F2K(4, 3, 2, 16, 2, 4) break;
    case 15: F2K(2, 2, 2, 16, 4, 3) break;  // the default before the fold moved to warp 1
    case 16: F2K(3, 2, 1, 16, 4, 3) break;
    default: F2K(2, 2, 1, 16, 4, 3) break;  // lag 1: beta_new is folded off the consumers' path
  }
#undef F2K
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel(k, dim3(p.S * p.Gc), dim3(F2_THREADS), args, p.smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("bs_cox_grad_xbeta: cooperative launch failed: %s", cudaGetErrorString(e));
    return F2_REFUSED;  // the caller falls back to two passes
  }
  cox_fused2_finish<<<int(std::min<int64_t>(ceil_div(m + 1, 256), 1024)), 256, 0, st>>>(xb_parts, l1_parts, p.Gc, m,
                                                                                         xb_out);
  return check_launch("bs_cox_grad_xbeta", 2);
}

}  // namespace bs
