// tcgen05 3xTF32 skinny GEMMs for float32 NMF (scenarios b and a).
//
//   scn b  P[i][k] = sum_j X[j][i] W[j][k]    A = X MN-major (i contiguous), K = j   (distlinalg.py:246-252)
//   scn a  C[j][k] = sum_i X[j][i] Vt[i][k]   A = X K-major  (i contiguous), K = i   (distlinalg.py:239-243)
//
// M = 128 rows per tile on the tensor cores, N = r padded to a multiple of 32
// (the MN-major SW128 atom of B), K in blocks of 32.  Precision: float32 via
// 3xTF32 — every operand x is split into hi = tf32(x) (mantissa truncated, an
// exact tf32 value) and lo = x - hi (exact in fp32), and the accumulator in
// TMEM collects hi*hi + hi*lo + lo*hi (the dropped lo*lo term is ~2^-22 relative).
//
// Warp roles (192 threads, one CTA per SM, persistent over (tile, k-split) units):
//   warp 0      TMA producer: X tile (16 KB) + B tile (r x 32) per stage, SWIZZLE_128B
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (3 MMAs per 8-wide k step)
//   warps 2-5   converters: split each landed stage in place (hi) and into a
//               parallel buffer (lo) with the same swizzled layout, then
//               epilogue: tcgen05.ld the 128 x N accumulator and store the
//               unit's partial rows into its split-K slab.
// X is read exactly once per GEMM; the split-K slabs are folded (in order) by
// the fused factor-update kernel that consumes them.
#include "bsb200.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

using namespace bs;

namespace {

constexpr int TC_THREADS = 192;
constexpr int BM = 128;
constexpr int BK = 32;
constexpr int A_STAGE_BYTES = BM * BK * 4;  // 16 KB
constexpr int SMEM_BUDGET = 220 * 1024;

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// Waits for phase `parity` of the barrier; traps after ~10 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if ((spin & 1023) == 1023) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ULL) __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor (tcgen05): start, LBO, SBO in 16-byte units, version 1, layout type.
// Layout types: 2 = SWIZZLE_128B (K-major tiles, Swizzle<3,4,3>, 8-row atoms);
// 1 = SWIZZLE_128B_BASE32B, the only MN-major layout tf32 accepts (Swizzle<2,5,2>,
// 4-row x 128 B atoms) — the TMA produces it with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
constexpr uint32_t LAYOUT_SW128 = 2, LAYOUT_SW128_32B = 1;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version (Blackwell)
  d |= uint64_t(layout) << 61;
  return d;
}

// MN-major operand slab (32 MN x 32 K of a stage): k step s covers rows 8s..8s+7 = two 512 B atoms.
__device__ __forceinline__ uint64_t mn_desc(uint32_t base, int s) {
  return sdesc(base + uint32_t(s) * 1024u, 4096, 512, LAYOUT_SW128_32B);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Splits 4 words in place: hi = tf32-truncated x (exact tf32), lo = x - hi (exact fp32).
__device__ __forceinline__ void split4(uint4* hi_p, uint4* lo_p) {
  uint4 v = *hi_p;
  uint4 h, l;
  h.x = v.x & 0xFFFFE000u;
  h.y = v.y & 0xFFFFE000u;
  h.z = v.z & 0xFFFFE000u;
  h.w = v.w & 0xFFFFE000u;
  l.x = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(h.x));
  l.y = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(h.y));
  l.z = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(h.z));
  l.w = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(h.w));
  *hi_p = h;
  *lo_p = l;
}

template <int NP>
struct TcCfg {
  static constexpr int B_BYTES = NP * BK * 4;                 // NP/32 MN-atoms of 32 rows x 128 B
  static constexpr int STAGE = 2 * A_STAGE_BYTES + 2 * B_BYTES;  // A hi, A lo, B hi, B lo
  static constexpr int STAGES = (SMEM_BUDGET - 2048) / STAGE > 6 ? 6 : (SMEM_BUDGET - 2048) / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 512 /*barriers*/;
  // two accumulator buffers of NP columns (power of two allocation)
  static constexpr int TMEM_COLS = 2 * NP <= 64 ? 64 : 2 * NP <= 128 ? 128 : 256;
};

// ---------------------------------------------------------------------------
// the kernel
//
// Accumulation precision: the tensor core adds each MMA into the fp32 TMEM
// accumulator with truncation, so a long K run drifts by ~6e-8 per MMA (measured:
// 7e-6 relative after K = 320).  The K range of a unit is therefore cut into
// groups of G k-blocks; each group accumulates into a fresh TMEM buffer (two
// buffers alternate) and the epilogue warps fold the group partial into fp32
// registers with round-to-nearest adds.  The error is then bounded by one group
// (12*G MMAs) instead of the whole K extent.
// ---------------------------------------------------------------------------

template <bool A_MN, int NP>
__global__ void __launch_bounds__(TC_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int K, int r,
               int tiles, int kb_per_split, int units, int G, float* __restrict__ out, int64_t slab) {
  using C = TcCfg<NP>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  // bars: full[STAGES], conv[STAGES], empty[STAGES], acc_full[2], acc_empty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_total = (K + BK - 1) / BK;

  auto stage_a = [&](int s) { return smem + s * C::STAGE; };
  auto stage_al = [&](int s) { return smem + s * C::STAGE + A_STAGE_BYTES; };
  auto stage_b = [&](int s) { return smem + s * C::STAGE + 2 * A_STAGE_BYTES; };
  auto stage_bl = [&](int s) { return smem + s * C::STAGE + 2 * A_STAGE_BYTES + C::B_BYTES; };
  auto full = [&](int s) { return smem_u32(bars + s); };
  auto conv = [&](int s) { return smem_u32(bars + STAGES + s); };
  auto empty = [&](int s) { return smem_u32(bars + 2 * STAGES + s); };
  auto acc_full = [&](int b) { return smem_u32(bars + 3 * STAGES + b); };
  auto acc_empty = [&](int b) { return smem_u32(bars + 3 * STAGES + 2 + b); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(conv(s), 128);
      mbar_init(empty(s), 1);
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
        const int split = u / tiles, tile = u % tiles;
        const int kb0 = split * kb_per_split;
        const int kb1 = min(kb_total, kb0 + kb_per_split);
        const int m0 = tile * BM;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          const uint32_t fb = full(stage);
          mbar_expect_tx(fb, A_STAGE_BYTES + C::B_BYTES);
          const int k0 = kb * BK;
          if constexpr (A_MN) {
#pragma unroll
            for (int a = 0; a < BM / 32; ++a) tma_load_2d(smem_u32(stage_a(stage) + a * 4096), &tmA, m0 + 32 * a, k0, fb);
          } else {
            tma_load_2d(smem_u32(stage_a(stage)), &tmA, k0, m0, fb);
          }
#pragma unroll
          for (int b = 0; b < NP / 32; ++b) tma_load_2d(smem_u32(stage_b(stage) + b * 4096), &tmB, 32 * b, k0, fb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // idesc: D f32, A/B tf32, A major (MN for scn b), B MN-major, N = NP, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) | (1u << 16) |
                           (uint32_t(NP >> 3) << 17) | (uint32_t(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t gi = 0;  // global group counter (shared sequence with the epilogue)
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles;
      const int kb0 = split * kb_per_split;
      const int kb1 = min(kb_total, kb0 + kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int in_group = (kb - kb0) % G;
        const uint32_t buf = gi & 1;
        if (in_group == 0) {
          mbar_wait(acc_empty(buf), ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(conv(stage), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t d = tmem + buf * NP;
          const uint32_t a = smem_u32(stage_a(stage)), al = smem_u32(stage_al(stage));
          const uint32_t b = smem_u32(stage_b(stage)), bl = smem_u32(stage_bl(stage));
#pragma unroll
          for (int s = 0; s < BK / 8; ++s) {
            uint64_t da, dal;
            if constexpr (A_MN) {
              da = mn_desc(a, s);
              dal = mn_desc(al, s);
            } else {
              da = sdesc(a + s * 32, 16, 1024, LAYOUT_SW128);
              dal = sdesc(al + s * 32, 16, 1024, LAYOUT_SW128);
            }
            const uint64_t db = mn_desc(b, s);
            const uint64_t dbl = mn_desc(bl, s);
            const uint32_t acc = (in_group > 0 || s > 0) ? 1u : 0u;
            mma_tf32(d, dal, db, idesc, acc);  // lo * hi (small terms first)
            mma_tf32(d, da, dbl, idesc, 1u);   // hi * lo
            mma_tf32(d, da, db, idesc, 1u);    // hi * hi
          }
          mma_commit(empty(stage));
          if (in_group == G - 1 || kb == kb1 - 1) mma_commit(acc_full(buf));
        }
        __syncwarp();
        if (in_group == G - 1 || kb == kb1 - 1) ++gi;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- converters + epilogue (warps 2..5) ----------------
    const int ct = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    int stage = 0;
    uint32_t phase = 0;
    uint32_t gi = 0;
    float acc[NP];
    // folds group `g` (buffer g & 1) of TMEM into acc[] and releases the buffer
    auto drain = [&](uint32_t g) {
      const uint32_t buf = g & 1;
      mbar_wait(acc_full(buf), (g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + buf * NP + uint32_t(c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[c0 + i] = __fadd_rn(acc[c0 + i], v[i]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty(buf));
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles, tile = u % tiles;
      const int kb0 = split * kb_per_split;
      const int kb1 = min(kb_total, kb0 + kb_per_split);
#pragma unroll
      for (int i = 0; i < NP; ++i) acc[i] = 0.f;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(full(stage), phase);
        uint4* a = reinterpret_cast<uint4*>(stage_a(stage));
        uint4* al = reinterpret_cast<uint4*>(stage_al(stage));
#pragma unroll
        for (int e = ct; e < A_STAGE_BYTES / 16; e += 128) split4(a + e, al + e);
        uint4* b = reinterpret_cast<uint4*>(stage_b(stage));
        uint4* bl = reinterpret_cast<uint4*>(stage_bl(stage));
#pragma unroll
        for (int e = ct; e < C::B_BYTES / 16; e += 128) split4(b + e, bl + e);
        fence_proxy_async_smem();
        mbar_arrive(conv(stage));
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        // the previous group finished while this stage was converted: fold it
        if ((kb - kb0) % G == 0 && kb > kb0) drain(gi++);
      }
      drain(gi++);  // last group of the unit
      const int row = tile * BM + q * 32 + lane;
      if (row < M) {
        float* dst = out + int64_t(split) * slab + int64_t(row) * r;
#pragma unroll
        for (int i = 0; i < NP; ++i)
          if (i < r) dst[i] = acc[i];
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const float* base, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {d0 * sizeof(float)};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

int pick_np(int r) { return r <= 32 ? 32 : r <= 64 ? 64 : r <= 96 ? 96 : r <= 128 ? 128 : 0; }

bool tc_enabled() {
  static int enabled = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("BS_DISABLE_TCGEN05");
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    enabled = (e && e[0] == '1') ? 0 : (major == 10 && minor == 0) ? 1 : 0;
  });
  return enabled == 1;
}

template <bool A_MN, int NP>
int launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, int M, int K, int r, int splits, float* out, int64_t slab,
              cudaStream_t st) {
  using C = TcCfg<NP>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(tc_gemm_kernel<A_MN, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
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
    group = (e && atoi(e) > 0) ? atoi(e) : 2;
  });
  tc_gemm_kernel<A_MN, NP><<<grid, TC_THREADS, C::SMEM, st>>>(ta, tb, M, K, r, tiles, kb_per, units, group, out, slab);
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
  return ws_bytes<float>(int64_t(TC_MAX_SPLITS) * m * r);
}
int64_t tc_vtx_workspace(int64_t m, int64_t n_loc, int r) {
  (void)m; (void)n_loc; (void)r;
  return 0;
}

#define BS_TC_DISPATCH(AMN)                                                                            \
  switch (np) {                                                                                        \
    case 32: S = launch_tc<AMN, 32>(ta, tb, M, K, r, nsplit, out, slab, st); break;                    \
    case 64: S = launch_tc<AMN, 64>(ta, tb, M, K, r, nsplit, out, slab, st); break;                    \
    case 96: S = launch_tc<AMN, 96>(ta, tb, M, K, r, nsplit, out, slab, st); break;                    \
    default: S = launch_tc<AMN, 128>(ta, tb, M, K, r, nsplit, out, slab, st); break;                   \
  }

// scn b: writes S partial slabs of P (r x m) into the workspace and folds them into P.
int tc_wxt(const float* X, const float* W, int64_t m, int64_t n_loc, int r, float* P, Workspace& ws, cudaStream_t st,
           bool* used) {
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
  if (S > 1) {
    launch_sum_slabs_f32(slabs, S, m * r, P, st);
    rc = check_launch("tc_wxt fold");
    if (rc != BS_OK) return rc;
  }
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
  BS_TC_DISPATCH(false)
  int rc = check_launch("tc_vtx");
  if (rc != BS_OK) return rc;
  *splits = S;
  *used = true;
  return BS_OK;
}

}  // namespace bs
