// Stage-2 contraction kernel: tcgen05 / TMEM 3xTF32 GEMM for sm_100a.
//
//   D = alpha * op(A) op(B) + beta * Cin          (fp32 in, fp32 out)
//   op(A)(m,k) = ta ? A[k*lda + m] : A[m*lda + k]
//   op(B)(k,n) = tb ? B[n*ldb + k] : B[k*ldb + n]
//   optional K-concatenated second product: + op(A2) op(B2)  (SYR2K)
//
// 3xTF32: x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi); the
// product is accumulated as lo*hi + hi*lo + hi*hi in the fp32 TMEM
// accumulator (the lo*lo term, ~2^-22 relative, is dropped).  This keeps the
// fp32 tolerance (1e-4 relative, BASELINE.json north_star) on tensor cores.
//
// Data path:
//   1. tc_pack: reads op(A)/op(B) in either major-ness, splits, and writes the
//      hi/lo operands as ready-made 128x32 K-major SWIZZLE_128B shared-memory
//      images (16 KB each), one per (row block, k block).
//   2. tc_gemm_kernel (128 threads, 1 CTA/SM, 128x128 output tile):
//        warp0.lane0  producer: 4 x cp.async.bulk (16 KB) per k block into a
//                     3-stage ring, completion via mbarrier complete_tx
//        warp1.lane0  MMA issuer: 4 k-steps x 3 tcgen05.mma.kind::tf32
//                     (M=128, N=128, K=8) per k block; tcgen05.commit frees
//                     the stage; a final commit signals the epilogue
//        warp2        TMEM allocator (128 columns)
//        warps0-3     epilogue: tcgen05.ld 32x32b.x32 -> alpha/beta -> global
#pragma once
#include "pf_common.cuh"

#include <algorithm>

namespace pf {

// 3xFP16 operands (tc_f16.cuh): x * s = hi + lo with hi = fp16_rn(x s),
// lo = fp16_rn(x s - hi), s a power of two per operand row putting
// max|x_row s| in [2^14, 2^15); images are K-major R x kp halfs.
struct F16Operands {
  const void* hi[4];   // op(A), op(B), op(A2), op(B2)
  const void* lo[4];
  int kp;              // image pitch (halfs, multiple of 8)
  const float* rinv;   // device [M (+pad)]: 1 / s of each row of op(A)   (output rows)
  const float* cinv;   // device [N (+pad)]: 1 / s of each row of op(B)^T (output columns)
};

struct TcGemmArgs {
  int M, N, K;
  float alpha, beta;
  const float* A;
  int lda;
  bool ta;
  const float* B;
  int ldb;
  bool tb;
  const float* A2;  // optional: K-concatenated second operand pair
  const float* B2;
  const float* Cin;  // may alias D; unused if beta == 0
  int ldc;
  float* D;
  int ldd;
  int upper_only;  // compute only output tiles with n-block >= m-block
  // pre-split operands (TMA path): lo = x - trunc_tf32(x) images with the
  // operands' own layouts (nullptr: the kernel's converter warps split)
  const float* Alo = nullptr;
  const float* Blo = nullptr;
  const float* A2lo = nullptr;
  const float* B2lo = nullptr;
  // split-K hand-over flags (Workspace::ensure_tile_flags) and this launch's
  // epoch; nullptr: split-K products use a beta pre-pass instead
  int* tile_flags = nullptr;
  int epoch = 0;
  // optional: the epilogue also writes lo = D - trunc_tf32(D) here (pitch ldd)
  // for a later product that consumes D as an operand
  float* Dlo = nullptr;
  // symmetric product (M == N, op(A) op(B) symmetric: SYRK, SYR2K): only tiles
  // on or above the diagonal are computed; off-diagonal tiles are also
  // added, transposed, below the diagonal (beta pre-pass + add-reductions)
  int sym = 0;
  // 3xFP16 operand images (nullptr: fp32 operands, 3xTF32)
  const F16Operands* f16 = nullptr;
  // D already holds its base on every tile the product writes -- beta * Cin,
  // or zeros when beta = 0: split-K partials and symmetric mirrors all
  // add-reduce, with no pre-pass and no ordered hand-over
  int d_base = 0;
};

constexpr int kTcBM = 128, kTcBN = 128, kTcBK = 32;
constexpr uint32_t kTcTile = 16384;  // one packed image: 128 rows x 32 fp32

// Tile configurations: BN = 128 (3-stage ring, 64 KB/stage) for small
// problems, BN = 256 (2-stage ring, 96 KB/stage; N=256 MMAs, 25% less operand
// traffic per flop) when there are enough output tiles to fill the GPU.
template <int BN>
struct TcCfg {
  static constexpr int kStages = BN == 256 ? 2 : 3;
  static constexpr uint32_t kBTiles = BN / 128;                       // packed 128-row images per B operand
  static constexpr uint32_t kStageBytes = (2 + 2 * kBTiles) * kTcTile;  // A hi/lo + B hi/lo
  static constexpr uint32_t kSmem = kStages * kStageBytes + 1024;
  static constexpr uint32_t kTmemCols = BN;
};

struct TcParams {
  const float* ahi;
  const float* alo;
  const float* bhi;
  const float* blo;
  int kblocks;      // k blocks of the whole reduction
  int kb_per_split; // k blocks per blockIdx.z (split-K; == kblocks when not split)
  int M, N;
  float alpha, beta;
  const float* Cin;
  int ldc;
  float* D;
  int ldd;
  int upper_only;
};

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (sm100 layout):
// start>>4 @[0,14), LBO>>4 @[16,30) (unused for swizzled K-major), SBO>>4
// @[32,46) = 1024 B between 8-row groups, version 1 @[46,48), layout 2 @[61,64).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32 (bit 4), A/B tf32 (2 @7, 2 @10),
// K-major A and B, N>>3 @[17,23), M>>4 @[24,29).
constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// kind::f16 (fp16 A/B, fp32 accumulate; K = 16 per instruction = 32 bytes,
// the same byte step as kind::tf32's K = 8)
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue of one warp: TMEM lanes (tile rows row0 .. row0+31) x ncols
// accumulator columns starting at TMEM column 0 / output column col0.
// tcgen05.ld gives lane = row, register j = column; the 32x32 block is
// transposed through a padded per-warp shared buffer (33-float rows: both
// phases conflict-free) so every global access is one 128-byte row segment
// (lane = column) instead of 32 rows x 4 bytes.
//   split:  D += alpha * acc          (D pre-scaled by beta; red.global.add)
//   else:   D  = alpha * acc + beta * Cin
__device__ __forceinline__ void epilogue_rows32(uint32_t taddr, int ncols, int row0, int col0, int M, int N,
                                                float alpha, float beta, const float* Cin, int ldc, float* D,
                                                int ldd, bool split, float* stage, int lane) {
#pragma unroll 1
  for (int c = 0; c < ncols / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + (uint32_t)(c * 32), r);
#pragma unroll
    for (int j = 0; j < 32; ++j) stage[lane * 33 + j] = __uint_as_float(r[j]);
    __syncwarp();
    const int col = col0 + c * 32 + lane;
    if (col < N) {
#pragma unroll 4
      for (int rr = 0; rr < 32; ++rr) {
        const int row = row0 + rr;
        if (row >= M) break;
        const float v = alpha * stage[rr * 33 + lane];
        float* d = D + (size_t)row * ldd + col;
        if (split) {
          atomicAdd(d, v);
        } else {
          *d = beta != 0.f ? fmaf(beta, Cin[(size_t)row * ldc + col], v) : v;
        }
      }
    }
    __syncwarp();
  }
}

// Lane-per-row epilogue (each lane stores 32 consecutive columns of its own
// row straight from its TMEM registers; no staging, uncoalesced across the
// warp).  Kept as the A/B alternative to epilogue_rows32 (PF_TC_DIAG bit 16).
__device__ __forceinline__ void epilogue_lane_rows(uint32_t taddr, int ncols, int row0, int col0, int M, int N,
                                                   float alpha, float beta, const float* Cin, int ldc, float* D,
                                                   int ldd, bool split, int lane) {
  const int row = row0 + lane;
#pragma unroll 1
  for (int c = 0; c < ncols / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + (uint32_t)(c * 32), r);
    const int cb = col0 + c * 32;
    if (row < M) {
      float* drow = D + (size_t)row * ldd;
      const float* crow = Cin + (size_t)row * ldc;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = cb + j;
        if (col < N) {
          const float v = alpha * __uint_as_float(r[j]);
          if (split)
            atomicAdd(drow + col, v);
          else
            drow[col] = beta != 0.f ? fmaf(beta, crow[col], v) : v;
        }
      }
    }
  }
}

}  // namespace tc

// Pack op(X) (R x K logical, rows = M for A / N for B) into hi/lo K-major
// SW128 tile images.  value(r,k) = kmajor ? X[r*ld + k] : X[k*ld + r];
// k >= K reads X2 at k-K (K-concatenation).  Zero padding to 128 x 32.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) tc_pack(const float* __restrict__ X, const float* __restrict__ X2, int ld,
                                               int kmajor, int R, int K, int ktot, int kblocks,
                                               float* __restrict__ hi, float* __restrict__ lo) {
  const int kb = blockIdx.x, rb = blockIdx.y;
  float* thi = hi + ((size_t)rb * kblocks + kb) * (kTcTile / 4);
  float* tlo = lo + ((size_t)rb * kblocks + kb) * (kTcTile / 4);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = threadIdx.x + 256 * i;  // 16-byte chunk id in the tile
    int r, c;
    if (kmajor) {
      r = q >> 3;
      c = q & 7;
    } else {
      r = q & 127;
      c = q >> 7;
    }
    const int gr = rb * kTcBM + r;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = kb * kTcBK + c * 4 + e;
      float x = 0.f;
      if (gr < R && k < ktot) {
        const float* src = X;
        if (k >= K) {
          src = X2;
          k -= K;
        }
        x = kmajor ? src[(size_t)gr * ld + k] : src[(size_t)k * ld + gr];
      }
      v[e] = x;
    }
    float4 h, l;
    h.x = tc::tf32_rna(v[0]);
    h.y = tc::tf32_rna(v[1]);
    h.z = tc::tf32_rna(v[2]);
    h.w = tc::tf32_rna(v[3]);
    l.x = tc::tf32_rna(v[0] - h.x);
    l.y = tc::tf32_rna(v[1] - h.y);
    l.z = tc::tf32_rna(v[2] - h.z);
    l.w = tc::tf32_rna(v[3] - h.w);
    const int off = (r >> 3) * 256 + (r & 7) * 32 + ((c ^ (r & 7)) << 2);  // in floats
    *reinterpret_cast<float4*>(thi + off) = h;
    *reinterpret_cast<float4*>(tlo + off) = l;
  }
}

template <BenchId Bn, int V, int BN>
__global__ void __launch_bounds__(128, 1) tc_gemm_kernel(TcParams p) {
  using Cfg = TcCfg<BN>;
  constexpr int kTcStages = Cfg::kStages;
  constexpr uint32_t kStageBytes = Cfg::kStageBytes;
  extern __shared__ uint8_t tc_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages], accum_bar;
  __shared__ uint32_t tmem_slot;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = blockIdx.y, nb = blockIdx.x;
  if (p.upper_only && (nb + 1) * BN <= mb * kTcBM) return;  // tile strictly below the diagonal

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(&accum_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nkb = min(p.kblocks - kb0, p.kb_per_split);
  const bool split = gridDim.z > 1;
  const size_t a_base = ((size_t)mb * p.kblocks + kb0) * (kTcTile / 4);
  // B row block nb spans kBTiles packed 128-row images (rb = nb*kBTiles + t)
  const size_t b_base = ((size_t)nb * Cfg::kBTiles * p.kblocks + kb0) * (kTcTile / 4);
  const size_t b_tile_stride = (size_t)p.kblocks * (kTcTile / 4);

  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kTcStages;
      const uint32_t ph = (kb / kTcStages) & 1;
      tc::mbar_wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
      const uint32_t fb = tc::smem_u32(&full_bar[s]);
      tc::mbar_expect_tx(fb, kStageBytes);
      // stage layout: [A hi][A lo][B hi (kBTiles images)][B lo (kBTiles images)]
      const uint32_t dst = tc::smem_u32(smem + (size_t)s * kStageBytes);
      const size_t ko = (size_t)kb * (kTcTile / 4);
      tc::bulk_g2s(dst, p.ahi + a_base + ko, kTcTile, fb);
      tc::bulk_g2s(dst + kTcTile, p.alo + a_base + ko, kTcTile, fb);
#pragma unroll
      for (uint32_t t = 0; t < Cfg::kBTiles; ++t) {
        tc::bulk_g2s(dst + (2 + t) * kTcTile, p.bhi + b_base + t * b_tile_stride + ko, kTcTile, fb);
        tc::bulk_g2s(dst + (2 + Cfg::kBTiles + t) * kTcTile, p.blo + b_base + t * b_tile_stride + ko, kTcTile, fb);
      }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = tc::idesc_tf32(kTcBM, BN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kTcStages;
      const uint32_t ph = (kb / kTcStages) & 1;
      tc::mbar_wait(tc::smem_u32(&full_bar[s]), ph);
      tc::fence_after();
      const uint32_t base = tc::smem_u32(smem + (size_t)s * kStageBytes);
#pragma unroll
      for (int kk = 0; kk < kTcBK / 8; ++kk) {
        const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
        const uint64_t ahi = tc::desc_sw128(base + koff);
        const uint64_t alo = tc::desc_sw128(base + kTcTile + koff);
        const uint64_t bhi = tc::desc_sw128(base + 2 * kTcTile + koff);
        const uint64_t blo = tc::desc_sw128(base + (2 + Cfg::kBTiles) * kTcTile + koff);
        tc::mma_tf32(tmem, alo, bhi, idesc, (kb | kk) != 0);
        tc::mma_tf32(tmem, ahi, blo, idesc, 1u);
        tc::mma_tf32(tmem, ahi, bhi, idesc, 1u);
      }
      tc::mma_commit(tc::smem_u32(&empty_bar[s]));
    }
    tc::mma_commit(tc::smem_u32(&accum_bar));
  }
  __syncwarp();

  // Epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w+31; the idle
  // stage ring (all MMAs retired) holds the per-warp transpose buffers.
  tc::mbar_wait(tc::smem_u32(&accum_bar), 0);
  tc::fence_after();
  tc::epilogue_rows32(tmem + ((uint32_t)(warp * 32) << 16), BN, mb * kTcBM + warp * 32, nb * BN, p.M, p.N, p.alpha,
                      p.beta, p.Cin, p.ldc, p.D, p.ldd, split, reinterpret_cast<float*>(smem) + warp * 32 * 33, lane);
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Split-K factor: small problems (fewer output tiles than SMs) spread their k
// blocks over blockIdx.z so that ~148 CTAs run; at least 2 k blocks per split.
inline int tc_bn(int64_t m, int64_t n) {
  // BN = 256 only when it still yields at least ~one wave of output tiles
  const int64_t tiles256 = ((m + kTcBM - 1) / kTcBM) * ((n + 255) / 256);
  return tiles256 >= 120 ? 256 : 128;
}

inline int tc_splits(int64_t m, int64_t n, int64_t ktot) {
  const int bn = tc_bn(m, n);
  const int64_t tiles = ((m + kTcBM - 1) / kTcBM) * ((n + bn - 1) / bn);
  const int64_t kblocks = (ktot + kTcBK - 1) / kTcBK;
  if (tiles >= 74) return 1;
  int64_t s = std::min<int64_t>(device_sms() / tiles, kblocks / 2);
  return (int)std::max<int64_t>(1, s);
}

// pack A, pack B, [pre-scale D when split], gemm
inline int64_t tc_gemm_launches(int64_t m, int64_t n, int64_t k, bool dual = false) {
  return 3 + (tc_splits(m, n, dual ? 2 * k : k) > 1 ? 1 : 0);
}
inline bool tc_gemm_supported(int64_t m, int64_t n, int64_t k) { return m > 0 && n > 0 && k > 0; }

// D = beta * Cin (or 0) before split-K partials are accumulated atomically.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) tc_prescale(float* D, int ldd, const float* Cin, int ldc, int M, int N,
                                                   float beta) {
  // the split-K GEMM launched after this kernel (programmatic dependent
  // launch) may start its mainloop now; it waits for this grid before its
  // first add-reduction onto D
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (n >= N) return;
  D[(size_t)m * ldd + n] = beta != 0.f ? beta * Cin[(size_t)m * ldc + n] : 0.f;
}

// Contiguous form (ldd == ldc == N, 16-byte aligned): float4, four loads in
// flight per thread, grid-stride.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) tc_prescale_flat(float4* __restrict__ D, const float4* __restrict__ Cin,
                                                        int64_t n4, float beta) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = Cin[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      D[i + u * stride] = make_float4(beta * v[u].x, beta * v[u].y, beta * v[u].z, beta * v[u].w);
  }
  for (; i < n4; i += stride) {
    const float4 v = Cin[i];
    D[i] = make_float4(beta * v.x, beta * v.y, beta * v.z, beta * v.w);
  }
}

template <BenchId Bn, int V, int BN>
inline void launch_tc_main(const TcParams& p, int np, int mp, int zs, cudaStream_t s) {
  set_smem_attr((const void*)tc_gemm_kernel<Bn, V, BN>, (int)TcCfg<BN>::kSmem);
  tc_gemm_kernel<Bn, V, BN><<<dim3(np / BN, mp / kTcBM, zs), 128, TcCfg<BN>::kSmem, s>>>(p);
}

template <BenchId Bn, int V>
inline void launch_tc_gemm(Workspace& ws, const TcGemmArgs& a, cudaStream_t s) {
  const int ktot = a.A2 ? 2 * a.K : a.K;
  const int bn = tc_bn(a.M, a.N);
  const int mp = round_up(a.M, kTcBM), np = round_up(a.N, bn), kp = round_up(ktot, kTcBK);
  const int kblocks = kp / kTcBK;
  const size_t asz = (size_t)mp * kp, bsz = (size_t)np * kp;
  float* scr = ws.ensure_scratch((2 * asz + 2 * bsz) * sizeof(float));
  if (!scr) {
    launch_failed("tcgen05 packed path: operand scratch allocation failed");
    return;
  }
  float* ahi = scr;
  float* alo = ahi + asz;
  float* bhi = alo + asz;
  float* blo = bhi + bsz;
  tc_pack<Bn, V><<<dim3(kblocks, mp / kTcBM), 256, 0, s>>>(a.A, a.A2, a.lda, a.ta ? 0 : 1, a.M, a.K, ktot, kblocks,
                                                            ahi, alo);
  tc_pack<Bn, V><<<dim3(kblocks, np / 128), 256, 0, s>>>(a.B, a.B2, a.ldb, a.tb ? 1 : 0, a.N, a.K, ktot, kblocks,
                                                          bhi, blo);
  const int splits = tc_splits(a.M, a.N, ktot);
  const int per = (kblocks + splits - 1) / splits;
  const int zs = (kblocks + per - 1) / per;
  if (zs > 1) tc_prescale<Bn, V><<<dim3(cdiv(a.N, 256), a.M), 256, 0, s>>>(a.D, a.ldd, a.Cin, a.ldc, a.M, a.N, a.beta);
  TcParams p{ahi, alo, bhi, blo, kblocks, per, a.M, a.N, a.alpha, a.beta, a.Cin, a.ldc, a.D, a.ldd, a.upper_only};
  if (bn == 256)
    launch_tc_main<Bn, V, 256>(p, np, mp, zs, s);
  else
    launch_tc_main<Bn, V, 128>(p, np, mp, zs, s);
}

}  // namespace pf
