// Stage-2 contraction kernels, TMA generation: tcgen05 / TMEM GEMM in two
// arithmetic modes -- 3xTF32 fed directly from the raw fp32 operands
// (kind::tf32), or 3xFP16 fed from row-scaled fp16 hi / lo images
// (kind::f16, tc_f16.cuh; TmaParams::f16).  A 128-row x 128-byte operand tile
// is byte-identical in both (32 fp32 or 64 fp16 of K), so the descriptors,
// ring and warp roles below are shared; the epilogue undoes the 3xFP16 row
// and column scales.
//
//   D = alpha * op(A) op(B) + beta * Cin        (same contract as tc_gemm.cuh)
//
// Operands:
//   * TMA tensor maps (cuTensorMapEncodeTiled, SWIZZLE_128B) load the raw fp32
//     tiles in either major-ness -- K-major tiles as one 128x32 box, MN-major
//     tiles as four 32x32 boxes -- straight into the canonical UMMA
//     shared-memory layouts;
//   * the tensor core truncates fp32 to TF32 when it reads an operand, so the
//     raw tile *is* the "hi" operand (hi = trunc_tf32(x)); the "lo" operand
//     x - trunc_tf32(x) is either TMA-loaded from a pre-split image in global
//     memory (products without split-K: tc_split_lo, or the previous product's
//     epilogue, or CORR's transpose pass) or computed by four converter warps
//     into the stage's lo buffers (split-K products).
// Precision: x = hi + lo exactly; the tensor core truncates lo to TF32
// (|error| <= 2^-10 |lo| <= 2^-20 |x|); the dropped lo*lo term is ~2^-20.
//
// Warp roles (192 threads, 1 CTA/SM, 3-stage ring of [A raw | B raw | A lo |
// B lo] = 64 KB):
//   warp 0 lane 0   TMA producer            full[s]  (expect_tx)
//   warps 2..5      lo converters (or a pass-through arrive when pre-split)
//                   -> ready[s]; then the epilogue (warp w reads TMEM lanes
//                   32*(w%4)): TMA Cin loads, alpha/beta in place in shared
//                   memory, TMA stores / add-reductions, optional lo image of D
//   warp 1 lane 0   MMA issuer: 4 k-steps x {lo*hi, hi*lo, hi*hi}; commit -> empty[s]
//   warp 1          TMEM allocation
// tc_tma_kernel: one CTA per 128x128 tile (cta_group::1); tc_tma2_kernel: a
// CTA pair per 256x256 tile (cta_group::2, each CTA streams half of B).
// Split-K: beta pre-pass + TMA add-reductions (the GEMM launched as a
// programmatic dependent launch), or for beta = 0 an in-kernel ordered
// hand-over through per-tile flags, or -- when the caller already wrote D's
// base (TcGemmArgs::d_base: zeros or beta * Cin) -- add-reductions only.
#pragma once
#include "pf_common.cuh"
#include "tc_gemm.cuh"
#include "tma_map.cuh"

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

namespace pf {

constexpr int kTmaStages = 3;
constexpr uint32_t kTmaTileBytes = 128 * 32 * 4;           // one 128-row x 32-k fp32 tile
constexpr uint32_t kTmaStageBytes = 4 * kTmaTileBytes;      // A raw, B raw, A lo, B lo
constexpr uint32_t kTmaSmem = kTmaStages * kTmaStageBytes + 1024;
constexpr int kTmaThreads = 192;

struct TmaParams {
  CUtensorMap ta, tb, ta2, tb2;  // 2nd pair: K-concatenated product (SYR2K)
  CUtensorMap tal, tbl, ta2l, tb2l;  // pre-split lo operands (valid iff presplit)
  int presplit;
  CUtensorMap tc, td;            // epilogue: Cin / D as 32x32 SWIZZLE_128B boxes (valid iff tma_epi)
  int tma_epi;
  CUtensorMap tdl;               // lo image of D (valid iff dlo)
  int dlo;
  int sym;                       // mirror off-diagonal tiles (add-reductions)
  int* tile_flags;               // ordered split-K: split 0 stores, the others add after its flag
  int epoch;
  int kblocks, kb_per_split, kb1;
  int a_mn, b_mn;                // operand is MN-major (contiguous along M / N)
  int M, N;
  float alpha, beta;
  const float* Cin;
  int ldc;
  float* D;
  int ldd;
  int upper_only;
  uint32_t mn_lbo, mn_sbo, mn_kstep;  // MN-major descriptor strides / k-step advance (bytes)
  int idesc_override;                 // probe only: -1 auto, else (a_major | b_major << 1)
  int sk_tiles, sk_pairs, sk_tiles_n;  // stream-K pair kernel (tc_sk2.cuh): pair tiles, pairs, tiles along N
  int f16;                            // operands are 3xFP16 images (hi/lo fp16, K-major): kind::f16 MMAs
  const float* f16_rinv;              // f16: 1 / row scale per output row (power of two)
  const float* f16_cinv;              // f16: 1 / row scale of op(B)^T per output column
  int diag;                           // diagnostics only (PF_TC_DIAG): 1 skip lo split, 2 skip MMAs, 4 skip loads, 8 skip epilogue, 16 lane-row epilogue, 32 smem-transpose epilogue
};

namespace tma {

__device__ __forceinline__ void load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// CTA-pair form: the destination is this CTA's shared memory, the completion
// mbarrier (a shared::cluster address) may be the pair leader's -- both CTAs'
// operand bytes then land on ONE barrier that the leader's MMA issuer waits on.
__device__ __forceinline__ void load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// UMMA shared-memory descriptors.
//   K-major (SWIZZLE_128B, layout 2): 8-row groups of 128-byte rows, SBO 1024 B.
//   MN-major: for TF32 the only legal MN-major layout is SWIZZLE_128B_BASE32B
//   (layout 1, Swizzle<2,5,2>: 32-byte chunks of a 128-byte row XORed with
//   row%4 -- CUTLASS sm100_common.inl); TMA produces it with
//   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.  128-byte rows hold 32 MN elements of
//   one K index; 4-row K groups at SBO = 512 B; 32-element MN slabs at
//   LBO = 4 KB (one 32x32 TMA box each).
__device__ __forceinline__ uint64_t desc(uint32_t saddr, bool mn_major, uint32_t lbo = 4096u, uint32_t sbo = 512u) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(mn_major ? ((lbo >> 4) & 0x3FFFu) : 1u) << 16;
  d |= (uint64_t)(((mn_major ? sbo : 1024u) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(mn_major ? 1u : 2u) << 61;
  return d;
}

// D f32 (bit 4); A/B format @7 / @10: tf32 = 2 (kind::tf32), f16 = 0 (kind::f16)
__device__ __forceinline__ uint32_t idesc(int m, int n, int a_mn, int b_mn, bool f16 = false) {
  const uint32_t fmt = f16 ? 0u : 2u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}



__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Converter warps (128 threads, t = 0..127): lo = x - trunc_tf32(x) for
// COUNT float4 per thread of a stage (raw at `raw`, lo image at `lo`), eight
// shared-memory loads in flight before their stores (the lds/sts asm
// statements are volatile, so a load-store-load order would serialise them).
template <int COUNT>
__device__ __forceinline__ void split_lo(uint32_t raw, uint32_t lo, int t) {
#pragma unroll
  for (int b = 0; b < COUNT; b += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b + u < COUNT) v[u] = lds128(raw + 16u * (uint32_t)(t + 128 * (b + u)));
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b + u < COUNT)
        sts128(lo + 16u * (uint32_t)(t + 128 * (b + u)),
               make_float4(v[u].x - trunc_tf32(v[u].x), v[u].y - trunc_tf32(v[u].y), v[u].z - trunc_tf32(v[u].z),
                           v[u].w - trunc_tf32(v[u].w)));
  }
}

__device__ __forceinline__ void store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void reduce_add_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}

// ar: alpha, or for 3xFP16 operands alpha / s_row of this lane's row (exact:
// powers of two); cs_s: the 3xFP16 column factors 1 / s_col of this tile's
// columns (shared memory, indexed from col0), or nullptr.
// Epilogue of one warp through TMA (the tile rows row0 .. row0+31 = TMEM
// lanes, ncols accumulator columns from col0).  The warp's Cin boxes (32x32,
// SWIZZLE_128B) are requested with one mbarrier before the first TMEM read;
// each 32-column chunk is combined in place -- lane = row, float4 chunk j at
// 16 * (j ^ (row % 8)), conflict-free -- and written back by one TMA store
// (or a TMA add-reduction onto the beta-prescaled D for split-K).  buf:
// 1024-byte aligned, ncols / 32 * 4 KB; bar: this warp's mbarrier (phase 0).
__device__ __forceinline__ void epilogue_tma(const TmaParams& p, float ar, const float* cs_s, uint32_t taddr,
                                             int ncols, int row0, int col0, bool split, uint8_t* buf, uint32_t bar,
                                             int lane,
                                             bool writes_done = false, uint8_t* lobuf = nullptr,
                                             bool mirror = false) {
  if (row0 >= p.M) return;  // warp-uniform
  const int nch = min(ncols / 32, (p.N - col0 + 31) / 32);
  const bool use_c = !split && p.beta != 0.f;
  const bool want_lo = p.dlo && !split && lobuf != nullptr;  // 4 x 4 KB ring of lo chunks
  const bool want_mirror = mirror && split && lobuf != nullptr;  // same ring: transposed chunks
  const uint32_t sbuf = tc::smem_u32(buf);
  const uint32_t slo = (want_lo || want_mirror) ? tc::smem_u32(lobuf) : 0u;

  if (use_c && lane == 0) {
    tc::mbar_expect_tx(bar, (uint32_t)nch * 4096u);
    for (int c = 0; c < nch; ++c) load_2d(sbuf + c * 4096, &p.tc, col0 + c * 32, row0, bar);
  }
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    uint32_t r[32];
    tc::tmem_ld32(taddr + (uint32_t)(c * 32), r);
    if (use_c && c == 0) tc::mbar_wait(bar, 0);
    float4* row = reinterpret_cast<float4*>(buf + c * 4096 + lane * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4* slot = row + (j ^ (lane & 7));
      float4 v = make_float4(ar * __uint_as_float(r[4 * j]), ar * __uint_as_float(r[4 * j + 1]),
                             ar * __uint_as_float(r[4 * j + 2]), ar * __uint_as_float(r[4 * j + 3]));
      if (cs_s) {  // 3xFP16: 1 / s_col, staged in shared memory before the accumulator wait
        const float4 cs = *reinterpret_cast<const float4*>(cs_s + c * 32 + 4 * j);
        v = make_float4(v.x * cs.x, v.y * cs.y, v.z * cs.z, v.w * cs.w);
      }
      if (use_c) {
        const float4 ci = *slot;
        v = make_float4(fmaf(p.beta, ci.x, v.x), fmaf(p.beta, ci.y, v.y), fmaf(p.beta, ci.z, v.z),
                        fmaf(p.beta, ci.w, v.w));
      }
      *slot = v;
      if ((want_lo || want_mirror) && j == 0 && c >= 4) {  // ring slot c % 4 is free once chunk c - 4's
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");  // stores have read it
        __syncwarp();
      }
      if (want_mirror) {  // transposed box: row = this column, column = lane (conflict-free 4-byte stores)
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int jr = 4 * j + e;
          *reinterpret_cast<float*>(lobuf + (c & 3) * 4096 + jr * 128 + (((lane >> 2) ^ (jr & 7)) << 4) +
                                    ((lane & 3) << 2)) = vv[e];
        }
      }
      if (want_lo) {
        float4* lslot = reinterpret_cast<float4*>(lobuf + (c & 3) * 4096 + lane * 128) + (j ^ (lane & 7));
        *lslot = make_float4(v.x - trunc_tf32(v.x), v.y - trunc_tf32(v.y), v.z - trunc_tf32(v.z),
                             v.w - trunc_tf32(v.w));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      if (split)
        reduce_add_2d(&p.td, sbuf + c * 4096, col0 + c * 32, row0);
      else
        store_2d(&p.td, sbuf + c * 4096, col0 + c * 32, row0);
      if (want_lo) store_2d(&p.tdl, slo + (c & 3) * 4096, col0 + c * 32, row0);
      if (want_mirror) reduce_add_2d(&p.td, slo + (c & 3) * 4096, row0, col0 + c * 32);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) {
    if (writes_done)  // the stores themselves complete (split-K hand-over), not just their smem reads
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    else
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
}

// 3xFP16: this warp's row factor alpha / s_row and its copy of the tile's
// column factors (ncols floats from col0), loaded while the mainloop runs.
__device__ __forceinline__ float stage_f16_scales(const TmaParams& p, int row, int col0, int ncols, float* cs_s,
                                                  int lane) {
  if (!p.f16) return p.alpha;
  for (int c = lane; c < ncols; c += 32) cs_s[c] = col0 + c < p.N ? __ldg(p.f16_cinv + col0 + c) : 1.f;
  __syncwarp();
  return p.alpha * __ldg(p.f16_rinv + min(row, p.M - 1));
}

// Ordered split-K hand-over.  Split 0 of an output tile writes
// alpha * acc + beta * Cin with plain TMA stores and then raises the tile's
// flag to this launch's epoch; every other split waits for that flag before
// its TMA add-reductions.  No beta pre-pass kernel, no extra launch.
__device__ __forceinline__ void split_wait(const TmaParams& p, int lane) {
  const int tile = blockIdx.y * gridDim.x + blockIdx.x;
  if (lane == 0) {
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.tile_flags + tile) : "memory");
    } while (v != p.epoch);
  }
  __syncwarp();
  asm volatile("fence.proxy.async.global;" ::: "memory");  // the add-reductions (async proxy) come after
}

__device__ __forceinline__ void split_publish(const TmaParams& p, int warp, int lane) {
  asm volatile("bar.sync 3, 128;" ::: "memory");  // the four epilogue warps' stores are complete
  if (warp == 2 && lane == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.tile_flags + tile), "r"(p.epoch) : "memory");
  }
}

// The A and B tiles of one k block (raw, or the pre-split lo images) into
// [base, base + 32 KB): K-major operands as one 128x32 box, MN-major ones as
// four 32x32 boxes.
__device__ __forceinline__ void load_operands(const TmaParams& p, bool second, bool lo, uint32_t base, int m0, int n0,
                                              int k0, uint32_t fb, bool pair_bar = false) {
  const CUtensorMap* ma = lo ? (second ? &p.ta2l : &p.tal) : (second ? &p.ta2 : &p.ta);
  const CUtensorMap* mb = lo ? (second ? &p.tb2l : &p.tbl) : (second ? &p.tb2 : &p.tb);
  auto ld = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
    if (pair_bar)
      load_2d_pair(dst, m, c0, c1, fb);
    else
      load_2d(dst, m, c0, c1, fb);
  };
  if (p.a_mn) {
#pragma unroll
    for (int j = 0; j < 4; ++j) ld(base + j * 4096, ma, m0 + 32 * j, k0);
  } else {
    ld(base, ma, k0, m0);
  }
  if (p.b_mn) {
#pragma unroll
    for (int j = 0; j < 4; ++j) ld(base + kTmaTileBytes + j * 4096, mb, n0 + 32 * j, k0);
  } else {
    ld(base + kTmaTileBytes, mb, k0, n0);
  }
}

}  // namespace tma

template <BenchId Bn, int V>
__global__ void __launch_bounds__(kTmaThreads, 1) tc_tma_kernel(const __grid_constant__ TmaParams p) {
  extern __shared__ uint8_t tma_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kTmaStages], ready_bar[kTmaStages], empty_bar[kTmaStages], accum_bar, epi_bar[4];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float epi_cs[4][256];  // 3xFP16 column factors, one copy per epilogue warp
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tma_smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = blockIdx.y, nb = blockIdx.x;
  if (p.upper_only && (nb + 1) * 128 <= mb * 128) return;
  const int m0 = mb * 128, n0 = nb * 128;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nkb = min(p.kblocks - kb0, p.kb_per_split);
  const bool split = gridDim.z > 1 || p.sym;  // sym: beta pre-pass + add-reductions

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&ready_bar[s]), 4);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(&accum_bar), 1);
    for (int q = 0; q < 4; ++q) tc::mbar_init(tc::smem_u32(&epi_bar[q]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma::prefetch_map(&p.ta);
    tma::prefetch_map(&p.tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)),
                 "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int kb = kb0 + i;
        const int s = i % kTmaStages;
        const uint32_t ph = (i / kTmaStages) & 1;
        tc::mbar_wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
        const uint32_t fb = tc::smem_u32(&full_bar[s]);
        if (p.diag & 4) {  // diagnostics: no operand loads
          tma::mbar_arrive(fb);
          continue;
        }
        tc::mbar_expect_tx(fb, (p.presplit ? 4 : 2) * kTmaTileBytes);
        const bool second = kb >= p.kb1;
        const int k0 = (second ? kb - p.kb1 : kb) * (p.f16 ? 64 : 32);  // elements per 128-byte k block
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
        tma::load_operands(p, second, false, base, m0, n0, k0, fb);
        if (p.presplit) tma::load_operands(p, second, true, base + 2 * kTmaTileBytes, m0, n0, k0, fb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = p.idesc_override < 0 ? tma::idesc(128, 128, p.a_mn, p.b_mn, p.f16)
                                               : tma::idesc(128, 128, p.idesc_override & 1, p.idesc_override >> 1);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kTmaStages;
        const uint32_t ph = (i / kTmaStages) & 1;
        // pre-split operands: nothing to convert, the MMAs wait for the TMA bytes
        tc::mbar_wait(tc::smem_u32(p.presplit ? &full_bar[s] : &ready_bar[s]), ph);
        tc::fence_after();
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ka = p.a_mn ? kk * p.mn_kstep : kk * 32u;
          const uint32_t kbo = p.b_mn ? kk * p.mn_kstep : kk * 32u;
          const uint64_t ahi = tma::desc(base + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t bhi = tma::desc(base + kTmaTileBytes + kbo, p.b_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t alo = tma::desc(base + 2 * kTmaTileBytes + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t blo = tma::desc(base + 3 * kTmaTileBytes + kbo, p.b_mn, p.mn_lbo, p.mn_sbo);
          if (p.diag & 2) continue;
          if (p.f16) {
            tc::mma_f16(tmem, alo, bhi, id, (i | kk) != 0);
            tc::mma_f16(tmem, ahi, blo, id, 1u);
            tc::mma_f16(tmem, ahi, bhi, id, 1u);
          } else {
            tc::mma_tf32(tmem, alo, bhi, id, (i | kk) != 0);
            tc::mma_tf32(tmem, ahi, blo, id, 1u);
            tc::mma_tf32(tmem, ahi, bhi, id, 1u);
          }
        }
        tc::mma_commit(tc::smem_u32(&empty_bar[s]));
      }
      tc::mma_commit(tc::smem_u32(&accum_bar));
    }
    __syncwarp();
  } else {
    // ---- converters: lo = x - trunc_tf32(x) for the A and B raw tiles
    const int ct = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < (p.presplit ? 0 : nkb); ++i) {
      const int s = i % kTmaStages;
      const uint32_t ph = (i / kTmaStages) & 1;
      tc::mbar_wait(tc::smem_u32(&full_bar[s]), ph);
      const uint32_t raw = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
      const uint32_t lo = raw + 2 * kTmaTileBytes;
      if (!((p.diag & 1) || p.presplit)) tma::split_lo<(int)(2 * kTmaTileBytes / 16 / 128)>(raw, lo, ct);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(tc::smem_u32(&ready_bar[s]));
    }
    // ---- epilogue: TMEM lanes 32*(warp%4) .. +31 are tile rows (coalesced
    // through the idle stage ring, see tc::epilogue_rows32)
    const int quad = warp & 3;
    const float ar = tma::stage_f16_scales(p, m0 + quad * 32 + lane, n0, 128, epi_cs[quad], lane);
    tc::mbar_wait(tc::smem_u32(&accum_bar), 0);
    tc::fence_after();
    if (p.tma_epi && !(p.diag & (8 | 16 | 32))) {
      const bool ordered = split && p.tile_flags != nullptr;
      if (ordered && blockIdx.z > 0) tma::split_wait(p, lane);
      if (split && !ordered) asm volatile("griddepcontrol.wait;" ::: "memory");  // the beta pre-pass is done
      tma::epilogue_tma(p, ar, p.f16 ? epi_cs[quad] : nullptr, tmem + ((uint32_t)(quad * 32) << 16), 128, m0 + quad * 32, n0,
                        split && !(ordered && blockIdx.z == 0), smem + (size_t)quad * 32768,
                        tc::smem_u32(&epi_bar[quad]), lane, ordered, smem + 131072 + (size_t)quad * 16384,
                        p.sym && nb != mb);
      if (ordered && blockIdx.z == 0) tma::split_publish(p, warp, lane);
    }
    else if (p.diag & 16)
      tc::epilogue_lane_rows(tmem + ((uint32_t)(quad * 32) << 16), 128, m0 + quad * 32, n0, p.M, p.N, p.alpha, p.beta,
                             p.Cin, p.ldc, p.D, p.ldd, split, lane);
    else if (!(p.diag & 8))
      tc::epilogue_rows32(tmem + ((uint32_t)(quad * 32) << 16), 128, m0 + quad * 32, n0, p.M, p.N, p.alpha, p.beta,
                          p.Cin, p.ldc, p.D, p.ldd, split, reinterpret_cast<float*>(smem) + quad * 32 * 33, lane);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
  }
}

// ---------------------------------------------------------------- CTA-pair kernel
// Same contract and per-CTA stage layout as tc_tma_kernel, but two CTAs of a
// cluster (one TPC) cooperate on a 256x256 tile with tcgen05.mma.cta_group::2
// (M = 256, N = 256): CTA r holds A rows m0 + 128r .. +127 and B columns
// n0 + 128r .. +127 of every k block, and accumulates its 128 rows x all 256
// columns in its own TMEM.  Each CTA streams half of the B tile the pair needs,
// so shared-memory operand traffic per FMA halves -- the single-CTA kernel is
// shared-memory-bandwidth bound (ncu, profiles/r01_ncu_tc_tma.md).
//   * each CTA: TMA producer (own full[s]) -> 4 converter warps (lo) -> one
//     arrive per warp on the LEADER's ready[s] (8 arrivals per phase);
//   * leader warp 1 lane 0 issues the MMAs; tcgen05.commit multicasts to
//     empty[s] / accum in both CTAs;
//   * TMEM: 256 columns allocated with cta_group::2 by warp 1 of both CTAs.
// Every wait is bounded (~10 s of clock64) and traps instead of hanging.
namespace tc2 {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t peer_addr(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
  if (try_wait(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t n = 1;; ++n) {
    if (try_wait(bar, parity)) return;
    if ((n & 1023u) == 0 && clock64() - t0 > 20000000000LL) __trap();
  }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void commit_both(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

}  // namespace tc2

template <BenchId Bn, int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTmaThreads, 1)
    tc_tma2_kernel(const __grid_constant__ TmaParams p) {
  extern __shared__ uint8_t tma_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kTmaStages], ready_bar[kTmaStages], empty_bar[kTmaStages], accum_bar, epi_bar[4];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float epi_cs[4][256];  // 3xFP16 column factors, one copy per epilogue warp
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tma_smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc2::cluster_rank();
  const int mb = blockIdx.y, nb = blockIdx.x >> 1;
  if (p.upper_only && nb < mb) return;  // the whole pair leaves together
  const int m0 = mb * 256 + (int)rank * 128;  // A rows / accumulator rows of this CTA
  const int nB = nb * 256 + (int)rank * 128;  // B columns streamed by this CTA
  const int n0 = nb * 256;                    // accumulator columns (both CTAs)
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nkb = min(p.kblocks - kb0, p.kb_per_split);
  const bool split = gridDim.z > 1 || p.sym;  // sym: beta pre-pass + add-reductions

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&ready_bar[s]), 8);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(&accum_bar), 1);
    for (int q = 0; q < 4; ++q) tc::mbar_init(tc::smem_u32(&epi_bar[q]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma::prefetch_map(&p.ta);
    tma::prefetch_map(&p.tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)),
                 "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before();
  tc2::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int kb = kb0 + i;
        const int s = i % kTmaStages;
        const uint32_t ph = (i / kTmaStages) & 1;
        tc2::wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
        const uint32_t fb = tc::smem_u32(&full_bar[s]);
        if (p.diag & 4) {  // diagnostics: no operand loads
          tma::mbar_arrive(fb);
          continue;
        }
        const bool second = kb >= p.kb1;
        const int k0 = (second ? kb - p.kb1 : kb) * (p.f16 ? 64 : 32);  // elements per 128-byte k block
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
        if (p.presplit) {
          // both CTAs' bytes complete on the LEADER's full[s]: its MMA issuer
          // waits on that one barrier (no converter hand-off, no remote arrive;
          // 2MM 2048: 0.187 -> 0.165 ms)
          const uint32_t lb = tc2::peer_addr(fb, 0);
          if (rank == 0) tc::mbar_expect_tx(fb, 2 * 4 * kTmaTileBytes);
          tma::load_operands(p, second, false, base, m0, nB, k0, lb, true);
          tma::load_operands(p, second, true, base + 2 * kTmaTileBytes, m0, nB, k0, lb, true);
          continue;
        }
        tc::mbar_expect_tx(fb, 2 * kTmaTileBytes);
        tma::load_operands(p, second, false, base, m0, nB, k0, fb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t id = tma::idesc(256, 256, p.a_mn, p.b_mn, p.f16);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kTmaStages;
        const uint32_t ph = (i / kTmaStages) & 1;
        tc2::wait(tc::smem_u32(p.presplit ? &full_bar[s] : &ready_bar[s]), ph);
        tc::fence_after();
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ka = p.a_mn ? kk * p.mn_kstep : kk * 32u;
          const uint32_t kbo = p.b_mn ? kk * p.mn_kstep : kk * 32u;
          const uint64_t ahi = tma::desc(base + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t bhi = tma::desc(base + kTmaTileBytes + kbo, p.b_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t alo = tma::desc(base + 2 * kTmaTileBytes + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t blo = tma::desc(base + 3 * kTmaTileBytes + kbo, p.b_mn, p.mn_lbo, p.mn_sbo);
          if (p.diag & 2) continue;
          if (p.f16) {
            tc2::mma_f16(tmem, alo, bhi, id, (i | kk) != 0);
            tc2::mma_f16(tmem, ahi, blo, id, 1u);
            tc2::mma_f16(tmem, ahi, bhi, id, 1u);
          } else {
            tc2::mma_tf32(tmem, alo, bhi, id, (i | kk) != 0);
            tc2::mma_tf32(tmem, ahi, blo, id, 1u);
            tc2::mma_tf32(tmem, ahi, bhi, id, 1u);
          }
        }
        tc2::commit_both(tc::smem_u32(&empty_bar[s]));
      }
      tc2::commit_both(tc::smem_u32(&accum_bar));
    }
    __syncwarp();
  } else {
    const int ct = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < (p.presplit ? 0 : nkb); ++i) {
      const int s = i % kTmaStages;
      const uint32_t ph = (i / kTmaStages) & 1;
      tc2::wait(tc::smem_u32(&full_bar[s]), ph);
      const uint32_t raw = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
      const uint32_t lo = raw + 2 * kTmaTileBytes;
      if (!((p.diag & 1) || p.presplit)) tma::split_lo<(int)(2 * kTmaTileBytes / 16 / 128)>(raw, lo, ct);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc2::arrive_remote(tc2::peer_addr(tc::smem_u32(&ready_bar[s]), 0));
    }
    // all MMAs of the pair (which read this CTA's ring) have retired once
    // accum fires, so the ring holds the epilogue transpose buffers
    const int quad = warp & 3;
    const float ar = tma::stage_f16_scales(p, m0 + quad * 32 + lane, n0, 256, epi_cs[quad], lane);
    tc2::wait(tc::smem_u32(&accum_bar), 0);
    tc::fence_after();
    if (p.tma_epi && !(p.diag & (8 | 16 | 32))) {
      const bool ordered = split && p.tile_flags != nullptr;
      if (ordered && blockIdx.z > 0) tma::split_wait(p, lane);
      if (split && !ordered) asm volatile("griddepcontrol.wait;" ::: "memory");  // the beta pre-pass is done
      tma::epilogue_tma(p, ar, p.f16 ? epi_cs[quad] : nullptr, tmem + ((uint32_t)(quad * 32) << 16), 256, m0 + quad * 32, n0,
                        split && !(ordered && blockIdx.z == 0), smem + (size_t)quad * 32768,
                        tc::smem_u32(&epi_bar[quad]), lane, ordered, smem + 131072 + (size_t)quad * 16384,
                        p.sym && nb != mb);
      if (ordered && blockIdx.z == 0) tma::split_publish(p, warp, lane);
    }
    else if (p.diag & 16)
      tc::epilogue_lane_rows(tmem + ((uint32_t)(quad * 32) << 16), 256, m0 + quad * 32, n0, p.M, p.N, p.alpha, p.beta,
                             p.Cin, p.ldc, p.D, p.ldd, split, lane);
    else if (!(p.diag & 8))
      tc::epilogue_rows32(tmem + ((uint32_t)(quad * 32) << 16), 256, m0 + quad * 32, n0, p.M, p.N, p.alpha, p.beta,
                          p.Cin, p.ldc, p.D, p.ldd, split, reinterpret_cast<float*>(smem) + quad * 32 * 33, lane);
  }
  tc::fence_before();
  tc2::cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
  }
}

// ---------------------------------------------------------------- host side
namespace tma {

// 2-D fp32 tensor map over X[outer][inner] (row pitch ld elements), box
// {box_inner, box_outer}, out-of-bounds reads as zero.  K-major tiles use
// SWIZZLE_128B, MN-major tiles SWIZZLE_128B_ATOM_32B (see desc()).
inline bool make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, uint32_t box_inner,
                     uint32_t box_outer, bool base32, bool f16 = false) {
  struct Key {
    const void* p;
    int64_t a, b, c;
    uint32_t d, e;
    bool f, h;
    bool operator==(const Key& o) const {
      return p == o.p && a == o.a && b == o.b && c == o.c && d == o.d && e == o.e && f == o.f && h == o.h;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      size_t h = std::hash<const void*>()(k.p);
      for (int64_t v : {k.a, k.b, k.c, (int64_t)k.d, (int64_t)k.e, (int64_t)k.f, (int64_t)k.h})
        h = h * 1000003u ^ std::hash<int64_t>()(v);
      return h;
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key key{ptr, inner, outer, ld, box_inner, box_outer, base32, f16};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return true;
  }
  EncodeFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (f16 ? 2u : 4u)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   base32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 4096) cache.clear();
  cache[key] = *map;
  return true;
}

// operand X of logical shape R x K: MN-major (X[k*ld + r]) or K-major (X[r*ld + k])
inline bool operand_map(CUtensorMap* map, const float* X, bool mn_major, int64_t R, int64_t K, int64_t ld) {
  if (reinterpret_cast<uintptr_t>(X) % 16 || (ld * 4) % 16) return false;
  return mn_major ? make_map(map, X, R, K, ld, 32, 32, true) : make_map(map, X, K, R, ld, 32, 128, false);
}

// 3xFP16 operand image (K-major R x K halfs, pitch ld): 128 rows x 64 halfs
// (128-byte rows, SWIZZLE_128B) -- byte-identical shared-memory layout to
// the fp32 K-major tile, so the same UMMA descriptors apply.
inline bool operand_map_f16(CUtensorMap* map, const void* X, int64_t R, int64_t K, int64_t ld) {
  if (reinterpret_cast<uintptr_t>(X) % 16 || (ld * 2) % 16) return false;
  return make_map(map, X, K, R, ld, 64, 128, false, true);
}

}  // namespace tma

// True when the TMA path can serve these operands (16-byte aligned bases and
// pitches); otherwise launch_tc_gemm's packed path is used.
struct TmaProbe {
  uint32_t lbo = 4096, sbo = 512, kstep = 1024;
  int idesc_override = -1;
};
inline TmaProbe& tma_probe() {
  static TmaProbe p;
  return p;
}

}  // namespace pf

#include "tc_splitk.cuh"  // small products: split-K in a cluster (needs the map helpers above)
#include "tc_f16.cuh"     // 3xFP16 operand images
#include "tc_sk2.cuh"     // stream-K pair kernel for plain 3xFP16 products

namespace pf {

// CTA-pair (256x256) tiles for products with at least one full pair tile;
// PF_TC_PAIR=0 in the environment forces the single-CTA kernel (A/B runs).
inline bool tc_pair_ok(int64_t m, int64_t n) {
  static const bool enabled = [] {
    const char* e = std::getenv("PF_TC_PAIR");
    return !(e && e[0] == '0');
  }();
  return enabled && m >= 256 && n >= 256;
}

// split-K factor: fill ~148 SMs when the output has too few (active) tiles;
// upper: only tiles on or above the block diagonal run (CORR/COVAR Gram)
inline int tc_tma_splits(int64_t m, int64_t n, int kblocks, bool pair, bool upper = false) {
  const int64_t bm = pair ? (m + 255) / 256 : (m + 127) / 128, bn = pair ? (n + 255) / 256 : (n + 127) / 128;
  int64_t tiles = bm * bn;
  if (upper) {
    tiles = 0;
    for (int64_t i = 0; i < bm; ++i) tiles += std::max<int64_t>(0, bn - i);
  }
  const int64_t ctas = pair ? 2 * tiles : tiles;
  static const int cap = [] {  // PF_TC_SPLITS=<n>: cap the split factor (A/B runs)
    const char* e = std::getenv("PF_TC_SPLITS");
    return e ? std::max(1, std::atoi(e)) : 1 << 30;
  }();
  int splits = 1;
  if (2 * ctas < device_sms()) splits = (int)std::max<int64_t>(1, std::min<int64_t>(device_sms() / ctas, kblocks / 2));
  splits = std::min(splits, cap);
  const int per = (kblocks + splits - 1) / splits;
  return (kblocks + per - 1) / per;
}

// Stream-K for plain 3xFP16 products (beta = 0, not symmetric, no split-K)
// whose pair tiles do not divide evenly over the SM pairs.  PF_TC_SK2=0
// keeps one tile per pair.
inline bool tc_sk2_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PF_TC_SK2");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline bool tc_sk2_wanted(int64_t m, int64_t n, int64_t k, bool dual, bool upper, bool sym, float beta) {
  if (!tc_sk2_enabled() || dual || upper || sym || beta != 0.f || m < 256 || n < 256) return false;
  const int64_t kb = (k + 63) / 64, tiles = ((m + 255) / 256) * ((n + 255) / 256);
  const int64_t pairs = std::max(1, device_sms() / 2);
  if (kb < 8) return false;
  // several waves with a partial last one (4096^2: 256 tiles on 74 pairs, 3.46
  // waves: 765 -> 710 us for 2MM).  A single partial wave (2048^2: 64 tiles) is
  // left alone: the product runs at the power-capped tensor rate there and
  // spreading it over all 74 pairs measured no faster (46.5 vs 47 us).
  return tiles > pairs && tiles % pairs != 0;
}

template <BenchId Bn, int V>
inline bool launch_tc_tma(const TcGemmArgs& a, cudaStream_t s, bool* dlo_written = nullptr) {
  if (dlo_written) *dlo_written = false;
  // small single products: split-K inside a cluster, DSMEM reduction (one launch)
  if (!a.f16 && !a.sym && !a.upper_only && !a.A2 && launch_tc_splitk<Bn, V>(a, s)) return true;
  TmaParams p;
  std::memset(&p, 0, sizeof(p));
  p.mn_lbo = tma_probe().lbo;
  p.mn_sbo = tma_probe().sbo;
  p.mn_kstep = tma_probe().kstep;
  p.idesc_override = tma_probe().idesc_override;
  static const int diag = [] {
    const char* e = std::getenv("PF_TC_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  p.diag = diag;
  if (a.f16) {
    // 3xFP16: K-major fp16 hi / lo images for every operand (tc_f16.cuh)
    const F16Operands& f = *a.f16;
    p.f16 = 1;
    p.f16_rinv = f.rinv;
    p.f16_cinv = f.cinv;
    p.presplit = 1;
    if (!tma::operand_map_f16(&p.ta, f.hi[0], a.M, a.K, f.kp) || !tma::operand_map_f16(&p.tal, f.lo[0], a.M, a.K, f.kp) ||
        !tma::operand_map_f16(&p.tb, f.hi[1], a.N, a.K, f.kp) || !tma::operand_map_f16(&p.tbl, f.lo[1], a.N, a.K, f.kp))
      return false;
    if (a.A2) {
      if (!tma::operand_map_f16(&p.ta2, f.hi[2], a.M, a.K, f.kp) ||
          !tma::operand_map_f16(&p.ta2l, f.lo[2], a.M, a.K, f.kp) ||
          !tma::operand_map_f16(&p.tb2, f.hi[3], a.N, a.K, f.kp) || !tma::operand_map_f16(&p.tb2l, f.lo[3], a.N, a.K, f.kp))
        return false;
    } else {
      p.ta2 = p.ta;
      p.tb2 = p.tb;
      p.ta2l = p.tal;
      p.tb2l = p.tbl;
    }
  } else {
  p.a_mn = a.ta ? 1 : 0;
  p.b_mn = a.tb ? 0 : 1;
  if (!tma::operand_map(&p.ta, a.A, p.a_mn, a.M, a.K, a.lda)) return false;
  if (!tma::operand_map(&p.tb, a.B, p.b_mn, a.N, a.K, a.ldb)) return false;
  if (a.A2) {
    if (!tma::operand_map(&p.ta2, a.A2, p.a_mn, a.M, a.K, a.lda)) return false;
    if (!tma::operand_map(&p.tb2, a.B2, p.b_mn, a.N, a.K, a.ldb)) return false;
  } else {
    p.ta2 = p.ta;
    p.tb2 = p.tb;
  }
  p.presplit = a.Alo && a.Blo && (!a.A2 || (a.A2lo && a.B2lo)) &&
               tma::operand_map(&p.tal, a.Alo, p.a_mn, a.M, a.K, a.lda) &&
               tma::operand_map(&p.tbl, a.Blo, p.b_mn, a.N, a.K, a.ldb) &&
               (!a.A2 || (tma::operand_map(&p.ta2l, a.A2lo, p.a_mn, a.M, a.K, a.lda) &&
                          tma::operand_map(&p.tb2l, a.B2lo, p.b_mn, a.N, a.K, a.ldb)));
  if (p.presplit && !a.A2) {
    p.ta2l = p.tal;
    p.tb2l = p.tbl;
  }
  }
  // TMA epilogue when D (and Cin, if read) are 16-byte aligned with 16-byte pitches
  p.tma_epi = (reinterpret_cast<uintptr_t>(a.D) % 16 == 0 && (a.ldd * 4) % 16 == 0 &&
               tma::make_map(&p.td, a.D, a.N, a.M, a.ldd, 32, 32, false))
                  ? 1
                  : 0;
  if (p.tma_epi && a.beta != 0.f)
    p.tma_epi = (a.Cin && reinterpret_cast<uintptr_t>(a.Cin) % 16 == 0 && (a.ldc * 4) % 16 == 0 &&
                 tma::make_map(&p.tc, a.Cin, a.N, a.M, a.ldc, 32, 32, false))
                    ? 1
                    : 0;
  if (a.f16 && !p.tma_epi) return false;  // the row-scale epilogue is the TMA one
  const int kb1 = a.f16 ? (a.K + 63) / 64 : (a.K + 31) / 32;  // 128-byte k blocks
  const int kblocks = a.A2 ? 2 * kb1 : kb1;
  // split-K problems: beta pre-pass + TMA add-reductions, or the ordered
  // hand-over for beta = 0.  (Reducing the partials inside a z-cluster through
  // DSMEM was measured slower on B200 -- 24.5 vs 15.3 us for GEMM 512^3 -- and
  // removed.)
  // symmetric products compute the upper tiles and mirror the rest (needs the
  // TMA epilogue; otherwise the full product is computed)
  p.sym = (a.sym && p.tma_epi && a.M == a.N) ? 1 : 0;
  // CTA pairs only for problems that fill the GPU without split-K (GEMM 512^3:
  // 128 single-CTA split-K tiles beat 64 split-K pair halves)
  const bool up = a.upper_only != 0 || p.sym;
  const bool pair = tc_pair_ok(a.M, a.N) && tc_tma_splits(a.M, a.N, kblocks, true, up) <= 2;
  const int zs = tc_tma_splits(a.M, a.N, kblocks, pair, up);
  const int per = (kblocks + zs - 1) / zs;
  p.dlo = (a.Dlo && !a.f16 && p.tma_epi && zs == 1 && !p.sym && reinterpret_cast<uintptr_t>(a.Dlo) % 16 == 0 &&
           tma::make_map(&p.tdl, a.Dlo, a.N, a.M, a.ldd, 32, 32, false))
              ? 1
              : 0;
  if (dlo_written) *dlo_written = p.dlo != 0;
  const int64_t grid_tiles = pair ? 2 * cdiv(a.N, 256) * (int64_t)cdiv(a.M, 256) : (int64_t)cdiv(a.N, 128) * cdiv(a.M, 128);
  // ordered hand-over only where the alternative pre-pass is a memset (beta
  // == 0): with beta != 0 split 0's Cin load + store serialise the splits
  // (GEMM 512^3: 17.4 us vs 15.3 us with the beta pre-pass)
  const bool zeroed = a.d_base && p.tma_epi && (p.sym || zs > 1);  // every write is an add-reduction
  const bool ordered = zs > 1 && !zeroed && !p.sym && p.tma_epi && a.tile_flags && grid_tiles <= kTileFlagsGemm &&
                       a.beta == 0.f;
  const bool prepass = (zs > 1 || p.sym) && !ordered && !zeroed;  // beta * Cin (or zero) before the adds
  p.tile_flags = ordered ? a.tile_flags : nullptr;
  p.epoch = a.epoch;
  if (prepass) {
    if (a.beta == 0.f)
      cudaMemset2DAsync(a.D, (size_t)a.ldd * sizeof(float), 0, (size_t)a.N * sizeof(float), a.M, s);
    else if (a.ldd == a.N && a.ldc == a.N && a.N % 4 == 0 && reinterpret_cast<uintptr_t>(a.D) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(a.Cin) % 16 == 0)
      tc_prescale_flat<Bn, V><<<4 * device_sms(), 256, 0, s>>>(reinterpret_cast<float4*>(a.D),
                                                       reinterpret_cast<const float4*>(a.Cin),
                                                       (int64_t)a.M * a.N / 4, a.beta);
    else
      tc_prescale<Bn, V><<<dim3(cdiv(a.N, 256), a.M), 256, 0, s>>>(a.D, a.ldd, a.Cin, a.ldc, a.M, a.N, a.beta);
  }
  p.kblocks = kblocks;
  p.kb_per_split = per;
  p.kb1 = kb1;
  p.M = a.M;
  p.N = a.N;
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.Cin = a.Cin;
  p.ldc = a.ldc;
  p.D = a.D;
  p.ldd = a.ldd;
  p.upper_only = a.upper_only || p.sym;
  if (a.f16 && a.d_base && pair && zs == 1 && !p.sym && !a.upper_only && !a.A2 && a.beta == 0.f && p.tma_epi &&
      tc_sk2_wanted(a.M, a.N, a.K, false, false, false, a.beta)) {
    const int tn = (int)cdiv(a.N, 256), tiles = tn * (int)cdiv(a.M, 256);
    p.sk_tiles = tiles;
    p.sk_tiles_n = tn;
    p.sk_pairs = (int)std::min<int64_t>(std::max(1, device_sms() / 2), (int64_t)tiles * kblocks);
    set_smem_attr((const void*)tc_tma2_sk_kernel<Bn, V>, (int)kSk2Smem);
    tc_tma2_sk_kernel<Bn, V><<<2 * p.sk_pairs, kTmaThreads, kSk2Smem, s>>>(p);
    if (cudaGetLastError() != cudaSuccess) launch_failed("tcgen05 stream-K contraction launch rejected");
    return true;
  }
  set_smem_attr((const void*)tc_tma_kernel<Bn, V>, (int)kTmaSmem);
  set_smem_attr((const void*)tc_tma2_kernel<Bn, V>, (int)kTmaSmem);
  {
    // after a beta pre-pass the GEMM is a programmatic dependent launch: its
    // prologue and mainloop overlap the pre-pass (griddepcontrol.wait gates
    // only the epilogue's add-reductions)
    const bool pdl = prepass;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = pair ? dim3(2 * cdiv(a.N, 256), cdiv(a.M, 256), zs) : dim3(cdiv(a.N, 128), cdiv(a.M, 128), zs);
    cfg.blockDim = dim3(kTmaThreads);
    cfg.dynamicSmemBytes = kTmaSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, tc_tma2_kernel<Bn, V>, p)
                               : cudaLaunchKernelEx(&cfg, tc_tma_kernel<Bn, V>, p);
    if (e != cudaSuccess) launch_failed("tcgen05 contraction launch rejected");
  }
  return true;
}

// launches of one TMA-path product: [prescale] + gemm
inline int64_t tc_tma_launches(int64_t m, int64_t n, int64_t k, bool dual = false, bool upper = false,
                               bool beta_zero = false) {
  if (tc_splitk_factor(m, n, k, dual, upper)) return 1;  // cluster split-K kernel
  const int kblocks = (int)((dual ? 2 : 1) * ((k + 31) / 32));
  const bool pair = tc_pair_ok(m, n) && tc_tma_splits(m, n, kblocks, true, upper) <= 2;
  const bool split = tc_tma_splits(m, n, kblocks, pair, upper) > 1;
  return split && !beta_zero ? 2 : 1;  // beta pre-pass, or the in-kernel ordered hand-over
}

}  // namespace pf

namespace pf {

// Dims-level predicate matching launch_tc_tma's pointer checks (cudaMalloc
// bases are 256-byte aligned): pitches and base offsets multiples of 4 floats.
inline bool tma_ok(int64_t lda, int64_t ldb, int64_t offset_elems = 0) {
  return lda % 4 == 0 && ldb % 4 == 0 && offset_elems % 4 == 0;
}

inline int64_t tc_launches(int64_t m, int64_t n, int64_t k, bool tma, bool dual = false, int operands = 2);

// One tensor-core contraction: TMA-fed raw-operand kernel when possible,
// otherwise the packed-operand kernel (tc_gemm.cuh).
// lo = x - trunc_tf32(x) over n floats (operand storage, pitch included)
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) tc_split_lo(const float* __restrict__ x, float* __restrict__ lo, int64_t n) {
  const int64_t n4 = n / 4, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {  // four 16-byte loads in flight per thread
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(x) + i + u * stride);  // the GEMM re-reads x from L2
#pragma unroll
    for (int u = 0; u < 4; ++u)
      reinterpret_cast<float4*>(lo)[i + u * stride] =
          make_float4(v[u].x - tma::trunc_tf32(v[u].x), v[u].y - tma::trunc_tf32(v[u].y),
                      v[u].z - tma::trunc_tf32(v[u].z), v[u].w - tma::trunc_tf32(v[u].w));
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
    reinterpret_cast<float4*>(lo)[i] = make_float4(v.x - tma::trunc_tf32(v.x), v.y - tma::trunc_tf32(v.y),
                                                   v.z - tma::trunc_tf32(v.z), v.w - tma::trunc_tf32(v.w));
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lo[i] = x[i] - tma::trunc_tf32(x[i]);
}

// Pre-split operands: one pass over global memory writes lo = x - trunc(x)
// next to each operand and the kernel TMA-loads both halves, so the converter
// warps' shared-memory round trip (64 KB per k block) and their proxy-fence
// hand-off leave the mainloop (2MM/3MM 2048: -11%, SYRK/SYR2K: -17-19% on
// B200).  Used when the product runs without split-K (a split-K product is
// latency-bound and the extra pass costs more than it saves: GEMM 512^3).
// PF_TC_PRESPLIT=0 / =1 force it off / on (A/B runs).
inline bool tc_presplit_wanted(int64_t m, int64_t n, int64_t k, bool dual, bool upper) {
  static const int mode = [] {
    const char* v = std::getenv("PF_TC_PRESPLIT");
    return v ? std::atoi(v) : -1;
  }();
  if (mode >= 0) return mode == 1;
  const int kblocks = (int)((dual ? 2 : 1) * ((k + 31) / 32));
  const bool pair = tc_pair_ok(m, n) && tc_tma_splits(m, n, kblocks, true, upper) <= 2;
  return tc_tma_splits(m, n, kblocks, pair, upper) == 1;
}

// 3xFP16 for the products that run pre-split (large enough for CTA pairs
// or symmetric), when the fp16 images fit the 16-byte TMA pitch rules
inline bool tc_f16_wanted(int64_t m, int64_t n, int64_t k, bool dual, bool upper, bool sym) {
  return tc_f16_enabled() && m >= 256 && n >= 256 && (sym || tc_presplit_wanted(m, n, k, dual, upper));
}
inline bool tc_f16_wanted(const TcGemmArgs& a) {
  return tc_f16_wanted(a.M, a.N, a.K, a.A2 != nullptr, a.upper_only != 0, a.sym != 0);
}

// launches of a 3xFP16 contraction: split [+ transposing split of an MN-major
// op(B), as in 2MM / 3MM] + [beta pre-pass] + gemm; symmetric products
// (K-major operands only): split + beta pre-pass + gemm
inline int64_t tc_f16_launches(int64_t m, int64_t n, int64_t k, bool dual, bool sym, bool beta_zero = false) {
  if (sym) return 2;  // split (+ the beta pre-pass in the same launch) + gemm
  const int kblocks = (int)((dual ? 2 : 1) * ((k + 63) / 64));
  const bool pair = tc_pair_ok(m, n) && tc_tma_splits(m, n, kblocks, true, false) <= 2;
  const bool split = tc_tma_splits(m, n, kblocks, pair, false) > 1;
  return 2 + 1 + (split && !beta_zero ? 1 : 0);  // [K-major rows, MN strips | rows + column maxima, tiles]
}

// launches of one contraction: [lo passes, one per distinct operand array] +
// [prescale] + gemm (TMA path), the 3xFP16 sequence, or the packed path's
inline int64_t tc_launches(int64_t m, int64_t n, int64_t k, bool tma, bool dual, int operands) {
  if (!tma) return tc_gemm_launches(m, n, k, dual);
  if (tc_f16_wanted(m, n, k, dual, false, false)) return tc_f16_launches(m, n, k, dual, false);
  return tc_tma_launches(m, n, k, dual) + (tc_presplit_wanted(m, n, k, dual, false) ? operands : 0);
}

// Returns true when the epilogue also wrote a0.Dlo (the lo image of D) for a
// later product; operand lo images passed in a0 (Alo, Blo, ...) are used as
// given and not recomputed.
template <BenchId Bn, int V>
inline bool launch_contraction(Workspace& ws, const TcGemmArgs& a0, cudaStream_t s) {
  TcGemmArgs a = a0;
  a.tile_flags = ws.ensure_tile_flags(s);
  a.epoch = ++ws.tile_epoch;
  bool dlo = false;
  // 3xFP16 operand images for the products that would run pre-split
  if (tc_f16_wanted(a)) {
    F16Operands f;
    // symmetric products (beta pre-pass + add-reductions): the pre-pass rides
    // in the operand-split launch when D and Cin are flat, aligned and identical in shape
    const bool flat_d = a.ldd == a.N && a.N % 4 == 0 && reinterpret_cast<uintptr_t>(a.D) % 16 == 0;
    const bool base_d = (a.sym && a.Cin && flat_d && a.ldc == a.N && reinterpret_cast<uintptr_t>(a.Cin) % 16 == 0) ||
                        // stream-K adds every partial tile onto D: zeros written by the split launch
                        (flat_d && tc_sk2_wanted(a.M, a.N, a.K, a.A2 != nullptr, a.upper_only != 0, a.sym != 0, a.beta));
    if (prepare_f16<Bn, V>(ws, a, f, s, base_d)) {
      TcGemmArgs b = a;
      b.f16 = &f;
      b.d_base = base_d ? 1 : 0;
      b.Alo = b.Blo = b.A2lo = b.B2lo = nullptr;
      b.Dlo = nullptr;
      if (launch_tc_tma<Bn, V>(b, s)) return false;
    }
  }
  // symmetric products split-K their upper tiles but still profit from the
  // pre-split operands (SYRK: one lo pass serves both operands)
  if ((a.sym || tc_presplit_wanted(a.M, a.N, a.K, a.A2 != nullptr, a.upper_only != 0)) && tma_ok(a.lda, a.ldb)) {
    // distinct operand arrays without a given lo image, and their storage extents (floats)
    const float* ops[4] = {a.A, a.B, a.A2, a.B2};
    const float* given[4] = {a.Alo, a.Blo, a.A2lo, a.B2lo};
    const int64_t ext_a = a.ta ? (int64_t)(a.K - 1) * a.lda + a.M : (int64_t)(a.M - 1) * a.lda + a.K;
    const int64_t ext_b = a.tb ? (int64_t)(a.N - 1) * a.ldb + a.K : (int64_t)(a.K - 1) * a.ldb + a.N;
    const int64_t e[4] = {ext_a, ext_b, a.A2 ? ext_a : 0, a.B2 ? ext_b : 0};
    int64_t off[4], total = 0;
    for (int i = 0; i < 4; ++i) {
      off[i] = -1;
      if (!ops[i] || given[i]) continue;
      for (int j = 0; j < i; ++j)
        if (!given[j] && ops[j] == ops[i] && e[j] == e[i]) off[i] = off[j];
      if (off[i] < 0) {
        off[i] = total;
        total += (e[i] + 63) / 64 * 64;  // 256-byte aligned images
      }
    }
    float* lo = total ? ws.ensure_scratch((size_t)total * sizeof(float)) : nullptr;
    if (lo || !total) {
      bool done[4] = {false, false, false, false};
      for (int i = 0; i < 4; ++i) {
        if (!ops[i] || given[i] || done[i]) continue;
        for (int j = i; j < 4; ++j)
          if (!given[j] && ops[j] == ops[i] && off[j] == off[i]) done[j] = true;
        tc_split_lo<Bn, V><<<4 * device_sms(), 256, 0, s>>>(ops[i], lo + off[i], e[i]);
      }
      TcGemmArgs b = a;
      for (int i = 0; i < 4; ++i) {
        const float* l = given[i] ? given[i] : (ops[i] ? lo + off[i] : nullptr);
        (i == 0 ? b.Alo : i == 1 ? b.Blo : i == 2 ? b.A2lo : b.B2lo) = l;
      }
      if (launch_tc_tma<Bn, V>(b, s, &dlo)) return dlo;
    }
  }
  a.Alo = a.Blo = a.A2lo = a.B2lo = nullptr;  // converter warps split in-kernel
  if (launch_tc_tma<Bn, V>(a, s, &dlo)) return dlo;
  launch_tc_gemm<Bn, V>(ws, a, s);
  return false;
}

}  // namespace pf
