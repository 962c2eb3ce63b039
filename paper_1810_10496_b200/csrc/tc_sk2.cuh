// Stream-K CTA-pair kernel for plain 3xFP16 products (D = alpha op(A) op(B),
// beta = 0, D pre-zeroed): included by tc_tma.cuh after its helpers.
//
// Why: a 4096^2 product has 256 pair tiles of 64 k blocks for 74 SM pairs:
// one tile per pair and wave takes 4 waves, the last one half empty.  Here
// the 256 x 64 (tile, k block) units are cut into 74 contiguous ranges, one
// per pair (221.4 units each), so every pair does the same MMA work (2MM
// 4096: 765 -> 710 us).  A range
// covers at most two or three tile segments; each segment accumulates in its
// own TMEM buffer (2 x 256 columns, double-buffered) and its epilogue --
// 4 warps per CTA, one 4 KB staging slot each -- adds it onto D with TMA
// add-reductions while the MMAs of the next segment run.  D starts at zero
// (written by the operand-split launch), so the partial tiles of adjacent
// ranges need no ordering.  (At 2048^2 -- 64 tiles, one partial wave -- the
// same balancing measured no faster: the product runs at the power-capped
// tensor rate, so it is not used there.)
//
// Roles per CTA (192 threads): warp 0 lane 0 TMA producer (both CTAs' bytes
// on the leader's full[s]); leader warp 1 lane 0 MMA issuer (waits tfree[b]
// before reusing TMEM buffer b); warps 2..5 epilogue (rows 32 (w % 4)).
#pragma once

namespace pf {

constexpr uint32_t kSk2EpiSlot = 4096;                         // 32 x 32 fp32 chunk per epilogue warp
constexpr uint32_t kSk2Smem = kTmaStages * kTmaStageBytes + 4 * kSk2EpiSlot + 1024;

namespace sk2 {

struct Range {
  int64_t u0, u1;
};

__device__ __forceinline__ Range range_of(const TmaParams& p, int pair) {
  const int64_t W = (int64_t)p.sk_tiles * p.kblocks;
  return Range{W * pair / p.sk_pairs, W * (pair + 1) / p.sk_pairs};
}

}  // namespace sk2

template <BenchId Bn, int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTmaThreads, 1)
    tc_tma2_sk_kernel(const __grid_constant__ TmaParams p) {
  extern __shared__ uint8_t tma_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kTmaStages], empty_bar[kTmaStages], accum_bar[2], tfree_bar[2];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float epi_cs[4][256];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tma_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + kTmaStages * kTmaStageBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc2::cluster_rank();
  const int pair = blockIdx.x >> 1;
  const sk2::Range rg = sk2::range_of(p, pair);
  const int kb = p.kblocks, tn = p.sk_tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tc::smem_u32(&accum_bar[b]), 1);
      tc::mbar_init(tc::smem_u32(&tfree_bar[b]), 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma::prefetch_map(&p.ta);
    tma::prefetch_map(&p.tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before();
  tc2::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int64_t u = rg.u0; u < rg.u1; ++u) {
        const int i = (int)(u - rg.u0), s = i % kTmaStages;
        const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
        const int tile = (int)(u / kb), k0 = (int)(u % kb) * 64;
        const int m0 = (tile / tn) * 256 + (int)rank * 128, nB = (tile % tn) * 256 + (int)rank * 128;
        tc2::wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
        const uint32_t fb = tc::smem_u32(&full_bar[s]);
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
        const uint32_t lb = tc2::peer_addr(fb, 0);
        if (rank == 0) tc::mbar_expect_tx(fb, 2 * 4 * kTmaTileBytes);
        tma::load_operands(p, false, false, base, m0, nB, k0, lb, true);
        tma::load_operands(p, false, true, base + 2 * kTmaTileBytes, m0, nB, k0, lb, true);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t id = tma::idesc(256, 256, 0, 0, true);
      int seg = 0;
      for (int64_t u = rg.u0; u < rg.u1; ++u) {
        const int i = (int)(u - rg.u0), s = i % kTmaStages;
        const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
        const bool first = u == rg.u0 || u % kb == 0;
        const bool last = u + 1 == rg.u1 || (u + 1) % kb == 0;
        const int b = seg & 1;
        if (first && seg >= 2) {  // TMEM buffer b: its previous segment's epilogue has read it out
          tc2::wait(tc::smem_u32(&tfree_bar[b]), (uint32_t)((seg >> 1) - 1) & 1u);
          tc::fence_after();
        }
        tc2::wait(tc::smem_u32(&full_bar[s]), ph);
        tc::fence_after();
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kTmaStageBytes);
        const uint32_t acc = tmem + (uint32_t)(b * 256);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ahi = tma::desc(base + kk * 32u, false);
          const uint64_t bhi = tma::desc(base + kTmaTileBytes + kk * 32u, false);
          const uint64_t alo = tma::desc(base + 2 * kTmaTileBytes + kk * 32u, false);
          const uint64_t blo = tma::desc(base + 3 * kTmaTileBytes + kk * 32u, false);
          tc2::mma_f16(acc, alo, bhi, id, (first && kk == 0) ? 0u : 1u);
          tc2::mma_f16(acc, ahi, blo, id, 1u);
          tc2::mma_f16(acc, ahi, bhi, id, 1u);
        }
        tc2::commit_both(tc::smem_u32(&empty_bar[s]));
        if (last) {
          tc2::commit_both(tc::smem_u32(&accum_bar[b]));
          ++seg;
        }
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: segment by segment, TMEM buffer seg % 2 -> add-reductions onto D
    const int quad = warp & 3;
    uint8_t* slot = epi + (size_t)quad * kSk2EpiSlot;
    const uint32_t sslot = tc::smem_u32(slot);
    const uint32_t leader_free0 = tc2::peer_addr(tc::smem_u32(&tfree_bar[0]), 0);
    const uint32_t leader_free1 = tc2::peer_addr(tc::smem_u32(&tfree_bar[1]), 0);
    int seg = 0;
    for (int64_t u = rg.u0; u < rg.u1; ++seg) {
      const int tile = (int)(u / kb);
      const int64_t uend = min(rg.u1, (int64_t)(tile + 1) * kb);
      u = uend;
      const int b = seg & 1;
      const int row0 = (tile / tn) * 256 + (int)rank * 128 + quad * 32, col0 = (tile % tn) * 256;
      const float ar = tma::stage_f16_scales(p, row0 + lane, col0, 256, epi_cs[quad], lane);
      tc2::wait(tc::smem_u32(&accum_bar[b]), (uint32_t)(seg >> 1) & 1u);
      tc::fence_after();
      if (row0 < p.M) {
        const int nch = min(8, (p.N - col0 + 31) / 32);
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * 256);
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          uint32_t r[32];
          tc::tmem_ld32(taddr + (uint32_t)(c * 32), r);
          if (c > 0) {  // the slot's previous chunk has been read by its add-reduction
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
          }
          float4* rowp = reinterpret_cast<float4*>(slot + lane * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 cs = *reinterpret_cast<const float4*>(epi_cs[quad] + c * 32 + 4 * j);
            rowp[j ^ (lane & 7)] =
                make_float4(ar * __uint_as_float(r[4 * j]) * cs.x, ar * __uint_as_float(r[4 * j + 1]) * cs.y,
                            ar * __uint_as_float(r[4 * j + 2]) * cs.z, ar * __uint_as_float(r[4 * j + 3]) * cs.w);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma::reduce_add_2d(&p.td, sslot, col0 + c * 32, row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      // this warp has read its rows of buffer b: let the leader reuse it
      tc::fence_before();
      if (lane == 0) tc2::arrive_remote(b ? leader_free1 : leader_free0);
      __syncwarp();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the add-reductions are done
    __syncwarp();
  }
  tc::fence_before();
  tc2::cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
  }
}

}  // namespace pf
