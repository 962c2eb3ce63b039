// Small contractions (too few output tiles to fill the GPU): split-K inside a
// thread-block cluster, partial sums exchanged through distributed shared
// memory.  Included by tc_tma.cuh after its host-side tensor-map helpers.
//
//   D = alpha * op(A) op(B) + beta * Cin,  one launch, no pre-pass, no atomics
//
// Grid (N/64, M/128, S), cluster (1, 1, S), S in {2, 4}: the S CTAs of a
// cluster share one 128 x 64 output tile and CTA r accumulates k blocks
// [r * per, (r + 1) * per) in TMEM (3xTF32, same operand handling as
// tc_tma_kernel: TMA-loaded raw fp32 tiles are the hi part, four converter
// warps write lo = x - trunc_tf32(x) next to them).  After the MMAs each CTA
// dumps its 128 x 64 partial into its own (idle) operand ring, one cluster
// barrier, and CTA r then owns rows [r * 128 / S, (r + 1) * 128 / S): it
// loads that slice from all S partials (DSMEM, every load in flight at once),
// sums in split order, applies alpha and beta * Cin (Cin prefetched into
// registers at kernel start) and writes D with coalesced 16-byte stores.  A
// relaxed cluster barrier keeps the partials alive until their readers are
// done.  (Pushing rows to their owners with st.async + mbarrier transaction
// counts instead measured slower: 2.4 vs ~1.8 us from accumulator to stores
// for GEMM 512^3 -- DSMEM runs at ~17 B/clk per SM either way.)
// Why: the 128 x 128 split-K 8 form of GEMM 512^3 spent its time on a beta
// pre-pass launch and 8 MB of TMA add-reductions into 1 MB of output (ncu:
// tensor pipe 0.4% active, barrier 30% of stalls); here the cross-split
// traffic is 24 KB of DSMEM stores per CTA.
#pragma once

namespace pf {

constexpr int kSkBN = 64;
constexpr int kSkStages = 4;
constexpr uint32_t kSkATile = 128 * 32 * 4;                   // A: 128 rows x 32 k
constexpr uint32_t kSkBTile = kSkBN * 32 * 4;                  // B: 64 cols x 32 k
constexpr uint32_t kSkStageBytes = 2 * (kSkATile + kSkBTile);  // raw A, raw B, lo A, lo B
constexpr uint32_t kSkSmem = kSkStages * kSkStageBytes + 1024;  // the partial reuses stage 0
constexpr int kSkThreads = 192;

struct SkParams {
  CUtensorMap ta, tb;
  int a_mn, b_mn;
  int kblocks, kb_per_split;
  int M, N;
  float alpha, beta;
  const float* Cin;
  int ldc;
  float* D;
  int ldd;
  uint32_t mn_lbo, mn_sbo, mn_kstep;
  int trace;  // PF_SK_TRACE=1: %globaltimer timeline per CTA into D (diagnostics; wrong results)
};

namespace sk {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// generic address of the same shared-memory location in cluster CTA `peer`
__device__ __forceinline__ const float4* peer_ptr(const void* local, uint32_t peer) {
  uint64_t remote;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(remote) : "l"(reinterpret_cast<uint64_t>(local)), "r"(peer));
  return reinterpret_cast<const float4*>(remote);
}

// byte offset of float4 chunk ch (0..15) of partial row `row` (256-byte rows;
// the XOR makes the TMEM dump and the slice reads conflict-free)
__device__ __forceinline__ uint32_t row_off(int row, int ch) {
  return (uint32_t)(row * 256 + ((ch ^ (row & 7)) << 4));
}

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace sk

template <BenchId Bn, int V, int S>
__global__ void __launch_bounds__(kSkThreads, 1) tc_splitk_kernel(const __grid_constant__ SkParams p) {
  extern __shared__ uint8_t sk_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kSkStages], ready_bar[kSkStages], empty_bar[kSkStages], accum_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ uint64_t trace_t[16];  // 0-8 phases, 9-12 stage landed, 13-15 stage converted
  constexpr int R = 128 / S;         // output rows this CTA finishes
  constexpr int NQ = R * 16 / 128;   // float4 chunks per epilogue thread
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sk_smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * kSkBN;
  const int r = (int)sk::cluster_rank();
  const int kb0 = r * p.kb_per_split;
  const int nkb = max(0, min(p.kblocks - kb0, p.kb_per_split));
  if (p.trace && threadIdx.x == 0) trace_t[0] = sk::gtime();

  // TMA producer (thread 0): barriers, then the first ring's loads right away
  // -- the tensor-map fetch and the operand latency overlap the TMEM
  // allocation and the setup barrier
  auto issue = [&](int i) {
    const int s = i % kSkStages;
    const uint32_t fb = tc::smem_u32(&full_bar[s]);
    tc::mbar_expect_tx(fb, kSkATile + kSkBTile);
    const int k0 = (kb0 + i) * 32;
    const uint32_t base = tc::smem_u32(smem + (size_t)s * kSkStageBytes);
    if (p.a_mn) {
#pragma unroll
      for (int j = 0; j < 4; ++j) tma::load_2d(base + j * 4096, &p.ta, m0 + 32 * j, k0, fb);
    } else {
      tma::load_2d(base, &p.ta, k0, m0, fb);
    }
    if (p.b_mn) {
#pragma unroll
      for (int j = 0; j < kSkBN / 32; ++j) tma::load_2d(base + kSkATile + j * 4096, &p.tb, n0 + 32 * j, k0, fb);
    } else {
      tma::load_2d(base + kSkATile, &p.tb, k0, n0, fb);
    }
  };
  if (threadIdx.x == 0) {
    tma::prefetch_map(&p.ta);
    tma::prefetch_map(&p.tb);
    for (int s = 0; s < kSkStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&ready_bar[s]), 4);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(&accum_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = 0; i < min(nkb, kSkStages); ++i) issue(i);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)),
                 "r"((uint32_t)kSkBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;
  if (p.trace && threadIdx.x == 0) trace_t[1] = sk::gtime();

  // epilogue threads (warps 2..5): chunk q = et + 128 j of this CTA's row slice
  const int et = (int)threadIdx.x - 64;
  float4 cin[NQ];
  if (warp >= 2 && p.beta != 0.f) {  // Cin of the slice, in flight while the mainloop runs
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int q = et + 128 * j, row = m0 + r * R + q / 16, col = n0 + 4 * (q % 16);
      cin[j] = (row < p.M && col < p.N) ? __ldg(reinterpret_cast<const float4*>(p.Cin + (size_t)row * p.ldc + col))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }

  if (warp == 0) {
    if (lane == 0) {
      for (int i = kSkStages; i < nkb; ++i) {
        tc::mbar_wait(tc::smem_u32(&empty_bar[i % kSkStages]), ((i / kSkStages) & 1) ^ 1);
        issue(i);
      }
      if (p.trace) trace_t[2] = sk::gtime();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = tma::idesc(128, kSkBN, p.a_mn, p.b_mn);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kSkStages;
        const uint32_t ph = (i / kSkStages) & 1;
        tc::mbar_wait(tc::smem_u32(&ready_bar[s]), ph);
        tc::fence_after();
        const uint32_t base = tc::smem_u32(smem + (size_t)s * kSkStageBytes);
        const uint32_t lo = base + kSkATile + kSkBTile;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ka = p.a_mn ? kk * p.mn_kstep : kk * 32u;
          const uint32_t kb = p.b_mn ? kk * p.mn_kstep : kk * 32u;
          const uint64_t ahi = tma::desc(base + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t bhi = tma::desc(base + kSkATile + kb, p.b_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t alo = tma::desc(lo + ka, p.a_mn, p.mn_lbo, p.mn_sbo);
          const uint64_t blo = tma::desc(lo + kSkATile + kb, p.b_mn, p.mn_lbo, p.mn_sbo);
          tc::mma_tf32(tmem, alo, bhi, id, (i | kk) != 0);
          tc::mma_tf32(tmem, ahi, blo, id, 1u);
          tc::mma_tf32(tmem, ahi, bhi, id, 1u);
        }
        tc::mma_commit(tc::smem_u32(&empty_bar[s]));
      }
      tc::mma_commit(tc::smem_u32(&accum_bar));  // also when nkb == 0: arrives at once
      if (p.trace) trace_t[4] = sk::gtime();
    }
    __syncwarp();
  } else {
    // ---- converters: lo = x - trunc_tf32(x) for the stage's A and B raw tiles
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kSkStages;
      const uint32_t ph = (i / kSkStages) & 1;
      tc::mbar_wait(tc::smem_u32(&full_bar[s]), ph);
      if (p.trace && et == 0) trace_t[i == 0 ? 3 : 9 + min(i, 3)] = sk::gtime();
      const uint32_t raw = tc::smem_u32(smem + (size_t)s * kSkStageBytes);
      const uint32_t lo = raw + kSkATile + kSkBTile;
      tma::split_lo<(int)((kSkATile + kSkBTile) / 16 / 128)>(raw, lo, et);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(tc::smem_u32(&ready_bar[s]));
      if (p.trace && et == 0 && i < 3) trace_t[13 + i] = sk::gtime();
    }
    // ---- partial: TMEM lane = tile row -> own shared memory (the operand
    // ring is idle: accum_bar follows every MMA's completion)
    tc::mbar_wait(tc::smem_u32(&accum_bar), 0);
    tc::fence_after();
    if (p.trace && et == 0) trace_t[5] = sk::gtime();
    const int row = 32 * (warp & 3) + lane;
#pragma unroll 1
    for (int c = 0; c < kSkBN / 32; ++c) {
      uint32_t v[32];
      if (nkb > 0) {
        tc::tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(c * 32), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(smem + sk::row_off(row, 8 * c + j)) =
            make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                        __uint_as_float(v[4 * j + 3]));
    }
  }
  tc::fence_before();
  __syncwarp();
  sk::cluster_sync();  // every partial of the cluster is in shared memory
  if (p.trace && threadIdx.x == 64) trace_t[6] = sk::gtime();
  if (warp >= 2) {
    // CTA r's slice summed over the S partials in split order; all NQ x S
    // remote loads are issued before the first add
    float4 v[NQ][S];
#pragma unroll
    for (int pr = 0; pr < S; ++pr) {
      const float4* peer = sk::peer_ptr(smem, (uint32_t)pr);
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int q = et + 128 * j;
        v[j][pr] = peer[sk::row_off(r * R + q / 16, q % 16) / 16];
      }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int q = et + 128 * j, ch = q % 16;
      const int orow = m0 + r * R + q / 16, col = n0 + 4 * ch;
      float4 acc = v[j][0];
#pragma unroll
      for (int pr = 1; pr < S; ++pr) {
        acc.x += v[j][pr].x;
        acc.y += v[j][pr].y;
        acc.z += v[j][pr].z;
        acc.w += v[j][pr].w;
      }
      float4 d = make_float4(p.alpha * acc.x, p.alpha * acc.y, p.alpha * acc.z, p.alpha * acc.w);
      if (p.beta != 0.f)
        d = make_float4(fmaf(p.beta, cin[j].x, d.x), fmaf(p.beta, cin[j].y, d.y), fmaf(p.beta, cin[j].z, d.z),
                        fmaf(p.beta, cin[j].w, d.w));
      if (orow < p.M && col < p.N) *reinterpret_cast<float4*>(p.D + (size_t)orow * p.ldd + col) = d;
    }
    if (p.trace && et == 0) trace_t[7] = sk::gtime();
  }
  __syncwarp();
  // no CTA leaves while a peer may still read its partial (the loads above
  // have returned their values, so no release is needed: relaxed arrive)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  if (p.trace && threadIdx.x == 0) {
    trace_t[8] = sk::gtime();
    uint32_t* o = reinterpret_cast<uint32_t*>(p.D + (size_t)(m0 + r * R) * p.ldd + n0);
    for (int e = 0; e < 16; ++e) {
      o[2 * e] = (uint32_t)trace_t[e];
      o[2 * e + 1] = (uint32_t)(trace_t[e] >> 32);
    }
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)kSkBN));
}

// Cluster split-K factor for a problem, or 0 when the cluster kernel does not
// apply: single products (no K-concatenation, not symmetric / upper-only)
// whose 128 x 64 tiles leave at least half the GPU idle, N and the output
// pitches multiples of 4 floats.  PF_TC_SK=0 disables it (A/B runs).
inline int tc_splitk_factor(int64_t m, int64_t n, int64_t k, bool dual, bool upper) {
  static const bool enabled = [] {
    const char* e = std::getenv("PF_TC_SK");
    return !(e && e[0] == '0');
  }();
  if (!enabled || dual || upper || n % 4) return 0;
  const int64_t tiles = (int64_t)cdiv(m, 128) * cdiv(n, kSkBN);
  const int64_t kblocks = (k + 31) / 32;
  // one wave of clusters: 4-CTA clusters strand SMs in the 16/18-SM GPCs
  // (<= 132 co-resident CTAs), 8-CTA clusters even more (measured: GEMM 384^3
  // with S = 8 ran its last two clusters as a second wave)
  if (4 * tiles <= 128 && kblocks >= 8) return 4;
  if (2 * tiles <= device_sms() && kblocks >= 4) return 2;
  return 0;
}

template <BenchId Bn, int V>
inline bool launch_tc_splitk(const TcGemmArgs& a, cudaStream_t s) {
  const int S = tc_splitk_factor(a.M, a.N, a.K, a.A2 != nullptr, a.upper_only != 0 || a.sym != 0);
  if (!S) return false;
  if (reinterpret_cast<uintptr_t>(a.D) % 16 || a.ldd % 4) return false;
  if (a.beta != 0.f && (!a.Cin || reinterpret_cast<uintptr_t>(a.Cin) % 16 || a.ldc % 4)) return false;
  SkParams p;
  std::memset(&p, 0, sizeof(p));
  p.a_mn = a.ta ? 1 : 0;
  p.b_mn = a.tb ? 0 : 1;
  if (!tma::operand_map(&p.ta, a.A, p.a_mn, a.M, a.K, a.lda)) return false;
  if (reinterpret_cast<uintptr_t>(a.B) % 16 || ((int64_t)a.ldb * 4) % 16) return false;
  if (!(p.b_mn ? tma::make_map(&p.tb, a.B, a.N, a.K, a.ldb, 32, 32, true)
               : tma::make_map(&p.tb, a.B, a.K, a.N, a.ldb, 32, kSkBN, false)))
    return false;
  p.mn_lbo = tma_probe().lbo;
  p.mn_sbo = tma_probe().sbo;
  p.mn_kstep = tma_probe().kstep;
  p.kblocks = (a.K + 31) / 32;
  p.kb_per_split = (p.kblocks + S - 1) / S;
  p.M = a.M;
  p.N = a.N;
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.Cin = a.Cin;
  p.ldc = a.ldc;
  p.D = a.D;
  p.ldd = a.ldd;
  static const int trace = [] {
    const char* e = std::getenv("PF_SK_TRACE");
    return e ? std::atoi(e) : 0;
  }();
  p.trace = trace;
  auto kern = S == 4 ? tc_splitk_kernel<Bn, V, 4> : tc_splitk_kernel<Bn, V, 2>;
  set_smem_attr((const void*)kern, (int)kSkSmem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cdiv(a.N, kSkBN), cdiv(a.M, 128), S);
  cfg.blockDim = dim3(kSkThreads);
  cfg.dynamicSmemBytes = kSkSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = S;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess)
    launch_failed("tcgen05 cluster split-K launch rejected");
  return true;
}

}  // namespace pf
