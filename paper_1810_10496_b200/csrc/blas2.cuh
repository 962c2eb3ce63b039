// Shared kernels for the memory-bound BLAS-2 set (ATAX, BICG, MVT, GESUMMV).
//
// stage 0  PolyBench/GPU shapes: thread-per-row loops (uncoalesced: a warp
//          touches 32 rows) and thread-per-column loops (coalesced), with the
//          store / unroll / lsr / vec knobs.
// stage 1  warp-per-row dot products (coalesced 512-byte row segments,
//          shuffle reduction) and row-split column products (enough CTAs to
//          fill 148 SMs, partials merged with vector atomics).
// stage 2  one persistent pass over A: every A row is loaded from HBM once
//          into registers and feeds both the row dot product (block
//          reduction) and the column accumulation (register partials,
//          merged once per CTA) -- 4N^2 compulsory bytes instead of 8N^2.
#pragma once
#include "pf_common.cuh"

#include <algorithm>

namespace pf {

// ---------------------------------------------------------------- stage 0
// dst (+)= sum_j A[row*lda + j] * v[j], j in [0, n).  zero: start from 0.
template <int kStore, int kUnroll, int kLsr, int kVec>
__device__ __forceinline__ void s0_row_dot(float* dst, const float* A, int lda, int row, const float* v, int n,
                                           bool zero) {
  Acc<kStore> acc;
  acc.init(dst, zero ? 0.0f : *dst);
  if constexpr (kVec) {
    const float4* a4 = reinterpret_cast<const float4*>(A + (size_t)row * lda);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    PF_UNROLL_IMPL(kUnroll)
    for (int q = 0; q < n / 4; ++q) {
      float4 a = a4[q], b = v4[q];
      acc.add(dst, a.x * b.x);
      acc.add(dst, a.y * b.y);
      acc.add(dst, a.z * b.z);
      acc.add(dst, a.w * b.w);
    }
  } else if constexpr (kLsr) {
    const float* pa = A + (size_t)row * lda;
    const float* pv = v;
    PF_UNROLL_IMPL(kUnroll)
    for (int j = n; j > 0; --j) acc.add(dst, *pa++ * *pv++);
  } else {
    PF_UNROLL_IMPL(kUnroll)
    for (int j = 0; j < n; j++) acc.add(dst, A[row * lda + j] * v[j]);
  }
  acc.finish(dst);
}

// dst[col+e] (+)= sum_i A[i*lda + col+e] * v[i], i in [0, m); e < (kVec ? 4 : 1).
template <int kStore, int kUnroll, int kLsr, int kVec>
__device__ __forceinline__ void s0_col_dot(float* dst, const float* A, int lda, int col, const float* v, int m,
                                           bool zero) {
  constexpr int W = kVec ? 4 : 1;
  Acc<kStore> acc[W];
#pragma unroll
  for (int e = 0; e < W; ++e) acc[e].init(dst + e, zero ? 0.0f : dst[e]);
  if constexpr (kVec) {
    PF_UNROLL_IMPL(kUnroll)
    for (int i = 0; i < m; i++) {
      float4 a = *reinterpret_cast<const float4*>(A + (size_t)i * lda + col);
      float vi = v[i];
      acc[0].add(dst + 0, a.x * vi);
      acc[1].add(dst + 1, a.y * vi);
      acc[2].add(dst + 2, a.z * vi);
      acc[3].add(dst + 3, a.w * vi);
    }
  } else if constexpr (kLsr) {
    const float* pa = A + col;
    const float* pv = v;
    PF_UNROLL_IMPL(kUnroll)
    for (int i = m; i > 0; --i) {
      acc[0].add(dst, *pa * *pv++);
      pa += lda;
    }
  } else {
    PF_UNROLL_IMPL(kUnroll)
    for (int i = 0; i < m; i++) acc[0].add(dst, A[i * lda + col] * v[i]);
  }
#pragma unroll
  for (int e = 0; e < W; ++e) acc[e].finish(dst + e);
}

// ---------------------------------------------------------------- stage 1
// Warp-per-row: out[row] = (init ? init[row] : 0) + sum_j A[row][j] v[j]
template <BenchId Bn, int V, int kUnroll, int kVec>
__global__ void __launch_bounds__(256) s1_row_dot(const float* __restrict__ A, int lda, const float* __restrict__ v,
                                                  int n, int rows, const float* init, float* out) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += warps) {
    const float* a = A + (size_t)row * lda;
    float s = 0.f;
    if constexpr (kVec) {
      const float4* a4 = reinterpret_cast<const float4*>(a);
      const float4* v4 = reinterpret_cast<const float4*>(v);
      PF_UNROLL_IMPL(kUnroll)
      for (int q = lane; q < n / 4; q += 32) {
        float4 x = __ldg(a4 + q), y = __ldg(v4 + q);
        s = fmaf(x.x, y.x, s);
        s = fmaf(x.y, y.y, s);
        s = fmaf(x.z, y.z, s);
        s = fmaf(x.w, y.w, s);
      }
    } else {
      PF_UNROLL_IMPL(kUnroll)
      for (int j = lane; j < n; j += 32) s = fmaf(__ldg(a + j), __ldg(v + j), s);
    }
    s = warp_sum(s);
    if (lane == 0) out[row] = (init ? init[row] : 0.f) + s;
  }
}

// Row-split column product: out[col] += sum_{i in split} A[i][col] v[i]
// (out holds its initial value; partials are added atomically).
template <BenchId Bn, int V, int kUnroll, int kVec>
__global__ void __launch_bounds__(256) s1_col_dot(const float* __restrict__ A, int lda, const float* __restrict__ v,
                                                  int m, int cols, int rows_per_split, float* out) {
  constexpr int W = kVec ? 4 : 1;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * W;
  if (col >= cols) return;
  const int i0 = blockIdx.y * rows_per_split;
  const int i1 = min(m, i0 + rows_per_split);
  float s[W];
#pragma unroll
  for (int e = 0; e < W; ++e) s[e] = 0.f;
  PF_UNROLL_IMPL(kUnroll)
  for (int i = i0; i < i1; ++i) {
    const float vi = __ldg(v + i);
    if constexpr (kVec) {
      float4 a = __ldg(reinterpret_cast<const float4*>(A + (size_t)i * lda + col));
      s[0] = fmaf(a.x, vi, s[0]);
      s[1] = fmaf(a.y, vi, s[1]);
      s[2] = fmaf(a.z, vi, s[2]);
      s[3] = fmaf(a.w, vi, s[3]);
    } else {
      s[0] = fmaf(__ldg(A + (size_t)i * lda + col), vi, s[0]);
    }
  }
  if constexpr (kVec)
    atomicAdd(reinterpret_cast<float4*>(out + col), make_float4(s[0], s[1], s[2], s[3]));
  else
    atomicAdd(out + col, s[0]);
}

template <BenchId Bn, int V, int kUnroll, int kVec>
inline void launch_s1_row_dot(const float* A, int lda, const float* v, int n, int rows, const float* init, float* out,
                              cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(((int64_t)rows + 7) / 8, device_sms() * 16);
  s1_row_dot<Bn, V, kUnroll, kVec><<<blocks, 256, 0, s>>>(A, lda, v, n, rows, init, out);
}

template <BenchId Bn, int V, int kUnroll, int kVec>
inline void launch_s1_col_dot(const float* A, int lda, const float* v, int m, int cols, float* out, cudaStream_t s) {
  constexpr int W = kVec ? 4 : 1;
  const int gx = (int)cdiv(cols, 256 * W);
  int splits = (int)cdiv(device_sms() * 4, gx);
  splits = std::max(1, std::min(splits, (m + 63) / 64));
  const int rps = (int)cdiv(m, splits);
  splits = (int)cdiv(m, rps);
  s1_col_dot<Bn, V, kUnroll, kVec><<<dim3(gx, splits), 256, 0, s>>>(A, lda, v, m, cols, rps, out);
}

// ---------------------------------------------------------------- stage 2
// One pass over A[rows][cols] (cols % 4 == 0), persistent CTAs (one per SM).
// Per row r:
//   dot_r = sum_j A[r][j] * xv[j]                  (if rowout)
//   rowout[r] = (rowinit ? rowinit[r] : 0) + dot_r
//   colacc[j] += A[r][j] * (colcoef ? colcoef[r] : dot_r)   (if colout)
// Rows stream HBM -> shared memory through a kFusedStages-deep ring of
// cp.async.bulk copies completing on mbarriers (UBLKCP): with 3 x 64 KB in
// flight per SM the memory pipe stays full without register staging.  Thread
// t owns the float4 column chunks q = t + T*c (c < C4); xv and the column
// partials live in its registers; the row dot product is a block reduction
// (one __syncthreads per row, which also releases the ring slot); per-CTA
// column partials are merged with float4 atomics at the end (colout holds its
// initial value).
struct FusedArgs {
  const float* A;
  int rows, cols;
  const float* xv;
  float* rowout;
  const float* rowinit;
  const float* colcoef;
  float* colout;
};

constexpr int kFusedThreads = 512;
constexpr int kFusedStages = 3;

namespace fused {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(0x12F0000000000000ull)  // evict-first policy
      : "memory");
}
}  // namespace fused

template <BenchId Bn, int V, int C4>
__global__ void __launch_bounds__(kFusedThreads, 1) s2_fused(FusedArgs p) {
  extern __shared__ __align__(128) float4 ring[];
  __shared__ __align__(8) uint64_t full[kFusedStages];
  __shared__ float red[2][kFusedThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nq = p.cols >> 2;
  const uint32_t row_bytes = (uint32_t)p.cols * 4u;
  const bool do_row = p.rowout != nullptr;
  const bool do_col = p.colout != nullptr;
  // rows of this CTA: r_k = blockIdx.x + k * gridDim.x
  const int nrows = p.rows > (int)blockIdx.x ? (p.rows - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (t == 0) {
    for (int s = 0; s < kFusedStages; ++s) fused::mbar_init(fused::smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < kFusedStages && k < nrows; ++k) {
      const uint32_t bar = fused::smem_u32(&full[k]);
      fused::mbar_expect_tx(bar, row_bytes);
      fused::bulk_row(fused::smem_u32(ring + (size_t)k * nq), p.A + (size_t)(blockIdx.x + k * gridDim.x) * p.cols,
                      row_bytes, bar);
    }
  }
  float4 xr[C4], acc[C4];
#pragma unroll
  for (int c = 0; c < C4; ++c) {
    const int q = t + kFusedThreads * c;
    xr[c] = (do_row && q < nq) ? __ldg(reinterpret_cast<const float4*>(p.xv) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  float coef_nxt = 0.f, init_nxt = 0.f;
  auto scalars = [&](int k) {
    if (k < nrows) {
      const int r = blockIdx.x + k * gridDim.x;
      coef_nxt = (do_col && p.colcoef) ? __ldg(p.colcoef + r) : 0.f;
      init_nxt = (t == 0 && p.rowinit) ? p.rowinit[r] : 0.f;
    }
  };
  scalars(0);
  for (int k = 0; k < nrows; ++k) {
    const int r = blockIdx.x + k * gridDim.x;
    const int s = k % kFusedStages;
    float coef = coef_nxt;
    const float init = init_nxt;
    scalars(k + 1);
    fused::mbar_wait(fused::smem_u32(&full[s]), (uint32_t)(k / kFusedStages) & 1u);
    const float4* row = ring + (size_t)s * nq;
    float4 v[C4];
#pragma unroll
    for (int c = 0; c < C4; ++c) {
      const int q = t + kFusedThreads * c;
      v[c] = q < nq ? row[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float tot = 0.f;
    if (do_row) {
      float d = 0.f;
#pragma unroll
      for (int c = 0; c < C4; ++c) {
        d = fmaf(v[c].x, xr[c].x, d);
        d = fmaf(v[c].y, xr[c].y, d);
        d = fmaf(v[c].z, xr[c].z, d);
        d = fmaf(v[c].w, xr[c].w, d);
      }
      d = warp_sum(d);
      if (lane == 0) red[k & 1][warp] = d;
    }
    __syncthreads();  // every thread has read ring slot s (and red is complete)
    if (t == 0 && k + kFusedStages < nrows) {
      const uint32_t bar = fused::smem_u32(&full[s]);
      fused::mbar_expect_tx(bar, row_bytes);
      fused::bulk_row(fused::smem_u32(ring + (size_t)s * nq),
                      p.A + (size_t)(blockIdx.x + (k + kFusedStages) * gridDim.x) * p.cols, row_bytes, bar);
    }
    if (do_row) {
#pragma unroll
      for (int w = 0; w < kFusedThreads / 32; ++w) tot += red[k & 1][w];
      if (t == 0) p.rowout[r] = init + tot;
      if (!p.colcoef) coef = tot;
    }
    if (do_col) {
#pragma unroll
      for (int c = 0; c < C4; ++c) {
        acc[c].x = fmaf(v[c].x, coef, acc[c].x);
        acc[c].y = fmaf(v[c].y, coef, acc[c].y);
        acc[c].z = fmaf(v[c].z, coef, acc[c].z);
        acc[c].w = fmaf(v[c].w, coef, acc[c].w);
      }
    }
  }
  if (do_col) {
#pragma unroll
    for (int c = 0; c < C4; ++c) {
      const int q = t + kFusedThreads * c;
      if (q < nq) atomicAdd(reinterpret_cast<float4*>(p.colout) + q, acc[c]);
    }
  }
}

inline int fused_c4(int cols) { return (int)cdiv(cols / 4, kFusedThreads); }

// Supported when cols % 4 == 0, the column vector fits in shared memory and
// C4 is one of the instantiated widths.
inline bool fused_supported(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 4 || cols % 4) return false;
  if (cols * 4 * kFusedStages > 196 * 1024) return false;
  return fused_c4((int)cols) <= 8;
}

template <BenchId Bn, int V, int C4>
inline void launch_fused_c4(const FusedArgs& p, cudaStream_t s) {
  const size_t smem = (size_t)kFusedStages * p.cols * sizeof(float);
  set_smem_attr((const void*)s2_fused<Bn, V, C4>, 200 * 1024);
  int grid = std::min(p.rows, device_sms());
  s2_fused<Bn, V, C4><<<grid, kFusedThreads, smem, s>>>(p);
}

template <BenchId Bn, int V>
inline void launch_fused(const FusedArgs& p, cudaStream_t s) {
  const int c4 = fused_c4(p.cols);
  if (c4 <= 1) launch_fused_c4<Bn, V, 1>(p, s);
  else if (c4 <= 2) launch_fused_c4<Bn, V, 2>(p, s);
  else if (c4 <= 4) launch_fused_c4<Bn, V, 4>(p, s);
  else launch_fused_c4<Bn, V, 8>(p, s);
}

}  // namespace pf
