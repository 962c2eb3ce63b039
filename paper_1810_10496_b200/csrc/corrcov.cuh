// Shared implementation of CORR and COVAR (PolyBench/GPU correlation.cu,
// covariance.cu).  Arrays are (N+1) x (M+1) with 1-based indexing.
//
// stage 0  PolyBench kernels: mean_kernel / std_kernel (thread per column,
//          accumulators in global memory), reduce_kernel (2-D elementwise),
//          corr_kernel / covar_kernel (thread per j1 walking the triangle
//          j2 >= j1 with symmat[j1][j2] read-modify-written in the i loop:
//          the paper's 5.4x CORR case).
// stage 1  row-split column statistics (atomics) and the Gram matrix D^T D
//          as an upper-triangle tiled SIMT GEMM + mirror.
// stage 2  3xFP16 Gram (m >= 256): the column-strip kernel (statistics,
//          centring and per-column scaled fp16 hi/lo operand rows in one
//          launch, strip_stats_f16; for n > kCSMaxRows: colpart + colfinal +
//          centre_split), the Gram on kind::f16 pair tiles, the scatter.
//          Otherwise (3xTF32)
//          four launches: (1) one pass over data accumulates every column's
//          sum and sum of squares in fp64 (row splits, fp64 atomics) and the
//          last block of each column finishes mean (and CORR's std) --
//          sum (x - mu)^2 = S2 - 2 mu S1 + n mu^2 exactly in fp64; (2) the
//          centred (scaled) data and its 3xTF32 lo image are written into an
//          aligned scratch (the data itself is not
//          written back: it is not in the compare set, and its pristine copy
//          is restored before every run anyway), transposed into a K-major
//          operand; (3) the Gram matrix on the TMA-fed tcgen05 3xTF32 kernel
//          with pre-split operands (upper-triangle pair tiles, 2-way split-K
//          with the ordered hand-over) into an aligned m x m scratch; (4) one
//          tiled pass scatters it into the 1-based symmat with the mirror
//          (and CORR's unit diagonal) folded in.
#pragma once
#include "pf_common.cuh"
#include "simt_gemm.cuh"
#include "tc_gemm.cuh"
#include "tc_tma.cuh"

#include <algorithm>

namespace pf {
namespace corrcov {

constexpr float kFloatN = 3214212.01f;
constexpr float kEps = 0.005f;

template <BenchId Bn, int V, int kStore, int kUnroll, int kLsr>
__global__ void __launch_bounds__(256) mean_s0(float* mean, const float* data, int m, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j < 1 || j >= m + 1) return;
  Acc<kStore> acc;
  acc.init(&mean[j], 0.0f);
  if constexpr (kLsr) {
    const float* p = data + (m + 1) + j;
    PF_UNROLL_IMPL(kUnroll)
    for (int i = n; i > 0; --i) {
      acc.add(&mean[j], *p);
      p += m + 1;
    }
  } else {
    PF_UNROLL_IMPL(kUnroll)
    for (int i = 1; i < n + 1; i++) acc.add(&mean[j], data[i * (m + 1) + j]);
  }
  acc.finish(&mean[j]);
  mean[j] /= kFloatN;
}

template <BenchId Bn, int V, int kStore, int kUnroll, int kLsr>
__global__ void __launch_bounds__(256) std_s0(const float* mean, float* stdv, const float* data, int m, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j < 1 || j >= m + 1) return;
  Acc<kStore> acc;
  acc.init(&stdv[j], 0.0f);
  if constexpr (kLsr) {
    const float* p = data + (m + 1) + j;
    PF_UNROLL_IMPL(kUnroll)
    for (int i = n; i > 0; --i) {
      const float d = *p - mean[j];
      acc.add(&stdv[j], d * d);
      p += m + 1;
    }
  } else {
    PF_UNROLL_IMPL(kUnroll)
    for (int i = 1; i < n + 1; i++)
      acc.add(&stdv[j], (data[i * (m + 1) + j] - mean[j]) * (data[i * (m + 1) + j] - mean[j]));
  }
  acc.finish(&stdv[j]);
  stdv[j] /= kFloatN;
  stdv[j] = sqrtf(stdv[j]);
  if (stdv[j] <= kEps) stdv[j] = 1.0f;
}

template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) reduce_s0(const float* mean, const float* stdv, float* data, int m, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int i = blockIdx.y * blockDim.y + threadIdx.y + 1;
  if (i >= 1 && i < n + 1 && j >= 1 && j < m + 1) {
    data[i * (m + 1) + j] -= mean[j];
    if constexpr (kCorr) data[i * (m + 1) + j] /= (sqrtf(kFloatN) * stdv[j]);
  }
}

// kCorr: j1 in [1, m), j2 in (j1, m], diagonal 1; else j1 in [1, m], j2 in [j1, m].
template <BenchId Bn, int V, int kStore, int kUnroll, int kLsr, bool kCorr>
__global__ void __launch_bounds__(256) gram_s0(float* sym, const float* data, int m, int n) {
  const int j1 = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j1 == 1 && kCorr) sym[m * (m + 1) + m] = 1.0f;
  if (j1 < 1 || j1 >= (kCorr ? m : m + 1)) return;
  if constexpr (kCorr) sym[j1 * (m + 1) + j1] = 1.0f;
  for (int j2 = j1 + (kCorr ? 1 : 0); j2 < m + 1; j2++) {
    float* dst = &sym[j1 * (m + 1) + j2];
    Acc<kStore> acc;
    acc.init(dst, 0.0f);
    if constexpr (kLsr) {
      const float* p1 = data + (m + 1) + j1;
      const float* p2 = data + (m + 1) + j2;
      PF_UNROLL_IMPL(kUnroll)
      for (int i = n; i > 0; --i) {
        acc.add(dst, *p1 * *p2);
        p1 += m + 1;
        p2 += m + 1;
      }
    } else {
      PF_UNROLL_IMPL(kUnroll)
      for (int i = 1; i < n + 1; i++) acc.add(dst, data[i * (m + 1) + j1] * data[i * (m + 1) + j2]);
    }
    acc.finish(dst);
    sym[j2 * (m + 1) + j1] = *dst;
  }
}

// ---- stage >= 1 helpers
// Partial column sums over a row split: out[j] += sum_i f(data[i][j]) with
// f = x (pass 0) or (x - mean[j])^2 (pass 1).  Columns 1..m, rows 1..n.
template <BenchId Bn, int V, int kPass>
__global__ void __launch_bounds__(256) colsum_split(const float* __restrict__ data, const float* __restrict__ mean,
                                                    float* out, int m, int n, int rows_per_split) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j > m) return;
  const int i0 = 1 + blockIdx.y * rows_per_split;
  const int i1 = min(n + 1, i0 + rows_per_split);
  const float mu = kPass ? mean[j] : 0.f;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;  // four loads in flight per thread
  int i = i0;
  for (; i + 3 < i1; i += 4) {
    const float a = __ldg(data + (size_t)i * (m + 1) + j) - mu;
    const float b = __ldg(data + (size_t)(i + 1) * (m + 1) + j) - mu;
    const float c = __ldg(data + (size_t)(i + 2) * (m + 1) + j) - mu;
    const float d = __ldg(data + (size_t)(i + 3) * (m + 1) + j) - mu;
    s0 += kPass ? a * a : a;
    s1 += kPass ? b * b : b;
    s2 += kPass ? c * c : c;
    s3 += kPass ? d * d : d;
  }
  for (; i < i1; ++i) {
    const float a = __ldg(data + (size_t)i * (m + 1) + j) - mu;
    s0 += kPass ? a * a : a;
  }
  atomicAdd(out + j, (s0 + s1) + (s2 + s3));
}

template <BenchId Bn, int V, int kPass>
__global__ void finalize_stat(float* v, int m) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j > m) return;
  if (kPass == 0) {
    v[j] = v[j] / kFloatN;
  } else {
    float s = sqrtf(v[j] / kFloatN);
    v[j] = s <= kEps ? 1.0f : s;
  }
}

template <BenchId Bn, int V>
__global__ void set_unit_diag(float* sym, int m) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (j <= m) sym[j * (m + 1) + j] = 1.0f;
}

template <BenchId Bn, int V, int kPass>
inline void launch_colstat(const float* data, const float* mean, float* out, int m, int n, cudaStream_t s) {
  const int gx = (int)cdiv(m, 256);
  int splits = std::max(1, std::min((int)cdiv(device_sms() * 4, gx), (n + 31) / 32));
  const int rps = (int)cdiv(n, splits);
  splits = (int)cdiv(n, rps);
  colsum_split<Bn, V, kPass><<<dim3(gx, splits), 256, 0, s>>>(data, mean, out, m, n, rps);
  finalize_stat<Bn, V, kPass><<<cdiv(m, 256), 256, 0, s>>>(out, m);
}

// 64x64 tiles of the symmat scatter (stage-2 fallback)
constexpr int kCT = 64;

// ---- stage 2: fused column statistics.  acc[0..m] = S1, acc[m+1..2m+1] = S2
// (fp64, zeroed before the launch), blockIdx.y = row split; the last block of
// a column split group (a per-column-block arrival counter) finishes the
// statistics for its 256 columns.
template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) colstats_fused(const float* __restrict__ data, double* acc, unsigned* arrivals,
                                                      float* mean, float* stdv, int m, int n, int rps) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int i0 = 1 + blockIdx.y * rps;
  const int i1 = min(n + 1, i0 + rps);
  if (j <= m) {
    double s1 = 0.0, s2 = 0.0;
    int i = i0;
    for (; i + 3 < i1; i += 4) {  // four loads in flight per thread
      const float a = __ldg(data + (size_t)i * (m + 1) + j), b = __ldg(data + (size_t)(i + 1) * (m + 1) + j);
      const float c = __ldg(data + (size_t)(i + 2) * (m + 1) + j), d = __ldg(data + (size_t)(i + 3) * (m + 1) + j);
      s1 += ((double)a + b) + ((double)c + d);
      if constexpr (kCorr) s2 += ((double)a * a + (double)b * b) + ((double)c * c + (double)d * d);
    }
    for (; i < i1; ++i) {
      const float a = __ldg(data + (size_t)i * (m + 1) + j);
      s1 += a;
      if constexpr (kCorr) s2 += (double)a * a;
    }
    atomicAdd(acc + j, s1);
    if constexpr (kCorr) atomicAdd(acc + (m + 1) + j, s2);
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(arrivals + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last || j > m) return;
  __threadfence();
  const double S1 = atomicAdd(acc + j, 0.0);  // coherent read of the completed sums
  const float mu = (float)(S1 / (double)kFloatN);
  mean[j] = mu;
  if constexpr (kCorr) {
    const double S2 = atomicAdd(acc + (m + 1) + j, 0.0);
    const double q = S2 - 2.0 * (double)mu * S1 + (double)n * (double)mu * (double)mu;
    const float sd = (float)sqrt(fmax(q, 0.0) / (double)kFloatN);
    stdv[j] = sd <= kEps ? 1.0f : sd;
  }
}

// Xt[j-1][i-1] = centred (CORR: scaled) data[i][j] -- the data transposed
// into a K-major m x n operand (pitch ldx, a multiple of 4) -- and its 3xTF32
// lo image.  Block (32, 8) on a 64x64 tile through shared memory: 16
// elements per thread, all loads issued before the first store.  (Writing X
// untransposed and running the Gram with MN-major operands measured slower:
// 68 vs 54 us for the 2048^2 Gram.)
template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) centre_transpose(const float* __restrict__ data, const float* __restrict__ mean,
                                                        const float* __restrict__ stdv, float* __restrict__ xt,
                                                        float* __restrict__ xt_lo, int m, int n, int ldx) {
  __shared__ float t[kCT][kCT + 1];
  const int j0 = blockIdx.x * kCT, i0 = blockIdx.y * kCT;
  float mu[2], sc[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int j = j0 + threadIdx.x + 32 * c + 1;
    mu[c] = j <= m ? mean[j] : 0.f;
    sc[c] = kCorr && j <= m ? sqrtf(kFloatN) * stdv[j] : 1.f;
  }
  float v[kCT / 8][2];
#pragma unroll
  for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = i0 + threadIdx.y + 8 * q + 1, j = j0 + threadIdx.x + 32 * c + 1;
      v[q][c] = (i <= n && j <= m) ? __ldg(data + (size_t)i * (m + 1) + j) : 0.f;
    }
#pragma unroll
  for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float x = v[q][c] - mu[c];
      if constexpr (kCorr) x /= sc[c];
      t[threadIdx.y + 8 * q][threadIdx.x + 32 * c] = x;
    }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = j0 + threadIdx.y + 8 * q, i = i0 + threadIdx.x + 32 * c;
      if (j < m && i < n) {
        const float x = t[threadIdx.x + 32 * c][threadIdx.y + 8 * q];
        xt[(size_t)j * ldx + i] = x;
        xt_lo[(size_t)j * ldx + i] = x - tma::trunc_tf32(x);
      }
    }
}

// ---- stage 2 (3xFP16 Gram, n <= kCSMaxRows): column statistics + centre/scale + operand
// split in ONE launch with no inter-CTA dependency.  A CTA owns a strip of
// kCS whole columns: all n rows of the strip land in shared memory through
// cp.async (every 4-byte load in flight at once, no registers), the fp64
// column sums and the mean / std are exact per CTA (sum (x - mu)^2 =
// S2 - 2 mu S1 + n mu^2 as before), the centred (scaled) column gets its own
// power-of-two scale from its max|x'|, and each column leaves as one K-major
// row of the Gram operand: n fp16 hi + n fp16 lo halfs, coalesced.  Data
// is read from HBM once; the Gram epilogue undoes the column scales.
constexpr int kCS = 16;              // columns per CTA
constexpr int kCSThreads = 256;      // 16 columns x 16 row groups
constexpr int kCSMaxRows = 2944;     // n * (kCS + 1) * 4 bytes <= 200 KB of shared memory

inline size_t strip_smem(int n) { return (size_t)n * (kCS + 1) * sizeof(float); }

template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(kCSThreads, 1)
    strip_stats_f16(const float* __restrict__ data, float* mean, float* stdv, __half* __restrict__ xh,
                    __half* __restrict__ xl, float* __restrict__ rinv, int m, int n, int ldx, float* __restrict__ G,
                    int ldg) {
  extern __shared__ float cs_smem[];  // [n][kCS + 1]
  __shared__ double r1[16][kCS], r2[16][kCS];
  __shared__ float rmax[16][kCS], mus[kCS], scs[kCS], s16[kCS];
  const int t = threadIdx.x, c = t % kCS, g = t / kCS;
  const int j0 = blockIdx.x * kCS;  // 0-based first column of the strip
  const int j = j0 + c + 1;         // 1-based data column of this thread
  const bool colok = j <= m;
  // ---- load: rows g, g + 16, ... of column c, straight into shared memory
  {
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(cs_smem));
    for (int i = g; i < n; i += 16) {
      if (colok)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sbase + 4u * (uint32_t)(i * (kCS + 1) + c)),
                     "l"(data + (size_t)(i + 1) * (m + 1) + j)
                     : "memory");
      else
        cs_smem[i * (kCS + 1) + c] = 0.f;
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  // ---- fp64 column sums (16 row groups, then a fixed-order combine)
  {
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int i = g; i < n; i += 16) {
      const float v = cs_smem[i * (kCS + 1) + c];
      s1 += v;
      if constexpr (kCorr) s2 += (double)v * v;
    }
    r1[g][c] = s1;
    if constexpr (kCorr) r2[g][c] = s2;
  }
  __syncthreads();
  if (t < kCS) {
    double S1 = 0.0, S2 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      S1 += r1[q][t];
      if constexpr (kCorr) S2 += r2[q][t];
    }
    const float mu = (float)(S1 / (double)kFloatN);
    float sc = 1.f;
    if (j0 + t + 1 <= m) {
      mean[j0 + t + 1] = mu;
      if constexpr (kCorr) {
        const double qq = S2 - 2.0 * (double)mu * S1 + (double)n * (double)mu * (double)mu;
        const float sdv = (float)sqrt(fmax(qq, 0.0) / (double)kFloatN);
        const float sd = sdv <= kEps ? 1.0f : sdv;
        stdv[j0 + t + 1] = sd;
        sc = sqrtf(kFloatN) * sd;
      }
    }
    mus[t] = mu;
    scs[t] = sc;
  }
  __syncthreads();
  // ---- centre (and scale) in place, per-column max|x'|
  {
    const float mu = mus[c], rsc = 1.f / scs[c];  // (x - mu) * (1 / sc): within an ulp of the division
    float mx = 0.f;
#pragma unroll 4
    for (int i = g; i < n; i += 16) {
      float x = cs_smem[i * (kCS + 1) + c] - mu;
      if constexpr (kCorr) x *= rsc;
      cs_smem[i * (kCS + 1) + c] = x;
      mx = fmaxf(mx, fabsf(x));
    }
    rmax[g][c] = mx;
  }
  __syncthreads();
  if (t < kCS) {
    float mx = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) mx = fmaxf(mx, rmax[q][t]);
    const float s = f16op::scale_of(mx);
    s16[t] = s;
    if (j0 + t < m) rinv[j0 + t] = 1.f / s;
  }
  __syncthreads();
  // ---- zero this strip's rows of the Gram's upper pair tiles (columns from the
  // row's 256-block on): both split-K halves then add-reduce, no ordered wait
  {
    const int w = t >> 5, lane = t & 31;
    for (int cc = w; cc < kCS; cc += kCSThreads / 32) {
      const int row = j0 + cc;
      if (row >= m) break;
      float4* g4 = reinterpret_cast<float4*>(G + (size_t)row * ldg);
      for (int c4 = (row / 256) * 64 + lane; c4 < ldg / 4; c4 += 32) g4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  // ---- each column -> one operand row (warp w: columns w, w + 8; lane: rows 2 lane + 64 e, +1)
  const int w = t >> 5, lane = t & 31;
#pragma unroll 1
  for (int cc = w; cc < kCS; cc += kCSThreads / 32) {
    if (j0 + cc >= m) break;
    const float s = s16[cc];
    __half* hrow = xh + (size_t)(j0 + cc) * ldx;
    __half* lrow = xl + (size_t)(j0 + cc) * ldx;
#pragma unroll 4
    for (int i = 2 * lane; i < n; i += 64) {
      __half2 hh, ll;
      f16op::split1(cs_smem[i * (kCS + 1) + cc], s, hh.x, ll.x);
      f16op::split1(i + 1 < n ? cs_smem[(i + 1) * (kCS + 1) + cc] : 0.f, s, hh.y, ll.y);
      *reinterpret_cast<__half2*>(hrow + i) = hh;  // ldx and i even: 4-byte aligned
      *reinterpret_cast<__half2*>(lrow + i) = ll;
    }
  }
}

// ---- stage 2 (3xFP16 Gram, n > kCSMaxRows): three fully parallel launches,
// data read from HBM once (the strip kernel above was measured faster at
// 2048^2: 62 vs 71 us for CORR).
//  (1) colpart: thread per column, 64-row blocks: fp64 S1 (and S2 for CORR)
//      and the float min / max of the block's rows into partial arrays
//      [row block][column] (every slot written once: no atomics, no memset).
//  (2) centre_split: 64 x 64 tiles.  Each CTA finishes the statistics of its
//      64 columns from the partials in a fixed order (deterministic; mean and
//      CORR's std exactly as before: sum (x - mu)^2 = S2 - 2 mu S1 + n mu^2
//      in fp64), bounds max|x'| by max(xmax - mu, mu - xmin) (/ sc for CORR)
//      to pick each column's power-of-two scale, centres (scales) its tile,
//      splits it into fp16 hi / lo and writes it transposed: column j of the
//      data becomes 64 halfs (128 B) of row j of the K-major Gram operand.
//      The Gram epilogue undoes the column scales exactly.
constexpr int kPB = 32;  // rows per partial block (all 32 loads of a thread in flight)

template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) colpart(const float* __restrict__ data, double* __restrict__ p1,
                                               double* __restrict__ p2, float* __restrict__ pmin,
                                               float* __restrict__ pmax, int m, int n) {
  const int j = blockIdx.x * 256 + threadIdx.x + 1;
  const int i0 = 1 + blockIdx.y * kPB, i1 = min(n + 1, i0 + kPB);
  if (j > m) return;
  double s1 = 0.0, s2 = 0.0;
  float lo = INFINITY, hi = -INFINITY;
  float v[kPB];
#pragma unroll
  for (int u = 0; u < kPB; ++u) v[u] = i0 + u < i1 ? __ldg(data + (size_t)(i0 + u) * (m + 1) + j) : 0.f;
#pragma unroll
  for (int u = 0; u < kPB; ++u)
    if (i0 + u < i1) {
      s1 += v[u];
      if constexpr (kCorr) s2 += (double)v[u] * v[u];
      lo = fminf(lo, v[u]);
      hi = fmaxf(hi, v[u]);
    }
  const size_t slot = (size_t)blockIdx.y * m + (j - 1);
  p1[slot] = s1;
  if constexpr (kCorr) p2[slot] = s2;
  pmin[slot] = lo;
  pmax[slot] = hi;
}

// Statistics of every column once, from the partials: a warp per column
// (lanes over the row blocks, fixed-order butterfly).  cst[3 j + 0..2] =
// mu, 1 / sc (CORR), fp16 scale s; mean / std / 1 / s (the Gram epilogue's
// column factor) written for the compare set and the epilogue.
template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) colfinal(const double* __restrict__ p1, const double* __restrict__ p2,
                                                const float* __restrict__ pmin, const float* __restrict__ pmax,
                                                float* mean, float* stdv, float* __restrict__ cst,
                                                float* __restrict__ rinv, int m, int n) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= m) return;
  const int nb = (n + kPB - 1) / kPB;
  double s1 = 0.0, s2 = 0.0;
  float lo = INFINITY, hi = -INFINITY;
  for (int b = lane; b < nb; b += 32) {
    const size_t slot = (size_t)b * m + j;
    s1 += p1[slot];
    if constexpr (kCorr) s2 += p2[slot];
    lo = fminf(lo, pmin[slot]);
    hi = fmaxf(hi, pmax[slot]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    if constexpr (kCorr) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane) return;
  const float mu = (float)(s1 / (double)kFloatN);
  float rsc = 1.f;
  if constexpr (kCorr) {
    const double qq = s2 - 2.0 * (double)mu * s1 + (double)n * (double)mu * (double)mu;
    const float sdv = (float)sqrt(fmax(qq, 0.0) / (double)kFloatN);
    const float sd = sdv <= kEps ? 1.0f : sdv;
    rsc = 1.f / (sqrtf(kFloatN) * sd);
    stdv[j + 1] = sd;
  }
  mean[j + 1] = mu;
  const float bound = fmaxf(fmaxf(hi - mu, mu - lo), 0.f) * rsc * 1.0001f;
  const float sc = f16op::scale_of(bound);
  cst[3 * j] = mu;
  cst[3 * j + 1] = rsc;
  cst[3 * j + 2] = sc;
  rinv[j] = 1.f / sc;
}

template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) centre_split(const float* __restrict__ data, const float* __restrict__ cst,
                                                    __half* __restrict__ xh, __half* __restrict__ xl, int m, int n,
                                                    int ldx) {
  __shared__ float t[64][65];
  __shared__ float mu_s[64], rsc_s[64], s16_s[64];
  const int j0 = blockIdx.x * 64, i0 = blockIdx.y * 64;  // 0-based tile origin (column j0 + c, row i0 + r)
  // ---- tile: rows i0 .. i0+63 (data rows i0+1 ..), columns j0 .. j0+63 -> transposed halfs;
  // its loads are issued before the column statistics are fetched
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  float v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int i = i0 + ty + 4 * u, j = j0 + tx;
    v[u] = (i < n && j < m) ? __ldg(data + (size_t)(i + 1) * (m + 1) + (j + 1)) : 0.f;
  }
  if (threadIdx.x < 64) {
    const int j = min(j0 + (int)threadIdx.x, m - 1);
    mu_s[threadIdx.x] = cst[3 * j];
    rsc_s[threadIdx.x] = cst[3 * j + 1];
    s16_s[threadIdx.x] = cst[3 * j + 2];
  }
  __syncthreads();
  {
    const float mu = mu_s[tx], rsc = rsc_s[tx];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      float x = v[u] - mu;
      if constexpr (kCorr) x *= rsc;
      t[ty + 4 * u][tx] = x;
    }
  }
  __syncthreads();
  // warp w: operand rows (columns) w, w + 8, ...; lane: halfs 2 lane, +1 of this tile's 64 (128 B)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 2
  for (int cc = w; cc < 64; cc += 8) {
    const int j = j0 + cc, i = i0 + 2 * lane;
    if (j >= m || i >= n) continue;
    const float s = s16_s[cc];
    __half2 hh, ll;
    f16op::split1(t[2 * lane][cc], s, hh.x, ll.x);
    f16op::split1(i + 1 < n ? t[2 * lane + 1][cc] : 0.f, s, hh.y, ll.y);
    *reinterpret_cast<__half2*>(xh + (size_t)j * ldx + i) = hh;  // ldx and i even: 4-byte aligned
    *reinterpret_cast<__half2*>(xl + (size_t)j * ldx + i) = ll;
  }
}

// symmat[1 + r][1 + c] = G[min(r,c)][max(r,c)] (pitch ldg) (only G's upper
// triangle is computed); CORR's diagonal is 1.  Block (32, 8), 64x64 tile:
// thread (x, y) owns tile rows y + 8q and columns x, x + 32.  Tiles above
// the diagonal copy straight from registers (no shared memory); tiles below
// it read the mirrored G tile (coalesced rows) and transpose through shared
// memory; diagonal tiles mirror within the tile.  Interior tiles take an
// unpredicated path with per-thread row pointers.
template <BenchId Bn, int V, bool kCorr>
__global__ void __launch_bounds__(256) sym_scatter(const float* __restrict__ G, int ldg, float* sym, int m) {
  __shared__ float t[kCT][kCT + 1];
  const int c0 = blockIdx.x * kCT, r0 = blockIdx.y * kCT;
  const int x = threadIdx.x, y = threadIdx.y;
  const bool lower = r0 > c0, diag = r0 == c0;
  const bool full = r0 + kCT <= m && c0 + kCT <= m;
  const int gr0 = lower ? c0 : r0, gc0 = lower ? r0 : c0;  // G tile origin (always on/above the diagonal)
  const size_t ls = (size_t)(m + 1);
  float v[kCT / 8][2];
  if (full) {
    const float* g = G + (size_t)(gr0 + y) * ldg + gc0 + x;
#pragma unroll
    for (int q = 0; q < kCT / 8; ++q) {
      v[q][0] = __ldg(g + (size_t)(8 * q) * ldg);
      v[q][1] = __ldg(g + (size_t)(8 * q) * ldg + 32);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int gr = gr0 + y + 8 * q, gc = gc0 + x + 32 * c;
        v[q][c] = (gr < m && gc < m) ? __ldg(G + (size_t)gr * ldg + gc) : 0.f;
      }
  }
  if (!lower && !diag) {  // strictly above the diagonal: symmat tile = G tile
    float* d = sym + (size_t)(r0 + y + 1) * ls + c0 + x + 1;
#pragma unroll
    for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (full || (r0 + y + 8 * q < m && c0 + x + 32 * c < m)) d[(size_t)(8 * q) * ls + 32 * c] = v[q][c];
    return;
  }
#pragma unroll
  for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
    for (int c = 0; c < 2; ++c) t[y + 8 * q][x + 32 * c] = v[q][c];
  __syncthreads();
  float* d = sym + (size_t)(r0 + y + 1) * ls + c0 + x + 1;
#pragma unroll
  for (int q = 0; q < kCT / 8; ++q)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int k = y + 8 * q, xx = x + 32 * c;  // tile row, tile column
      if (!full && (r0 + k >= m || c0 + xx >= m)) continue;
      float val = (lower || k > xx) ? t[xx][k] : t[k][xx];
      if (kCorr && diag && k == xx) val = 1.0f;
      d[(size_t)(8 * q) * ls + 32 * c] = val;
    }
}

// One variant run.  arrays: data, mean, [std,] symmat
template <BenchId Bn, int V, bool kCorr, int kStage, int kStore, int kUnroll, int kLsr>
inline void run(Workspace& ws, cudaStream_t s) {
  const int m = (int)ws.dims.d[0], n = (int)ws.dims.d[1];
  float* data = ws.a.p[0];
  float* mean = ws.a.p[1];
  float* stdv = kCorr ? ws.a.p[2] : nullptr;
  float* sym = ws.a.p[kCorr ? 3 : 2];
  if constexpr (kStage == 0) {
    mean_s0<Bn, V, kStore, kUnroll, kLsr><<<cdiv(m, kB1), kB1, 0, s>>>(mean, data, m, n);
    if constexpr (kCorr) std_s0<Bn, V, kStore, kUnroll, kLsr><<<cdiv(m, kB1), kB1, 0, s>>>(mean, stdv, data, m, n);
    reduce_s0<Bn, V, kCorr><<<dim3(cdiv(m, kBX), cdiv(n, kBY)), dim3(kBX, kBY), 0, s>>>(mean, stdv, data, m, n);
    gram_s0<Bn, V, kStore, kUnroll, kLsr, kCorr><<<cdiv(m, kB1), kB1, 0, s>>>(sym, data, m, n);
  } else {
    if constexpr (kStage == 2) {
      // scratch: Xt and Xt_lo (m x np: the K-major Gram operand; 16-byte
      // pitch for the TMA maps, the K tail reads as zero), G (m x mp: split
      // 0's partial sums, or the whole Gram for the scatter fallback), then
      // the fp64 column sums and the per-column-block arrival counters
      const int mp = (m + 3) / 4 * 4, np = (n + 7) / 8 * 8;
      const size_t xs = (size_t)m * np, gs = (size_t)m * mp;
      const int gx = (int)cdiv(m, 256);
      const int nb = (n + kPB - 1) / kPB;
      float* X = ws.ensure_scratch((2 * xs + gs) * sizeof(float) + 2 * (m + 1) * sizeof(double) + 64 * 4 +
                                   gx * sizeof(unsigned) + (m + 64) * sizeof(float) + 512 +
                                   (size_t)nb * m * (2 * sizeof(double) + 2 * sizeof(float)) + 3 * (size_t)m * sizeof(float));
      if (!X) {
        launch_failed("CORR/COVAR stage 2: scratch allocation failed");
        return;
      }
      float* Xlo = X + xs;
      float* G = Xlo + xs;
      double* acc = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(G + gs) + 255) & ~uintptr_t(255));
      unsigned* arrivals = reinterpret_cast<unsigned*>(acc + 2 * (m + 1));
      float* rinv = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(arrivals + gx) + 255) & ~uintptr_t(255));
      // 3xFP16 Gram (PF_TC_F16=0: 3xTF32) when the column strips fit in
      // shared memory: statistics, centring and the operand split in one
      // launch (strip_stats_f16); else the two-launch fp32 preparation
      const bool f16 = tc_f16_enabled() && m >= 256;
      F16Operands f16ops;
      if (f16 && n <= kCSMaxRows) {
        __half* xh = reinterpret_cast<__half*>(X);
        __half* xl = xh + xs;
        set_smem_attr((const void*)strip_stats_f16<Bn, V, kCorr>, (int)strip_smem(n));
        strip_stats_f16<Bn, V, kCorr><<<cdiv(m, kCS), kCSThreads, strip_smem(n), s>>>(data, mean, stdv, xh, xl,
                                                                                     rinv, m, n, np, G, mp);
        f16ops.hi[0] = f16ops.hi[1] = xh;
        f16ops.lo[0] = f16ops.lo[1] = xl;
        f16ops.hi[2] = f16ops.hi[3] = f16ops.lo[2] = f16ops.lo[3] = nullptr;
        f16ops.kp = np;
        f16ops.rinv = f16ops.cinv = rinv;
      } else if (f16) {
        // fp16 images inside X (halfs); column partials after the scale vector
        __half* xh = reinterpret_cast<__half*>(X);
        __half* xl = xh + xs;
        double* p1 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(rinv + m + 64) + 255) & ~uintptr_t(255));
        double* p2 = p1 + (size_t)nb * m;
        float* pmin = reinterpret_cast<float*>(p2 + (size_t)nb * m);
        float* pmax = pmin + (size_t)nb * m;
        float* cst = pmax + (size_t)nb * m;  // [m][3]
        colpart<Bn, V, kCorr><<<dim3(cdiv(m, 256), nb), 256, 0, s>>>(data, p1, p2, pmin, pmax, m, n);
        colfinal<Bn, V, kCorr><<<cdiv(m, 8), 256, 0, s>>>(p1, p2, pmin, pmax, mean, stdv, cst, rinv, m, n);
        centre_split<Bn, V, kCorr><<<dim3(cdiv(m, 64), cdiv(n, 64)), 256, 0, s>>>(data, cst, xh, xl, m, n, np);
        f16ops.hi[0] = f16ops.hi[1] = xh;
        f16ops.lo[0] = f16ops.lo[1] = xl;
        f16ops.hi[2] = f16ops.hi[3] = f16ops.lo[2] = f16ops.lo[3] = nullptr;
        f16ops.kp = np;
        f16ops.rinv = f16ops.cinv = rinv;
      } else {
        cudaMemsetAsync(acc, 0, 2 * (m + 1) * sizeof(double) + gx * sizeof(unsigned), s);
        int splits = std::max(1, std::min((int)cdiv(device_sms() * 4, gx), (n + 31) / 32));
        const int rps = (int)cdiv(n, splits);
        splits = (int)cdiv(n, rps);
        colstats_fused<Bn, V, kCorr><<<dim3(gx, splits), 256, 0, s>>>(data, acc, arrivals, mean, stdv, m, n, rps);
        centre_transpose<Bn, V, kCorr><<<dim3(cdiv(m, kCT), cdiv(n, kCT)), dim3(32, 8), 0, s>>>(data, mean, stdv, X,
                                                                                              Xlo, m, n, np);
      }
      // Xt Xt^T with K-major operands
      TcGemmArgs g{m, m, n, 1.f, 0.f, X, np, false, X, np, true, nullptr, nullptr, nullptr, mp, G, mp, 1};
      if (f16) {
        g.f16 = &f16ops;
        g.d_base = n <= kCSMaxRows;  // the strip kernel zeroed G's upper tiles (beta = 0)
      } else {
        g.Alo = Xlo;
        g.Blo = Xlo;
      }
      g.tile_flags = ws.ensure_tile_flags(s);
      g.epoch = ++ws.tile_epoch;
      if (!launch_tc_tma<Bn, V>(g, s)) {
        launch_failed("CORR/COVAR stage 2: TMA operand maps rejected");
        return;
      }
      // (Writing symmat from the Gram epilogue instead -- plain stores of
      // each tile and its mirror, 256x128 pair tiles without split-K -- was
      // measured slower on B200: 68.7 us vs 47.1 us Gram + 8.5 us scatter;
      // the unaligned 1-based rows turn the epilogue's stores into partial
      // sector writes.)
      sym_scatter<Bn, V, kCorr><<<dim3(cdiv(m, kCT), cdiv(m, kCT)), dim3(32, 8), 0, s>>>(G, mp, sym, m);
      return;
    }
    launch_colstat<Bn, V, 0>(data, nullptr, mean, m, n, s);
    if constexpr (kCorr) launch_colstat<Bn, V, 1>(data, mean, stdv, m, n, s);
    reduce_s0<Bn, V, kCorr><<<dim3(cdiv(m, kBX), cdiv(n, kBY)), dim3(kBX, kBY), 0, s>>>(mean, stdv, data, m, n);
    const float* d1 = data + (m + 1) + 1;  // data[1][1]
    float* s1 = sym + (m + 1) + 1;         // symmat[1][1]
    launch_simt_gemm<Bn, V, true, false, false>(
        SimtGemmArgs{m, m, n, 1.f, 0.f, d1, m + 1, d1, m + 1, nullptr, nullptr, nullptr, m + 1, s1, m + 1, 1}, s);
    launch_mirror<Bn, V>(s1, m, m + 1, s);
    if constexpr (kCorr) set_unit_diag<Bn, V><<<cdiv(m, 256), 256, 0, s>>>(sym, m);
  }
}

inline int64_t launches(bool corr, int stage, int64_t m, int64_t n) {
  if (stage == 0) return corr ? 4 : 3;
  const int64_t stats = corr ? 4 : 2;
  if (stage == 2) {  // 3xFP16: partials, statistics, centre + split; else stats, centre; Gram; scatter
    const bool f16 = tc_f16_enabled() && m >= 256;
    return (f16 ? (n <= kCSMaxRows ? 1 : 3) : 2) + tc_tma_launches(m, m, n, false, true, true) + 1;
  }
  return stats + 1 + 1 + 1 + (corr ? 1 : 0);
}

}  // namespace corrcov
}  // namespace pf
