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
// stage 2  the Gram matrix on tcgen05 3xTF32 (MN-major operands straight
//          from the 1-based array) + mirror.
#pragma once
#include "pf_common.cuh"
#include "simt_gemm.cuh"
#include "tc_gemm.cuh"

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
  float s0 = 0.f, s1 = 0.f;
  int i = i0;
  for (; i + 1 < i1; i += 2) {
    const float a = __ldg(data + (size_t)i * (m + 1) + j) - mu;
    const float b = __ldg(data + (size_t)(i + 1) * (m + 1) + j) - mu;
    s0 += kPass ? a * a : a;
    s1 += kPass ? b * b : b;
  }
  if (i < i1) {
    const float a = __ldg(data + (size_t)i * (m + 1) + j) - mu;
    s0 += kPass ? a * a : a;
  }
  atomicAdd(out + j, s0 + s1);
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
  int splits = std::max(1, std::min((int)cdiv(148 * 4, gx), (n + 31) / 32));
  const int rps = (int)cdiv(n, splits);
  splits = (int)cdiv(n, rps);
  colsum_split<Bn, V, kPass><<<dim3(gx, splits), 256, 0, s>>>(data, mean, out, m, n, rps);
  finalize_stat<Bn, V, kPass><<<cdiv(m, 256), 256, 0, s>>>(out, m);
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
    launch_colstat<Bn, V, 0>(data, nullptr, mean, m, n, s);
    if constexpr (kCorr) launch_colstat<Bn, V, 1>(data, mean, stdv, m, n, s);
    reduce_s0<Bn, V, kCorr><<<dim3(cdiv(m, kBX), cdiv(n, kBY)), dim3(kBX, kBY), 0, s>>>(mean, stdv, data, m, n);
    const float* d1 = data + (m + 1) + 1;  // data[1][1]
    float* s1 = sym + (m + 1) + 1;         // symmat[1][1]
    if constexpr (kStage == 1) {
      launch_simt_gemm<Bn, V, true, false, false>(
          SimtGemmArgs{m, m, n, 1.f, 0.f, d1, m + 1, d1, m + 1, nullptr, nullptr, nullptr, m + 1, s1, m + 1, 1}, s);
    } else {
      launch_tc_gemm<Bn, V>(ws, TcGemmArgs{m, m, n, 1.f, 0.f, d1, m + 1, true, d1, m + 1, false, nullptr, nullptr,
                                           nullptr, m + 1, s1, m + 1, 1}, s);
    }
    launch_mirror<Bn, V>(s1, m, m + 1, s);
    if constexpr (kCorr) set_unit_diag<Bn, V><<<cdiv(m, 256), 256, 0, s>>>(sym, m);
  }
}

inline int64_t launches(bool corr, int stage, int64_t m, int64_t n) {
  if (stage == 0) return corr ? 4 : 3;
  const int64_t stats = corr ? 4 : 2;
  const int64_t gram = stage == 1 ? 1 : tc_gemm_launches(m, m, n);
  return stats + 1 + gram + 1 + (corr ? 1 : 0);
}

}  // namespace corrcov
}  // namespace pf
