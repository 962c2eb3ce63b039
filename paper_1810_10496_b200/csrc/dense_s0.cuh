// Stage-0 (PolyBench/GPU shape) dot loop shared by the matmul-type kernels:
// one thread per output element, the accumulation target `dst` handled by the
// store knob (RMW in global memory / register / local depot).
//
//   dst = init + sum_k alpha * a_row[k] * bval(k)
//   bval(k) = kBT ? b[j*ldb + k]   (second operand row j, SYRK-style A A^T)
//                 : b[k*ldb + j]   (column j of a row-major matrix)
//   init  = beta_scale ? dst*beta : 0
#pragma once
#include "pf_common.cuh"

namespace pf {

template <int kStore, int kUnroll, int kLsr, int kVec, bool kBT>
__device__ __forceinline__ void s0_dot(float* dst, const float* a_row, const float* b, int j, int ldb, int nk,
                                       float alpha, bool beta_scale, float beta) {
  Acc<kStore> acc;
  acc.init(dst, beta_scale ? *dst * beta : 0.0f);
  if constexpr (kVec) {
    const float4* a4 = reinterpret_cast<const float4*>(a_row);
    PF_UNROLL_IMPL(kUnroll)
    for (int k4 = 0; k4 < nk / 4; ++k4) {
      const float4 av = a4[k4];
      const int k = 4 * k4;
      if constexpr (kBT) {
        const float4 bv = *reinterpret_cast<const float4*>(b + (size_t)j * ldb + k);
        acc.add(dst, alpha * av.x * bv.x);
        acc.add(dst, alpha * av.y * bv.y);
        acc.add(dst, alpha * av.z * bv.z);
        acc.add(dst, alpha * av.w * bv.w);
      } else {
        acc.add(dst, alpha * av.x * b[k * ldb + j]);
        acc.add(dst, alpha * av.y * b[(k + 1) * ldb + j]);
        acc.add(dst, alpha * av.z * b[(k + 2) * ldb + j]);
        acc.add(dst, alpha * av.w * b[(k + 3) * ldb + j]);
      }
    }
  } else if constexpr (kLsr) {
    const float* pa = a_row;
    const float* pb = kBT ? b + (size_t)j * ldb : b + j;
    const int step = kBT ? 1 : ldb;
    PF_UNROLL_IMPL(kUnroll)
    for (int k = nk; k > 0; --k) {
      acc.add(dst, alpha * *pa * *pb);
      pa += 1;
      pb += step;
    }
  } else {
    PF_UNROLL_IMPL(kUnroll)
    for (int k = 0; k < nk; k++) acc.add(dst, alpha * a_row[k] * (kBT ? b[j * ldb + k] : b[k * ldb + j]));
  }
  acc.finish(dst);
}

// out[i][j] = (beta_scale ? beta*out : 0) + alpha * sum_k a[i][k] * b(k, j)
template <BenchId Bn, int V, int kStore, int kUnroll, int kLsr, int kVec, bool kBT>
__global__ void __launch_bounds__(256) s0_mm(const float* a, int lda, const float* b, int ldb, float* out, int ldo,
                                             int ni, int nj, int nk, float alpha, int beta_scale, float beta) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= ni || j >= nj) return;
  s0_dot<kStore, kUnroll, kLsr, kVec, kBT>(&out[i * ldo + j], a + (size_t)i * lda, b, j, ldb, nk, alpha,
                                           beta_scale != 0, beta);
}

template <BenchId Bn, int V, int kStore, int kUnroll, int kLsr, int kVec, bool kBT>
inline void launch_s0_mm(const float* a, int lda, const float* b, int ldb, float* out, int ldo, int ni, int nj, int nk,
                         float alpha, int beta_scale, float beta, cudaStream_t s) {
  dim3 block(kBX, kBY), grid(cdiv(nj, kBX), cdiv(ni, kBY));
  s0_mm<Bn, V, kStore, kUnroll, kLsr, kVec, kBT><<<grid, block, 0, s>>>(a, lda, b, ldb, out, ldo, ni, nj, nk, alpha,
                                                                        beta_scale, beta);
}

}  // namespace pf
