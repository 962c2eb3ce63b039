// Stage-1 contraction kernel: shared-memory tiled, register-blocked SIMT
// fp32 GEMM (128x128x8 tiles, 256 threads, 8x8 outputs per thread).
//
//   D = alpha * (op(A) op(B) [+ op(A2) op(B2)]) + beta * Cin
//   op(A)(m,k) = TA ? A[k*lda + m] : A[m*lda + k]
//   op(B)(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n]
//
// Used by GEMM, 2MM, 3MM, SYRK, SYR2K, CORR, COVAR.  Every kernel carries the
// (bench, variant) template prefix so the artifact extractor can attribute
// its SASS to a variant (tools/gen_artifacts.py).
#pragma once
#include "pf_common.cuh"

namespace pf {

struct SimtGemmArgs {
  int M, N, K;
  float alpha, beta;
  const float* A;
  int lda;
  const float* B;
  int ldb;
  const float* A2;  // DUAL only
  const float* B2;
  const float* Cin;  // may alias D; ignored when beta == 0
  int ldc;
  float* D;
  int ldd;
  int upper_only;  // 1: skip tiles strictly below the diagonal (symmetric outputs)
};

constexpr int kSgBM = 128, kSgBN = 128, kSgBK = 8;

template <bool TA, bool TB>
__device__ __forceinline__ void sg_load_tiles(const float* __restrict__ A, int lda, const float* __restrict__ B,
                                              int ldb, int M, int N, int K, int m0, int n0, int k0,
                                              float (*As)[kSgBM + 4], float (*Bs)[kSgBN + 4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int m, k;
    if (TA) {  // m contiguous: 32 threads x 4 along m, 8 rows of k
      k = t / 32;
      m = (t % 32) * 4 + r;
    } else {  // k contiguous: 2 threads x 4 along k per row m
      m = t / 2;
      k = (t % 2) * 4 + r;
    }
    int gm = m0 + m, gk = k0 + k;
    float v = 0.f;
    if (gm < M && gk < K) v = TA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk];
    As[k][m] = v;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int n, k;
    if (TB) {  // k contiguous
      n = t / 2;
      k = (t % 2) * 4 + r;
    } else {  // n contiguous
      k = t / 32;
      n = (t % 32) * 4 + r;
    }
    int gn = n0 + n, gk = k0 + k;
    float v = 0.f;
    if (gn < N && gk < K) v = TB ? B[(size_t)gn * ldb + gk] : B[(size_t)gk * ldb + gn];
    Bs[k][n] = v;
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void sg_mainloop(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
                                            int M, int N, int K, int m0, int n0, float (*As)[kSgBM + 4],
                                            float (*Bs)[kSgBN + 4], float (&acc)[8][8]) {
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int k0 = 0; k0 < K; k0 += kSgBK) {
    sg_load_tiles<TA, TB>(A, lda, B, ldb, M, N, K, m0, n0, k0, As, Bs);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSgBK; ++k) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[k][ty * 4 + i];
        a[4 + i] = As[k][64 + ty * 4 + i];
        b[i] = Bs[k][tx * 4 + i];
        b[4 + i] = Bs[k][64 + tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
}

template <BenchId Bn, int V, bool TA, bool TB, bool DUAL>
__global__ void __launch_bounds__(256) simt_gemm(SimtGemmArgs p) {
  __shared__ float As[kSgBK][kSgBM + 4];
  __shared__ float Bs[kSgBK][kSgBN + 4];
  const int m0 = blockIdx.y * kSgBM, n0 = blockIdx.x * kSgBN;
  if (p.upper_only && n0 + kSgBN <= m0) return;  // tile strictly below the diagonal
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  sg_mainloop<TA, TB>(p.A, p.lda, p.B, p.ldb, p.M, p.N, p.K, m0, n0, As, Bs, acc);
  if (DUAL) sg_mainloop<TA, TB>(p.A2, p.lda, p.B2, p.ldb, p.M, p.N, p.K, m0, n0, As, Bs, acc);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= p.N) continue;
      float v = p.alpha * acc[i][j];
      if (p.beta != 0.f) v = fmaf(p.beta, p.Cin[(size_t)m * p.ldc + n], v);
      p.D[(size_t)m * p.ldd + n] = v;
    }
  }
}

template <BenchId Bn, int V, bool TA, bool TB, bool DUAL>
inline void launch_simt_gemm(const SimtGemmArgs& p, cudaStream_t s) {
  dim3 grid(cdiv(p.N, kSgBN), cdiv(p.M, kSgBM));
  simt_gemm<Bn, V, TA, TB, DUAL><<<grid, 256, 0, s>>>(p);
}

// Mirror the upper triangle into the lower one (symmetric outputs).
template <BenchId Bn, int V>
__global__ void mirror_upper(float* S, int n, int ld) {
  __shared__ float tile[32][33];
  int bx = blockIdx.x, by = blockIdx.y;
  if (bx < by) return;  // source tile (by, bx) in the upper triangle, bx >= by
  int r = by * 32 + threadIdx.y, c = bx * 32 + threadIdx.x;
  for (int yy = 0; yy < 32; yy += 8)
    if (r + yy < n && c < n) tile[threadIdx.y + yy][threadIdx.x] = S[(size_t)(r + yy) * ld + c];
  __syncthreads();
  // write transposed into tile (bx, by)
  int r2 = bx * 32 + threadIdx.y, c2 = by * 32 + threadIdx.x;
  for (int yy = 0; yy < 32; yy += 8) {
    int rr = r2 + yy;
    if (rr < n && c2 < n && rr > c2) S[(size_t)rr * ld + c2] = tile[threadIdx.x][threadIdx.y + yy];
  }
}

template <BenchId Bn, int V>
inline void launch_mirror(float* S, int n, int ld, cudaStream_t s) {
  dim3 grid(cdiv(n, 32), cdiv(n, 32));
  mirror_upper<Bn, V><<<grid, dim3(32, 8), 0, s>>>(S, n, ld);
}

}  // namespace pf
