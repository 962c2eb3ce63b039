// Probe: tcgen05 TMA kernel with an MN-major B (GEMM C = A*B, B[k][n]) under
// alternative MN-major descriptor encodings; prints max relative error each.
#include "../paper_1810_10496_b200/csrc/tc_tma.cuh"
#include <cstdio>
#include <vector>
#include <cmath>

namespace pf {
void register_bench(int, const BenchDesc*) {}
float* Workspace::ensure_scratch(size_t) { return nullptr; }
}
using namespace pf;

int main() {
  const int M = 128, N = 128, K = 64;
  std::vector<float> A(M * K), B(K * N), C(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 37) % 101) / 101.f;
  for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 53) % 97) / 97.f;
  std::vector<double> ref(M * N, 0.0);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < N; ++j) ref[i * N + j] += (double)A[i * K + k] * B[k * N + j];
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  // A MN-major (At[k][m]) with K-major B, and both MN-major
  std::vector<float> At(K * M);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) At[k * M + i] = A[i * K + k];
  float* dAt;
  cudaMalloc(&dAt, At.size() * 4);
  cudaMemcpy(dAt, At.data(), At.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<float> Bt(N * K);
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < N; ++j) Bt[j * K + k] = B[k * N + j];
    float* dBt;
    cudaMalloc(&dBt, Bt.size() * 4);
    cudaMemcpy(dBt, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0, C.size() * 4);
    tma_probe().idesc_override = mode == 2 ? 0 : -1;
    TcGemmArgs a = mode == 0 ? TcGemmArgs{M, N, K, 1.f, 0.f, dAt, M, true, dBt, K, true, nullptr, nullptr, nullptr, N, dC, N, 0}
                 : mode == 1 ? TcGemmArgs{M, N, K, 1.f, 0.f, dAt, M, true, dB, N, false, nullptr, nullptr, nullptr, N, dC, N, 0}
                             : TcGemmArgs{M, N, K, 1.f, 0.f, dA, K, false, dB, N, false, nullptr, nullptr, nullptr, N, dC, N, 0};
    launch_tc_tma<B_GEMM, 997>(a, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0, asum = 0;
    for (int i = 0; i < M * N; ++i) {
      worst = std::fmax(worst, std::fabs(C[i] - ref[i]) / std::fmax(1e-3, std::fabs(ref[i])));
      asum += std::fabs(C[i]);
    }
    printf("mode %d (%s): err=%s max_rel=%.3e sum|C|=%.3e C[1]=%f\n", mode,
           mode == 0 ? "A MN-major, B K-major" : mode == 1 ? "A MN, B MN" : "B MN data, idesc majors forced 0",
           cudaGetErrorString(e), worst, asum, C[1]);
  }
  tma_probe().idesc_override = -1;
  uint32_t combos[][3] = {{4096, 512, 1024}, {512, 4096, 1024}, {4096, 512, 512}};
  // control: K-major B (B stored N x K), the SYRK-style path
  {
    std::vector<float> Bt(N * K);
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < N; ++j) Bt[j * K + k] = B[k * N + j];
    float* dBt;
    cudaMalloc(&dBt, Bt.size() * 4);
    cudaMemcpy(dBt, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0, C.size() * 4);
    TcGemmArgs a{M, N, K, 1.f, 0.f, dA, K, false, dBt, K, true, nullptr, nullptr, nullptr, N, dC, N, 0};
    bool ok = launch_tc_tma<B_GEMM, 998>(a, 0);
    cudaError_t le = cudaGetLastError();
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int i = 0; i < M * N; ++i) worst = std::fmax(worst, std::fabs(C[i] - ref[i]) / std::fmax(1e-3, std::fabs(ref[i])));
    printf("control K-major B: launched=%d launch_err=%s sync=%s max_rel=%.3e C[0]=%f ref=%f\n", ok, cudaGetErrorString(le),
           cudaGetErrorString(e), worst, C[1], ref[1]);
  }
  for (auto& c : combos) {
    tma_probe().lbo = c[0]; tma_probe().sbo = c[1]; tma_probe().kstep = c[2];
    cudaMemset(dC, 0, C.size() * 4);
    TcGemmArgs a{M, N, K, 1.f, 0.f, dA, K, false, dB, N, false, nullptr, nullptr, nullptr, N, dC, N, 0};
    bool ok = launch_tc_tma<B_GEMM, 999>(a, 0);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) printf("launch error: %s\n", cudaGetErrorString(le));
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int i = 0; i < M * N; ++i) worst = std::fmax(worst, std::fabs(C[i] - ref[i]) / std::fmax(1e-3, std::fabs(ref[i])));
    printf("lbo=%u sbo=%u kstep=%u launched=%d err=%s max_rel=%.3e C[1]=%f ref=%f\n", c[0], c[1], c[2], ok,
           cudaGetErrorString(e), worst, C[1], ref[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
