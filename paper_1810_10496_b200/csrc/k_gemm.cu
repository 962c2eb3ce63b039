// GEMM (PolyBench/GPU gemm.cu):  C = beta*C + alpha*A*B,  NI x NJ x NK.
//
// Baseline (variant 0) keeps the PolyBench/GPU CUDA shape: one thread per
// C element on 32x8 blocks, `c *= BETA` then `c += ALPHA*a*b` read-modify-
// written in global memory inside the k loop (no __restrict__, so nvcc cannot
// prove the store does not alias a/b and keeps it in the loop -- PAPER.md:400).
// Stage-0 variants apply the phase-order transformations (store promotion,
// depot, unroll, strength reduction, 128-bit A loads); stage 1 is the tiled
// SIMT kernel; stage 2 the tcgen05 3xTF32 kernel (tc_gemm.cuh).
#include "pf_common.cuh"
#include "simt_gemm.cuh"
#include "tc_tma.cuh"

namespace pf {
namespace {

constexpr float kAlpha = 32412.0f;
constexpr float kBeta = 2123.0f;

constexpr auto kTab = make_variants<2, 1, 1, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t ni, nj, nk;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) {  // A[i][k] = i*k / NI
      int64_t i = idx / nk, k = idx % nk;
      return fdiv(fmul(i2f(i), i2f(k)), i2f(ni));
    }
    if (array == 1) {  // B[k][j] = (k*j + 1) / NJ
      int64_t k = idx / nj, j = idx % nj;
      return fdiv(fadd(fmul(i2f(k), i2f(j)), 1.0f), i2f(nj));
    }
    int64_t i = idx / nj, j = idx % nj;  // C[i][j] = (i*j + 2) / NJ
    return fdiv(fadd(fmul(i2f(i), i2f(j)), 2.0f), i2f(nj));
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], d.d[1], d.d[2], stock, stream_key(seed, B_GEMM, array, inst)}, s);
}

// Stage 0: PolyBench thread mapping (j = x, i = y), knobs from the variant.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gemm_s0(const float* a, const float* b, float* c, int ni, int nj, int nk,
                                               float alpha, float beta) {
  constexpr Knobs K = kTab.v[V];
  constexpr int U = K.unroll;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= ni || j >= nj) return;
  float* dst = &c[i * nj + j];
  Acc<K.store> acc;
  acc.init(dst, *dst * beta);
  if constexpr (K.vec) {
    const float4* pa = reinterpret_cast<const float4*>(a + (size_t)i * nk);
    const float* pb = b + j;
    PF_UNROLL_IMPL(U)
    for (int k4 = 0; k4 < nk / 4; ++k4) {
      float4 av = pa[k4];
      if constexpr (K.lsr) {
        acc.add(dst, alpha * av.x * pb[0]);
        acc.add(dst, alpha * av.y * pb[nj]);
        acc.add(dst, alpha * av.z * pb[2 * nj]);
        acc.add(dst, alpha * av.w * pb[3 * nj]);
        pb += 4 * nj;
      } else {
        int k = 4 * k4;
        acc.add(dst, alpha * av.x * b[k * nj + j]);
        acc.add(dst, alpha * av.y * b[(k + 1) * nj + j]);
        acc.add(dst, alpha * av.z * b[(k + 2) * nj + j]);
        acc.add(dst, alpha * av.w * b[(k + 3) * nj + j]);
      }
    }
  } else if constexpr (K.lsr) {
    const float* pa = a + (size_t)i * nk;
    const float* pb = b + j;
    PF_UNROLL_IMPL(U)
    for (int k = nk; k > 0; --k) {
      acc.add(dst, alpha * *pa * *pb);
      pa += 1;
      pb += nj;
    }
  } else {
    PF_UNROLL_IMPL(U)
    for (int k = 0; k < nk; k++) acc.add(dst, alpha * a[i * nk + k] * b[k * nj + j]);
  }
  acc.finish(dst);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int ni = (int)ws.dims.d[0], nj = (int)ws.dims.d[1], nk = (int)ws.dims.d[2];
    const float* A = ws.a.p[0];
    const float* B = ws.a.p[1];
    float* C = ws.a.p[2];
    if constexpr (K.stage == 0) {
      dim3 block(kBX, kBY), grid(cdiv(nj, kBX), cdiv(ni, kBY));
      gemm_s0<B_GEMM, V><<<grid, block, 0, s>>>(A, B, C, ni, nj, nk, kAlpha, kBeta);
    } else if constexpr (K.stage == 1) {
      SimtGemmArgs p{ni, nj, nk, kAlpha, kBeta, A, nk, B, nj, nullptr, nullptr, C, nj, C, nj, 0};
      launch_simt_gemm<B_GEMM, V, false, false, false>(p, s);
    } else {
      TcGemmArgs p{ni, nj, nk, kAlpha, kBeta, A, nk, false, B, nj, false, nullptr, nullptr, C, nj, C, nj, 0};
      launch_contraction<B_GEMM, V>(ws, p, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int array, const Dims& d) {
  const int64_t ni = d.d[0], nj = d.d[1], nk = d.d[2];
  return array == 0 ? ni * nk : array == 1 ? nk * nj : ni * nj;
}

int64_t launches(int v, const Dims& d) {
  return kTab.v[v].stage == 2 ? tc_launches(d.d[0], d.d[1], d.d[2], tma_ok(d.d[2], d.d[1])) : 1;
}

double alg_bytes(const Dims& d) {
  const double ni = d.d[0], nj = d.d[1], nk = d.d[2];
  return 4.0 * (ni * nk + nk * nj + 2.0 * ni * nj);
}

double alg_flops(const Dims& d) { return 2.0 * d.d[0] * d.d[1] * d.d[2]; }

int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.stage == 0 && k.vec && d.d[2] % 4) return 1;
  if (k.stage == 2 && !tc_gemm_supported(d.d[0], d.d[1], d.d[2])) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "GEMM", 3, {"ni", "nj", "nk"}, 3,
    {{"A", IN, 0}, {"B", IN, 0}, {"C", INOUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_GEMM, &kDesc);

}  // namespace
}  // namespace pf
