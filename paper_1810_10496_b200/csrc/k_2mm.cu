// 2MM (PolyBench/GPU 2mm.cu): C = A B ; E = C D.
//
// Baseline: mm2_kernel1/2, one thread per output on 32x8 blocks, the
// accumulator zeroed and updated in global memory inside the k loop; the
// paper's best order (-cfl-anders-aa -dse -loop-reduce -licm -instcombine)
// moves the store out of the loop (1.63x over OpenCL, 1.56x over CUDA,
// PAPER.md:360-371).  Stage 1: tiled SIMT; stage 2: tcgen05 3xTF32.
#include "pf_common.cuh"
#include "dense_s0.cuh"
#include "simt_gemm.cuh"
#include "tc_tma.cuh"

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 1, 1, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t ni, nj, nk, nl;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) return fdiv(fmul(i2f(idx / nk), i2f(idx % nk)), i2f(ni));      // A = i*k/NI
    if (array == 1) return fdiv(fmul(i2f(idx / nj), i2f(idx % nj + 1)), i2f(nj));  // B = k*(j+1)/NJ
    return fdiv(fmul(i2f(idx / nl), i2f(idx % nl + 2)), i2f(nk));                  // D = j*(l+2)/NK
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], d.d[1], d.d[2], d.d[3], stock, stream_key(seed, B_2MM, array, inst)}, s);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int ni = (int)ws.dims.d[0], nj = (int)ws.dims.d[1], nk = (int)ws.dims.d[2], nl = (int)ws.dims.d[3];
    const float* A = ws.a.p[0];
    const float* B = ws.a.p[1];
    float* C = ws.a.p[2];
    const float* D = ws.a.p[3];
    float* E = ws.a.p[4];
    if constexpr (K.stage == 0) {
      launch_s0_mm<B_2MM, V, K.store, K.unroll, K.lsr, K.vec, false>(A, nk, B, nj, C, nj, ni, nj, nk, 1.0f, 0, 0.f, s);
      launch_s0_mm<B_2MM, V, K.store, K.unroll, K.lsr, K.vec, false>(C, nj, D, nl, E, nl, ni, nl, nj, 1.0f, 0, 0.f, s);
    } else if constexpr (K.stage == 1) {
      launch_simt_gemm<B_2MM, V, false, false, false>(
          SimtGemmArgs{ni, nj, nk, 1.f, 0.f, A, nk, B, nj, nullptr, nullptr, nullptr, nj, C, nj, 0}, s);
      launch_simt_gemm<B_2MM, V, false, false, false>(
          SimtGemmArgs{ni, nl, nj, 1.f, 0.f, C, nj, D, nl, nullptr, nullptr, nullptr, nl, E, nl, 0}, s);
    } else {
      // C's lo image comes out of the first product's epilogue (when it runs
      // pre-split, without split-K), so the second product splits only D
      float* clo = ws.ensure_aux((size_t)ni * nj * sizeof(float));
      TcGemmArgs p1{ni, nj, nk, 1.f, 0.f, A, nk, false, B, nj, false, nullptr, nullptr, nullptr, nj, C, nj, 0};
      p1.Dlo = clo;
      const bool have_clo = launch_contraction<B_2MM, V>(ws, p1, s);
      TcGemmArgs p2{ni, nl, nj, 1.f, 0.f, C, nj, false, D, nl, false, nullptr, nullptr, nullptr, nl, E, nl, 0};
      if (have_clo) p2.Alo = clo;
      launch_contraction<B_2MM, V>(ws, p2, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) {
  const int64_t ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3];
  const int64_t s[5] = {ni * nk, nk * nj, ni * nj, nj * nl, ni * nl};
  return s[a];
}
int64_t launches(int v, const Dims& d) {
  if (kTab.v[v].stage != 2) return 2;
  return tc_launches(d.d[0], d.d[1], d.d[2], tma_ok(d.d[2], d.d[1])) +
         tc_launches(d.d[0], d.d[3], d.d[1], tma_ok(d.d[1], d.d[3]), false, 1);  // C's lo from the first epilogue
}
double alg_bytes(const Dims& d) {
  const double ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3];
  return 4.0 * (ni * nk + nk * nj + nj * nl + ni * nl);
}
double alg_flops(const Dims& d) {
  const double ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3];
  return 2.0 * ni * nj * nk + 2.0 * ni * nl * nj;
}
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.stage == 0 && k.vec && (d.d[2] % 4 || d.d[1] % 4)) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "2MM", 4, {"ni", "nj", "nk", "nl"}, 5,
    {{"A", IN, 0}, {"B", IN, 0}, {"C", OUT, 0}, {"D", IN, 0}, {"E", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_2MM, &kDesc);

}  // namespace
}  // namespace pf
