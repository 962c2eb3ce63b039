// 3MM (PolyBench/GPU 3mm.cu): E = A B ; F = C D ; G = E F.
//
// Baseline: mm3_kernel1/2/3 with the accumulator in global memory inside the
// k loop.  Paper: 1.55x over CUDA / 1.82x over OpenCL, from moving the store
// out of the loop.  Stage 1: tiled SIMT; stage 2: tcgen05.
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
  int64_t ni, nj, nk, nl, nm;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) return fdiv(fmul(i2f(idx / nk), i2f(idx % nk)), i2f(ni));      // A = i*k/NI
    if (array == 1) return fdiv(fmul(i2f(idx / nj), i2f(idx % nj + 1)), i2f(nj));  // B = k*(j+1)/NJ
    if (array == 2) return fdiv(fmul(i2f(idx / nm), i2f(idx % nm + 3)), i2f(nl));  // C = j*(m+3)/NL
    return fdiv(fmul(i2f(idx / nl), i2f(idx % nl + 2)), i2f(nk));                  // D = m*(l+2)/NK
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n,
                   Init{array, d.d[0], d.d[1], d.d[2], d.d[3], d.d[4], stock, stream_key(seed, B_3MM, array, inst)}, s);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int ni = (int)ws.dims.d[0], nj = (int)ws.dims.d[1], nk = (int)ws.dims.d[2], nl = (int)ws.dims.d[3],
              nm = (int)ws.dims.d[4];
    const float* A = ws.a.p[0];
    const float* B = ws.a.p[1];
    const float* C = ws.a.p[2];
    const float* D = ws.a.p[3];
    float* E = ws.a.p[4];
    float* F = ws.a.p[5];
    float* G = ws.a.p[6];
    if constexpr (K.stage == 0) {
      launch_s0_mm<B_3MM, V, K.store, K.unroll, K.lsr, K.vec, false>(A, nk, B, nj, E, nj, ni, nj, nk, 1.f, 0, 0.f, s);
      launch_s0_mm<B_3MM, V, K.store, K.unroll, K.lsr, K.vec, false>(C, nm, D, nl, F, nl, nj, nl, nm, 1.f, 0, 0.f, s);
      launch_s0_mm<B_3MM, V, K.store, K.unroll, K.lsr, K.vec, false>(E, nj, F, nl, G, nl, ni, nl, nj, 1.f, 0, 0.f, s);
    } else if constexpr (K.stage == 1) {
      launch_simt_gemm<B_3MM, V, false, false, false>(
          SimtGemmArgs{ni, nj, nk, 1.f, 0.f, A, nk, B, nj, nullptr, nullptr, nullptr, nj, E, nj, 0}, s);
      launch_simt_gemm<B_3MM, V, false, false, false>(
          SimtGemmArgs{nj, nl, nm, 1.f, 0.f, C, nm, D, nl, nullptr, nullptr, nullptr, nl, F, nl, 0}, s);
      launch_simt_gemm<B_3MM, V, false, false, false>(
          SimtGemmArgs{ni, nl, nj, 1.f, 0.f, E, nj, F, nl, nullptr, nullptr, nullptr, nl, G, nl, 0}, s);
    } else {
      // E's and F's lo images come out of their products' epilogues (when
      // those run pre-split), so G = E F needs no split pass of its own
      float* elo = ws.ensure_aux(((size_t)ni * nj + (size_t)nj * nl) * sizeof(float));
      float* flo = elo ? elo + (size_t)ni * nj : nullptr;  // no aux buffer: both products split in-kernel
      TcGemmArgs p1{ni, nj, nk, 1.f, 0.f, A, nk, false, B, nj, false, nullptr, nullptr, nullptr, nj, E, nj, 0};
      p1.Dlo = elo;
      const bool have_elo = launch_contraction<B_3MM, V>(ws, p1, s);
      TcGemmArgs p2{nj, nl, nm, 1.f, 0.f, C, nm, false, D, nl, false, nullptr, nullptr, nullptr, nl, F, nl, 0};
      p2.Dlo = flo;
      const bool have_flo = launch_contraction<B_3MM, V>(ws, p2, s);
      TcGemmArgs p3{ni, nl, nj, 1.f, 0.f, E, nj, false, F, nl, false, nullptr, nullptr, nullptr, nl, G, nl, 0};
      if (have_elo) p3.Alo = elo;
      if (have_flo) p3.Blo = flo;
      launch_contraction<B_3MM, V>(ws, p3, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) {
  const int64_t ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3], nm = d.d[4];
  const int64_t s[7] = {ni * nk, nk * nj, nj * nm, nm * nl, ni * nj, nj * nl, ni * nl};
  return s[a];
}
int64_t launches(int v, const Dims& d) {
  if (kTab.v[v].stage != 2) return 3;
  const int64_t ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3], nm = d.d[4];
  return tc_launches(ni, nj, nk, tma_ok(nk, nj)) + tc_launches(nj, nl, nm, tma_ok(nm, nl)) +
         tc_launches(ni, nl, nj, tma_ok(nj, nl), false, 0);  // E's and F's lo from the earlier epilogues
}
double alg_bytes(const Dims& d) {
  const double ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3], nm = d.d[4];
  return 4.0 * (ni * nk + nk * nj + nj * nm + nm * nl + ni * nl);
}
double alg_flops(const Dims& d) {
  const double ni = d.d[0], nj = d.d[1], nk = d.d[2], nl = d.d[3], nm = d.d[4];
  return 2.0 * (ni * nj * nk + nj * nl * nm + ni * nl * nj);
}
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.stage == 0 && k.vec && (d.d[2] % 4 || d.d[4] % 4 || d.d[1] % 4)) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "3MM", 5, {"ni", "nj", "nk", "nl", "nm"}, 7,
    {{"A", IN, 0}, {"B", IN, 0}, {"C", IN, 0}, {"D", IN, 0}, {"E", OUT, 0}, {"F", OUT, 0}, {"G", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_3MM, &kDesc);

}  // namespace
}  // namespace pf
