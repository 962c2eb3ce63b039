// MVT (PolyBench/GPU mvt.cu): x1 += A y1 ; x2 += A^T y2.   A is N x N.
//
// Baseline: mvt_kernel1 one thread per row (`x1[i] += a[i][j]*y1[j]`,
// uncoalesced), mvt_kernel2 one thread per i reading column i
// (`x2[i] += a[j][i]*y2[j]`, coalesced); stores inside the loops.  Paper:
// 1.32x over CUDA from store extraction.  Stage 2 reads A once.
#include "pf_common.cuh"
#include "blas2.cuh"

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 4, 2, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t n;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) return fdiv(fmul(i2f(idx / n), i2f(idx % n)), i2f(n));  // A = i*j/N
    const int off[5] = {0, 0, 1, 3, 4};                                      // x1, x2, y1, y2
    return fdiv(i2f(idx + off[array]), i2f(n));
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], stock, stream_key(seed, B_MVT, array, inst)}, s);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) mvt_k1(const float* a, float* x1, const float* y1, int n) {
  constexpr Knobs K = kTab.v[V];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) s0_row_dot<K.store, K.unroll, K.lsr, K.vec>(&x1[i], a, n, i, y1, n, false);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) mvt_k2(const float* a, float* x2, const float* y2, int n) {
  constexpr Knobs K = kTab.v[V];
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * (K.vec ? 4 : 1);
  if (i < n) s0_col_dot<K.store, K.unroll, K.lsr, K.vec>(&x2[i], a, n, i, y2, n, false);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int n = (int)ws.dims.d[0];
    const float* A = ws.a.p[0];
    float* x1 = ws.a.p[1];
    float* x2 = ws.a.p[2];
    const float* y1 = ws.a.p[3];
    const float* y2 = ws.a.p[4];
    if constexpr (K.stage == 0) {
      mvt_k1<B_MVT, V><<<cdiv(n, kB1), kB1, 0, s>>>(A, x1, y1, n);
      mvt_k2<B_MVT, V><<<cdiv(n, kB1 * (K.vec ? 4 : 1)), kB1, 0, s>>>(A, x2, y2, n);
    } else if constexpr (K.stage == 1) {
      launch_s1_row_dot<B_MVT, V, K.unroll, K.vec>(A, n, y1, n, n, x1, x1, s);
      launch_s1_col_dot<B_MVT, V, K.unroll, K.vec>(A, n, y2, n, n, x2, s);
    } else {
      launch_fused<B_MVT, V>(FusedArgs{A, n, n, y1, x1, x1, y2, x2}, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) { return a == 0 ? d.d[0] * d.d[0] : d.d[0]; }
int64_t launches(int v, const Dims&) { return kTab.v[v].stage == 2 ? 1 : 2; }
double alg_bytes(const Dims& d) { return 4.0 * ((double)d.d[0] * d.d[0] + 6.0 * d.d[0]); }
double alg_flops(const Dims& d) { return 4.0 * (double)d.d[0] * d.d[0]; }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.vec && d.d[0] % 4) return 1;
  if (k.stage == 2 && !fused_supported(d.d[0], d.d[0])) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "MVT", 1, {"n"}, 5,
    {{"A", IN, 0}, {"x1", INOUT, 1}, {"x2", INOUT, 1}, {"y1", IN, 0}, {"y2", IN, 0}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_MVT, &kDesc);

}  // namespace
}  // namespace pf
