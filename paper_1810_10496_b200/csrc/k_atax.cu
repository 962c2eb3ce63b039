// ATAX (PolyBench/GPU atax.cu): tmp = A x ; y = A^T tmp.   A is NX x NY.
//
// Baseline: atax_kernel1 one thread per row i (`tmp[i] += A[i][j]*x[j]`, a
// warp touches 32 different rows -> uncoalesced), atax_kernel2 one thread per
// column j (`y[j] += A[i][j]*tmp[i]`, coalesced); both accumulate in global
// memory inside the loop.  The paper's phase orders move the stores out of
// the loops (1.47x over OpenCL).  Stage 2 reads A once.
#include "pf_common.cuh"
#include "blas2.cuh"

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 4, 2, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t nx, ny;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) return fdiv(fmul(i2f(idx / ny), i2f(idx % ny)), i2f(nx));  // A = i*j/NX
    return __double2float_rn((double)idx * 3.14159265358979323846);            // x = j*pi
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], d.d[1], stock, stream_key(seed, B_ATAX, array, inst)}, s);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) atax_k1(const float* A, const float* x, float* tmp, int nx, int ny) {
  constexpr Knobs K = kTab.v[V];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nx) s0_row_dot<K.store, K.unroll, K.lsr, K.vec>(&tmp[i], A, ny, i, x, ny, false);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) atax_k2(const float* A, float* y, const float* tmp, int nx, int ny) {
  constexpr Knobs K = kTab.v[V];
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) * (K.vec ? 4 : 1);
  if (j < ny) s0_col_dot<K.store, K.unroll, K.lsr, K.vec>(&y[j], A, ny, j, tmp, nx, false);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1];
    const float* A = ws.a.p[0];
    const float* x = ws.a.p[1];
    float* y = ws.a.p[2];
    float* tmp = ws.a.p[3];
    if constexpr (K.stage == 0) {
      atax_k1<B_ATAX, V><<<cdiv(nx, kB1), kB1, 0, s>>>(A, x, tmp, nx, ny);
      atax_k2<B_ATAX, V><<<cdiv(ny, kB1 * (K.vec ? 4 : 1)), kB1, 0, s>>>(A, y, tmp, nx, ny);
    } else if constexpr (K.stage == 1) {
      launch_s1_row_dot<B_ATAX, V, K.unroll, K.vec>(A, ny, x, ny, nx, nullptr, tmp, s);
      launch_s1_col_dot<B_ATAX, V, K.unroll, K.vec>(A, ny, tmp, nx, ny, y, s);
    } else {
      launch_fused<B_ATAX, V>(FusedArgs{A, nx, ny, x, tmp, nullptr, nullptr, y}, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) {
  const int64_t s[4] = {d.d[0] * d.d[1], d.d[1], d.d[1], d.d[0]};
  return s[a];
}
int64_t launches(int v, const Dims&) { return kTab.v[v].stage == 2 ? 1 : 2; }
double alg_bytes(const Dims& d) { return 4.0 * ((double)d.d[0] * d.d[1] + 2.0 * d.d[1]); }
double alg_flops(const Dims& d) { return 4.0 * (double)d.d[0] * d.d[1]; }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.vec && d.d[1] % 4) return 1;
  if (k.stage == 2 && !fused_supported(d.d[0], d.d[1])) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "ATAX", 2, {"nx", "ny"}, 4,
    {{"A", IN, 0}, {"x", IN, 0}, {"y", OUT, 1}, {"tmp", OUT, 0}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_ATAX, &kDesc);

}  // namespace
}  // namespace pf
