// BICG (PolyBench/GPU bicg.cu): s = A^T r ; q = A p.   A is NX x NY.
//
// Baseline: bicgKernel1 one thread per column j (`s[j] = 0; s[j] += r[i]*A[i][j]`,
// coalesced), bicgKernel2 one thread per row i (`q[i] = 0; q[i] += A[i][j]*p[j]`,
// uncoalesced); stores inside the loops.  Paper: 1.48x over OpenCL from store
// removal + unrolling.  Stage 2 computes both products from a
// single read of A.
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
    return __double2float_rn((double)idx * 3.14159265358979323846);            // r, p = i*pi
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], d.d[1], stock, stream_key(seed, B_BICG, array, inst)}, s);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) bicg_k1(const float* A, const float* r, float* s, int nx, int ny) {
  constexpr Knobs K = kTab.v[V];
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) * (K.vec ? 4 : 1);
  if (j < ny) s0_col_dot<K.store, K.unroll, K.lsr, K.vec>(&s[j], A, ny, j, r, nx, true);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) bicg_k2(const float* A, const float* p, float* q, int nx, int ny) {
  constexpr Knobs K = kTab.v[V];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nx) s0_row_dot<K.store, K.unroll, K.lsr, K.vec>(&q[i], A, ny, i, p, ny, true);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t st) {
    constexpr Knobs K = kTab.v[V];
    const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1];
    const float* A = ws.a.p[0];
    const float* r = ws.a.p[1];
    const float* p = ws.a.p[2];
    float* s = ws.a.p[3];
    float* q = ws.a.p[4];
    if constexpr (K.stage == 0) {
      bicg_k1<B_BICG, V><<<cdiv(ny, kB1 * (K.vec ? 4 : 1)), kB1, 0, st>>>(A, r, s, nx, ny);
      bicg_k2<B_BICG, V><<<cdiv(nx, kB1), kB1, 0, st>>>(A, p, q, nx, ny);
    } else if constexpr (K.stage == 1) {
      launch_s1_col_dot<B_BICG, V, K.unroll, K.vec>(A, ny, r, nx, ny, s, st);
      launch_s1_row_dot<B_BICG, V, K.unroll, K.vec>(A, ny, p, ny, nx, nullptr, q, st);
    } else {
      launch_fused<B_BICG, V>(FusedArgs{A, nx, ny, p, q, nullptr, r, s}, st);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) {
  const int64_t s[5] = {d.d[0] * d.d[1], d.d[0], d.d[1], d.d[1], d.d[0]};
  return s[a];
}
int64_t launches(int v, const Dims&) { return kTab.v[v].stage == 2 ? 1 : 2; }
double alg_bytes(const Dims& d) { return 4.0 * ((double)d.d[0] * d.d[1] + 2.0 * (d.d[0] + d.d[1])); }
double alg_flops(const Dims& d) { return 4.0 * (double)d.d[0] * d.d[1]; }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.vec && d.d[1] % 4) return 1;
  if (k.stage == 2 && !fused_supported(d.d[0], d.d[1])) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "BICG", 2, {"nx", "ny"}, 5,
    {{"A", IN, 0}, {"r", IN, 0}, {"p", IN, 0}, {"s", OUT, 1}, {"q", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_BICG, &kDesc);

}  // namespace
}  // namespace pf
