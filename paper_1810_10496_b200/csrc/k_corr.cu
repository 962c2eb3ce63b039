// CORR (PolyBench/GPU correlation.cu): Pearson correlation matrix of the M columns of
// the 1-based (N+1) x (M+1) data array (mean, std, normalise, D^T D).
// See corrcov.cuh for the variant stages.
#include "corrcov.cuh"

namespace pf {
namespace {

constexpr auto kTab = make_variants<1, 1, 1, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t m;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    return fdiv(fmul(i2f(idx / (m + 1)), i2f(idx % (m + 1))), i2f(m + 1));
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], stock, stream_key(seed, B_CORR, array, inst)}, s);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    corrcov::run<B_CORR, V, true, K.stage, K.store, K.unroll, K.lsr>(ws, s);
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) {
  const int64_t m = d.d[0], n = d.d[1];
  if (a == 0) return (n + 1) * (m + 1);
  if (a == 4 - 1) return (m + 1) * (m + 1);
  return m + 1;
}
int64_t launches(int v, const Dims& d) { return corrcov::launches(true, kTab.v[v].stage, d.d[0], d.d[1]); }
double alg_bytes(const Dims& d) {
  const double m = d.d[0], n = d.d[1];
  return 4.0 * ((n + 1) * (m + 1) + (m + 1) * (m + 1));
}
double alg_flops(const Dims& d) {
  const double m = d.d[0], n = d.d[1];
  return double(m) * m * n + 5.0 * m * n;
}
int check(int, const Dims&) { return 0; }

const BenchDesc kDesc = {
    "CORR", 2, {"m", "n"}, 4,
    {{"data", INOUT, 0}, {"mean", OUT, 0}, {"std", OUT, 0}, {"symmat", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_CORR, &kDesc);

}  // namespace
}  // namespace pf
