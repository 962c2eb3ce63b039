// GESUMMV (PolyBench/GPU gesummv.cu): y = alpha*A*x + beta*B*x,  N x N.
//
// Baseline: gesummv_kernel one thread per row (`tmp[i] += a[i][j]*x[j];
// y[i] += b[i][j]*x[j]` in global memory, uncoalesced), then
// `y[i] = ALPHA*tmp[i] + BETA*y[i]`.  Paper: 1.02-1.07x;
// the Table-1 order (-instcombine -reg2mem -mem2reg) has no licm, so the
// phase-ordered variant keeps its stores.  Both matrices must be streamed
// once: 8N^2 compulsory bytes.
#include "pf_common.cuh"
#include "blas2.cuh"

namespace pf {
namespace {

constexpr float kAlpha = 43532.0f;
constexpr float kBeta = 12313.0f;

constexpr auto kTab = make_variants<2, 4, 2, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t n;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array <= 1) return fdiv(fmul(i2f(idx / n), i2f(idx % n)), i2f(n));  // A, B = i*j/N
    return fdiv(i2f(idx), i2f(n));                                           // x = i/N
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], stock, stream_key(seed, B_GESUMMV, array, inst)}, s);
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gesummv_s0(const float* a, const float* b, const float* x, float* y,
                                                  float* tmp, int n) {
  constexpr Knobs K = kTab.v[V];
  constexpr int U = K.unroll;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Acc<K.store> at, ay;
  at.init(&tmp[i], tmp[i]);
  ay.init(&y[i], y[i]);
  if constexpr (K.vec) {
    const float4* a4 = reinterpret_cast<const float4*>(a + (size_t)i * n);
    const float4* b4 = reinterpret_cast<const float4*>(b + (size_t)i * n);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    PF_UNROLL_IMPL(U)
    for (int q = 0; q < n / 4; ++q) {
      float4 av = a4[q], bv = b4[q], xv = x4[q];
      at.add(&tmp[i], av.x * xv.x);
      ay.add(&y[i], bv.x * xv.x);
      at.add(&tmp[i], av.y * xv.y);
      ay.add(&y[i], bv.y * xv.y);
      at.add(&tmp[i], av.z * xv.z);
      ay.add(&y[i], bv.z * xv.z);
      at.add(&tmp[i], av.w * xv.w);
      ay.add(&y[i], bv.w * xv.w);
    }
  } else if constexpr (K.lsr) {
    const float* pa = a + (size_t)i * n;
    const float* pb = b + (size_t)i * n;
    const float* px = x;
    PF_UNROLL_IMPL(U)
    for (int j = n; j > 0; --j) {
      at.add(&tmp[i], *pa++ * *px);
      ay.add(&y[i], *pb++ * *px++);
    }
  } else {
    PF_UNROLL_IMPL(U)
    for (int j = 0; j < n; j++) {
      at.add(&tmp[i], a[i * n + j] * x[j]);
      ay.add(&y[i], b[i * n + j] * x[j]);
    }
  }
  at.finish(&tmp[i]);
  ay.finish(&y[i]);
  y[i] = kAlpha * tmp[i] + kBeta * y[i];
}

// Stage 1: warp per row, both matrices streamed with coalesced loads.
template <BenchId Bn, int V, int kUnroll, int kVec>
__global__ void __launch_bounds__(256) gesummv_s1(const float* __restrict__ a, const float* __restrict__ b,
                                                  const float* __restrict__ x, float* y, float* tmp, int n) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += warps) {
    float sa = 0.f, sb = 0.f;
    if constexpr (kVec) {
      const float4* a4 = reinterpret_cast<const float4*>(a + (size_t)row * n);
      const float4* b4 = reinterpret_cast<const float4*>(b + (size_t)row * n);
      const float4* x4 = reinterpret_cast<const float4*>(x);
      PF_UNROLL_IMPL(kUnroll)
      for (int q = lane; q < n / 4; q += 32) {
        float4 av = __ldg(a4 + q), bv = __ldg(b4 + q), xv = __ldg(x4 + q);
        sa = fmaf(av.x, xv.x, fmaf(av.y, xv.y, fmaf(av.z, xv.z, fmaf(av.w, xv.w, sa))));
        sb = fmaf(bv.x, xv.x, fmaf(bv.y, xv.y, fmaf(bv.z, xv.z, fmaf(bv.w, xv.w, sb))));
      }
    } else {
      PF_UNROLL_IMPL(kUnroll)
      for (int j = lane; j < n; j += 32) {
        const float xv = __ldg(x + j);
        sa = fmaf(__ldg(a + (size_t)row * n + j), xv, sa);
        sb = fmaf(__ldg(b + (size_t)row * n + j), xv, sb);
      }
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      tmp[row] = sa;
      y[row] = kAlpha * sa + kBeta * sb;
    }
  }
}

// Stage 2: persistent warp-per-row with x staged in shared memory and 4
// independent 128-bit streaming loads per matrix in flight per lane.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(512) gesummv_s2(const float* __restrict__ a, const float* __restrict__ b,
                                                  const float* __restrict__ x, float* y, float* tmp, int n) {
  extern __shared__ float4 xs[];
  const int nq = n >> 2;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) xs[q] = __ldg(reinterpret_cast<const float4*>(x) + q);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += warps) {
    const float4* a4 = reinterpret_cast<const float4*>(a + (size_t)row * n);
    const float4* b4 = reinterpret_cast<const float4*>(b + (size_t)row * n);
    float sa0 = 0.f, sa1 = 0.f, sb0 = 0.f, sb1 = 0.f;
    int q = lane;
    for (; q + 96 < nq; q += 128) {
      float4 av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = __ldcs(a4 + q + 32 * u);
        bv[u] = __ldcs(b4 + q + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 xv = xs[q + 32 * u];
        float& sa = (u & 1) ? sa1 : sa0;
        float& sb = (u & 1) ? sb1 : sb0;
        sa = fmaf(av[u].x, xv.x, fmaf(av[u].y, xv.y, fmaf(av[u].z, xv.z, fmaf(av[u].w, xv.w, sa))));
        sb = fmaf(bv[u].x, xv.x, fmaf(bv[u].y, xv.y, fmaf(bv[u].z, xv.z, fmaf(bv[u].w, xv.w, sb))));
      }
    }
    for (; q < nq; q += 32) {
      const float4 av = __ldcs(a4 + q), bv = __ldcs(b4 + q), xv = xs[q];
      sa0 = fmaf(av.x, xv.x, fmaf(av.y, xv.y, fmaf(av.z, xv.z, fmaf(av.w, xv.w, sa0))));
      sb0 = fmaf(bv.x, xv.x, fmaf(bv.y, xv.y, fmaf(bv.z, xv.z, fmaf(bv.w, xv.w, sb0))));
    }
    const float sa = warp_sum(sa0 + sa1), sb = warp_sum(sb0 + sb1);
    if (lane == 0) {
      tmp[row] = sa;
      y[row] = kAlpha * sa + kBeta * sb;
    }
  }
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int n = (int)ws.dims.d[0];
    const float* A = ws.a.p[0];
    const float* B = ws.a.p[1];
    const float* x = ws.a.p[2];
    float* y = ws.a.p[3];
    float* tmp = ws.a.p[4];
    if constexpr (K.stage == 0) {
      gesummv_s0<B_GESUMMV, V><<<cdiv(n, kB1), kB1, 0, s>>>(A, B, x, y, tmp, n);
    } else if constexpr (K.stage == 1) {
      int blocks = (int)std::min<int64_t>((n + 7) / 8, device_sms() * 16);
      gesummv_s1<B_GESUMMV, V, K.unroll, K.vec><<<blocks, 256, 0, s>>>(A, B, x, y, tmp, n);
    } else {
      set_smem_attr((const void*)gesummv_s2<B_GESUMMV, V>, 100 * 1024);
      int blocks = (int)std::min<int64_t>((n + 15) / 16, device_sms() * 2);
      gesummv_s2<B_GESUMMV, V><<<blocks, 512, n * sizeof(float), s>>>(A, B, x, y, tmp, n);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) { return a <= 1 ? d.d[0] * d.d[0] : d.d[0]; }
int64_t launches(int, const Dims&) { return 1; }
double alg_bytes(const Dims& d) { return 4.0 * (2.0 * d.d[0] * d.d[0] + 2.0 * d.d[0]); }
double alg_flops(const Dims& d) { return 4.0 * (double)d.d[0] * d.d[0] + 3.0 * d.d[0]; }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if ((k.vec || k.stage == 2) && d.d[0] % 4) return 1;
  if (k.stage == 2 && d.d[0] * 4 > 100 * 1024) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "GESUMMV", 1, {"n"}, 5,
    {{"A", IN, 0}, {"B", IN, 0}, {"x", IN, 0}, {"y", OUT, 1}, {"tmp", OUT, 0}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_GESUMMV, &kDesc);

}  // namespace
}  // namespace pf
