// FDTD-2D (PolyBench/GPU fdtd2d.cu): 2-D Yee scheme, TMAX time steps on
// NX x NY fields ex, ey, hz.
//
// Baseline: three kernels per time step (ey update with the _fict_ source
// row, ex update, hz update), i.e. 3*TMAX launches.  Phase ordering had no
// effect on the paper's GPU.  Stage 1: one fused kernel per
// step on double-buffered fields (each thread recomputes the two neighbour
// updates hz needs), TMAX launches; stage 2: the stage-1 sequence captured
// once as a CUDA graph.  At 2048^2 the six 16 MiB fields stay L2-resident.
#include "pf_common.cuh"

#include <algorithm>

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 1, 1, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int array;
  int64_t nx, ny;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    if (array == 0) return i2f(idx);  // _fict_[t] = t
    const int64_t i = idx / ny, j = idx % ny;
    if (array == 1) return fdiv(fadd(fmul(i2f(i), i2f(j + 1)), 1.0f), i2f(nx));     // ex
    if (array == 2) return fdiv(fadd(fmul(i2f(i - 1), i2f(j + 2)), 2.0f), i2f(nx));  // ey
    return fdiv(fadd(fmul(i2f(i - 9), i2f(j + 4)), 3.0f), i2f(nx));                  // hz
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{array, d.d[0], d.d[1], stock, stream_key(seed, B_FDTD2D, array, inst)}, s);
}

__device__ __forceinline__ float upd_e(float e, float h1, float h0) { return e - 0.5f * (h1 - h0); }
__device__ __forceinline__ float upd_h(float h, float exr, float exc, float eyd, float eyc) {
  return h - 0.7f * (exr - exc + eyd - eyc);
}

// ---- stage 0: the three PolyBench kernels (vec: 4 consecutive j per thread)
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) step1(const float* fict, float* ey, const float* hz, int nx, int ny, int t) {
  constexpr int W = kTab.v[V].vec ? 4 : 1;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) * W + e;
    if ((i < nx) && (j < ny)) {
      if (i == 0)
        ey[i * ny + j] = fict[t];
      else
        ey[i * ny + j] = upd_e(ey[i * ny + j], hz[i * ny + j], hz[(i - 1) * ny + j]);
    }
  }
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) step2(float* ex, const float* hz, int nx, int ny) {
  constexpr int W = kTab.v[V].vec ? 4 : 1;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) * W + e;
    if ((i < nx) && (j < ny) && (j > 0)) ex[i * ny + j] = upd_e(ex[i * ny + j], hz[i * ny + j], hz[i * ny + (j - 1)]);
  }
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) step3(const float* ex, const float* ey, float* hz, int nx, int ny) {
  constexpr int W = kTab.v[V].vec ? 4 : 1;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) * W + e;
    if ((i < (nx - 1)) && (j < (ny - 1)))
      hz[i * ny + j] = upd_h(hz[i * ny + j], ex[i * ny + (j + 1)], ex[i * ny + j], ey[(i + 1) * ny + j], ey[i * ny + j]);
  }
}

// ---- stage 1: one fused step, fields read from (ex0, ey0, hz0), written to (ex1, ey1, hz1)
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) step_fused(const float* __restrict__ fict, const float* __restrict__ ex0,
                                                  const float* __restrict__ ey0, const float* __restrict__ hz0,
                                                  float* __restrict__ ex1, float* __restrict__ ey1,
                                                  float* __restrict__ hz1, int nx, int ny, int t) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const size_t c = (size_t)i * ny + j;
  const float h = hz0[c];
  float ey_c, ex_c;
  if (i == 0)
    ey_c = __ldg(fict + t);
  else
    ey_c = upd_e(ey0[c], h, hz0[c - ny]);
  if (j == 0)
    ex_c = ex0[c];
  else
    ex_c = upd_e(ex0[c], h, hz0[c - 1]);
  float h_new = h;
  if (i < nx - 1 && j < ny - 1) {
    const float ex_r = upd_e(ex0[c + 1], hz0[c + 1], h);      // ex'(i, j+1), j+1 >= 1
    const float ey_d = upd_e(ey0[c + ny], hz0[c + ny], h);    // ey'(i+1, j), i+1 >= 1
    h_new = upd_h(h, ex_r, ex_c, ey_d, ey_c);
  }
  ey1[c] = ey_c;
  ex1[c] = ex_c;
  hz1[c] = h_new;
}

// 4 consecutive j per thread (ny % 4 == 0): 128-bit loads/stores, the
// neighbour values shared in registers instead of 9 scalar loads per point.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) step_fused4(const float* __restrict__ fict, const float* __restrict__ ex0,
                                                   const float* __restrict__ ey0, const float* __restrict__ hz0,
                                                   float* __restrict__ ex1, float* __restrict__ ey1,
                                                   float* __restrict__ hz1, int nx, int ny, int t) {
  const int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j0 >= ny) return;
  const size_t c = (size_t)i * ny + j0;
  const float4 hc = *reinterpret_cast<const float4*>(hz0 + c);
  const float h[6] = {j0 > 0 ? hz0[c - 1] : 0.f, hc.x, hc.y, hc.z, hc.w, j0 + 4 < ny ? hz0[c + 4] : 0.f};
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 hu4 = i > 0 ? *reinterpret_cast<const float4*>(hz0 + c - ny) : zero;
  const bool has_down = i < nx - 1;
  const float4 hd4 = has_down ? *reinterpret_cast<const float4*>(hz0 + c + ny) : zero;
  const float4 ex4 = *reinterpret_cast<const float4*>(ex0 + c);
  const float ex_next = j0 + 4 < ny ? ex0[c + 4] : 0.f;
  const float4 ey4 = *reinterpret_cast<const float4*>(ey0 + c);
  const float4 eyd4 = has_down ? *reinterpret_cast<const float4*>(ey0 + c + ny) : zero;
  const float hu[4] = {hu4.x, hu4.y, hu4.z, hu4.w}, hd[4] = {hd4.x, hd4.y, hd4.z, hd4.w};
  const float exv[5] = {ex4.x, ex4.y, ex4.z, ex4.w, ex_next};
  const float eyv[4] = {ey4.x, ey4.y, ey4.z, ey4.w}, eyd[4] = {eyd4.x, eyd4.y, eyd4.z, eyd4.w};
  const float src = i == 0 ? __ldg(fict + t) : 0.f;
  float oey[4], oex[4], ohz[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int j = j0 + e;
    const float hh = h[e + 1];
    float ey_c, ex_c;
    if (i == 0)
      ey_c = src;
    else
      ey_c = upd_e(eyv[e], hh, hu[e]);
    if (j == 0)
      ex_c = exv[e];
    else
      ex_c = upd_e(exv[e], hh, h[e]);
    float hn = hh;
    if (has_down && j < ny - 1) {
      const float ex_r = upd_e(exv[e + 1], h[e + 2], hh);
      const float ey_d = upd_e(eyd[e], hd[e], hh);
      hn = upd_h(hh, ex_r, ex_c, ey_d, ey_c);
    }
    oey[e] = ey_c;
    oex[e] = ex_c;
    ohz[e] = hn;
  }
  *reinterpret_cast<float4*>(ey1 + c) = make_float4(oey[0], oey[1], oey[2], oey[3]);
  *reinterpret_cast<float4*>(ex1 + c) = make_float4(oex[0], oex[1], oex[2], oex[3]);
  *reinterpret_cast<float4*>(hz1 + c) = make_float4(ohz[0], ohz[1], ohz[2], ohz[3]);
}

template <BenchId Bn, int V>
void fused_sequence(Workspace& ws, cudaStream_t s) {
  const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1], tmax = (int)ws.dims.d[2];
  const size_t n = (size_t)nx * ny;
  float* scratch = ws.ensure_scratch(3 * n * sizeof(float));
  float* buf[2][3] = {{ws.a.p[1], ws.a.p[2], ws.a.p[3]}, {scratch, scratch + n, scratch + 2 * n}};
  const bool vec = ny % 4 == 0;
  dim3 block(kBX, kBY), grid(cdiv(ny, kBX), cdiv(nx, kBY));
  dim3 block4(64, 4), grid4(cdiv(ny / 4, 64), cdiv(nx, 4));
  for (int t = 0; t < tmax; ++t) {
    float** src = buf[t & 1];
    float** dst = buf[(t + 1) & 1];
    if (vec)
      step_fused4<Bn, V><<<grid4, block4, 0, s>>>(ws.a.p[0], src[0], src[1], src[2], dst[0], dst[1], dst[2], nx, ny,
                                                  t);
    else
      step_fused<Bn, V><<<grid, block, 0, s>>>(ws.a.p[0], src[0], src[1], src[2], dst[0], dst[1], dst[2], nx, ny, t);
  }
  if (tmax & 1)
    for (int f = 0; f < 3; ++f) cudaMemcpyAsync(buf[0][f], buf[1][f], n * sizeof(float), cudaMemcpyDeviceToDevice, s);
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1], tmax = (int)ws.dims.d[2];
    const float* fict = ws.a.p[0];
    float* ex = ws.a.p[1];
    float* ey = ws.a.p[2];
    float* hz = ws.a.p[3];
    if constexpr (K.stage == 0) {
      dim3 block(kBX, kBY), grid(cdiv(ny, kBX * (K.vec ? 4 : 1)), cdiv(nx, kBY));
      for (int t = 0; t < tmax; ++t) {
        step1<B_FDTD2D, V><<<grid, block, 0, s>>>(fict, ey, hz, nx, ny, t);
        step2<B_FDTD2D, V><<<grid, block, 0, s>>>(ex, hz, nx, ny);
        step3<B_FDTD2D, V><<<grid, block, 0, s>>>(ex, ey, hz, nx, ny);
      }
    } else if constexpr (K.stage == 1) {
      fused_sequence<B_FDTD2D, V>(ws, s);
    } else {
      ws.ensure_scratch(3 * (size_t)nx * ny * sizeof(float));  // allocate before capture
      cudaGraphExec_t g = cached_graph(ws, V, &fused_sequence<B_FDTD2D, V>);
      cudaGraphLaunch(g, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) { return a == 0 ? d.d[2] : d.d[0] * d.d[1]; }
int64_t launches(int v, const Dims& d) {
  const int st = kTab.v[v].stage;
  return st == 0 ? 3 * d.d[2] : d.d[2];
}
// fused compulsory traffic per step: read ex, ey, hz, write ex, ey, hz
double alg_bytes(const Dims& d) { return 4.0 * 6.0 * (double)d.d[0] * d.d[1] * d.d[2]; }
double alg_flops(const Dims& d) { return 11.0 * (double)d.d[0] * d.d[1] * d.d[2]; }
int check(int v, const Dims& d) {
  if (kTab.v[v].vec && d.d[1] % 4) return 1;
  return d.d[0] < 2 || d.d[1] < 2;
}

const BenchDesc kDesc = {
    "FDTD-2D", 3, {"nx", "ny", "tmax"}, 4,
    {{"fict", IN, 0}, {"ex", INOUT, 1}, {"ey", INOUT, 1}, {"hz", INOUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_FDTD2D, &kDesc);

}  // namespace
}  // namespace pf
