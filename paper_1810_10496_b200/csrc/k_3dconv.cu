// 3DCONV (PolyBench/GPU 3DConvolution.cu): 15-tap 3-D stencil (PolyBench's
// repeated taps kept) on the interior of an NI x NJ x NK array.
//
// Baseline: the host launches convolution3D_kernel once per plane i
// (NI-2 launches of a (k, j) grid), 15 global loads per point.  No order
// helped on the paper's GPU.  Stage 1: one launch, each
// thread streams a 16-plane chunk of i with the 7 distinct (j, k) taps of a
// plane kept in a 3-plane register ring (7 loads per output); stage 2: 4
// outputs along k per thread with 128-bit loads.
#include "pf_common.cuh"

#include <algorithm>

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 1, 1, 1>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

constexpr float c11 = 2, c12 = -3, c13 = 4, c21 = 5, c22 = 6, c23 = 7, c31 = -8, c32 = -9, c33 = 10;

struct Init {
  int64_t nj, nk;
  int stock;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    if (!stock) return unit_float(key, idx);
    const int64_t i = idx / (nj * nk), j = (idx / nk) % nj, k = idx % nk;
    return (float)(i % 12 + 2 * (j % 7) + 3 * (k % 13));
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  launch_init_with(out, n, Init{d.d[1], d.d[2], stock, stream_key(seed, B_3DCONV, array, inst)}, s);
}

// PolyBench evaluation order of the 15 taps.
// m: plane i-1, z: plane i, p: plane i+1; offsets (dj, dk).
struct Taps {
  float m_mm, m_mp, m_zp, m_pp;  // (j-1,k-1) (j-1,k+1) (j,k+1) (j+1,k+1) in plane i-1
  float z_mz, z_zz, z_pz;        // (j-1,k) (j,k) (j+1,k) in plane i
  float p_mm, p_mp, p_zp, p_pp;  // same as m_* in plane i+1
};

__device__ __forceinline__ float eval15(const Taps& t) {
  return c11 * t.m_mm + c13 * t.p_mm + c21 * t.m_mm + c23 * t.p_mm + c31 * t.m_mm + c33 * t.p_mm + c12 * t.z_mz +
         c22 * t.z_zz + c32 * t.z_pz + c11 * t.m_mp + c13 * t.p_mp + c21 * t.m_zp + c23 * t.p_zp + c31 * t.m_pp +
         c33 * t.p_pp;
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) conv3d_s0(const float* A, float* B, int ni, int nj, int nk, int i) {
  constexpr Knobs K = kTab.v[V];
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int kk = (blockIdx.x * blockDim.x + threadIdx.x) * (K.vec ? 4 : 1);
#pragma unroll
  for (int e = 0; e < (K.vec ? 4 : 1); ++e) {
    const int k = kk + e;
    if ((i < (ni - 1)) && (j < (nj - 1)) && (k < (nk - 1)) && (i > 0) && (j > 0) && (k > 0)) {
      if constexpr (K.lsr) {
        const float* m = A + ((size_t)(i - 1) * nj + j) * nk + k;
        const float* z = m + (size_t)nj * nk;
        const float* p = z + (size_t)nj * nk;
        Taps t{m[-nk - 1], m[-nk + 1], m[1], m[nk + 1], z[-nk], z[0], z[nk], p[-nk - 1], p[-nk + 1], p[1], p[nk + 1]};
        B[((size_t)i * nj + j) * nk + k] = eval15(t);
      } else {
        B[i * (nk * nj) + j * nk + k] =
            c11 * A[(i - 1) * (nk * nj) + (j - 1) * nk + (k - 1)] + c13 * A[(i + 1) * (nk * nj) + (j - 1) * nk + (k - 1)] +
            c21 * A[(i - 1) * (nk * nj) + (j - 1) * nk + (k - 1)] + c23 * A[(i + 1) * (nk * nj) + (j - 1) * nk + (k - 1)] +
            c31 * A[(i - 1) * (nk * nj) + (j - 1) * nk + (k - 1)] + c33 * A[(i + 1) * (nk * nj) + (j - 1) * nk + (k - 1)] +
            c12 * A[(i + 0) * (nk * nj) + (j - 1) * nk + (k + 0)] + c22 * A[(i + 0) * (nk * nj) + (j + 0) * nk + (k + 0)] +
            c32 * A[(i + 0) * (nk * nj) + (j + 1) * nk + (k + 0)] + c11 * A[(i - 1) * (nk * nj) + (j - 1) * nk + (k + 1)] +
            c13 * A[(i + 1) * (nk * nj) + (j - 1) * nk + (k + 1)] + c21 * A[(i - 1) * (nk * nj) + (j + 0) * nk + (k + 1)] +
            c23 * A[(i + 1) * (nk * nj) + (j + 0) * nk + (k + 1)] + c31 * A[(i - 1) * (nk * nj) + (j + 1) * nk + (k + 1)] +
            c33 * A[(i + 1) * (nk * nj) + (j + 1) * nk + (k + 1)];
      }
    }
  }
}

// The 7 distinct (j, k) taps of one plane for output column (j, k).
struct Plane7 {
  float mm, mp, zp, pp, mz, zz, pz;
};

__device__ __forceinline__ Plane7 load_plane(const float* __restrict__ A, size_t base, int nk) {
  // base = index of (plane, j, k)
  return Plane7{__ldg(A + base - nk - 1), __ldg(A + base - nk + 1), __ldg(A + base + 1), __ldg(A + base + nk + 1),
                __ldg(A + base - nk), __ldg(A + base), __ldg(A + base + nk)};
}

// planes per CTA in the streaming kernels (i split into chunks for parallelism)
constexpr int kChunk = 16;

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) conv3d_s1(const float* __restrict__ A, float* __restrict__ B, int ni, int nj,
                                                 int nk) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (j <= 0 || j >= nj - 1 || k <= 0 || k >= nk - 1) return;
  const size_t plane = (size_t)nj * nk;
  const size_t col = (size_t)j * nk + k;
  const int i0 = 1 + blockIdx.z * kChunk, i1 = min(ni - 1, i0 + kChunk);
  Plane7 pm = load_plane(A, (size_t)(i0 - 1) * plane + col, nk);
  Plane7 pz = load_plane(A, (size_t)i0 * plane + col, nk);
  for (int i = i0; i < i1; ++i) {
    const Plane7 pp = load_plane(A, (size_t)(i + 1) * plane + col, nk);
    Taps t{pm.mm, pm.mp, pm.zp, pm.pp, pz.mz, pz.zz, pz.pz, pp.mm, pp.mp, pp.zp, pp.pp};
    B[(size_t)i * plane + col] = eval15(t);
    pm = pz;
    pz = pp;
  }
}

// 4 consecutive k per thread: per plane row offset dj, a float4 at k0 plus the
// k0-1 and k0+4 halo scalars.
struct Row6 {
  float v[6];  // k0-1 .. k0+4
};

__device__ __forceinline__ Row6 load_row6(const float* __restrict__ A, size_t rowbase, int k0, int nk) {
  Row6 r;
  const float4 c = __ldg(reinterpret_cast<const float4*>(A + rowbase + k0));
  r.v[0] = k0 > 0 ? __ldg(A + rowbase + k0 - 1) : 0.f;
  r.v[1] = c.x;
  r.v[2] = c.y;
  r.v[3] = c.z;
  r.v[4] = c.w;
  r.v[5] = k0 + 4 < nk ? __ldg(A + rowbase + k0 + 4) : 0.f;
  return r;
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(128) conv3d_s2(const float* __restrict__ A, float* __restrict__ B, int ni, int nj,
                                                 int nk) {
  const int k0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (j <= 0 || j >= nj - 1 || k0 >= nk) return;
  const size_t plane = (size_t)nj * nk;
  const int i0 = 1 + blockIdx.z * kChunk, i1 = min(ni - 1, i0 + kChunk);
  // rows (j-1, j, j+1) of planes i-1 and i
  Row6 m[3], z[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    m[d] = load_row6(A, (size_t)(i0 - 1) * plane + (size_t)(j - 1 + d) * nk, k0, nk);
    z[d] = load_row6(A, (size_t)i0 * plane + (size_t)(j - 1 + d) * nk, k0, nk);
  }
  // plane i+1 rows are prefetched one iteration ahead (plane i+2 requested
  // while plane i is computed): two planes of loads in flight per thread
  Row6 p[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) p[d] = load_row6(A, (size_t)(i0 + 1) * plane + (size_t)(j - 1 + d) * nk, k0, nk);
  for (int i = i0; i < i1; ++i) {
    Row6 q[3];
    if (i + 2 < ni) {
#pragma unroll
      for (int d = 0; d < 3; ++d) q[d] = load_row6(A, (size_t)(i + 2) * plane + (size_t)(j - 1 + d) * nk, k0, nk);
    }
    float out[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // output k = k0 + e -> index e+1 in Row6; k-1 -> e, k+1 -> e+2
      Taps t{m[0].v[e], m[0].v[e + 2], m[1].v[e + 2], m[2].v[e + 2], z[0].v[e + 1], z[1].v[e + 1], z[2].v[e + 1],
             p[0].v[e], p[0].v[e + 2], p[1].v[e + 2], p[2].v[e + 2]};
      out[e] = eval15(t);
    }
    float* brow = B + (size_t)i * plane + (size_t)j * nk;
    if (k0 > 0 && k0 + 4 < nk) {
      __stcs(reinterpret_cast<float4*>(brow + k0), make_float4(out[0], out[1], out[2], out[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (k0 + e > 0 && k0 + e < nk - 1) brow[k0 + e] = out[e];
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      m[d] = z[d];
      z[d] = p[d];
      p[d] = q[d];
    }
  }
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int ni = (int)ws.dims.d[0], nj = (int)ws.dims.d[1], nk = (int)ws.dims.d[2];
    const float* A = ws.a.p[0];
    float* B = ws.a.p[1];
    if constexpr (K.stage == 0) {
      dim3 block(kBX, kBY), grid(cdiv(nk, kBX * (K.vec ? 4 : 1)), cdiv(nj, kBY));
      for (int i = 1; i < ni - 1; ++i) conv3d_s0<B_3DCONV, V><<<grid, block, 0, s>>>(A, B, ni, nj, nk, i);
    } else if constexpr (K.stage == 1) {
      conv3d_s1<B_3DCONV, V><<<dim3(cdiv(nk, 32), cdiv(nj, 8), cdiv(ni - 2, kChunk)), dim3(32, 8), 0, s>>>(A, B, ni, nj,
                                                                                                    nk);
    } else {
      conv3d_s2<B_3DCONV, V><<<dim3(cdiv(nk, 4 * 32), cdiv(nj, 4), cdiv(ni - 2, kChunk)), dim3(32, 4), 0, s>>>(
          A, B, ni, nj, nk);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int, const Dims& d) { return d.d[0] * d.d[1] * d.d[2]; }
int64_t launches(int v, const Dims& d) { return kTab.v[v].stage == 0 ? std::max<int64_t>(d.d[0] - 2, 0) : 1; }
double alg_bytes(const Dims& d) {
  return 4.0 * ((double)d.d[0] * d.d[1] * d.d[2] + (double)(d.d[0] - 2) * (d.d[1] - 2) * (d.d[2] - 2));
}
double alg_flops(const Dims& d) { return 29.0 * (double)(d.d[0] - 2) * (d.d[1] - 2) * (d.d[2] - 2); }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if ((k.vec || k.stage == 2) && d.d[2] % 4) return 1;
  if (d.d[0] < 3 || d.d[1] < 3 || d.d[2] < 3) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "3DCONV", 3, {"ni", "nj", "nk"}, 2,
    {{"A", IN, 0}, {"B", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_3DCONV, &kDesc);

}  // namespace
}  // namespace pf
