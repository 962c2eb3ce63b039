// FDTD-2D (PolyBench/GPU fdtd2d.cu): 2-D Yee scheme, TMAX time steps on
// NX x NY fields ex, ey, hz.
//
// Baseline: three kernels per time step (ey update with the _fict_ source
// row, ex update, hz update), i.e. 3*TMAX launches.  Phase ordering had no
// effect on the paper's GPU.  Stage 1: one fused kernel per
// step on double-buffered fields (each thread recomputes the two neighbour
// updates hz needs), TMAX launches; stage 2: temporal blocking in registers
// (6 time steps per launch on 64 x 128 regions held in registers, 6-cell
// halo), the launch sequence captured once as a CUDA graph.  At 2048^2 the
// six 16 MiB fields stay L2-resident.
#include "pf_common.cuh"

#include <algorithm>
#include <cstdlib>

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

// ---- stage 2: temporal blocking.  A CTA loads a (64 + 2T)^2 region of the
// three fields into shared memory, advances it kTB time steps there (ey/ex
// phase, barrier, hz phase, barrier -- the per-cell arithmetic of the fused
// step), and writes back the central 64 x 64 tile, whose values depend only on
// cells inside the region: every step the valid area shrinks by at most one
// cell per side (global boundary rules need no neighbours, so they do not
// shrink).  L2 traffic per time step falls from 6 field passes to
// ~(6 * 1.27) / kTB.
// kTB: time steps per launch = halo width; kTR: region edge (float4 rows);
// output tile edge kTR - 2 kTB; kTBThreads threads, kTR^2 / 4 / kTBThreads
// row-quads per thread per phase
template <int kTR>
constexpr size_t tb_smem() {
  return 3ull * kTR * kTR * sizeof(float);
}

template <BenchId Bn, int V, int kTB, int kTR, int kTBThreads>
__global__ void __launch_bounds__(kTBThreads) step_tb(const float* __restrict__ fict, const float* __restrict__ ex0,
                                                      const float* __restrict__ ey0, const float* __restrict__ hz0,
                                                      float* __restrict__ ex1, float* __restrict__ ey1,
                                                      float* __restrict__ hz1, int nx, int ny, int t0, int steps) {
  constexpr int kTT = kTR - 2 * kTB;
  extern __shared__ __align__(16) float tb_smem[];
  float* sex = tb_smem;
  float* sey = sex + kTR * kTR;
  float* shz = sey + kTR * kTR;
  const int gi0 = blockIdx.y * kTT - kTB, gj0 = blockIdx.x * kTT - kTB;  // region origin (global)
  constexpr int kQ = kTR / 4;                                           // float4 per region row
  constexpr int kItems = kTR * kQ / kTBThreads;
  // ---- load (ny % 4 == 0 and gj0 % 4 == 0: a float4 is all in or all out of the domain)
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int item = threadIdx.x + kTBThreads * r, li = item / kQ, lj = 4 * (item % kQ);
    const int gi = gi0 + li, gj = gj0 + lj;
    float4 vx = make_float4(0.f, 0.f, 0.f, 0.f), vy = vx, vz = vx;
    if (gi >= 0 && gi < nx && gj >= 0 && gj < ny) {
      const size_t c = (size_t)gi * ny + gj;
      vx = __ldcg(reinterpret_cast<const float4*>(ex0 + c));
      vy = __ldcg(reinterpret_cast<const float4*>(ey0 + c));
      vz = __ldcg(reinterpret_cast<const float4*>(hz0 + c));
    }
    *reinterpret_cast<float4*>(sex + li * kTR + lj) = vx;
    *reinterpret_cast<float4*>(sey + li * kTR + lj) = vy;
    *reinterpret_cast<float4*>(shz + li * kTR + lj) = vz;
  }
  __syncthreads();
  // Cells outside the domain hold garbage after a step, but no in-domain cell
  // ever reads them (row 0 takes _fict_, column 0 keeps ex, the last row and
  // column keep hz), and region-edge garbage moves inward one cell per step.
  for (int st = 0; st < steps; ++st) {
    const float src = __ldg(fict + t0 + st);
    // ey / ex phase (reads hz only: in place)
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const int item = threadIdx.x + kTBThreads * r, li = item / kQ, lj = 4 * (item % kQ);
      const int gi = gi0 + li, gj = gj0 + lj;
      const int l = li * kTR + lj;
      const float4 h = *reinterpret_cast<const float4*>(shz + l);
      if (li > 0 || gi == 0) {
        float4 e = *reinterpret_cast<const float4*>(sey + l);
        if (gi == 0) {
          e = make_float4(src, src, src, src);
        } else {
          const float4 hu = *reinterpret_cast<const float4*>(shz + l - kTR);
          e = make_float4(upd_e(e.x, h.x, hu.x), upd_e(e.y, h.y, hu.y), upd_e(e.z, h.z, hu.z), upd_e(e.w, h.w, hu.w));
        }
        *reinterpret_cast<float4*>(sey + l) = e;
      }
      if (lj > 0 || gj > 0) {
        float4 x = *reinterpret_cast<const float4*>(sex + l);
        const float hl = lj > 0 ? shz[l - 1] : 0.f;  // lj == 0 < gj: region edge, garbage allowed
        const float nx0 = gj == 0 ? x.x : upd_e(x.x, h.x, hl);
        x = make_float4(nx0, upd_e(x.y, h.y, h.x), upd_e(x.z, h.z, h.y), upd_e(x.w, h.w, h.z));
        *reinterpret_cast<float4*>(sex + l) = x;
      }
    }
    __syncthreads();
    // hz phase (reads the new ex / ey)
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const int item = threadIdx.x + kTBThreads * r, li = item / kQ, lj = 4 * (item % kQ);
      const int gi = gi0 + li, gj = gj0 + lj;
      if (li >= kTR - 1 || gi >= nx - 1) continue;
      const int l = li * kTR + lj;
      float4 h = *reinterpret_cast<const float4*>(shz + l);
      const float4 x = *reinterpret_cast<const float4*>(sex + l);
      const float xr = lj + 4 < kTR ? sex[l + 4] : 0.f;
      const float4 e = *reinterpret_cast<const float4*>(sey + l);
      const float4 ed = *reinterpret_cast<const float4*>(sey + l + kTR);
      const float hv[4] = {h.x, h.y, h.z, h.w}, xv[5] = {x.x, x.y, x.z, x.w, xr};
      const float ev[4] = {e.x, e.y, e.z, e.w}, edv[4] = {ed.x, ed.y, ed.z, ed.w};
      float o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        o[q] = gj + q < ny - 1 ? upd_h(hv[q], xv[q + 1], xv[q], edv[q], ev[q]) : hv[q];
      h = make_float4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<float4*>(shz + l) = h;
    }
    __syncthreads();
  }
  // ---- store the central tile
  constexpr int kT4 = kTT / 4;
  for (int idx = threadIdx.x; idx < kTT * kT4; idx += kTBThreads) {
    const int oi = idx / kT4, oj = 4 * (idx % kT4);
    const int gi = gi0 + kTB + oi, gj = gj0 + kTB + oj;
    if (gi >= nx || gj >= ny) continue;
    const int l = (kTB + oi) * kTR + kTB + oj;
    const size_t c = (size_t)gi * ny + gj;
    __stcg(reinterpret_cast<float4*>(ex1 + c), *reinterpret_cast<const float4*>(sex + l));
    __stcg(reinterpret_cast<float4*>(ey1 + c), *reinterpret_cast<const float4*>(sey + l));
    __stcg(reinterpret_cast<float4*>(hz1 + c), *reinterpret_cast<const float4*>(shz + l));
  }
}

template <BenchId Bn, int V, int kTB, int kTR, int kTBThreads>
void tb_sequence(Workspace& ws, cudaStream_t s) {
  constexpr int kTT = kTR - 2 * kTB;
  constexpr size_t smem = tb_smem<kTR>();
  const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1], tmax = (int)ws.dims.d[2];
  const size_t n = (size_t)nx * ny;
  float* scratch = ws.ensure_scratch(3 * n * sizeof(float));
  if (!scratch) {
    launch_failed("FDTD-2D: double-buffer allocation failed");
    return;
  }
  float* buf[2][3] = {{ws.a.p[1], ws.a.p[2], ws.a.p[3]}, {scratch, scratch + n, scratch + 2 * n}};
  set_smem_attr((const void*)step_tb<Bn, V, kTB, kTR, kTBThreads>, (int)smem);
  const dim3 grid(cdiv(ny, kTT), cdiv(nx, kTT));
  int launches = 0;
  for (int t = 0; t < tmax; t += kTB, ++launches) {
    float** src = buf[launches & 1];
    float** dst = buf[(launches + 1) & 1];
    step_tb<Bn, V, kTB, kTR, kTBThreads><<<grid, kTBThreads, smem, s>>>(
        ws.a.p[0], src[0], src[1], src[2], dst[0], dst[1], dst[2], nx, ny, t, std::min(kTB, tmax - t));
  }
  if (launches & 1)
    for (int f = 0; f < 3; ++f) cudaMemcpyAsync(buf[0][f], buf[1][f], n * sizeof(float), cudaMemcpyDeviceToDevice, s);
}

// ---- stage 2, register-tiled temporal blocking.  A 128-thread CTA holds a
// 32-row x 128-column region of the three fields in REGISTERS: warp w owns
// rows 8w .. 8w+7, lane l columns 4l .. 4l+3 (one float4 per row and field).
// Neighbours along j come from the adjacent lane (shuffles), along i from the
// thread's own registers, and across warps from one shared row per warp and
// field (hz's last row before the ey/ex phase, ey's first row before the hz
// phase): two block barriers per time step and no per-cell shared-memory
// traffic.  kRT steps per launch.  A region edge is wrong after one step and
// the error advances one row and one column per step (ey/hz couple rows i-1/i+1,
// ex/hz columns j-1/j+1), so the halo is kRT rows and kH = ceil(kRT/4) float4s
// of columns per side: the CTA writes rows kRT .. kRows-1-kRT and lanes
// kH .. 31-kH, i.e. 128 - 8*kH columns per column tile.
template <BenchId Bn, int V, int kRT, int kW>
__global__ void __launch_bounds__(32 * kW) step_rt(const float* __restrict__ fict, const float* __restrict__ ex0,
                                               const float* __restrict__ ey0, const float* __restrict__ hz0,
                                               float* __restrict__ ex1, float* __restrict__ ey1,
                                               float* __restrict__ hz1, int nx, int ny, int t0, int steps) {
  constexpr int kR = 8, kRows = kR * kW, kOutRows = kRows - 2 * kRT;
  constexpr int kH = (kRT + 3) / 4, kCols = 128 - 8 * kH;
  __shared__ float4 hz_last[kW][32], ey_first[kW][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi0 = blockIdx.y * kOutRows - kRT + warp * kR;  // global row of this thread's r = 0
  const int gj = blockIdx.x * kCols - 4 * kH + 4 * lane;   // global column of this thread's c = 0
  const bool col_in = gj >= 0 && gj < ny;                    // ny % 4 == 0: a float4 is all in or all out
  float ex[kR][4], ey[kR][4], hz[kR][4];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int gi = gi0 + r;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a;
    if (col_in && gi >= 0 && gi < nx) {
      const size_t o = (size_t)gi * ny + gj;
      a = __ldcg(reinterpret_cast<const float4*>(ex0 + o));
      b = __ldcg(reinterpret_cast<const float4*>(ey0 + o));
      c = __ldcg(reinterpret_cast<const float4*>(hz0 + o));
    }
    ex[r][0] = a.x, ex[r][1] = a.y, ex[r][2] = a.z, ex[r][3] = a.w;
    ey[r][0] = b.x, ey[r][1] = b.y, ey[r][2] = b.z, ey[r][3] = b.w;
    hz[r][0] = c.x, hz[r][1] = c.y, hz[r][2] = c.z, hz[r][3] = c.w;
  }
  for (int st = 0; st < steps; ++st) {
    const float src = __ldg(fict + t0 + st);
    // hz row above this warp's first row (region edge for warp 0: garbage allowed)
    hz_last[warp][lane] = make_float4(hz[kR - 1][0], hz[kR - 1][1], hz[kR - 1][2], hz[kR - 1][3]);
    __syncthreads();
    const float4 hu = warp > 0 ? hz_last[warp - 1][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    // ey / ex phase
#pragma unroll
    for (int r = kR - 1; r >= 0; --r) {  // bottom-up: hz is not modified here, order is free
      const int gi = gi0 + r;
      const float up[4] = {r > 0 ? hz[r - 1][0] : hu.x, r > 0 ? hz[r - 1][1] : hu.y, r > 0 ? hz[r - 1][2] : hu.z,
                           r > 0 ? hz[r - 1][3] : hu.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) ey[r][c] = gi == 0 ? src : upd_e(ey[r][c], hz[r][c], up[c]);
      const float hl = __shfl_up_sync(0xffffffffu, hz[r][3], 1);  // lane 0: region edge
      ex[r][0] = gj == 0 ? ex[r][0] : upd_e(ex[r][0], hz[r][0], hl);
#pragma unroll
      for (int c = 1; c < 4; ++c) ex[r][c] = upd_e(ex[r][c], hz[r][c], hz[r][c - 1]);
    }
    // ey row below this warp's last row (region edge for warp 3)
    ey_first[warp][lane] = make_float4(ey[0][0], ey[0][1], ey[0][2], ey[0][3]);
    __syncthreads();
    const float4 ed = warp < kW - 1 ? ey_first[warp + 1][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    // hz phase
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int gi = gi0 + r;
      const float down[4] = {r < kR - 1 ? ey[r + 1][0] : ed.x, r < kR - 1 ? ey[r + 1][1] : ed.y,
                             r < kR - 1 ? ey[r + 1][2] : ed.z, r < kR - 1 ? ey[r + 1][3] : ed.w};
      const float xr = __shfl_down_sync(0xffffffffu, ex[r][0], 1);  // lane 31: region edge
      if (gi < nx - 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float xn = c < 3 ? ex[r][c + 1] : xr;
          if (gj + c < ny - 1) hz[r][c] = upd_h(hz[r][c], xn, ex[r][c], down[c], ey[r][c]);
        }
      }
    }
  }
  // ---- store rows kRT .. kRows-1-kRT of the region, lanes kH .. 31-kH
  if (lane < kH || lane > 31 - kH || !col_in) return;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int lr = warp * kR + r, gi = gi0 + r;
    if (lr < kRT || lr >= kRows - kRT || gi < 0 || gi >= nx) continue;
    const size_t o = (size_t)gi * ny + gj;
    __stcg(reinterpret_cast<float4*>(ex1 + o), make_float4(ex[r][0], ex[r][1], ex[r][2], ex[r][3]));
    __stcg(reinterpret_cast<float4*>(ey1 + o), make_float4(ey[r][0], ey[r][1], ey[r][2], ey[r][3]));
    __stcg(reinterpret_cast<float4*>(hz1 + o), make_float4(hz[r][0], hz[r][1], hz[r][2], hz[r][3]));
  }
}

template <BenchId Bn, int V, int kRT, int kW>
void rt_sequence(Workspace& ws, cudaStream_t s) {
  const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1], tmax = (int)ws.dims.d[2];
  const size_t n = (size_t)nx * ny;
  float* scratch = ws.ensure_scratch(3 * n * sizeof(float));
  if (!scratch) {
    launch_failed("FDTD-2D: double-buffer allocation failed");
    return;
  }
  float* buf[2][3] = {{ws.a.p[1], ws.a.p[2], ws.a.p[3]}, {scratch, scratch + n, scratch + 2 * n}};
  constexpr int kCols = 128 - 8 * ((kRT + 3) / 4);
  const dim3 grid(cdiv(ny, kCols), cdiv(nx, 8 * kW - 2 * kRT));
  int launches = 0;
  for (int t = 0; t < tmax; t += kRT, ++launches) {
    float** src = buf[launches & 1];
    float** dst = buf[(launches + 1) & 1];
    step_rt<Bn, V, kRT, kW><<<grid, 32 * kW, 0, s>>>(ws.a.p[0], src[0], src[1], src[2], dst[0], dst[1], dst[2], nx, ny, t,
                                            std::min(kRT, tmax - t));
  }
  if (launches & 1)
    for (int f = 0; f < 3; ++f) cudaMemcpyAsync(buf[0][f], buf[1][f], n * sizeof(float), cudaMemcpyDeviceToDevice, s);
}

// Stage 2 = the register-tiled temporal blocking (kRTSteps time steps per
// launch on (8*kRTWarps)-row x 128-column register regions).  Measured on
// B200 for 2048^2 x 500 steps with the ceil(steps/4)-float4 column halo
// (round 2; round 1's one-float4 halo was only correct up to 4 steps): 4/6/8/
// 10/12 steps x 8 warps 2.81/2.32/2.12/-/- ms, 8/10/12 steps x 16 warps
// 2.50/2.20/2.06 ms; the shared-memory blocking (64x64 regions, 4 steps,
// PF_FDTD_TB=4) 5.77 ms and the per-step fused sequence (PF_FDTD_TB=0)
// 6.16 ms.
constexpr int kRTSteps = 12, kRTWarps = 16;
inline int fdtd_tb_depth() {
  static const int d = [] {
    const char* e = std::getenv("PF_FDTD_TB");
    const int v = e ? std::atoi(e) : -1;
    return (v == 0 || v == 4) ? v : -1;
  }();
  return d;
}
// register-tiled steps per launch and warps per CTA (A/B switches
// PF_FDTD_RT=4|6|8|10|12, PF_FDTD_RW=8|16; defaults kRTSteps, kRTWarps)
inline int fdtd_rt_steps() {
  static const int d = [] {
    const char* e = std::getenv("PF_FDTD_RT");
    const int v = e ? std::atoi(e) : kRTSteps;
    return (v == 4 || v == 6 || v == 8 || v == 10 || v == 12) ? v : kRTSteps;
  }();
  return d;
}
inline int fdtd_rt_warps() {
  static const int w = [] {
    const char* e = std::getenv("PF_FDTD_RW");
    const int v = e ? std::atoi(e) : kRTWarps;
    return (v == 8 || v == 16) ? v : kRTWarps;
  }();
  return w;
}
template <BenchId Bn, int V, int kW>
cudaGraphExec_t rt_graph(Workspace& ws) {
  switch (fdtd_rt_steps()) {
    case 4: return cached_graph(ws, V, &rt_sequence<Bn, V, 4, kW>);
    case 6: return cached_graph(ws, V, &rt_sequence<Bn, V, 6, kW>);
    case 10: return cached_graph(ws, V, &rt_sequence<Bn, V, 10, kW>);
    case 12: return cached_graph(ws, V, &rt_sequence<Bn, V, 12, kW>);
    default: return cached_graph(ws, V, &rt_sequence<Bn, V, 8, kW>);
  }
}
// time steps per stage-2 launch
inline int fdtd_steps_per_launch() {
  const int d = fdtd_tb_depth();
  return d == 0 ? 1 : d == 4 ? 4 : fdtd_rt_steps();
}
inline bool fdtd_tb_disabled() { return fdtd_tb_depth() == 0; }

template <BenchId Bn, int V>
void fused_sequence(Workspace& ws, cudaStream_t s) {
  const int nx = (int)ws.dims.d[0], ny = (int)ws.dims.d[1], tmax = (int)ws.dims.d[2];
  const size_t n = (size_t)nx * ny;
  float* scratch = ws.ensure_scratch(3 * n * sizeof(float));
  if (!scratch) {
    launch_failed("FDTD-2D: double-buffer allocation failed");
    return;
  }
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
      const bool tb = ny % 4 == 0 && !fdtd_tb_disabled();
      const int d = fdtd_tb_depth();
      cudaGraphExec_t g = !tb      ? cached_graph(ws, V + 1000, &fused_sequence<B_FDTD2D, V>)
                          : d == 4 ? cached_graph(ws, V + 2000, &tb_sequence<B_FDTD2D, V, 4, 64, 256>)
                          : fdtd_rt_warps() == 16 ? rt_graph<B_FDTD2D, V, 16>(ws)
                                                  : rt_graph<B_FDTD2D, V, 8>(ws);
      cudaGraphLaunch(g, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) { return a == 0 ? d.d[2] : d.d[0] * d.d[1]; }
int64_t launches(int v, const Dims& d) {
  const int st = kTab.v[v].stage;
  if (st == 2 && d.d[1] % 4 == 0 && !fdtd_tb_disabled()) {
    const int steps = fdtd_steps_per_launch();
    return (d.d[2] + steps - 1) / steps;
  }
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
