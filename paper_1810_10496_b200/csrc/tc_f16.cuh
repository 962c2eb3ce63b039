// 3xFP16 operand preparation for the tcgen05 contractions (kind::f16).
//
// Why: kind::f16 runs at twice the kind::tf32 rate and a 16-bit operand tile
// holds twice the K depth per shared-memory byte, so the same three-product
// split that holds fp32 tolerance costs half the tensor-core time and half the
// operand traffic.
//
// Split, per operand ROW (a row of op(A) or of op(B)^T: one output row /
// column): s = 2^e with max|x_row| s in [2^14, 2^15), then
//   hi = fp16_rn(x s),  lo = fp16_rn(x s - hi)
// x s is exact (power of two), |x s - hi| <= 2^-11 |x s|, and lo carries
// the next 11 bits, so hi + lo = x s to 2^-22 relative -- the same 22
// operand bits as 3xTF32 (whose lo is truncated to TF32 by the tensor core).
// Elements below 2^-17 of their row's max lose low bits of lo to fp16
// subnormals; their absolute error stays below 2^-39 of the row max.  The
// product accumulates lo*hi + hi*lo + hi*hi in the fp32 TMEM accumulator and
// the epilogue multiplies by alpha / (s_row s_col), exactly (powers of two).
// Per-row scales need no global reduction: a K-major row is scaled by the
// warp that converts it, an MN-major column by the CTA that holds its strip;
// MN-major operands with K > kStripMaxK (or unaligned) take a second launch
// (column maxima of 32-row blocks, then 64 x 64 tiles transposed).  K-concatenated products (SYR2K: A B^T + B A^T)
// share one scale per row index across both arrays, so both pairs carry the
// same s_i s_j.
#pragma once
#include "pf_common.cuh"
#include "tc_gemm.cuh"

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace pf {
namespace f16op {

constexpr int kMaxOps = 4;

struct Op {
  const float* x;   // storage: mn ? K rows x R cols : R rows x K cols, pitch ld (floats)
  const float* x2;  // K-major only: second array sharing the row scales (K-concatenated pair), or nullptr
  int mn;
  int R, K, ld;
  __half* hi;       // image: R rows x K halfs, pitch kp
  __half* lo;
  __half* hi2;      // image of x2
  __half* lo2;
  float* rinv;      // [R] 1 / s_row
  float* part;      // MN-major: per-64-row-block column maxima [ceil(K / 64)][R]
};

struct Ops {
  Op op[kMaxOps];
  int n;
  int kp;
  int strips;  // MN-major operands as shared-memory strips (else column maxima + transposed tiles)
  // optional beta pre-pass riding along in the blockIdx.y == n slice: D = beta * Cin (zeros without Cin)
  float4* pre_d;
  const float4* pre_c;
  int64_t pre_n4;
  float pre_beta;
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) v = warp_max(lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f);
  return v;  // valid in warp 0
}

// power-of-two scale: max|x| s in [2^14, 2^15)
__device__ __forceinline__ float scale_of(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 1.f;
  int ex;
  frexpf(amax, &ex);  // amax = f 2^ex, f in [0.5, 1)
  return ldexpf(1.f, 15 - ex);
}

__device__ __forceinline__ void split1(float x, float s, __half& h, __half& l) {
  const float y = x * s;
  h = __float2half_rn(y);
  l = __float2half_rn(y - __half2float(h));
}

__device__ __forceinline__ float amax4(float4 v) {
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

__device__ __forceinline__ void store4(__half* hi, __half* lo, float4 v, float s) {
  __half h[4], l[4];
  split1(v.x, s, h[0], l[0]);
  split1(v.y, s, h[1], l[1]);
  split1(v.z, s, h[2], l[2]);
  split1(v.w, s, h[3], l[3]);
  *reinterpret_cast<uint2*>(hi) = *reinterpret_cast<const uint2*>(h);
  *reinterpret_cast<uint2*>(lo) = *reinterpret_cast<const uint2*>(l);
}

// K-major row r of op (and of x2): warp-cooperative, 2048-float chunks with
// 16 float4 loads per lane in flight.  Rows of up to 2048 floats stay in
// registers between the max and the conversion; longer rows are read twice
// (max pass, then a conversion pass that hits L2).
template <bool kDual>
__device__ __forceinline__ void load_chunk(const Op& o, const float* row, const float* row2, int k0, int lane,
                                           float4 (&v)[16], float4 (&v2)[16]) {
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int k = k0 + 4 * lane + 128 * u;
    v[u] = k < o.K ? __ldg(reinterpret_cast<const float4*>(row + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (kDual)
      v2[u] = k < o.K ? __ldg(reinterpret_cast<const float4*>(row2 + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <bool kDual>
__device__ __forceinline__ void store_chunk(const Op& o, int kp, int r, int k0, int lane, float s,
                                            const float4 (&v)[16], const float4 (&v2)[16]) {
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int k = k0 + 4 * lane + 128 * u;
    if (k < o.K) {
      store4(o.hi + (size_t)r * kp + k, o.lo + (size_t)r * kp + k, v[u], s);
      if constexpr (kDual) store4(o.hi2 + (size_t)r * kp + k, o.lo2 + (size_t)r * kp + k, v2[u], s);
    }
  }
}

template <bool kDual>
__device__ __forceinline__ void split_row(const Op& o, int kp, int r, int lane) {
  const float* row = o.x + (size_t)r * o.ld;
  const float* row2 = kDual ? o.x2 + (size_t)r * o.ld : nullptr;
  const bool vec = (o.ld % 4 == 0) && (o.K % 4 == 0) && (reinterpret_cast<uintptr_t>(o.x) % 16 == 0) &&
                   (!kDual || reinterpret_cast<uintptr_t>(o.x2) % 16 == 0);
  float m = 0.f;
  if (vec) {
    float4 v[16], v2[16];
    for (int k0 = 0; k0 < o.K; k0 += 2048) {
      load_chunk<kDual>(o, row, row2, k0, lane, v, v2);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        m = fmaxf(m, amax4(v[u]));
        if constexpr (kDual) m = fmaxf(m, amax4(v2[u]));
      }
    }
    const float s = scale_of(warp_max(m));
    if (lane == 0) o.rinv[r] = 1.f / s;
    if (o.K <= 2048) {
      store_chunk<kDual>(o, kp, r, 0, lane, s, v, v2);
      return;
    }
    for (int k0 = 0; k0 < o.K; k0 += 2048) {
      load_chunk<kDual>(o, row, row2, k0, lane, v, v2);
      store_chunk<kDual>(o, kp, r, k0, lane, s, v, v2);
    }
    return;
  }
  // unaligned rows: scalar max pass, then a conversion pass
  for (int k = lane; k < o.K; k += 32) {
    m = fmaxf(m, fabsf(__ldg(row + k)));
    if constexpr (kDual) m = fmaxf(m, fabsf(__ldg(row2 + k)));
  }
  const float s = scale_of(warp_max(m));
  if (lane == 0) o.rinv[r] = 1.f / s;
  for (int k = lane; k < o.K; k += 32) {
    split1(__ldg(row + k), s, o.hi[(size_t)r * kp + k], o.lo[(size_t)r * kp + k]);
    if constexpr (kDual) split1(__ldg(row2 + k), s, o.hi2[(size_t)r * kp + k], o.lo2[(size_t)r * kp + k]);
  }
}

constexpr int kStrip = 16;  // MN-major strips: columns per CTA

// MN-major strip (K <= kStripMaxK): storage X[k][r], columns r0 .. r0+15 ->
// image rows r0 .. r0+15 (K halfs each).  The whole K x 16 strip lands in
// shared memory through 16-byte cp.async (pitch 20 floats; a warp request
// covers 8 rows x 64 B, so the load is not limited by outstanding 4-byte
// requests as the first, pitch-17 form was: 15 us for a 2048^2 operand),
// per-column max, then 256-row chunks are converted row-wise (float4 reads)
// into a transposed half buffer and leave as 16-byte stores of image rows.
constexpr int kStripMaxK = 2048;  // K * 20 * 4 + 2 * 16 * 256 * 2 bytes <= 180 KB
constexpr int kSP = 20;           // strip pitch (floats): 16-byte aligned rows
constexpr int kSC = 256;          // rows per conversion chunk
inline size_t strip_smem_bytes(int K) {
  return (size_t)K * kSP * sizeof(float) + 2 * (size_t)kStrip * (kSC + 8) * sizeof(__half);
}

__device__ __forceinline__ void split_strip(const Op& o, int kp, int r0, float* strip) {
  __shared__ float red[16][kStrip + 1];
  __shared__ float sc[kStrip];
  __half* th = reinterpret_cast<__half*>(strip + (size_t)o.K * kSP);  // [16][kSC + 8]
  __half* tl = th + kStrip * (kSC + 8);
  const int t = threadIdx.x;
  {  // load: thread (chunk q, row group g): 16 bytes at rows g, g + 64, ...
    const int q = t & 3, g = t >> 2;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(strip));
    const int valid = min(4, max(0, o.R - (r0 + 4 * q)));  // columns of this chunk inside the operand
    for (int k = g; k < o.K; k += 64) {
      const float* src = o.x + (size_t)k * o.ld + r0 + 4 * q;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sbase + 4u * (uint32_t)(k * kSP + 4 * q)),
                   "l"(valid ? src : o.x), "r"(4 * valid)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  {
    const int c = t % kStrip, g = t / kStrip;  // 16 x 16
    float m = 0.f;
#pragma unroll 4
    for (int k = g; k < o.K; k += 16) m = fmaxf(m, fabsf(strip[k * kSP + c]));
    red[g][c] = m;
  }
  __syncthreads();
  if (t < kStrip) {
    float mm = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) mm = fmaxf(mm, red[q][t]);
    const float s = scale_of(mm);
    sc[t] = s;
    if (r0 + t < o.R) o.rinv[r0 + t] = 1.f / s;
  }
  __syncthreads();
  const int q = t & 3;
  const float s0 = sc[4 * q], s1 = sc[4 * q + 1], s2 = sc[4 * q + 2], s3 = sc[4 * q + 3];
  for (int k0 = 0; k0 < o.K; k0 += kSC) {
    // row-wise conversion: thread (chunk q, row t / 4 + 64 u) -> transposed halfs
#pragma unroll
    for (int u = 0; u < kSC / 64; ++u) {
      const int kk = (t >> 2) + 64 * u, k = k0 + kk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < o.K) v = *reinterpret_cast<const float4*>(strip + k * kSP + 4 * q);
      split1(v.x, s0, th[(4 * q + 0) * (kSC + 8) + kk], tl[(4 * q + 0) * (kSC + 8) + kk]);
      split1(v.y, s1, th[(4 * q + 1) * (kSC + 8) + kk], tl[(4 * q + 1) * (kSC + 8) + kk]);
      split1(v.z, s2, th[(4 * q + 2) * (kSC + 8) + kk], tl[(4 * q + 2) * (kSC + 8) + kk]);
      split1(v.w, s3, th[(4 * q + 3) * (kSC + 8) + kk], tl[(4 * q + 3) * (kSC + 8) + kk]);
    }
    __syncthreads();
    // 16 image rows x kSC halfs per array: thread -> row t / 16, 16-byte pieces (t % 16) + 16 e
    const int rr = t / 16, piece = t % 16;
    if (r0 + rr < o.R) {
#pragma unroll
      for (int e = 0; e < kSC / 8 / 16; ++e) {
        const int kk = 8 * (piece + 16 * e), k = k0 + kk;
        if (k < o.K) {  // kp is a multiple of 8: whole 16-byte pieces stay inside the row
          *reinterpret_cast<uint4*>(o.hi + (size_t)(r0 + rr) * kp + k) =
              *reinterpret_cast<const uint4*>(th + rr * (kSC + 8) + kk);
          *reinterpret_cast<uint4*>(o.lo + (size_t)(r0 + rr) * kp + k) =
              *reinterpret_cast<const uint4*>(tl + rr * (kSC + 8) + kk);
        }
      }
    }
    __syncthreads();
  }
}

// MN-major operands with K > kStripMaxK (storage X[k][r], r contiguous) in
// two fully parallel passes: f16_split computes per-column maxima of 64-row blocks into
// partials [block][r] (thread per column, 16 loads in flight), then
// f16_tsplit converts 64 x 64 tiles: each CTA reduces its 64 columns'
// partials (fixed order), scales, splits and writes the tile transposed
// (column r -> 128-byte segment of image row r).
constexpr int kMB = 32;  // rows per partial-max block (all 32 loads of a thread in flight)

__device__ __forceinline__ void colmax_part(const Op& o, float* part, int bx, int nbx) {
  const int nb = (o.K + kMB - 1) / kMB, nc = (o.R + 255) / 256;
  for (int job = bx; job < nb * nc; job += nbx) {
    const int b = job / nc, r = (job % nc) * 256 + threadIdx.x;
    if (r >= o.R) continue;
    const int k0 = b * kMB, k1 = min(o.K, k0 + kMB);
    float m = 0.f, v[kMB];
#pragma unroll
    for (int u = 0; u < kMB; ++u) v[u] = k0 + u < k1 ? __ldg(o.x + (size_t)(k0 + u) * o.ld + r) : 0.f;
#pragma unroll
    for (int u = 0; u < kMB; ++u) m = fmaxf(m, fabsf(v[u]));
    part[(size_t)b * o.R + r] = m;
  }
}

// blockIdx.y = operand.  K-major operands: one warp per row (8 rows per
// CTA); MN-major operands: one 16-column strip per CTA.
template <BenchId Bn, int V, bool kDual>
__global__ void __launch_bounds__(256) f16_split(const Ops ops) {
  if ((int)blockIdx.y == ops.n) {  // the contraction's beta pre-pass (symmetric products), 4 loads in flight
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < ops.pre_n4; i += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ops.pre_c ? __ldg(ops.pre_c + i + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        ops.pre_d[i + u * stride] = make_float4(ops.pre_beta * v[u].x, ops.pre_beta * v[u].y,
                                                ops.pre_beta * v[u].z, ops.pre_beta * v[u].w);
    }
    for (; i < ops.pre_n4; i += stride) {
      const float4 v = ops.pre_c ? __ldg(ops.pre_c + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      ops.pre_d[i] = make_float4(ops.pre_beta * v.x, ops.pre_beta * v.y, ops.pre_beta * v.z, ops.pre_beta * v.w);
    }
    return;
  }
  const Op& o = ops.op[blockIdx.y];
  if (o.mn) {
    extern __shared__ float f16_strip[];  // strip_smem_bytes(K) when ops.strips
    if (ops.strips)
      for (int r0 = blockIdx.x * kStrip; r0 < o.R; r0 += gridDim.x * kStrip) split_strip(o, ops.kp, r0, f16_strip);
    else
      colmax_part(o, o.part, blockIdx.x, gridDim.x);  // pass 1 (f16_tsplit follows)
    return;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + w; r < o.R; r += gridDim.x * 8) split_row<kDual>(o, ops.kp, r, lane);
}

// pass 2 of the MN-major operands: blockIdx.y = operand (K-major ones exit)
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) f16_tsplit(const Ops ops) {
  const Op& o = ops.op[blockIdx.y];
  if (!o.mn) return;
  __shared__ float t[64][65];
  __shared__ float sc[64];
  __shared__ float red[64][4];
  const int tr = (o.R + 63) / 64, tk = (o.K + 63) / 64, nb = (o.K + kMB - 1) / kMB;
  for (int tile = blockIdx.x; tile < tr * tk; tile += gridDim.x) {
    const int r0 = (tile % tr) * 64, k0 = (tile / tr) * 64;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
    float v[16];  // the tile's loads go out before the partials are reduced
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int k = k0 + ty + 4 * u, r = r0 + tx;
      v[u] = (k < o.K && r < o.R) ? __ldg(o.x + (size_t)k * o.ld + r) : 0.f;
    }
    {  // column scales: 4 threads per column over the row-block partials
      const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
      float m = 0.f;
      if (r0 + c < o.R)
        for (int b0 = q; b0 < nb; b0 += 4 * 16) {  // 16 partials per thread in flight
          float pm[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) pm[u] = b0 + 4 * u < nb ? o.part[(size_t)(b0 + 4 * u) * o.R + r0 + c] : 0.f;
#pragma unroll
          for (int u = 0; u < 16; ++u) m = fmaxf(m, pm[u]);
        }
      red[c][q] = m;
      __syncthreads();
      if (threadIdx.x < 64) {
        const int cc = threadIdx.x;
        const float s = scale_of(fmaxf(fmaxf(red[cc][0], red[cc][1]), fmaxf(red[cc][2], red[cc][3])));
        sc[cc] = s;
        if (k0 == 0 && r0 + cc < o.R) o.rinv[r0 + cc] = 1.f / s;
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) t[ty + 4 * u][tx] = v[u];
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 2
    for (int cc = w; cc < 64; cc += 8) {
      const int r = r0 + cc, k = k0 + 2 * lane;
      if (r >= o.R || k >= o.K) continue;
      const float s = sc[cc];
      __half2 hh, ll;
      split1(t[2 * lane][cc], s, hh.x, ll.x);
      split1(k + 1 < o.K ? t[2 * lane + 1][cc] : 0.f, s, hh.y, ll.y);
      *reinterpret_cast<__half2*>(o.hi + (size_t)r * ops.kp + k) = hh;  // kp and k even: 4-byte aligned
      *reinterpret_cast<__half2*>(o.lo + (size_t)r * ops.kp + k) = ll;
    }
    __syncthreads();
  }
}

}  // namespace f16op

// 3xFP16 contractions: on by default for the products that run pre-split
// (PF_TC_F16=0 keeps 3xTF32 everywhere, A/B runs).
inline bool tc_f16_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PF_TC_F16");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Prepares the 3xFP16 images and per-row inverse scales of a contraction's
// operands in the workspace scratch (ONE launch) and describes them in
// `out`.  Distinct operand arrays get one image each (SYRK's A serves both
// sides); a K-concatenated product (A2, B2 = B, A: SYR2K) converts A and B
// as one paired operand with shared row scales.
// base_d: also write D = beta * Cin (flat, same shape) inside the K-major
// launch -- the beta pre-pass of a symmetric product, off the critical path
// of its own launch; the caller then marks D as based (TcGemmArgs::d_base).
template <BenchId Bn, int V>
inline bool prepare_f16(Workspace& ws, const TcGemmArgs& a, F16Operands& out, cudaStream_t s, bool base_d = false) {
  const bool dual = a.A2 != nullptr;
  if (dual && !(a.A2 == a.B && a.B2 == a.A && !a.ta && a.tb && a.M == a.N && a.lda == a.ldb))
    return false;  // only the symmetric K-concatenation (A B^T + B A^T) shares row scales
  const int kp = (a.K + 7) / 8 * 8;
  const size_t img = ((size_t)std::max(a.M, a.N) * kp * 2 + 255) / 256 * 256;
  const size_t vec = ((size_t)std::max(a.M, a.N) + 64) * sizeof(float);  // inverse scales (padded)
  const bool same = !dual && a.A == a.B && a.ta == !a.tb && a.M == a.N && a.lda == a.ldb;  // SYRK: A A^T
  const int nimg = dual ? 2 : (same ? 1 : 2);
  const size_t partb = (((size_t)(a.K + f16op::kMB - 1) / f16op::kMB) * std::max(a.M, a.N) * sizeof(float) + 255) /
                       256 * 256;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws.ensure_scratch(2 * nimg * img + 2 * vec + 2 * partb + 256));
  if (!base) return false;
  auto H = [&](int i) { return reinterpret_cast<__half*>(base + i * img); };
  float* rinv_a = reinterpret_cast<float*>(base + 2 * nimg * img);
  float* rinv_b = reinterpret_cast<float*>(base + 2 * nimg * img + vec);
  f16op::Ops ops;
  std::memset(&ops, 0, sizeof(ops));
  ops.kp = kp;
  if (dual) {  // one paired K-major operand: rows of A and B, shared scales
    f16op::Op& o = ops.op[0];
    o.x = a.A;
    o.x2 = a.B;
    o.mn = 0;
    o.R = a.M;
    o.K = a.K;
    o.ld = a.lda;
    o.hi = H(0), o.lo = H(1), o.hi2 = H(2), o.lo2 = H(3);
    o.rinv = rinv_a;
    ops.n = 1;
    out.hi[0] = H(0), out.lo[0] = H(1);  // op(A)  = A
    out.hi[1] = H(2), out.lo[1] = H(3);  // op(B)  = B
    out.hi[2] = H(2), out.lo[2] = H(3);  // op(A2) = B
    out.hi[3] = H(0), out.lo[3] = H(1);  // op(B2) = A
    out.rinv = rinv_a;
    out.cinv = rinv_a;
  } else {
    f16op::Op& oa = ops.op[0];
    oa.x = a.A, oa.mn = a.ta ? 1 : 0, oa.R = a.M, oa.K = a.K, oa.ld = a.lda;
    oa.hi = H(0), oa.lo = H(1), oa.rinv = rinv_a;
    oa.part = reinterpret_cast<float*>(base + 2 * nimg * img + 2 * vec);
    ops.n = 1;
    out.hi[0] = H(0), out.lo[0] = H(1);
    out.rinv = rinv_a;
    if (same) {
      out.hi[1] = H(0), out.lo[1] = H(1);
      out.cinv = rinv_a;
    } else {
      f16op::Op& ob = ops.op[1];
      ob.x = a.B, ob.mn = a.tb ? 0 : 1, ob.R = a.N, ob.K = a.K, ob.ld = a.ldb;
      ob.hi = H(2), ob.lo = H(3), ob.rinv = rinv_b;
      ob.part = reinterpret_cast<float*>(base + 2 * nimg * img + 2 * vec + partb);
      ops.n = 2;
      out.hi[1] = H(2), out.lo[1] = H(3);
      out.cinv = rinv_b;
    }
    out.hi[2] = out.hi[3] = out.lo[2] = out.lo[3] = nullptr;
  }
  out.kp = kp;
  const int rows = std::max(a.M, a.N);
  bool any_mn = false, any_k = false;
  for (int i = 0; i < ops.n; ++i) (ops.op[i].mn ? any_mn : any_k) = true;
  bool aligned = true;  // 16-byte cp.async of the MN-major operands
  for (int i = 0; i < ops.n; ++i)
    if (ops.op[i].mn) aligned &= reinterpret_cast<uintptr_t>(ops.op[i].x) % 16 == 0 && ops.op[i].ld % 4 == 0;
  const bool strips = any_mn && aligned && a.K <= f16op::kStripMaxK;
  ops.strips = strips ? 1 : 0;
  const int kgrid = std::min((rows + 7) / 8, 8 * device_sms());  // K-major rows: 8 per CTA
  const int pre = base_d ? 1 : 0;
  if (base_d) {
    ops.pre_d = reinterpret_cast<float4*>(a.D);
    ops.pre_c = a.beta != 0.f ? reinterpret_cast<const float4*>(a.Cin) : nullptr;  // beta = 0: zeros
    ops.pre_n4 = (int64_t)a.M * a.N / 4;
    ops.pre_beta = a.beta;
  }
  if (dual) {
    f16op::f16_split<Bn, V, true><<<dim3(kgrid, ops.n + pre), 256, 0, s>>>(ops);
    return true;
  }
  if (strips) {
    // two launches: the strips' shared memory would hold the K-major CTAs to
    // one per SM (2MM 2048: 21 us for one shared launch)
    // The two launches are independent: the K-major rows go on the
    // workspace's side stream and overlap the strips (joined before the GEMM).
    f16op::Ops km = ops, mn = ops;
    km.n = mn.n = 0;
    for (int i = 0; i < ops.n; ++i) (ops.op[i].mn ? mn.op[mn.n++] : km.op[km.n++]) = ops.op[i];
    mn.pre_n4 = 0;
    const size_t smem = f16op::strip_smem_bytes(a.K);
    set_smem_attr((const void*)f16op::f16_split<Bn, V, false>, (int)smem);
    if (km.n || pre) {
      cudaStream_t ss = ws.fork(s);
      f16op::f16_split<Bn, V, false><<<dim3(kgrid, km.n + pre), 256, 0, ss>>>(km);
    }
    f16op::f16_split<Bn, V, false><<<dim3(std::min((rows + f16op::kStrip - 1) / f16op::kStrip, 8 * device_sms()), mn.n),
                                     256, smem, s>>>(mn);
    if (km.n || pre) ws.join(s);
    return true;
  }
  // K-major rows and (for long K) the column-max pass in one launch, then the transposed tiles
  const int jobs_mn = any_mn ? (int)(((a.K + f16op::kMB - 1) / f16op::kMB) * ((rows + 255) / 256)) : 0;
  f16op::f16_split<Bn, V, false><<<dim3(std::min(std::max(kgrid, jobs_mn), 8 * device_sms()), ops.n + pre), 256, 0,
                                   s>>>(ops);
  if (any_mn) {
    const int tiles = ((rows + 63) / 64) * ((a.K + 63) / 64);
    f16op::f16_tsplit<Bn, V><<<dim3(std::min(tiles, 8 * device_sms()), ops.n), 256, 0, s>>>(ops);
  }
  (void)any_k;
  return true;
}

}  // namespace pf
