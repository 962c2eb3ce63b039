// 3xFP16 operand preparation for the tcgen05 contractions (kind::f16).
//
// Why: kind::f16 runs at twice the kind::tf32 rate and a 16-bit operand tile
// holds twice the K depth per shared-memory byte, so the same three-product
// split that holds fp32 tolerance costs half the tensor-core time and half the
// operand traffic.
//
// Split: s = 2^e per operand group with max|x| * s in [2^14, 2^15), then
//   hi = fp16_rn(x s),  lo = fp16_rn(x s - hi)
// x s is exact (power of two), |x s - hi| <= 2^-11 |x s|, and lo carries
// the next 11 bits, so hi + lo = x s to 2^-22 relative -- the same 22
// operand bits as 3xTF32 (whose lo is truncated to TF32 by the tensor core).
// Elements below 2^-17 max|x| lose low bits of lo to fp16 subnormals; their
// absolute error stays below 2^-40 max|x|.  The product is accumulated as
// lo*hi + hi*lo + hi*hi in the fp32 TMEM accumulator and the epilogue
// multiplies alpha by 1 / (sA sB) (exact).
//
// Launches per contraction: f16_absmax (every operand, one arrival counter,
// the last block turns the maxima into the scales) and f16_split (every
// distinct operand: K-major rows converted in place order, MN-major operands
// transposed through shared memory into K-major images).
#pragma once
#include "pf_common.cuh"
#include "tc_gemm.cuh"

#include <cuda_fp16.h>

#include <algorithm>

namespace pf {
namespace f16op {

constexpr int kMaxOps = 4;

struct Op {
  const float* x;  // storage: mn ? K rows x R cols : R rows x K cols, pitch ld (floats)
  int mn;
  int R, K, ld;
  __half* hi;      // image: R rows x K halfs, pitch kp
  __half* lo;
  int grp;         // scale group (0 or 1)
};

struct Ops {
  Op op[kMaxOps];
  int n;
  int kp;
  float* partial;  // [n][gridDim.x] block maxima
  unsigned* counter;
  float* scale;    // [2]
};

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;  // valid in warp 0
}

// power-of-two scale: max|x| s in [2^14, 2^15)
__device__ __forceinline__ float scale_of(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 1.f;
  int ex;
  frexpf(amax, &ex);  // amax = f 2^ex, f in [0.5, 1)
  return ldexpf(1.f, 15 - ex);
}

// blockIdx.y = operand; grid-stride over its storage rectangle
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) f16_absmax(const Ops ops) {
  __shared__ float red[8];
  __shared__ bool last;
  const Op& o = ops.op[blockIdx.y];
  const int rows = o.mn ? o.K : o.R, cols = o.mn ? o.R : o.K;
  float m = 0.f;
  const bool vec = (o.ld % 4 == 0) && (cols % 4 == 0) && (reinterpret_cast<uintptr_t>(o.x) % 16 == 0);
  if (vec) {
    const int c4 = cols / 4;
    const int64_t n4 = (int64_t)rows * c4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / c4, c = i % c4;
      const float4 v = __ldg(reinterpret_cast<const float4*>(o.x + r * o.ld) + c);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  } else {
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      m = fmaxf(m, fabsf(__ldg(o.x + (i / cols) * o.ld + i % cols)));
  }
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    ops.partial[blockIdx.y * gridDim.x + blockIdx.x] = m;
    __threadfence();
    last = atomicAdd(ops.counter, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: per-group maxima -> scales; reset the counter for the next launch
  if (threadIdx.x < 32) {
    float g[2] = {0.f, 0.f};
    for (int j = 0; j < ops.n; ++j)
      for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
        const float v = __ldcg(ops.partial + j * gridDim.x + b);
        if (ops.op[j].grp) g[1] = fmaxf(g[1], v); else g[0] = fmaxf(g[0], v);
      }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) g[q] = fmaxf(g[q], __shfl_xor_sync(0xffffffffu, g[q], s));
    if (threadIdx.x == 0) {
      ops.scale[0] = scale_of(g[0]);
      ops.scale[1] = scale_of(g[1]);
      atomicExch(ops.counter, 0u);
    }
  }
}

__device__ __forceinline__ void split1(float x, float s, __half& h, __half& l) {
  const float y = x * s;
  h = __float2half_rn(y);
  l = __float2half_rn(y - __half2float(h));
}

// blockIdx.y = operand.  K-major: each warp converts rows, 4 floats per lane
// per step.  MN-major: 64 (k) x 64 (r) tiles transposed through shared memory.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) f16_split(const Ops ops) {
  __shared__ float t[64][65];
  const Op& o = ops.op[blockIdx.y];
  if (!o.hi) return;  // duplicate operand: its image is written by an earlier slot
  const float s = __ldcg(ops.scale + o.grp);
  const int kp = ops.kp;
  if (!o.mn) {
    const bool vec = (o.ld % 4 == 0) && (o.K % 4 == 0) && (reinterpret_cast<uintptr_t>(o.x) % 16 == 0);
    const int warps = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = blockIdx.x * warps + w; r < o.R; r += gridDim.x * warps) {
      const float* row = o.x + (size_t)r * o.ld;
      __half* hrow = o.hi + (size_t)r * kp;
      __half* lrow = o.lo + (size_t)r * kp;
      if (vec) {
        for (int k = 4 * lane; k < o.K; k += 128) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(row + k));
          __half h[4], l[4];
          split1(v.x, s, h[0], l[0]);
          split1(v.y, s, h[1], l[1]);
          split1(v.z, s, h[2], l[2]);
          split1(v.w, s, h[3], l[3]);
          *reinterpret_cast<uint2*>(hrow + k) = *reinterpret_cast<const uint2*>(h);
          *reinterpret_cast<uint2*>(lrow + k) = *reinterpret_cast<const uint2*>(l);
        }
      } else {
        for (int k = lane; k < o.K; k += 32) split1(__ldg(row + k), s, hrow[k], lrow[k]);
      }
    }
    return;
  }
  // MN-major storage X[k][r] -> image[r][k]
  const int tk = (o.K + 63) / 64, tr = (o.R + 63) / 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (int tile = blockIdx.x; tile < tk * tr; tile += gridDim.x) {
    const int k0 = (tile / tr) * 64, r0 = (tile % tr) * 64;
#pragma unroll 4
    for (int q = ty; q < 64; q += 4) {
      const int k = k0 + q, r = r0 + tx;
      t[q][tx] = (k < o.K && r < o.R) ? __ldg(o.x + (size_t)k * o.ld + r) : 0.f;
    }
    __syncthreads();
    // thread: image row r0 + q, halfs k0 + 2 tx2, +1 (32 lanes x 4 bytes = 128 B per row)
    const int tx2 = threadIdx.x & 31, ty2 = threadIdx.x >> 5;  // 32 x 8
#pragma unroll 2
    for (int q = ty2; q < 64; q += 8) {
      const int r = r0 + q, k = k0 + 2 * tx2;
      if (r < o.R && k < o.K) {
        __half2 h, l;
        split1(t[2 * tx2][q], s, h.x, l.x);
        if (k + 1 < o.K) {
          split1(t[2 * tx2 + 1][q], s, h.y, l.y);
          *reinterpret_cast<__half2*>(o.hi + (size_t)r * kp + k) = h;
          *reinterpret_cast<__half2*>(o.lo + (size_t)r * kp + k) = l;
        } else {
          o.hi[(size_t)r * kp + k] = h.x;
          o.lo[(size_t)r * kp + k] = l.x;
        }
      }
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

// Prepares the 3xFP16 images of a contraction's operands (two launches) in
// the workspace scratch and describes them in `out`.  Distinct operand
// arrays get one image each (SYRK's A serves both sides).  One scale group
// for K-concatenated products (both pairs must share sA sB), else A and B
// are scaled independently.
template <BenchId Bn, int V>
inline bool prepare_f16(Workspace& ws, const TcGemmArgs& a, F16Operands& out, cudaStream_t s) {
  const bool dual = a.A2 != nullptr;
  const int nops = dual ? 4 : 2;
  const float* ptr[4] = {a.A, a.B, a.A2, a.B2};
  const int mn[4] = {a.ta ? 1 : 0, a.tb ? 0 : 1, a.ta ? 1 : 0, a.tb ? 0 : 1};
  const int R[4] = {a.M, a.N, a.M, a.N};
  const int ld[4] = {a.lda, a.ldb, a.lda, a.ldb};
  const int kp = (a.K + 7) / 8 * 8;
  int img[4], nimg = 0, first[4];
  for (int i = 0; i < nops; ++i) {
    img[i] = -1;
    for (int j = 0; j < i; ++j)
      if (ptr[j] == ptr[i] && mn[j] == mn[i] && R[j] == R[i] && ld[j] == ld[i]) img[i] = img[j];
    if (img[i] < 0) {
      first[nimg] = i;
      img[i] = nimg++;
    }
  }
  int* flags = ws.ensure_tile_flags(s);
  if (!flags) return false;
  const int G = 2 * device_sms();
  const size_t per = ((size_t)std::max(a.M, a.N) * kp * 2 + 255) / 256 * 256;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws.ensure_scratch(2 * nimg * per + (size_t)nimg * G * 4 + 256));
  if (!base) return false;
  f16op::Ops ops;
  std::memset(&ops, 0, sizeof(ops));
  ops.n = nimg;
  ops.kp = kp;
  ops.partial = reinterpret_cast<float*>(base + 2 * nimg * per);
  ops.scale = ops.partial + (size_t)nimg * G;
  ops.counter = reinterpret_cast<unsigned*>(flags + kF16Counter);
  const bool b_own = !dual && img[1] != img[0];
  for (int q = 0; q < nimg; ++q) {
    const int i = first[q];
    f16op::Op& o = ops.op[q];
    o.x = ptr[i];
    o.mn = mn[i];
    o.R = R[i];
    o.K = a.K;
    o.ld = ld[i];
    o.hi = reinterpret_cast<__half*>(base + 2 * q * per);
    o.lo = reinterpret_cast<__half*>(base + (2 * q + 1) * per);
    o.grp = (b_own && i == 1) ? 1 : 0;
  }
  for (int i = 0; i < nops; ++i) {
    out.hi[i] = ops.op[img[i]].hi;
    out.lo[i] = ops.op[img[i]].lo;
  }
  for (int i = nops; i < 4; ++i) out.hi[i] = out.lo[i] = nullptr;
  out.kp = kp;
  out.scale = ops.scale;
  out.sb = b_own ? 1 : 0;
  f16op::f16_absmax<Bn, V><<<dim3(G, nimg), 256, 0, s>>>(ops);
  f16op::f16_split<Bn, V><<<dim3(G, nimg), 256, 0, s>>>(ops);
  return true;
}

}  // namespace pf
