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
#include "tc_gemm.cuh"
#include "tma_map.cuh"

#include <algorithm>
#include <cstdlib>

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

// Stage 2: TMA-fed plane streaming.  A CTA walks a contiguous run of
// (column tile, plane) units -- column tile = 128 k x 16 j outputs -- and a
// producer warp streams the input planes of that run (box 136 k x 18 j with
// the halo, negative / past-the-end coordinates zero-filled by TMA) through
// a kNS-deep shared-memory ring, several planes ahead of the math.  Each
// input plane is read from shared memory once: it finishes the outputs of
// the previous plane (its p-taps), adds its z-taps to the current plane and
// starts the next plane (its m-taps).  Runs are balanced to +-1 plane over a
// grid of exactly the resident CTAs (SMs x occupancy).
constexpr int kTK = 128, kTJ = 16;          // output column tile
constexpr int kBoxK = kTK + 8, kBoxJ = kTJ + 2;  // input box: k0-4 .. k0+131, j0-1 .. j0+16
constexpr int kNS = 6;                       // planes in the ring
constexpr uint32_t kSlotBytes = (kBoxK * kBoxJ * 4 + 127) / 128 * 128;
constexpr int kConsumerWarps = kTJ / 2;      // warp w: output rows j0+2w, j0+2w+1; lane: 4 k
constexpr int kS2Threads = 32 * (kConsumerWarps + 1);

struct S2Params {
  CUtensorMap map;
  float* B;
  int ni, nj, nk;
  int tiles_k, tiles;   // column tiles along k, total column tiles
  int64_t units;        // tiles * (ni - 2)
};



template <BenchId Bn, int V>
__global__ void __launch_bounds__(kS2Threads) conv3d_s2(const __grid_constant__ S2Params p) {
  extern __shared__ __align__(128) uint8_t c3_smem[];
  __shared__ __align__(8) uint64_t full[kNS], empty[kNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int planes = p.ni - 2;
  const int64_t u0 = p.units * blockIdx.x / gridDim.x, u1 = p.units * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const uint32_t base = tc::smem_u32(c3_smem);

  if (warp == kConsumerWarps) {
    // ---- producer: every input plane of every segment of [u0, u1)
    if (lane == 0) {
      int n = 0;
      for (int64_t u = u0; u < u1;) {
        const int t = (int)(u / planes), i_begin = 1 + (int)(u % planes);
        const int i_end = (int)(i_begin + (u1 - u) < (int64_t)planes + 1 ? i_begin + (u1 - u) : (int64_t)planes + 1);  // exclusive output plane
        const int k0 = (t % p.tiles_k) * kTK, j0 = 1 + (t / p.tiles_k) * kTJ;
        for (int q = i_begin - 1; q <= i_end; ++q, ++n) {
          const int s = n % kNS;
          tc::mbar_wait(tc::smem_u32(&empty[s]), ((n / kNS) & 1) ^ 1);
          const uint32_t fb = tc::smem_u32(&full[s]);
          tc::mbar_expect_tx(fb, kBoxK * kBoxJ * 4);
          tma::load_3d(base + s * kSlotBytes, &p.map, k0 - 4, j0 - 1, q, fb);
        }
        u += i_end - i_begin;
      }
    }
    return;
  }

  // ---- consumers
  int n = 0;
  for (int64_t u = u0; u < u1;) {
    const int t = (int)(u / planes), i_begin = 1 + (int)(u % planes);
    const int i_end = (int)(i_begin + (u1 - u) < (int64_t)planes + 1 ? i_begin + (u1 - u) : (int64_t)planes + 1);
    const int k0 = (t % p.tiles_k) * kTK, j0 = 1 + (t / p.tiles_k) * kTJ;
    const int kq = k0 + 4 * lane;       // first of this thread's 4 k
    const int jr = j0 + 2 * warp;       // first of this thread's 2 rows
    float mz[2][4] = {}, mn[2][4] = {};
    for (int q = i_begin - 1; q <= i_end; ++q, ++n) {
      const int s = n % kNS;
      tc::mbar_wait(tc::smem_u32(&full[s]), (n / kNS) & 1);
      const float* slot = reinterpret_cast<const float*>(c3_smem + s * kSlotBytes);
      // rows j-1 .. j+2 of the two output rows: smem rows 2w .. 2w+3
      float v[4][6];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const float* row = slot + (2 * warp + rr) * kBoxK;
        const float4 c = *reinterpret_cast<const float4*>(row + 4 + 4 * lane);
        float left = __shfl_up_sync(0xffffffffu, c.w, 1);
        float right = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0) left = row[3];
        if (lane == 31) right = row[4 + kTK];
        v[rr][0] = left;
        v[rr][1] = c.x;
        v[rr][2] = c.y;
        v[rr][3] = c.z;
        v[rr][4] = c.w;
        v[rr][5] = right;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[s])) : "memory");
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float out[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // (j-1, k-1) (j-1, k+1) (j, k+1) (j+1, k+1) and (j-1, k) (j, k) (j+1, k)
          const float xmm = v[r][e], xmp = v[r][e + 2], xzp = v[r + 1][e + 2], xpp = v[r + 2][e + 2];
          const float xmz = v[r][e + 1], xzz = v[r + 1][e + 1], xpz = v[r + 2][e + 1];
          // folded repeated taps, 11 FMAs per output (as in the direct form)
          out[e] = fmaf(c33, xpp, fmaf(c23, xzp, fmaf(c13, xmp, fmaf(c13 + c23 + c33, xmm, mz[r][e]))));
          mz[r][e] = fmaf(c32, xpz, fmaf(c22, xzz, fmaf(c12, xmz, mn[r][e])));
          mn[r][e] = fmaf(c31, xpp, fmaf(c21, xzp, fmaf(c11, xmp, (c11 + c21 + c31) * xmm)));
        }
        const int i = q - 1, j = jr + r;
        if (q > i_begin && j <= p.nj - 2 && kq < p.nk) {
          float* brow = p.B + ((size_t)i * p.nj + j) * p.nk;
          if (kq >= 1 && kq + 4 <= p.nk - 1) {
            __stcs(reinterpret_cast<float4*>(brow + kq), make_float4(out[0], out[1], out[2], out[3]));
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (kq + e >= 1 && kq + e <= p.nk - 2) brow[kq + e] = out[e];
          }
        }
      }
    }
    u += i_end - i_begin;
  }
}

// Stage 2, direct form: no shared memory.  A thread owns 4 consecutive k
// (one float4) x kR rows j and streams a chunk of kCH output planes along i.
// Every input plane q is consumed once as it arrives (its p-taps finish
// output q-1, its z-taps extend output q, its m-taps start output q+1), so
// only two partial-sum planes stay in registers; the loads of plane q + kPD
// are issued before plane q is consumed (register prefetch ring of kPD
// planes), keeping kPD x (kR + 2) x 16 B of loads in flight per thread.
// The repeated PolyBench taps are folded ((c11+c21+c31) A[i-1][j-1][k-1],
// (c13+c23+c33) A[i+1][j-1][k-1]): 11 FMAs per output.

template <int R, int KV>
struct PlaneRows {
  float v[R + 2][4 * KV + 2];  // rows j-1 .. j+R, columns k-1 .. k+4KV
};

// Loads of one input plane: row offsets and halo offsets are fixed per
// thread (clamped once, outside the plane loop), so the loop body carries no
// predicates -- a clamped halo only ever feeds a border output that is not
// stored.
template <int R, int KV>
__device__ __forceinline__ void load_rows(PlaneRows<R, KV>& P, const float* __restrict__ plane,
                                          const int (&roff)[R + 2], int offL, int offR) {
#pragma unroll
  for (int rr = 0; rr < R + 2; ++rr) {
    const float* rp = plane + roff[rr];
    P.v[rr][0] = __ldg(rp + offL);
#pragma unroll
    for (int h = 0; h < KV; ++h) {
      const float4 c = __ldcs(reinterpret_cast<const float4*>(rp) + h);
      P.v[rr][4 * h + 1] = c.x;
      P.v[rr][4 * h + 2] = c.y;
      P.v[rr][4 * h + 3] = c.z;
      P.v[rr][4 * h + 4] = c.w;
    }
    P.v[rr][4 * KV + 1] = __ldg(rp + offR);
  }
}

// Linear grid, i-chunk slowest: concurrently resident CTAs stream the same
// planes (DRAM page locality).  PF_C3_ZFAST=1 (A/B runs) puts the chunk
// index fastest so a chunk's two halo planes hit L2 when its neighbour reads
// them -- measured slower at 512^3 (213.0 vs 201.7 us; DRAM reads are 1.03x
// the algorithmic bytes either way) and equal at 256^3.
template <BenchId Bn, int V, int R, int PD, int CH, int TX, int TY, int KV>
__global__ void __launch_bounds__(TX * TY) conv3d_s2d(const float* __restrict__ A, float* __restrict__ B, int ni,
                                                      int nj, int nk, int nchunk, int nbx, int nbxy) {
  constexpr int W = 4 * KV;  // outputs along k per thread
  // nbxy > 0: chunk slowest (default); nbxy == 0: chunk fastest (PF_C3_ZFAST=1)
  const int chunk = nbxy ? blockIdx.x / nbxy : blockIdx.x % nchunk;
  const int bxy = nbxy ? blockIdx.x % nbxy : blockIdx.x / nchunk;
  const int kq = W * ((bxy % nbx) * TX + threadIdx.x);
  const int jr = 1 + ((bxy / nbx) * TY + threadIdx.y) * R;
  if (kq >= nk || jr > nj - 2) return;
  const int i0 = 1 + chunk * CH, i1 = min(ni - 1, i0 + CH);  // outputs [i0, i1), inputs i0-1 .. i1
  const int plane = nj * nk;                                      // < 2^31 (checked on the host)
  int roff[R + 2];
#pragma unroll
  for (int rr = 0; rr < R + 2; ++rr) roff[rr] = min(jr - 1 + rr, nj - 1) * nk + kq;
  const int offL = kq > 0 ? -1 : 0, offR = kq + W < nk ? W : W - 1;
  const bool full = kq >= 1 && kq + W <= nk - 1;
  constexpr float cM = c11 + c21 + c31, cP = c13 + c23 + c33;
  const float* src = A + (size_t)(i0 - 1) * plane;
  float* dst = B + (size_t)i0 * plane + jr * nk + kq;  // row jr of output plane i0
  const int nq = i1 - i0 + 2;
  PlaneRows<R, KV> ring[PD];
#pragma unroll
  for (int d = 0; d < PD; ++d)
    if (d < nq) load_rows<R, KV>(ring[d], src + d * plane, roff, offL, offR);
  float mz[R][W], mn[R][W];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int e = 0; e < W; ++e) mz[r][e] = mn[r][e] = 0.f;
  for (int q0 = 0; q0 < nq; q0 += PD) {
#pragma unroll
    for (int d = 0; d < PD; ++d) {
      const int q = q0 + d;
      if (q >= nq) break;
      const PlaneRows<R, KV>& cur = ring[d];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float out[W];
#pragma unroll
        for (int e = 0; e < W; ++e) {
          const float xmm = cur.v[r][e], xmz = cur.v[r][e + 1], xmp = cur.v[r][e + 2];
          const float xzz = cur.v[r + 1][e + 1], xzp = cur.v[r + 1][e + 2];
          const float xpz = cur.v[r + 2][e + 1], xpp = cur.v[r + 2][e + 2];
          // this plane as i+1 of output q-1, as i of output q, as i-1 of output q+1
          out[e] = fmaf(c33, xpp, fmaf(c23, xzp, fmaf(c13, xmp, fmaf(cP, xmm, mz[r][e]))));
          mz[r][e] = fmaf(c32, xpz, fmaf(c22, xzz, fmaf(c12, xmz, mn[r][e])));
          mn[r][e] = fmaf(c31, xpp, fmaf(c21, xzp, fmaf(c11, xmp, cM * xmm)));
        }
        if (q >= 2 && jr + r <= nj - 2) {  // relative input q finishes output plane i0 + q - 2
          float* o = dst + (size_t)(q - 2) * plane + r * nk;
          if (full) {
#pragma unroll
            for (int h = 0; h < KV; ++h)
              __stcs(reinterpret_cast<float4*>(o) + h,
                     make_float4(out[4 * h], out[4 * h + 1], out[4 * h + 2], out[4 * h + 3]));
          } else {
#pragma unroll
            for (int e = 0; e < W; ++e)
              if (kq + e >= 1 && kq + e <= nk - 2) o[e] = out[e];
          }
        }
      }
      // the slot is free once consumed: refill it PD planes ahead
      if (q + PD < nq) load_rows<R, KV>(ring[d], src + (size_t)(q + PD) * plane, roff, offL, offR);
    }
  }
}

template <int V, int R, int PD, int CH, int TX, int TY, int KV>
void launch_s2d(const float* A, float* B, int ni, int nj, int nk, cudaStream_t s) {
  if constexpr (KV > 1) {
    if (nk % (4 * KV)) {  // rows must hold whole KV-float4 groups
      launch_s2d<V, R, PD, CH, TX, TY, 1>(A, B, ni, nj, nk, s);
      return;
    }
  }
  static const bool zslow = [] {
    const char* e = std::getenv("PF_C3_ZFAST");
    return !(e && e[0] == '1');
  }();
  const int nbx = (int)cdiv(nk, 4 * KV * TX), nby = (int)cdiv(nj - 2, TY * R), nchunk = (int)cdiv(ni - 2, CH);
  conv3d_s2d<B_3DCONV, V, R, PD, CH, TX, TY, KV><<<(unsigned)nbx * nby * nchunk, dim3(TX, TY), 0, s>>>(
      A, B, ni, nj, nk, nchunk, nbx, zslow ? nbx * nby : 0);
}

// PF_C3=t (A/B runs) selects the TMA plane-streaming kernel (38.9 us at 256^3,
// issue-bound); default: the direct form (2 rows x float4 per thread, 8-plane
// chunks, 2 planes of register prefetch: 28.6 us).  Shapes measured and
// dropped: 4- and 32-plane chunks, 1 or 4 rows, 3-4 planes of prefetch, two
// float4 per thread, and a cp.async shared-memory ring (37 us).
inline int c3_mode() {
  static const int m = [] {
    const char* e = std::getenv("PF_C3");
    if (!e || !e[0]) return 0;
    return e[0] == 't' ? -1 : std::atoi(e);
  }();
  return m;
}

template <int V>
void launch_s2(const float* A, float* B, int ni, int nj, int nk, cudaStream_t s) {
  const int grid =
      std::max(1, occupancy((const void*)conv3d_s2<B_3DCONV, V>, kS2Threads, kNS * kSlotBytes)) * device_sms();
  S2Params p;
  if (!tma::make_map_3d(&p.map, A, nk, nj, ni, kBoxK, kBoxJ, 1)) {  // check() guarantees nk % 4 == 0
    launch_failed("3DCONV stage 2: cuTensorMapEncodeTiled rejected the input plane map");
    return;
  }
  p.B = B;
  p.ni = ni;
  p.nj = nj;
  p.nk = nk;
  p.tiles_k = (int)cdiv(nk, kTK);
  p.tiles = p.tiles_k * (int)cdiv(nj - 2, kTJ);
  p.units = (int64_t)p.tiles * (ni - 2);
  const int g = (int)std::min<int64_t>(grid, p.units);
  conv3d_s2<B_3DCONV, V><<<g, kS2Threads, kNS * kSlotBytes, s>>>(p);
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
    } else if ((int64_t)nj * nk >= (int64_t(1) << 31)) {  // int32 plane offsets in the direct form
      launch_s2<V>(A, B, ni, nj, nk, s);
    } else {
      // Direct-form shapes measured in round 2 (256^3 / 512^3, default 30.7 / 202.8 us):
      // TY=4 47.1 / 303.1, CH=16 32.8 / 198.7, CH=4 TY=4 49.1 / 337.9, TX=32 TY=4 30.7 / 200.7,
      // CH=6 30.7 / 206.9 -- none better at the config size.
      switch (c3_mode()) {
        case -1: launch_s2<V>(A, B, ni, nj, nk, s); break;
        default: launch_s2d<V, 2, 2, 8, 64, 2, 1>(A, B, ni, nj, nk, s); break;
      }
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
