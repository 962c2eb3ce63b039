// GRAMSCHM (PolyBench/GPU gramschmidt.cu): modified Gram-Schmidt QR of an
// M x N matrix A (A is overwritten; outputs A, R, Q).
//
// Baseline, per column k (3N launches): gramschmidt_kernel1 with a single
// thread summing the column norm, kernel2 normalising Q[:,k], kernel3 one
// thread per trailing column j computing R[k][j] (accumulated in global
// memory inside the i loop) then updating A[:,j].  Paper: 1.49x over CUDA
// from store motion.  Stage 1: block-parallel norm fused
// with the Q column, the R row as a split-i vector-matrix product, and a
// 2-D elementwise trailing update; stage 2: the stage-1 sequence captured as
// one CUDA graph (vec=0) or a persistent cooperative kernel with each CTA
// owning a shared-memory-resident 16-column panel of A and pivot columns
// handed over through release/acquire flags (vec=1).
//
// Input deviation (documented): PolyBench's A = (i+1)(j+1)/(M+1)
// is rank 1; here A = U[0,1) + N*I so the factorisation is well conditioned.
#include "pf_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace pf {
namespace {

constexpr auto kTab = make_variants<2, 1, 1, 2>();
constexpr int kNV = sizeof(kTab.v) / sizeof(Knobs);

struct Init {
  int64_t n;
  uint64_t key;
  __device__ float operator()(int64_t idx) const {
    float u = unit_float(key, idx);
    if (idx / n == idx % n) u = fadd(u, i2f(n));
    return u;
  }
};

void launch_init(float* out, int array, int64_t n, const Dims& d, int stock, uint64_t seed, int64_t inst,
                 cudaStream_t s) {
  const uint64_t key = stock ? stream_key(1729, B_GRAMSCHM, array, -2) : stream_key(seed, B_GRAMSCHM, array, inst);
  launch_init_with(out, n, Init{d.d[1], key}, s);
}

// ---- stage 0 (PolyBench shape)
template <BenchId Bn, int V>
__global__ void gs_k1(const float* a, float* r, int m, int n, int k) {
  constexpr Knobs K = kTab.v[V];
  if (threadIdx.x == 0) {
    float nrm = 0.0f;
    if constexpr (K.lsr) {
      const float* p = a + k;
      PF_UNROLL_IMPL(K.unroll)
      for (int i = m; i > 0; --i) {
        nrm += *p * *p;
        p += n;
      }
    } else {
      PF_UNROLL_IMPL(K.unroll)
      for (int i = 0; i < m; i++) nrm += a[i * n + k] * a[i * n + k];
    }
    r[k * n + k] = sqrtf(nrm);
  }
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gs_k2(const float* a, const float* r, float* q, int m, int n, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) q[i * n + k] = a[i * n + k] / r[k * n + k];
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gs_k3(float* a, float* r, const float* q, int m, int n, int k) {
  constexpr Knobs K = kTab.v[V];
  constexpr int W = K.vec ? 4 : 1;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * W;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const int j = j0 + e;
    if ((j > k) && (j < n)) {
      float* dst = &r[k * n + j];
      Acc<K.store> acc;
      acc.init(dst, 0.0f);
      if constexpr (K.lsr) {
        const float* pq = q + k;
        const float* pa = a + j;
        PF_UNROLL_IMPL(K.unroll)
        for (int i = m; i > 0; --i) {
          acc.add(dst, *pq * *pa);
          pq += n;
          pa += n;
        }
      } else {
        PF_UNROLL_IMPL(K.unroll)
        for (int i = 0; i < m; i++) acc.add(dst, q[i * n + k] * a[i * n + j]);
      }
      acc.finish(dst);
      PF_UNROLL_IMPL(K.unroll)
      for (int i = 0; i < m; i++) a[i * n + j] -= q[i * n + k] * acc.get(dst);
    }
  }
}

// ---- stage 1
// Column norm with a block reduction, then Q[:,k] = A[:,k] / R[k][k].
template <BenchId Bn, int V>
__global__ void __launch_bounds__(1024) gs_norm_q(const float* __restrict__ a, float* r, float* q, int m, int n,
                                                  int k) {
  __shared__ float part[32];
  __shared__ float rkk;
  float s = 0.f;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const float v = a[(size_t)i * n + k];
    s = fmaf(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) {
      rkk = sqrtf(t);
      r[(size_t)k * n + k] = rkk;
    }
  }
  __syncthreads();
  const float inv = rkk;
  for (int i = threadIdx.x; i < m; i += blockDim.x) q[(size_t)i * n + k] = a[(size_t)i * n + k] / inv;
}

// R[k][j] += sum_{i in split} Q[i][k] A[i][j], j > k (R row k starts at 0).
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gs_rrow(const float* __restrict__ a, float* r, const float* __restrict__ q,
                                               int m, int n, int k, int rows_per_split) {
  const int j = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int i0 = blockIdx.y * rows_per_split, i1 = min(m, i0 + rows_per_split);
  float s0 = 0.f, s1 = 0.f;
  int i = i0;
  for (; i + 1 < i1; i += 2) {
    s0 = fmaf(__ldg(q + (size_t)i * n + k), a[(size_t)i * n + j], s0);
    s1 = fmaf(__ldg(q + (size_t)(i + 1) * n + k), a[(size_t)(i + 1) * n + j], s1);
  }
  if (i < i1) s0 = fmaf(__ldg(q + (size_t)i * n + k), a[(size_t)i * n + j], s0);
  atomicAdd(r + (size_t)k * n + j, s0 + s1);
}

// A[i][j] -= Q[i][k] R[k][j] for j > k.
template <BenchId Bn, int V>
__global__ void __launch_bounds__(256) gs_update(float* a, const float* __restrict__ r, const float* __restrict__ q,
                                                 int m, int n, int k) {
  const int j = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (j >= n || i >= m) return;
  a[(size_t)i * n + j] -= __ldg(q + (size_t)i * n + k) * __ldg(r + (size_t)k * n + j);
}

template <BenchId Bn, int V>
void s1_sequence(Workspace& ws, cudaStream_t s) {
  const int m = (int)ws.dims.d[0], n = (int)ws.dims.d[1];
  float* A = ws.a.p[0];
  float* R = ws.a.p[1];
  float* Q = ws.a.p[2];
  for (int k = 0; k < n; ++k) {
    gs_norm_q<Bn, V><<<1, 1024, 0, s>>>(A, R, Q, m, n, k);
    const int cols = n - k - 1;
    if (cols <= 0) continue;
    const int gx = (int)cdiv(cols, 256);
    int splits = std::max(1, std::min((int)cdiv(device_sms() * 2, gx), (m + 127) / 128));
    const int rps = (int)cdiv(m, splits);
    splits = (int)cdiv(m, rps);
    gs_rrow<Bn, V><<<dim3(gx, splits), 256, 0, s>>>(A, R, Q, m, n, k, rps);
    gs_update<Bn, V><<<dim3(cdiv(cols, 32), cdiv(m, 8)), dim3(32, 8), 0, s>>>(A, R, Q, m, n, k);
  }
}

// ---- stage 2, vec=1: persistent panel MGS
// CTA b owns columns [b*W, b*W+W) of A, resident in shared memory (column
// major, leading dimension m+1 to avoid bank conflicts) for the whole run.
// Inside a CTA, warp w owns panel columns 2w and 2w+1, so every dot product is
// a warp reduction.  Step k: the warp owning column k (fully updated by then,
// since all updates of a column are applied by its owner in step order)
// computes R[k][k] and q_k into shared memory and a contiguous scratch vector
// and releases flag[k]; every CTA with columns > k acquires the flag, stages
// q_k (L2, bypassing L1) in shared memory and each warp applies the rank-1
// update to its columns.  Two block barriers per step.  All CTAs must be
// co-resident: launched cooperatively with grid = ceil(n/W) <= #SMs.
constexpr int kPanelW = 16;
constexpr int kPanelThreads = 256;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <BenchId Bn, int V>
__global__ void __launch_bounds__(kPanelThreads, 1) gs_panel(float* __restrict__ A, float* __restrict__ R,
                                                             float* __restrict__ Q, float* __restrict__ qbuf,
                                                             int* __restrict__ flags, int m, int n) {
  // shared: S [W][m+1] (column-major panel) then qs [m] (q_k of the current step)
  extern __shared__ float S[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ld = m + 1;
  float* qs = S + (size_t)kPanelW * ld;
  const int c0 = blockIdx.x * kPanelW;
  const int w = min(kPanelW, n - c0);
  for (int idx = t; idx < m * kPanelW; idx += kPanelThreads) {
    const int i = idx / kPanelW, jj = idx % kPanelW;
    if (jj < w) S[jj * ld + i] = A[(size_t)i * n + c0 + jj];
  }
  // warp `warp` owns panel columns 2*warp and 2*warp+1
  constexpr int kCols = kPanelW / (kPanelThreads / 32);
  const int last = c0 + w;
  for (int k = 0; k < last; ++k) {
    __syncthreads();  // previous step's updates (and reads of qs) are complete
    if (k >= c0) {
      const int jj = k - c0;
      if (warp == jj / kCols) {
        const float* col = S + jj * ld;
        float nrm = 0.f;
        for (int i = lane; i < m; i += 32) nrm = fmaf(col[i], col[i], nrm);
        nrm = warp_sum(nrm);
        const float rkk = sqrtf(nrm);
        for (int i = lane; i < m; i += 32) {
          const float q = col[i] / rkk;
          qs[i] = q;
          qbuf[(size_t)k * m + i] = q;
        }
        __syncwarp();
        if (lane == 0) {
          R[(size_t)k * n + k] = rkk;
          __threadfence();
          st_release(flags + k, 1);
        }
      }
    } else {
      if (t == 0)
        while (ld_acquire(flags + k) == 0) {
        }
      __syncthreads();
      for (int i = t; i < m; i += kPanelThreads) qs[i] = __ldcg(qbuf + (size_t)k * m + i);
    }
    __syncthreads();  // qs holds q_k
    if (k >= c0 && warp == (k - c0) / kCols) {
      // the pivot warp also stores the strided Q column (off the other CTAs' critical path)
      for (int i = lane; i < m; i += 32) Q[(size_t)i * n + k] = qs[i];
    }
#pragma unroll
    for (int cc = 0; cc < kCols; ++cc) {
      const int jj = warp * kCols + cc;
      if (jj >= w || c0 + jj <= k) continue;
      float* col = S + jj * ld;
      float r = 0.f;
      for (int i = lane; i < m; i += 32) r = fmaf(qs[i], col[i], r);
      r = warp_sum(r);
      if (lane == 0) R[(size_t)k * n + c0 + jj] = r;
      for (int i = lane; i < m; i += 32) col[i] = fmaf(-qs[i], r, col[i]);
    }
  }
  __syncthreads();
  for (int idx = t; idx < m * kPanelW; idx += kPanelThreads) {
    const int i = idx / kPanelW, jj = idx % kPanelW;
    if (jj < w) A[(size_t)i * n + c0 + jj] = S[jj * ld + i];
  }
}

inline size_t panel_smem(int m) { return ((size_t)kPanelW * (m + 1) + m) * sizeof(float); }

inline bool panel_supported(int64_t m, int64_t n) {
  return panel_smem((int)m) <= 200 * 1024 &&
         (n + kPanelW - 1) / kPanelW <= 148 && m >= 1 && n >= 1;
}

template <BenchId Bn, int V>
void launch_panel(Workspace& ws, cudaStream_t s) {
  const int m = (int)ws.dims.d[0], n = (int)ws.dims.d[1];
  float* scratch = ws.ensure_scratch((size_t)n * m * sizeof(float) + (size_t)n * sizeof(int));
  if (!scratch) {
    launch_failed("GRAMSCHM panel: scratch allocation failed");
    return;
  }
  float* qbuf = scratch;
  int* flags = reinterpret_cast<int*>(scratch + (size_t)n * m);
  cudaMemsetAsync(flags, 0, (size_t)n * sizeof(int), s);
  set_smem_attr((const void*)gs_panel<Bn, V>, 200 * 1024);
  float* A = ws.a.p[0];
  float* R = ws.a.p[1];
  float* Q = ws.a.p[2];
  void* args[] = {&A, &R, &Q, &qbuf, &flags, (void*)&m, (void*)&n};
  const int grid = (n + kPanelW - 1) / kPanelW;
  cudaLaunchCooperativeKernel((const void*)gs_panel<Bn, V>, dim3(grid), dim3(kPanelThreads), args, panel_smem(m), s);
}

// ---- stage 2, vec=1 (m <= 2048): persistent register-resident panels with
// panel-granular hand-over.  CTA b owns columns [16b, 16b+16); warp w holds
// panel columns 2w, 2w+1 in registers (lane: rows 128*(t/4) + 4*lane + t%4,
// t < 64; rows >= m are zero and stay zero).  The arithmetic per column is
// exactly the per-column kernel's (MGS: r = q_k . a_j on the current a_j, then
// a_j -= r q_k, k ascending); only the synchronisation changes: CTA b waits
// once per earlier PANEL (flag[p], release/acquire) and applies that panel's
// 16 q vectors back to back, q_{k+1} prefetched from L2 into registers while
// q_k is applied (one block barrier per q, double-buffered in shared memory),
// then factors its own panel and publishes its 16 q vectors (qbuf, 2048-row
// stride) with one flag.  Q = A * (1 / R[k][k]) (reciprocal once per column).
constexpr int kP2Rows = 2048;  // max m: 64 rows per lane

// Warp dot product of two 64-row lane slices: 4 independent FMA chains, then
// the butterfly sum.
__device__ __forceinline__ float dot64(const float (&x)[64], const float (&y)[64]) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int i = 0; i < 64; i += 4) {
    s0 = fmaf(x[i], y[i], s0);
    s1 = fmaf(x[i + 1], y[i + 1], s1);
    s2 = fmaf(x[i + 2], y[i + 2], s2);
    s3 = fmaf(x[i + 3], y[i + 3], s3);
  }
  return warp_sum((s0 + s1) + (s2 + s3));
}

// Diagnostics (PF_GS_TRACE=1, timing studies only -- it overwrites zeros of
// R's strict lower triangle): globaltimer in microseconds (mod 2^24) at
// three points of CTA b, stored in R[n-1][3b .. 3b+2] when 3b+2 < n-1.
__device__ __forceinline__ void gs_trace(float* R, int n, int b, int slot) {
  if (3 * b + 2 >= n - 1) return;
  uint64_t ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  R[(size_t)(n - 1) * n + 3 * b + slot] = (float)((ns / 1000) & 0xFFFFFF);
}

// Diagnostics: step-level timeline of CTA 5's own-panel factorisation in R's
// row n-2 (strict lower triangle): [3kk] pivot done, [3kk+1] last warp past
// the barrier, [3kk+2] last warp's update done, [3kk+3] pivot warp starts its
// pivot (microseconds, mod 2^24; layout 4 per step).
__device__ __forceinline__ void gs_trace_step(float* R, int n, int kk, int slot) {
  if (4 * kk + slot >= n - 2) return;
  uint64_t ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  R[(size_t)(n - 2) * n + 4 * kk + slot] = (float)((ns / 10) & 0xFFFFFF) * 0.01f;
}

// One MGS step on a warp's two register columns: r_c = q . a_c (8
// interleaved FMA chains, both butterflies interleaved), a_c -= r_c q, R row
// entries stored by lane 0.  A column with use_c == false is left exactly
// unchanged (r = 0) and its R entry is not written.
__device__ __forceinline__ void update2(const float (&q)[64], float (&a)[2][64], bool use0, bool use1, float* rrow,
                                        int lane) {
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 64; i += 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s[e] = fmaf(q[i + e], a[0][i + e], s[e]);
      s[4 + e] = fmaf(q[i + e], a[1][i + e], s[4 + e]);
    }
  }
  float r0 = (s[0] + s[1]) + (s[2] + s[3]), r1 = (s[4] + s[5]) + (s[6] + s[7]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r0 += __shfl_xor_sync(0xffffffffu, r0, o);
    r1 += __shfl_xor_sync(0xffffffffu, r1, o);
  }
  r0 = use0 ? r0 : 0.f;
  r1 = use1 ? r1 : 0.f;
  if (lane == 0) {
    if (use0) rrow[0] = r0;
    if (use1) rrow[1] = r1;
  }
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    a[0][i] = fmaf(-q[i], r0, a[0][i]);
    a[1][i] = fmaf(-q[i], r1, a[1][i]);
  }
}

// update2 for one register column (same summation order as update2's
// column 0): the pivot warp's second column after its first column's pivot,
// the step on the critical path of the own-panel factorisation.
__device__ __forceinline__ void update1(const float (&q)[64], float (&a)[64], float* rdst, int lane) {
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 64; i += 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = fmaf(q[i + e], a[i + e], s[e]);
  }
  float r = (s[0] + s[1]) + (s[2] + s[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  if (lane == 0) *rdst = r;
#pragma unroll
  for (int i = 0; i < 64; ++i) a[i] = fmaf(-q[i], r, a[i]);
}

template <BenchId Bn, int V, int W>
__global__ void __launch_bounds__(16 * W, 1) gs_panel2(float* __restrict__ A, float* __restrict__ R,
                                                              float* __restrict__ Q, float* __restrict__ qbuf,
                                                              int* __restrict__ flags, int m, int n, int trace) {
  constexpr int NT = 16 * W;  // W/2 warps, two register columns each
  int* colflags = flags + n;  // per-column flags (the next panel's owner), after the per-panel ones
  extern __shared__ __align__(16) float qpan[];  // [16][2048]: a panel's q vectors
  __shared__ __align__(8) uint64_t slot_bar[W];  // own panel: slot kk holds q_{c0+kk}
  __shared__ float rbuf[W * W];                  // own panel's R block, written out after the factorisation
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int b = blockIdx.x, c0 = b * W, w = min(W, n - c0);
  const bool named_bar = (trace & 2) != 0;  // PF_GS_NB=1: the own-panel steps meet at named barriers
  trace &= 1;
  float* st = qpan;  // staging for the panel load / store: 128 rows x (W + 1)
  if (t < W) {  // ordered before use by the load loop's barriers
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&slot_bar[t]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  }
  float a[2][64];

  // ---- load the panel (coalesced 16-float row segments through shared memory)
#pragma unroll
  for (int P = 0; P < kP2Rows / 128; ++P) {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = t + NT * e, row = 128 * P + idx / W, col = idx % W;
      st[(idx / W) * (W + 1) + col] = (row < m && col < w) ? A[(size_t)row * n + c0 + col] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int c = 0; c < 2; ++c) a[c][4 * P + e] = st[(4 * lane + e) * (W + 1) + 2 * warp + c];
  }
  __syncthreads();

  if (trace && t == 0) gs_trace(R, n, b, 0);
  // ---- apply earlier panels: the whole panel's 16 q vectors (128 KB) are
  // copied into shared memory with cp.async behind one flag acquire, then
  // every warp applies them back to back with no further block barriers
  // The panel right before this one is the critical path: its q vectors are
  // consumed column by column (per-column flags) while its owner is still
  // factoring, so only the last column's hand-over is exposed.
  for (int pb = 0; pb < b; ++pb) {
    if (pb == b - 1) {
      // software pipeline, one block barrier per column: at iteration it the
      // flag of column it is acquired and its copy issued (cp.async into its
      // own slot), while column it-2 -- landed by now -- is applied
      const uint32_t qs0 = static_cast<uint32_t>(__cvta_generic_to_shared(qpan));
      for (int it = 0; it < W + 2; ++it) {
        if (it < W && t == 0)
          while (ld_acquire(colflags + pb * W + it) == 0) {
          }
        if (it < W)
          asm volatile("cp.async.wait_group 1;" ::: "memory");  // own part of column it-2 landed
        else if (it == W)
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        else
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (it < W) {
          const float4* qsrc = reinterpret_cast<const float4*>(qbuf + (size_t)(pb * W + it) * kP2Rows);
          const uint32_t d = qs0 + (uint32_t)(it * kP2Rows * 4);
#pragma unroll
          for (int u = 0; u < kP2Rows / 4 / NT; ++u)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16u * (NT * u + t)),
                         "l"(qsrc + NT * u + t)
                         : "memory");
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if (it < 2) continue;
        const int kk = it - 2, k = pb * W + kk;
        const float* qb = qpan + kk * kP2Rows;
        float q[64];
#pragma unroll
        for (int g = 0; g < 16; ++g) {
          const float4 v = reinterpret_cast<const float4*>(qb)[32 * g + lane];
          q[4 * g] = v.x;
          q[4 * g + 1] = v.y;
          q[4 * g + 2] = v.z;
          q[4 * g + 3] = v.w;
        }
        update2(q, a, 2 * warp < w, 2 * warp + 1 < w, R + (size_t)k * n + c0 + 2 * warp, lane);
      }
      __syncthreads();  // qpan is reused below
      continue;
    }
    if (t == 0)
      while (ld_acquire(flags + pb) == 0) {
      }
    __syncthreads();  // also: every warp is done with the previous panel's q
    const float4* src = reinterpret_cast<const float4*>(qbuf + (size_t)pb * W * kP2Rows);
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(qpan));
#pragma unroll 8
    for (int e = 0; e < W * kP2Rows / 4 / NT; ++e) {
      const int idx = t + NT * e;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * idx), "l"(src + idx) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int kk = 0; kk < W; ++kk) {
      const int k = pb * W + kk;
      const float* qb = qpan + kk * kP2Rows;
      float q[64];
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const float4 v = reinterpret_cast<const float4*>(qb)[32 * g + lane];
        q[4 * g] = v.x;
        q[4 * g + 1] = v.y;
        q[4 * g + 2] = v.z;
        q[4 * g + 3] = v.w;
      }
      update2(q, a, 2 * warp < w, 2 * warp + 1 < w, R + (size_t)k * n + c0 + 2 * warp, lane);
    }
  }
  __syncthreads();  // qpan is reused by the factorisation below

  if (trace && t == 0) gs_trace(R, n, b, 1);
  // ---- factor the own panel.  Pivot warp kk/2 normalises column kk into
  // shared slot kk (qpan is free again: 16 slots, never reused) and meets only
  // the warps that still own a column > kk at a named barrier (bar.arrive if
  // it is not one of them); finished warps drop out.  Warp 0, done after
  // step 1, becomes the publisher: it copies ready slots to qbuf in batches,
  // fences once per batch and raises their column flags, keeping the
  // device-scope fence off the factorisation's critical path.
  float rdiag[2] = {1.f, 1.f};  // 1 / R[k][k] of the two own columns
  const int last_warp = (w - 1) / 2;
  for (int kk = 0; kk < w; ++kk) {
    const int pw = kk / 2;
    const int my_last = min(2 * warp + 1, w - 1);  // highest own column
    const bool consumer = 2 * warp < w && my_last > kk;
    const bool producer = warp == pw;
    if (!consumer && !producer) break;
    float* qb = qpan + kk * kP2Rows;
    if (producer) {
      if (trace && b == 5 && lane == 0) gs_trace_step(R, n, kk, 3);
      // the pivot column's register slice is selected by a compile-time index
      // (a runtime a[kk & 1] would demote the whole panel to local memory)
      // One warp runs this while the others wait, so it is kept short: rows
      // >= m are exactly zero in every register column (loaded as zero, and
      // q is zero there), so no row masks; 1/R[k][k] from one MUFU.RSQ.
      auto pivot = [&](float(&col)[64], float& rinv) {
        const float nrm = dot64(col, col);
        const float inv = rsqrtf(nrm);
        const float rkk = nrm * inv;
        rinv = inv;
#pragma unroll
        for (int g = 0; g < 16; ++g)
          reinterpret_cast<float4*>(qb)[32 * g + lane] =
              make_float4(col[4 * g] * inv, col[4 * g + 1] * inv, col[4 * g + 2] * inv, col[4 * g + 3] * inv);
        if (lane == 0) rbuf[kk * W + kk] = rkk;  // R entries of the own panel are staged in shared memory:
        __syncwarp();                           // no global store ahead of the barrier on the critical path
        if (lane == 0) {
          const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&slot_bar[kk]));
          asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
        }
      };
      if (kk & 1)
        pivot(a[1], rdiag[1]);
      else
        pivot(a[0], rdiag[0]);
      if (trace && b == 5 && lane == 0) gs_trace_step(R, n, kk, 0);
    }
    if (named_bar) {
      const int nthreads = 32 * (last_warp - pw + 1);  // the pivot warp and every warp after it
      if (consumer)
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (kk & 1)), "r"(nthreads) : "memory");
      else
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + (kk & 1)), "r"(nthreads) : "memory");
    } else if (consumer && !producer) {
      // slots are written once, so a consumer only waits for slot kk's
      // mbarrier (the pivot's release); no warp waits for a slower consumer
      const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&slot_bar[kk]));
      uint32_t ok = 0;
      do {
        asm volatile(
            "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], 0;\n\t"
            "selp.b32 %0, 1, 0, P;\n\t}"
            : "=r"(ok)
            : "r"(bar)
            : "memory");
      } while (!ok);
    }
    if (!consumer) continue;  // (a pure producer has no later column: it leaves at the next check)
    if (trace && b == 5 && warp == last_warp && lane == 0) gs_trace_step(R, n, kk, 1);
    float q[64];
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      const float4 v = reinterpret_cast<const float4*>(qb)[32 * g + lane];
      q[4 * g] = v.x;
      q[4 * g + 1] = v.y;
      q[4 * g + 2] = v.z;
      q[4 * g + 3] = v.w;
    }
    if (2 * warp > kk || named_bar)
      update2(q, a, 2 * warp < w && 2 * warp > kk, 2 * warp + 1 < w && 2 * warp + 1 > kk, rbuf + kk * W + 2 * warp,
              lane);
    else  // the warp's first column is factored; its second (a consumer's last column > kk) pivots next
      update1(q, a[1], rbuf + kk * W + 2 * warp + 1, lane);
    if (trace && b == 5 && warp == last_warp && lane == 0) gs_trace_step(R, n, kk, 2);
  }
  if (warp == 0) {  // publisher
    auto ready = [&](int j, bool block) {
      const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&slot_bar[j]));
      uint32_t ok = 0;
      do {
        if (block)
          asm volatile(
              "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], 0;\n\t"
              "selp.b32 %0, 1, 0, P;\n\t}"
              : "=r"(ok)
              : "r"(bar)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P, [%1], 0;\n\t"
              "selp.b32 %0, 1, 0, P;\n\t}"
              : "=r"(ok)
              : "r"(bar)
              : "memory");
      } while (block && !ok);
      return ok != 0;
    };
    for (int next = 0; next < w;) {
      ready(next, true);
      int last = next;
      while (last + 1 < w && last + 1 < next + 4 && ready(last + 1, false)) ++last;
      for (int j = next; j <= last; ++j) {
        const float4* src = reinterpret_cast<const float4*>(qpan + j * kP2Rows);
        float4* dst = reinterpret_cast<float4*>(qbuf + (size_t)(c0 + j) * kP2Rows);
#pragma unroll
        for (int g = 0; g < 16; ++g) dst[32 * g + lane] = src[32 * g + lane];
      }
      __threadfence();
      __syncwarp();
      if (lane == 0)
        for (int j = next; j <= last; ++j) st_release(colflags + c0 + j, 1);
      next = last + 1;
    }
  }
  // ---- publish the panel's q vectors
  __threadfence();
  __syncthreads();
  if (t == 0) st_release(flags + b, 1);
  for (int idx = t; idx < W * W; idx += NT) {
    const int kk = idx / W, j = idx % W;
    if (kk < w && j < w && j >= kk) R[(size_t)(c0 + kk) * n + c0 + j] = rbuf[idx];
  }
  if (trace && t == 0) gs_trace(R, n, b, 2);

  // ---- write back A (final columns) and Q = A / R[k][k] (coalesced through shared memory)
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    float* dst = which ? Q : A;
#pragma unroll
    for (int P = 0; P < kP2Rows / 128; ++P) {
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          st[(4 * lane + e) * (W + 1) + 2 * warp + c] = which ? a[c][4 * P + e] * rdiag[c] : a[c][4 * P + e];
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = t + NT * e, row = 128 * P + idx / W, col = idx % W;
        if (row < m && col < w) dst[(size_t)row * n + c0 + col] = st[(idx / W) * (W + 1) + col];
      }
    }
  }
}

template <BenchId Bn, int V, int W>
bool try_launch_panel2(void** args, int n, cudaStream_t s) {
  constexpr int NT = 16 * W;
  constexpr size_t smem = (size_t)W * kP2Rows * sizeof(float);
  const int per_sm = occupancy((const void*)gs_panel2<Bn, V, W>, NT, smem), sms = device_sms();
  const int grid = (n + W - 1) / W;
  if ((int64_t)per_sm * sms < grid) return false;  // the panels must all be co-resident
  if (cudaLaunchCooperativeKernel((const void*)gs_panel2<Bn, V, W>, dim3(grid), dim3(NT), args, smem, s) !=
      cudaSuccess)
    launch_failed("GRAMSCHM panel2: cooperative launch rejected");
  return true;
}

// 16-column panels (one CTA per SM).  PF_GS_W=8: 8-column panels, two CTAs per
// SM, when they fit co-resident -- half the per-column update work, twice the
// panels (3.14 vs 3.07 ms at 2048^2).  Also measured and dropped: a row-slice
// layout (warp = 256 rows of all 16 columns, every MGS step shared by the 8
// warps through a reduce-scatter and one block barrier): 4.69 ms.
template <BenchId Bn, int V>
void launch_panel2(Workspace& ws, cudaStream_t s) {
  const int m = (int)ws.dims.d[0], n = (int)ws.dims.d[1];
  float* scratch = ws.ensure_scratch((size_t)n * kP2Rows * sizeof(float) + 2 * (size_t)n * sizeof(int));
  if (!scratch) {
    launch_failed("GRAMSCHM panel2: scratch allocation failed");
    return;
  }
  float* qbuf = scratch;
  int* flags = reinterpret_cast<int*>(scratch + (size_t)n * kP2Rows);  // [n] panel flags, [n] column flags
  cudaMemsetAsync(flags, 0, 2 * (size_t)n * sizeof(int), s);
  float* A = ws.a.p[0];
  float* R = ws.a.p[1];
  float* Q = ws.a.p[2];
  static const int trace = [] {
    const char* e = std::getenv("PF_GS_TRACE");
    const char* nb = std::getenv("PF_GS_NB");
    return (e && e[0] == '1' ? 1 : 0) | (nb && nb[0] == '1' ? 2 : 0);
  }();
  static const int width = [] {
    const char* e = std::getenv("PF_GS_W");
    return e ? std::atoi(e) : 16;
  }();
  void* args[] = {&A, &R, &Q, &qbuf, &flags, (void*)&m, (void*)&n, (void*)&trace};
  if (width == 8 && try_launch_panel2<Bn, V, 8>(args, n, s)) return;  // else the 16-column panels
  if (!try_launch_panel2<Bn, V, 16>(args, n, s)) launch_failed("GRAMSCHM panel2: panels do not fit co-resident");
}

// PF_GS_PANEL=1 forces the per-column panel kernel (A/B runs).
inline bool panel_v1_forced() {
  static const bool f = [] {
    const char* e = std::getenv("PF_GS_PANEL");
    return e && e[0] == '1';
  }();
  return f;
}

template <int V>
struct Run {
  static void run(Workspace& ws, cudaStream_t s) {
    constexpr Knobs K = kTab.v[V];
    const int m = (int)ws.dims.d[0], n = (int)ws.dims.d[1];
    float* A = ws.a.p[0];
    float* R = ws.a.p[1];
    float* Q = ws.a.p[2];
    if constexpr (K.stage == 0) {
      for (int k = 0; k < n; ++k) {
        gs_k1<B_GRAMSCHM, V><<<1, kB1, 0, s>>>(A, R, m, n, k);
        gs_k2<B_GRAMSCHM, V><<<cdiv(m, kB1), kB1, 0, s>>>(A, R, Q, m, n, k);
        gs_k3<B_GRAMSCHM, V><<<cdiv(n, kB1 * (K.vec ? 4 : 1)), kB1, 0, s>>>(A, R, Q, m, n, k);
      }
    } else if constexpr (K.stage == 1) {
      s1_sequence<B_GRAMSCHM, V>(ws, s);
    } else if constexpr (K.vec == 0) {
      cudaGraphExec_t g = cached_graph(ws, V, &s1_sequence<B_GRAMSCHM, V>);
      cudaGraphLaunch(g, s);
    } else if (m <= kP2Rows && !panel_v1_forced()) {
      launch_panel2<B_GRAMSCHM, V>(ws, s);
    } else {
      launch_panel<B_GRAMSCHM, V>(ws, s);
    }
  }
};

constexpr auto kRun = make_run_table<Run>(std::make_integer_sequence<int, kNV>{});

int64_t elems(int a, const Dims& d) { return a == 1 ? d.d[1] * d.d[1] : d.d[0] * d.d[1]; }
int64_t launches(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.stage == 2 && k.vec) return 1;
  return k.stage == 0 ? 3 * d.d[1] : 3 * d.d[1] - 2;
}
double alg_bytes(const Dims& d) {
  const double m = d.d[0], n = d.d[1];
  return 4.0 * (2.0 * m * n + n * n + m * n);
}
double alg_flops(const Dims& d) { return 2.0 * (double)d.d[0] * d.d[1] * d.d[1]; }
int check(int v, const Dims& d) {
  const Knobs& k = kTab.v[v];
  if (k.stage == 0 && k.vec && d.d[1] % 4) return 1;
  if (k.stage == 2 && k.vec && !panel_supported(d.d[0], d.d[1])) return 1;
  return 0;
}

const BenchDesc kDesc = {
    "GRAMSCHM", 2, {"m", "n"}, 3,
    {{"A", INOUT, 1}, {"R", OUT, 1}, {"Q", OUT, 1}},
    elems, launch_init, kNV, kTab.v, kRun.f, launches, alg_bytes, alg_flops, check,
};
Registrar reg(B_GRAMSCHM, &kDesc);

}  // namespace
}  // namespace pf
