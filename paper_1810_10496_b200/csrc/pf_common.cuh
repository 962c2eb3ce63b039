// Shared infrastructure for the PolyBench/GPU variant library (sm_100a).
//
// Every benchmark module (k_*.cu) provides:
//   * a BenchDesc: array table, dims meaning, output list, variant table;
//   * a device init function  float init_<b>(array, idx, dims, stock)  used by
//     the generic on-device input generator (bit-exact with oracle/polybench_cpu.c);
//   * one host "run" function per variant (template on the variant index V)
//     that enqueues the variant's kernel sequence on a stream.
//
// Variant knobs:
//   stage 0 -- PolyBench/GPU thread mapping, with the transformations LLVM
//              phase orders expose in PTX:
//              store  RMW   accumulate into global memory inside the loop (baseline shape)
//                     REG   scalar-replaced accumulator, one store after the loop (LICM promotion)
//                     DEPOT accumulator in a per-thread local slot (reg2mem, no mem2reg/sroa)
//              unroll 0 = nvcc default (baseline only), else #pragma unroll N
//              lsr    strength-reduced pointer walk instead of recomputed 32-bit index math
//              vec    128-bit loads where a thread walks contiguous memory
//   stage 1 -- Blackwell re-mapping: warp-cooperative/coalesced reductions,
//              smem-tiled SIMT, single-launch streaming
//   stage 2 -- Blackwell staging: fused single-pass kernels, tcgen05/TMEM tiles
//              for contractions (3xFP16 on kind::f16, or 3xTF32), CUDA-graph /
//              persistent sequences
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <utility>

namespace pf {

enum Store : int { RMW = 0, REG = 1, DEPOT = 2 };

struct Knobs {
  int stage;
  int store;
  int unroll;  // 0: compiler default
  int lsr;
  int vec;
};

constexpr int kMaxDims = 6;
constexpr int kMaxArrays = 8;

enum Role : int {
  IN = 0,     // generated, read-only
  INOUT = 1,  // generated, modified in place -> restored from a pristine copy before every run
  OUT = 2,    // zeroed before every run
};

struct Dims {
  int64_t d[kMaxDims];
};

struct Workspace;
using RunFn = void (*)(Workspace&, cudaStream_t);

// Per-array device pointers as seen by run functions.
struct Arrays {
  float* p[kMaxArrays];
};

struct ArraySpec {
  const char* name;
  int role;
  int is_output;  // reported by pf_read / validation outputs
};

struct BenchDesc {
  const char* name;          // PolyBench/GPU benchmark id, e.g. "GEMM"
  int ndims;
  const char* dim_names[kMaxDims];
  int narrays;
  ArraySpec arrays[kMaxArrays];
  int64_t (*array_elems)(int array, const Dims&);
  // generic on-device input generator, launched by abi.cu
  void (*launch_init)(float* out, int array, int64_t n, const Dims& dims, int stock,
                      uint64_t seed, int64_t instance, cudaStream_t s);
  int nvariants;
  const Knobs* variants;
  const RunFn* run;
  // launch-count per variant run (for gpu_launches accounting)
  int64_t (*launches)(int variant, const Dims&);
  // algorithmic work per run (roofline basis)
  double (*alg_bytes)(const Dims&);
  double (*alg_flops)(const Dims&);
  // optional: static validation (dims sanity / alignment constraints per variant)
  int (*check)(int variant, const Dims&);
};

// Device workspace of one benchmark instance (the C-ABI's opaque pf_ws).
struct Workspace {
  int device;
  int bench;
  const BenchDesc* desc;
  Dims dims;
  Arrays a;
  float* pristine[kMaxArrays];
  int64_t elems[kMaxArrays];
  cudaStream_t stream;
  cudaEvent_t ev0, ev1;
  void* graphs;          // per-variant cached cudaGraphExec_t (graph-staged variants)
  float* scratch;        // lazily grown temporary buffer for variants that need one
  size_t scratch_bytes;
  float* ensure_scratch(size_t bytes);  // defined in abi.cu; only called outside timed regions' first use
  // split-K tile hand-over flags (tcgen05 contractions): kTileFlags ints,
  // zeroed once; each launch uses a fresh epoch value (runs on a workspace
  // are serialised on its stream, so epochs never interleave)
  int* tile_flags;
  int tile_epoch;
  int* ensure_tile_flags(cudaStream_t s);  // defined in abi.cu; zeroed on s, before the launch that uses them
  // second lazily grown buffer for data a variant hands from one launch to a
  // later one while the first scratch is reused in between (3xTF32 lo images
  // of chained products)
  float* aux;
  size_t aux_bytes;
  float* ensure_aux(size_t bytes);  // defined in abi.cu
  // a side stream for independent work inside one run (abi.cu): fork(s)
  // returns it ordered after everything enqueued on s so far; join(s) makes
  // s wait for everything enqueued on the side stream.  Event-timed runs on
  // s therefore include the side work.
  cudaStream_t side;
  cudaEvent_t fork_ev, join_ev;
  cudaStream_t fork(cudaStream_t s);
  void join(cudaStream_t s);
};
constexpr int kTileFlags = 4096;
constexpr int kTileFlagsGemm = kTileFlags;  // split-K tile flags

// Graph-staged variants: capture `body` once per (workspace, key) and return
// the executable graph (abi.cu).  Launch with cudaGraphLaunch(exec, stream).
cudaGraphExec_t cached_graph(Workspace& ws, int key, void (*body)(Workspace&, cudaStream_t));

// Per-context function setup (abi.cu).  A dynamic shared-memory limit above
// 48 KB is an attribute of a function *in one context*: it has to be set on
// every device a process drives and again after pf_device_reset re-creates
// the context.  set_smem_attr caches by (function, device, context
// generation), so calling it before every launch costs a map lookup.
void set_smem_attr(const void* fn, int bytes);
// SM count of the current device (cached per device).
int device_sms();
// cudaOccupancyMaxActiveBlocksPerMultiprocessor on the current device, after
// set_smem_attr(fn, smem); cached like set_smem_attr.
int occupancy(const void* fn, int threads, size_t smem);
void note_context_reset(int device);  // pf_device_reset: invalidates the caches above

// Registration: each k_*.cu module registers its descriptor at load time.
void register_bench(int id, const BenchDesc* desc);
struct Registrar {
  Registrar(int id, const BenchDesc* d) { register_bench(id, d); }
};

enum BenchId : int {
  B_2DCONV = 0, B_3DCONV, B_2MM, B_3MM, B_ATAX, B_BICG, B_CORR, B_COVAR, B_FDTD2D,
  B_GEMM, B_GESUMMV, B_GRAMSCHM, B_MVT, B_SYR2K, B_SYRK, B_COUNT
};

// Generic init kernel: out[i] = F(array, i) for a device functor F.
template <class F>
__global__ void init_kernel(float* out, int64_t n, F f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = f(i);
}

template <class F>
inline void launch_init_with(float* out, int64_t n, F f, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;  // grid-stride: any device, 32 CTAs per B200 SM
  if (blocks < 1) blocks = 1;
  init_kernel<<<(unsigned)blocks, 256, 0, s>>>(out, n, f);
}

// ---------------------------------------------------------------- RNG
// splitmix64 finaliser over (key, index): counter-based, order independent,
// reproduced bit-for-bit by oracle/polybench_cpu.c.
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t stream_key(uint64_t seed, int bench, int array, int64_t instance) {
  uint64_t k = mix64(seed + 0x9e3779b97f4a7c15ULL);
  k = mix64(k ^ (uint64_t)(bench + 1) * 0x100000001b3ULL);
  k = mix64(k ^ (uint64_t)(array + 1) * 0xc2b2ae3d27d4eb4fULL);
  k = mix64(k ^ (uint64_t)(instance + 2) * 0x165667b19e3779f9ULL);
  return k;
}

// U[0,1) with 24 random bits: exactly representable in fp32.
__host__ __device__ inline float unit_float(uint64_t key, int64_t idx) {
  uint64_t h = mix64(key + (uint64_t)idx * 0x9e3779b97f4a7c15ULL);
  return (float)(h >> 40) * (1.0f / 16777216.0f);
}

// ---------------------------------------------------------------- fp32 helpers
// Inputs are generated with explicitly rounded operations so no FMA
// contraction can change a bit between device and the CPU oracle.
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float i2f(int64_t i) { return __ll2float_rn(i); }

// ---------------------------------------------------------------- variant tables
// Stage-0 family: the baseline first, then store x unroll x lsr x vec.
template <int kNVec>
struct Stage0 {
  static constexpr int kCount = 1 + 3 * 4 * 2 * kNVec;
};

// LLVM-path unroll ladder: the paper's phase-ordered PTX is unrolled x2 without a
// loop-unroll pass; each loop-unroll doubles it.
constexpr int kUnrolls[4] = {2, 4, 8, 16};

template <size_t N>
struct VariantTable {
  Knobs v[N];
};

// Builds: [baseline] + stage0 grid + stage1 grid (unroll x vec) + stage2 grid.
template <int kNVec0, int kNUnroll1, int kNVec1, int kNStage2>
constexpr auto make_variants() {
  constexpr size_t n = 1 + 3 * 4 * 2 * kNVec0 + kNUnroll1 * kNVec1 + kNStage2;
  VariantTable<n> t{};
  size_t i = 0;
  t.v[i++] = Knobs{0, RMW, 0, 0, 0};
  for (int st = 0; st < 3; ++st)
    for (int u = 0; u < 4; ++u)
      for (int l = 0; l < 2; ++l)
        for (int vv = 0; vv < kNVec0; ++vv) t.v[i++] = Knobs{0, st, kUnrolls[u], l, vv};
  for (int u = 0; u < kNUnroll1; ++u)
    for (int vv = 0; vv < kNVec1; ++vv) t.v[i++] = Knobs{1, REG, kNUnroll1 == 1 ? 1 : kUnrolls[u], 0, vv};
  for (int s = 0; s < kNStage2; ++s) t.v[i++] = Knobs{2, REG, 1, 0, s};
  return t;
}

// Host-side table of run functions for variants 0..N-1.
template <template <int> class Runner, int... Vs>
constexpr auto make_run_table(std::integer_sequence<int, Vs...>) {
  struct T { RunFn f[sizeof...(Vs)]; };
  return T{{&Runner<Vs>::run...}};
}

// ---------------------------------------------------------------- launch helpers
// Host-side launch failures inside a variant's run function (e.g. a TMA map
// the driver refuses): recorded here and turned into PF_ECUDA by abi.cu right
// after the run, so a variant never silently skips its kernel.
inline thread_local const char* g_launch_error = nullptr;
inline void launch_failed(const char* why) { g_launch_error = why; }
inline const char* take_launch_error() {
  const char* w = g_launch_error;
  g_launch_error = nullptr;
  return w;
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// 32x8 blocks: the PolyBench/GPU DIM_THREAD_BLOCK_X/Y default
constexpr int kBX = 32;
constexpr int kBY = 8;
// 1-D PolyBench launches use 256 threads
constexpr int kB1 = 256;

// Accumulation helper reproducing the three store shapes.
//   RMW   : *dst is read-modified-written inside the loop (volatile-free but
//           aliasing-unsafe pointers keep nvcc from promoting it)
//   REG   : register accumulator
//   DEPOT : local-memory slot (the reg2mem __local_depot shape)
template <int kStore>
struct Acc;

template <>
struct Acc<REG> {
  float v;
  __device__ __forceinline__ void init(float* /*dst*/, float x) { v = x; }
  __device__ __forceinline__ void add(float* /*dst*/, float x) { v += x; }
  __device__ __forceinline__ float get(float* /*dst*/) const { return v; }
  __device__ __forceinline__ void finish(float* dst) { *dst = v; }
};

// The slot index is produced by an opaque instruction so NVVM and ptxas cannot
// resolve it: the accumulator stays in the __local_depot (ld/st.local per
// iteration), which is exactly what a reg2mem-without-mem2reg order leaves.
template <>
struct Acc<DEPOT> {
  float slot[2];
  int which;
  __device__ __forceinline__ void init(float*, float x) {
    asm volatile("mov.u32 %0, 0;" : "=r"(which));
    slot[which] = x;
  }
  __device__ __forceinline__ void add(float*, float x) { slot[which] = slot[which] + x; }
  __device__ __forceinline__ float get(float*) const { return slot[which]; }
  __device__ __forceinline__ void finish(float* dst) { *dst = slot[which]; }
};

template <>
struct Acc<RMW> {
  __device__ __forceinline__ void init(float* dst, float x) { *dst = x; }
  __device__ __forceinline__ void add(float* dst, float x) { *dst += x; }
  __device__ __forceinline__ float get(float* dst) const { return *dst; }
  __device__ __forceinline__ void finish(float*) {}
};

// Warp reduction (stage >= 1 kernels)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace pf

// Unroll pragma with a template constant: N==0 means "compiler default".
#define PF_PRAGMA(x) _Pragma(#x)
#define PF_UNROLL_IMPL(n) PF_PRAGMA(unroll n)
