/*
 * polybench_cpu.c -- CPU ORACLE (test infrastructure only).
 *
 * This file is the checker, never the product: only tests/, __graft_entry__
 * .smoke() and bench.py's cpu_baseline / --impl reference leg load it.
 *
 * It restates, independently of the CUDA sources, the 15 PolyBench/GPU 1.0
 * kernels of arXiv 1810.10496 and the input generators.
 * PolyBench/GPU itself is NOT part of /root/reference: the
 * definitions follow oracle/SPEC.md, which freezes the recalled PolyBench/GPU
 * semantics plus the documented deviations.  PARITY
 * UNPINNED for kernel arithmetic: no reference test or golden vector pins
 * kernel outputs (the reference's runners are stubs, conftest.py:106-133).
 * The pin used instead is agreement with a second, independent numpy
 * restatement (oracle/polybench_np.py) at small sizes.
 *
 * Numerics: inputs are fp32 and generated bit-exactly like the device
 * (explicitly rounded fp32 operations; build with -ffp-contract=off); every
 * dot product / reduction accumulates in fp64 and is rounded once to fp32
 * when stored, so the oracle is at least as accurate as any variant.
 * Arrays that the GPU stores between phases (2MM's C, 3MM's E/F, CORR's
 * normalised data, FDTD's fields, GRAMSCHM's A/Q/R) are stored as fp32 here
 * too, so both sides see the same intermediate precision.
 *
 * Entry points (ctypes, see oracle/oracle.py):
 *   orc_array_elems(bench, dims, array)        -> elements
 *   orc_generate(bench, dims, array, stock, seed, instance, out)
 *   orc_run(bench, dims, arrays)               -> runs the kernel in place
 *   orc_set_threads(n)                         -> worker threads (0 = all online CPUs)
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <pthread.h>
#include <stdatomic.h>
#include <string.h>
#include <unistd.h>

/* ---------------------------------------------------------------- threads
 * A minimal dynamic parallel-for over [0, n) (no OpenMP runtime in this
 * image): workers pull fixed-size chunks from an atomic counter. */
static int g_threads = 1;

typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t n, chunk;
  atomic_llong next;
} pfor_t;

static void* pfor_worker(void* p) {
  pfor_t* job = (pfor_t*)p;
  for (;;) {
    int64_t lo = atomic_fetch_add(&job->next, job->chunk);
    if (lo >= job->n) break;
    int64_t hi = lo + job->chunk < job->n ? lo + job->chunk : job->n;
    job->fn(job->ctx, lo, hi);
  }
  return NULL;
}

static void par_for(int64_t n, range_fn fn, void* ctx) {
  if (n <= 0) return;
  int t = g_threads < 256 ? g_threads : 256;
  if (t > n) t = (int)n;
  if (t <= 1) {
    fn(ctx, 0, n);
    return;
  }
  pfor_t job;
  job.fn = fn;
  job.ctx = ctx;
  job.n = n;
  job.chunk = n / ((int64_t)t * 8) > 0 ? n / ((int64_t)t * 8) : 1;
  atomic_init(&job.next, 0);
  pthread_t th[256];
  for (int i = 1; i < t; ++i) pthread_create(&th[i], NULL, pfor_worker, &job);
  pfor_worker(&job);
  for (int i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

enum {
  B_2DCONV = 0, B_3DCONV, B_2MM, B_3MM, B_ATAX, B_BICG, B_CORR, B_COVAR, B_FDTD2D,
  B_GEMM, B_GESUMMV, B_GRAMSCHM, B_MVT, B_SYR2K, B_SYRK, B_COUNT
};

#define STOCK_SEED 1729ULL
#define STOCK_INSTANCE (-2)

/* ---------------------------------------------------------------- RNG */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static uint64_t stream_key(uint64_t seed, int bench, int array, int64_t instance) {
  uint64_t k = mix64(seed + 0x9e3779b97f4a7c15ULL);
  k = mix64(k ^ (uint64_t)(bench + 1) * 0x100000001b3ULL);
  k = mix64(k ^ (uint64_t)(array + 1) * 0xc2b2ae3d27d4eb4fULL);
  k = mix64(k ^ (uint64_t)(instance + 2) * 0x165667b19e3779f9ULL);
  return k;
}

static float unit_float(uint64_t key, int64_t idx) {
  uint64_t h = mix64(key + (uint64_t)idx * 0x9e3779b97f4a7c15ULL);
  return (float)(h >> 40) * (1.0f / 16777216.0f);
}

/* fp32 helpers: separate statements keep every rounding explicit */
static float f_ij_over(int64_t i, int64_t j, float add, int64_t n) {
  float p = (float)i * (float)j;
  float s = p + add;
  return s / (float)n;
}

static float pi_times(int64_t i) { return (float)((double)i * 3.14159265358979323846); }

/* ---------------------------------------------------------------- sizes */
int64_t orc_array_elems(int bench, const int64_t* d, int a) {
  switch (bench) {
    case B_2DCONV: return d[0] * d[1];
    case B_3DCONV: return d[0] * d[1] * d[2];
    case B_2MM: { /* A ni*nk, B nk*nj, C ni*nj, D nj*nl, E ni*nl */
      int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3];
      int64_t s[5] = {ni * nk, nk * nj, ni * nj, nj * nl, ni * nl};
      return a < 5 ? s[a] : -1;
    }
    case B_3MM: { /* A ni*nk, B nk*nj, C nj*nm, D nm*nl, E ni*nj, F nj*nl, G ni*nl */
      int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3], nm = d[4];
      int64_t s[7] = {ni * nk, nk * nj, nj * nm, nm * nl, ni * nj, nj * nl, ni * nl};
      return a < 7 ? s[a] : -1;
    }
    case B_ATAX: { /* A nx*ny, x ny, y ny, tmp nx */
      int64_t s[4] = {d[0] * d[1], d[1], d[1], d[0]};
      return a < 4 ? s[a] : -1;
    }
    case B_BICG: { /* A nx*ny, r nx, p ny, s ny, q nx */
      int64_t s[5] = {d[0] * d[1], d[0], d[1], d[1], d[0]};
      return a < 5 ? s[a] : -1;
    }
    case B_CORR: { /* data (n+1)*(m+1), mean m+1, std m+1, symmat (m+1)^2 */
      int64_t m = d[0], n = d[1];
      int64_t s[4] = {(n + 1) * (m + 1), m + 1, m + 1, (m + 1) * (m + 1)};
      return a < 4 ? s[a] : -1;
    }
    case B_COVAR: { /* data, mean, symmat */
      int64_t m = d[0], n = d[1];
      int64_t s[3] = {(n + 1) * (m + 1), m + 1, (m + 1) * (m + 1)};
      return a < 3 ? s[a] : -1;
    }
    case B_FDTD2D: { /* fict tmax, ex, ey, hz nx*ny */
      int64_t s[4] = {d[2], d[0] * d[1], d[0] * d[1], d[0] * d[1]};
      return a < 4 ? s[a] : -1;
    }
    case B_GEMM: { /* A ni*nk, B nk*nj, C ni*nj */
      int64_t s[3] = {d[0] * d[2], d[2] * d[1], d[0] * d[1]};
      return a < 3 ? s[a] : -1;
    }
    case B_GESUMMV: { /* A, B n*n, x, y, tmp n */
      int64_t n = d[0];
      int64_t s[5] = {n * n, n * n, n, n, n};
      return a < 5 ? s[a] : -1;
    }
    case B_GRAMSCHM: { /* A m*n, R n*n, Q m*n */
      int64_t m = d[0], n = d[1];
      int64_t s[3] = {m * n, n * n, m * n};
      return a < 3 ? s[a] : -1;
    }
    case B_MVT: { /* A n*n, x1, x2, y1, y2 n */
      int64_t n = d[0];
      int64_t s[5] = {n * n, n, n, n, n};
      return a < 5 ? s[a] : -1;
    }
    case B_SYR2K: { /* A n*m, B n*m, C n*n */
      int64_t n = d[0], m = d[1];
      int64_t s[3] = {n * m, n * m, n * n};
      return a < 3 ? s[a] : -1;
    }
    case B_SYRK: { /* A n*m, C n*n */
      int64_t n = d[0], m = d[1];
      int64_t s[2] = {n * m, n * n};
      return a < 2 ? s[a] : -1;
    }
  }
  return -1;
}

/* role: 0 generated input, 1 generated + modified in place, 2 zeroed output/temporary */
int orc_array_role(int bench, int a) {
  static const int roles[B_COUNT][8] = {
      /* 2DCONV  */ {0, 2},
      /* 3DCONV  */ {0, 2},
      /* 2MM     */ {0, 0, 2, 0, 2},
      /* 3MM     */ {0, 0, 0, 0, 2, 2, 2},
      /* ATAX    */ {0, 0, 2, 2},
      /* BICG    */ {0, 0, 0, 2, 2},
      /* CORR    */ {1, 2, 2, 2},
      /* COVAR   */ {1, 2, 2},
      /* FDTD-2D */ {0, 1, 1, 1},
      /* GEMM    */ {0, 0, 1},
      /* GESUMMV */ {0, 0, 0, 2, 2},
      /* GRAMSCHM*/ {1, 2, 2},
      /* MVT     */ {0, 1, 1, 0, 0},
      /* SYR2K   */ {0, 0, 1},
      /* SYRK    */ {0, 1},
  };
  return roles[bench][a];
}

/* ---------------------------------------------------------------- inputs */
static float stock_value(int bench, const int64_t* d, int a, int64_t idx) {
  switch (bench) {
    case B_2DCONV: return unit_float(stream_key(STOCK_SEED, bench, a, STOCK_INSTANCE), idx);
    case B_3DCONV: {
      int64_t nj = d[1], nk = d[2];
      int64_t i = idx / (nj * nk), j = (idx / nk) % nj, k = idx % nk;
      return (float)(i % 12 + 2 * (j % 7) + 3 * (k % 13));
    }
    case B_2MM: {
      int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3];
      if (a == 0) return f_ij_over(idx / nk, idx % nk, 0.0f, ni);             /* A = i*k/ni */
      if (a == 1) return f_ij_over(idx / nj, idx % nj + 1, 0.0f, nj);         /* B = k*(j+1)/nj */
      if (a == 3) return f_ij_over(idx / nl, idx % nl + 2, 0.0f, nk);         /* D = j*(l+2)/nk */
      return 0.0f;
    }
    case B_3MM: {
      int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3], nm = d[4];
      if (a == 0) return f_ij_over(idx / nk, idx % nk, 0.0f, ni);             /* A = i*k/ni */
      if (a == 1) return f_ij_over(idx / nj, idx % nj + 1, 0.0f, nj);         /* B = k*(j+1)/nj */
      if (a == 2) return f_ij_over(idx / nm, idx % nm + 3, 0.0f, nl);         /* C = j*(m+3)/nl */
      if (a == 3) return f_ij_over(idx / nl, idx % nl + 2, 0.0f, nk);         /* D = m*(l+2)/nk */
      return 0.0f;
    }
    case B_ATAX: {
      int64_t nx = d[0], ny = d[1];
      if (a == 0) return f_ij_over(idx / ny, idx % ny, 0.0f, nx);             /* A = i*j/nx */
      if (a == 1) return pi_times(idx);                                       /* x = j*pi */
      return 0.0f;
    }
    case B_BICG: {
      int64_t nx = d[0], ny = d[1];
      if (a == 0) return f_ij_over(idx / ny, idx % ny, 0.0f, nx);             /* A = i*j/nx */
      if (a == 1 || a == 2) return pi_times(idx);                             /* r, p = i*pi */
      return 0.0f;
    }
    case B_CORR: {
      int64_t m = d[0];
      if (a == 0) return f_ij_over(idx / (m + 1), idx % (m + 1), 0.0f, m + 1); /* data = i*j/(m+1) */
      return 0.0f;
    }
    case B_COVAR: {
      int64_t m = d[0];
      if (a == 0) return f_ij_over(idx / (m + 1), idx % (m + 1), 0.0f, m);     /* data = i*j/m */
      return 0.0f;
    }
    case B_FDTD2D: {
      int64_t nx = d[0], ny = d[1];
      int64_t i = idx / ny, j = idx % ny;
      if (a == 0) return (float)idx;                                          /* fict[t] = t */
      if (a == 1) return f_ij_over(i, j + 1, 1.0f, nx);                       /* ex = (i(j+1)+1)/nx */
      if (a == 2) return f_ij_over(i - 1, j + 2, 2.0f, nx);                   /* ey = ((i-1)(j+2)+2)/nx */
      return f_ij_over(i - 9, j + 4, 3.0f, nx);                               /* hz = ((i-9)(j+4)+3)/nx */
    }
    case B_GEMM: {
      int64_t ni = d[0], nj = d[1], nk = d[2];
      if (a == 0) return f_ij_over(idx / nk, idx % nk, 0.0f, ni);             /* A = i*k/ni */
      if (a == 1) return f_ij_over(idx / nj, idx % nj, 1.0f, nj);             /* B = (k*j+1)/nj */
      return f_ij_over(idx / nj, idx % nj, 2.0f, nj);                         /* C = (i*j+2)/nj */
    }
    case B_GESUMMV: {
      int64_t n = d[0];
      if (a == 0 || a == 1) return f_ij_over(idx / n, idx % n, 0.0f, n);      /* A, B = i*j/n */
      if (a == 2) return (float)idx / (float)n;                               /* x = i/n */
      return 0.0f;
    }
    case B_GRAMSCHM: {
      int64_t n = d[1];
      if (a == 0) {                                                           /* A = U[0,1) + n*I */
        float u = unit_float(stream_key(STOCK_SEED, bench, a, STOCK_INSTANCE), idx);
        int64_t i = idx / n, j = idx % n;
        if (i == j) u = u + (float)n;
        return u;
      }
      return 0.0f;
    }
    case B_MVT: {
      int64_t n = d[0];
      if (a == 0) return f_ij_over(idx / n, idx % n, 0.0f, n);                /* A = i*j/n */
      if (a == 1) return (float)idx / (float)n;                               /* x1 = i/n */
      if (a == 2) return (float)(idx + 1) / (float)n;                         /* x2 = (i+1)/n */
      if (a == 3) return (float)(idx + 3) / (float)n;                         /* y1 = (i+3)/n */
      return (float)(idx + 4) / (float)n;                                     /* y2 = (i+4)/n */
    }
    case B_SYR2K: {
      int64_t n = d[0], m = d[1];
      if (a == 0) return f_ij_over(idx / m, idx % m, 1.0f, n);                /* A = (i*k+1)/n */
      if (a == 1) return f_ij_over(idx / m, idx % m, 2.0f, n);                /* B = (i*k+2)/n */
      return f_ij_over(idx / n, idx % n, 2.0f, n);                            /* C = (i*j+2)/n */
    }
    case B_SYRK: {
      int64_t n = d[0], m = d[1];
      if (a == 0) return f_ij_over(idx / m, idx % m, 0.0f, n);                /* A = i*k/n */
      return f_ij_over(idx / n, idx % n, 2.0f, n);                            /* C = (i*j+2)/n */
    }
  }
  return 0.0f;
}

static float random_value(int bench, const int64_t* d, int a, uint64_t seed, int64_t instance, int64_t idx) {
  float u = unit_float(stream_key(seed, bench, a, instance), idx);
  if (bench == B_GRAMSCHM && a == 0) {
    int64_t n = d[1];
    if (idx / n == idx % n) u = u + (float)n;
  }
  return u;
}

typedef struct {
  int bench;
  const int64_t* d;
  int a, stock;
  uint64_t seed;
  int64_t instance;
  float* out;
} gen_ctx_t;

static void gen_range(void* p, int64_t lo, int64_t hi) {
  gen_ctx_t* c = (gen_ctx_t*)p;
  for (int64_t i = lo; i < hi; ++i)
    c->out[i] = c->stock ? stock_value(c->bench, c->d, c->a, i)
                         : random_value(c->bench, c->d, c->a, c->seed, c->instance, i);
}

int orc_generate(int bench, const int64_t* d, int a, int stock, uint64_t seed, int64_t instance, float* out) {
  int64_t n = orc_array_elems(bench, d, a);
  if (n < 0) return -1;
  if (orc_array_role(bench, a) == 2) {
    memset(out, 0, (size_t)n * sizeof(float));
    return 0;
  }
  gen_ctx_t ctx = {bench, d, a, stock, seed, instance, out};
  par_for(n, gen_range, &ctx);
  return 0;
}

/* ---------------------------------------------------------------- kernels
 * Each parallel loop is a range function over its outer index; `K` is the
 * kernel's dims/arrays context. */
typedef struct {
  const int64_t* d;
  float** x;
  /* matmul / extra operands */
  int64_t ni, nj, nk, lda, ldb;
  double alpha, beta;
  const float* a;
  const float* b;
  const float* cin;
  float* out;
  int64_t step;  /* time step / k index for sequential outer loops */
} K;

static void conv2d_rows(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t ni = c->d[0], nj = c->d[1];
  const float* A = c->x[0];
  float* B = c->x[1];
  const double c11 = 0.2f, c21 = 0.5f, c31 = -0.8f, c12 = -0.3f, c22 = 0.6f, c32 = -0.9f, c13 = 0.4f, c23 = 0.7f,
               c33 = 0.10f;
  for (int64_t i = lo < 1 ? 1 : lo; i < hi && i < ni - 1; ++i) {
    const float* up = A + (i - 1) * nj;
    const float* mid = A + i * nj;
    const float* dn = A + (i + 1) * nj;
    for (int64_t j = 1; j < nj - 1; ++j) {
      double v = c11 * up[j - 1] + c12 * mid[j - 1] + c13 * dn[j - 1] + c21 * up[j] + c22 * mid[j] + c23 * dn[j] +
                 c31 * up[j + 1] + c32 * mid[j + 1] + c33 * dn[j + 1];
      B[i * nj + j] = (float)v;
    }
  }
}

static void conv3d_planes(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t ni = c->d[0], nj = c->d[1], nk = c->d[2];
  const float* A = c->x[0];
  float* B = c->x[1];
  const double c11 = 2, c12 = -3, c13 = 4, c21 = 5, c22 = 6, c23 = 7, c31 = -8, c32 = -9, c33 = 10;
#define A3(i, j, k) ((double)A[((i) * nj + (j)) * nk + (k)])
  for (int64_t i = lo < 1 ? 1 : lo; i < hi && i < ni - 1; ++i)
    for (int64_t j = 1; j < nj - 1; ++j)
      for (int64_t k = 1; k < nk - 1; ++k) {
        double v = c11 * A3(i - 1, j - 1, k - 1) + c13 * A3(i + 1, j - 1, k - 1) + c21 * A3(i - 1, j - 1, k - 1) +
                   c23 * A3(i + 1, j - 1, k - 1) + c31 * A3(i - 1, j - 1, k - 1) + c33 * A3(i + 1, j - 1, k - 1) +
                   c12 * A3(i, j - 1, k) + c22 * A3(i, j, k) + c32 * A3(i, j + 1, k) +
                   c11 * A3(i - 1, j - 1, k + 1) + c13 * A3(i + 1, j - 1, k + 1) + c21 * A3(i - 1, j, k + 1) +
                   c23 * A3(i + 1, j, k + 1) + c31 * A3(i - 1, j + 1, k + 1) + c33 * A3(i + 1, j + 1, k + 1);
        B[(i * nj + j) * nk + k] = (float)v;
      }
#undef A3
}

/* out[i][j] = alpha * sum_k a[i][k] b[k][j] + beta * cin[i][j] (row-major, fp64 accumulators) */
static void matmul_rows(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  double acc[4096];
  for (int64_t j0 = 0; j0 < c->nj; j0 += 4096) {
    const int64_t jn = c->nj - j0 < 4096 ? c->nj - j0 : 4096;
    for (int64_t i = lo; i < hi; ++i) {
      for (int64_t j = 0; j < jn; ++j) acc[j] = 0.0;
      for (int64_t k = 0; k < c->nk; ++k) {
        const double aik = c->a[i * c->lda + k];
        const float* brow = c->b + k * c->ldb + j0;
        for (int64_t j = 0; j < jn; ++j) acc[j] += aik * brow[j];
      }
      for (int64_t j = 0; j < jn; ++j) {
        double v = c->alpha * acc[j];
        if (c->cin) v += c->beta * (double)c->cin[i * c->nj + j0 + j];
        c->out[i * c->nj + j0 + j] = (float)v;
      }
    }
  }
}

static void matmul(int64_t ni, int64_t nj, int64_t nk, double alpha, const float* a, int64_t lda, const float* b,
                   int64_t ldb, double beta, const float* cin, float* out) {
  K c = {0};
  c.ni = ni;
  c.nj = nj;
  c.nk = nk;
  c.lda = lda;
  c.ldb = ldb;
  c.alpha = alpha;
  c.beta = beta;
  c.a = a;
  c.b = b;
  c.cin = cin;
  c.out = out;
  par_for(ni, matmul_rows, &c);
}

static void mm2(const int64_t* d, float** x) {
  const int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3];
  matmul(ni, nj, nk, 1.0, x[0], nk, x[1], nj, 0.0, NULL, x[2]); /* C = A B */
  matmul(ni, nl, nj, 1.0, x[2], nj, x[3], nl, 0.0, NULL, x[4]); /* E = C D */
}

static void mm3(const int64_t* d, float** x) {
  const int64_t ni = d[0], nj = d[1], nk = d[2], nl = d[3], nm = d[4];
  matmul(ni, nj, nk, 1.0, x[0], nk, x[1], nj, 0.0, NULL, x[4]); /* E = A B */
  matmul(nj, nl, nm, 1.0, x[2], nm, x[3], nl, 0.0, NULL, x[5]); /* F = C D */
  matmul(ni, nl, nj, 1.0, x[4], nj, x[5], nl, 0.0, NULL, x[6]); /* G = E F */
}

static void gemm(const int64_t* d, float** x) {
  matmul(d[0], d[1], d[2], 32412.0, x[0], d[2], x[1], d[1], 2123.0, x[2], x[2]);
}

/* out[i] = init[i] + sum_j A[i][j] v[j] over rows [lo, hi) */
static void rowdot_range(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  for (int64_t i = lo; i < hi; ++i) {
    double s = c->cin ? (double)c->cin[i] : 0.0;
    const float* row = c->a + i * c->lda;
    for (int64_t j = 0; j < c->nj; ++j) s += (double)row[j] * c->b[j];
    c->out[i] = (float)s;
  }
}

/* out[j] = init[j] + sum_i A[i][j] v[i] over columns [lo, hi): rows streamed, fp64 column accumulators */
static void coldot_range(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  double acc[2048];
  for (int64_t j0 = lo; j0 < hi; j0 += 2048) {
    const int64_t jn = hi - j0 < 2048 ? hi - j0 : 2048;
    for (int64_t j = 0; j < jn; ++j) acc[j] = c->cin ? (double)c->cin[j0 + j] : 0.0;
    for (int64_t i = 0; i < c->ni; ++i) {
      const double vi = c->b[i];
      const float* row = c->a + i * c->lda + j0;
      for (int64_t j = 0; j < jn; ++j) acc[j] += row[j] * vi;
    }
    for (int64_t j = 0; j < jn; ++j) c->out[j0 + j] = (float)acc[j];
  }
}

static void rowdot(int64_t rows, int64_t cols, const float* A, const float* v, const float* init, float* out) {
  K c = {0};
  c.nj = cols;
  c.lda = cols;
  c.a = A;
  c.b = v;
  c.cin = init;
  c.out = out;
  par_for(rows, rowdot_range, &c);
}

static void coldot(int64_t rows, int64_t cols, const float* A, const float* v, const float* init, float* out) {
  K c = {0};
  c.ni = rows;
  c.lda = cols;
  c.a = A;
  c.b = v;
  c.cin = init;
  c.out = out;
  par_for(cols, coldot_range, &c);
}

static void atax(const int64_t* d, float** x) {
  const int64_t nx = d[0], ny = d[1];
  rowdot(nx, ny, x[0], x[1], NULL, x[3]); /* tmp = A x */
  coldot(nx, ny, x[0], x[3], NULL, x[2]); /* y = A^T tmp */
}

static void bicg(const int64_t* d, float** x) {
  const int64_t nx = d[0], ny = d[1];
  coldot(nx, ny, x[0], x[1], NULL, x[3]); /* s = A^T r */
  rowdot(nx, ny, x[0], x[2], NULL, x[4]); /* q = A p */
}

static void mvt(const int64_t* d, float** x) {
  const int64_t n = d[0];
  rowdot(n, n, x[0], x[3], x[1], x[1]); /* x1 += A y1 */
  coldot(n, n, x[0], x[4], x[2], x[2]); /* x2 += A^T y2 */
}

static void gesummv_rows(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t n = c->d[0];
  const float* A = c->x[0];
  const float* B = c->x[1];
  const float* xv = c->x[2];
  for (int64_t i = lo; i < hi; ++i) {
    double t = 0.0, s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      t += (double)A[i * n + j] * xv[j];
      s += (double)B[i * n + j] * xv[j];
    }
    c->x[4][i] = (float)t;
    c->x[3][i] = (float)(43532.0 * t + 12313.0 * s);
  }
}

static void gesummv(const int64_t* d, float** x) {
  K c = {0};
  c.d = d;
  c.x = x;
  par_for(d[0], gesummv_rows, &c);
}

/* C[i][j] = beta C + alpha sum_k (A[i][k] B'[j][k] [+ B[i][k] A'[j][k]]) over rows [lo, hi) */
static void syrk_rows(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t n = c->d[0], m = c->d[1];
  const int dual = c->step != 0;
  const float* A = c->x[0];
  const float* B = dual ? c->x[1] : c->x[0];
  float* C = dual ? c->x[2] : c->x[1];
  for (int64_t i = lo; i < hi; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < m; ++k) {
        s += (double)A[i * m + k] * B[j * m + k];
        if (dual) s += (double)B[i * m + k] * A[j * m + k];
      }
      C[i * n + j] = (float)(4546.0 * C[i * n + j] + 12435.0 * s);
    }
}

static void syrk(const int64_t* d, float** x) {
  K c = {0};
  c.d = d;
  c.x = x;
  c.step = 0;
  par_for(d[0], syrk_rows, &c);
}

static void syr2k(const int64_t* d, float** x) {
  K c = {0};
  c.d = d;
  c.x = x;
  c.step = 1;
  par_for(d[0], syrk_rows, &c);
}

#define FLOAT_N 3214212.01f
#define EPS 0.005f

/* columns j in [lo+1, hi+1): mean (phase 0), std (phase 1) */
static void colstats_range(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t m = c->d[0], n = c->d[1];
  const float* data = c->x[0];
  float* mean = c->x[1];
  for (int64_t j = lo + 1; j < hi + 1; ++j) {
    double s = 0.0;
    for (int64_t i = 1; i <= n; ++i) s += data[i * (m + 1) + j];
    mean[j] = (float)(s / (double)FLOAT_N);
    if (c->step) { /* CORR: standard deviation */
      float* stdv = c->x[2];
      double q = 0.0;
      for (int64_t i = 1; i <= n; ++i) {
        double v = (double)data[i * (m + 1) + j] - mean[j];
        q += v * v;
      }
      stdv[j] = (float)sqrt(q / (double)FLOAT_N);
      if (stdv[j] <= EPS) stdv[j] = 1.0f;
    }
  }
}

/* rows i in [lo+1, hi+1): centre (and scale for CORR) */
static void centre_range(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t m = c->d[0];
  float* data = c->x[0];
  const float* mean = c->x[1];
  const double sqrt_n = sqrt((double)FLOAT_N);
  for (int64_t i = lo + 1; i < hi + 1; ++i)
    for (int64_t j = 1; j <= m; ++j) {
      if (c->step)
        data[i * (m + 1) + j] = (float)(((double)data[i * (m + 1) + j] - mean[j]) / (sqrt_n * c->x[2][j]));
      else
        data[i * (m + 1) + j] = data[i * (m + 1) + j] - mean[j];
    }
}

/* symmat rows j1 in [lo+1, hi+1): sum_i data[i][j1] data[i][j2], j2 >= j1 (> for CORR), mirrored */
static void gram_range(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t m = c->d[0], n = c->d[1];
  const float* data = c->x[0];
  float* sym = c->out;
  double acc[2048];
  for (int64_t j1 = lo + 1; j1 < hi + 1; ++j1) {
    const int64_t first = j1 + (c->step ? 1 : 0);
    for (int64_t j0 = first; j0 <= m; j0 += 2048) {
      const int64_t jn = m + 1 - j0 < 2048 ? m + 1 - j0 : 2048;
      for (int64_t t = 0; t < jn; ++t) acc[t] = 0.0;
      for (int64_t i = 1; i <= n; ++i) {
        const double a = data[i * (m + 1) + j1];
        const float* row = data + i * (m + 1) + j0;
        for (int64_t t = 0; t < jn; ++t) acc[t] += a * row[t];
      }
      for (int64_t t = 0; t < jn; ++t) {
        sym[j1 * (m + 1) + j0 + t] = (float)acc[t];
        sym[(j0 + t) * (m + 1) + j1] = (float)acc[t];
      }
    }
  }
}

static void covar(const int64_t* d, float** x) {
  const int64_t m = d[0], n = d[1];
  K c = {0};
  c.d = d;
  c.x = x;
  c.out = x[2];
  c.step = 0;
  par_for(m, colstats_range, &c);
  par_for(n, centre_range, &c);
  par_for(m, gram_range, &c);
}

static void corr(const int64_t* d, float** x) {
  const int64_t m = d[0], n = d[1];
  K c = {0};
  c.d = d;
  c.x = x;
  c.out = x[3];
  c.step = 1;
  par_for(m, colstats_range, &c);
  par_for(n, centre_range, &c);
  par_for(m - 1, gram_range, &c); /* j1 = 1..m-1 (corr_kernel bound j1 < M) */
  for (int64_t j = 1; j <= m; ++j) x[3][j * (m + 1) + j] = 1.0f;
}

/* FDTD phases over rows: step = t; phase chosen by c->ni (1: ey, 2: ex, 3: hz) */
static void fdtd_rows(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t nx = c->d[0], ny = c->d[1], t = c->step;
  const float* fict = c->x[0];
  float* ex = c->x[1];
  float* ey = c->x[2];
  float* hz = c->x[3];
  for (int64_t i = lo; i < hi; ++i) {
    if (c->ni == 1) {
      for (int64_t j = 0; j < ny; ++j) {
        if (i == 0)
          ey[j] = fict[t];
        else
          ey[i * ny + j] = (float)((double)ey[i * ny + j] - 0.5 * ((double)hz[i * ny + j] - hz[(i - 1) * ny + j]));
      }
    } else if (c->ni == 2) {
      for (int64_t j = 1; j < ny; ++j)
        ex[i * ny + j] = (float)((double)ex[i * ny + j] - 0.5 * ((double)hz[i * ny + j] - hz[i * ny + j - 1]));
    } else if (i < nx - 1) {
      for (int64_t j = 0; j < ny - 1; ++j)
        hz[i * ny + j] = (float)((double)hz[i * ny + j] - 0.7 * ((double)ex[i * ny + j + 1] - ex[i * ny + j] +
                                                                  ey[(i + 1) * ny + j] - ey[i * ny + j]));
    }
  }
}

static void fdtd(const int64_t* d, float** x) {
  K c = {0};
  c.d = d;
  c.x = x;
  for (int64_t t = 0; t < d[2]; ++t) {
    c.step = t;
    for (int phase = 1; phase <= 3; ++phase) {
      c.ni = phase;
      par_for(d[0], fdtd_rows, &c);
    }
  }
}

/* GRAMSCHM step k, columns j in (k, n): R[k][j] = q_k . a_j ; a_j -= q_k R[k][j] */
static void mgs_cols(void* p, int64_t lo, int64_t hi) {
  K* c = (K*)p;
  const int64_t m = c->d[0], n = c->d[1], k = c->step;
  float* A = c->x[0];
  float* R = c->x[1];
  const float* Q = c->x[2];
  for (int64_t j = k + 1 + lo; j < k + 1 + hi; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += (double)Q[i * n + k] * A[i * n + j];
    R[k * n + j] = (float)s;
    const double rkj = R[k * n + j];
    for (int64_t i = 0; i < m; ++i) A[i * n + j] = (float)(A[i * n + j] - (double)Q[i * n + k] * rkj);
  }
}

static void gramschmidt(const int64_t* d, float** x) {
  const int64_t m = d[0], n = d[1];
  float* A = x[0];
  float* R = x[1];
  float* Q = x[2];
  K c = {0};
  c.d = d;
  c.x = x;
  for (int64_t k = 0; k < n; ++k) {
    double nrm = 0.0;
    for (int64_t i = 0; i < m; ++i) nrm += (double)A[i * n + k] * A[i * n + k];
    R[k * n + k] = (float)sqrt(nrm);
    const double rkk = R[k * n + k];
    for (int64_t i = 0; i < m; ++i) Q[i * n + k] = (float)(A[i * n + k] / rkk);
    c.step = k;
    par_for(n - k - 1, mgs_cols, &c);
  }
}

int orc_run(int bench, const int64_t* d, float** x) {
  K c = {0};
  c.d = d;
  c.x = x;
  switch (bench) {
    case B_2DCONV: par_for(d[0], conv2d_rows, &c); return 0;
    case B_3DCONV: par_for(d[0], conv3d_planes, &c); return 0;
    case B_2MM: mm2(d, x); return 0;
    case B_3MM: mm3(d, x); return 0;
    case B_ATAX: atax(d, x); return 0;
    case B_BICG: bicg(d, x); return 0;
    case B_CORR: corr(d, x); return 0;
    case B_COVAR: covar(d, x); return 0;
    case B_FDTD2D: fdtd(d, x); return 0;
    case B_GEMM: gemm(d, x); return 0;
    case B_GESUMMV: gesummv(d, x); return 0;
    case B_GRAMSCHM: gramschmidt(d, x); return 0;
    case B_MVT: mvt(d, x); return 0;
    case B_SYR2K: syr2k(d, x); return 0;
    case B_SYRK: syrk(d, x); return 0;
  }
  return -1;
}

int orc_set_threads(int n) {
  if (n <= 0) n = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 256) n = 256;
  g_threads = n;
  return n;
}

int orc_get_threads(void) { return g_threads; }
