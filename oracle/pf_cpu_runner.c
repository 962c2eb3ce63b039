/*
 * pf_cpu_runner.c -- the CPU kernel runner of the reference arm (test /
 * baseline infrastructure only; never part of the product).
 *
 * The reference's ToolchainBackend executes every artifact by spawning a
 * runner process from the template `{artifact} {data} {kind}` and parsing its
 * report (/root/reference/pkg/src/phaseforge/backend/toolchain.py:216-273,
 * grammar :178-213; pkg/README.md:108-120).  PolyBench/GPU is not part of the
 * reference, so the runner of the reference's CPU path computes the kernel
 * with this repository's CPU oracle (polybench_cpu.c, all host threads) on
 * the input the data descriptor names:
 *
 *   data  = "<BENCH>:<dim>=<v>,...[#n]"   (registry.describe; "#n" is the
 *           n-th random input, toolchain.py:231-233; otherwise the stock
 *           PolyBench initialisation), seed 1729 as the B200 backend
 *   kind  = validation | measurement
 *   report: "TIME <kernel seconds>", "OUT <n>", then the n output values
 *           (validation runs; measurement runs report OUT 0 -- the engine
 *           never reads measurement outputs, explorer.py:210-214).
 *
 * Exit status 2 on a malformed command line or descriptor.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

int64_t orc_array_elems(int bench, const int64_t* d, int a);
int orc_array_role(int bench, int a);
int orc_generate(int bench, const int64_t* d, int a, int stock, uint64_t seed, int64_t instance, float* out);
int orc_run(int bench, const int64_t* d, float** x);
int orc_set_threads(int n);

static const char* kNames[15] = {"2DCONV", "3DCONV", "2MM",      "3MM", "ATAX",  "BICG",  "CORR", "COVAR",
                                 "FDTD-2D", "GEMM",  "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK"};
static const int kNArrays[15] = {2, 2, 5, 7, 4, 5, 4, 3, 4, 3, 5, 3, 5, 3, 2};
/* output arrays (PolyBench/GPU compareResults), as oracle/oracle.py OUTPUTS */
static const int kOut[15][3] = {{1, -1, -1}, {1, -1, -1}, {4, -1, -1}, {6, -1, -1}, {2, -1, -1},
                                {3, 4, -1},  {3, -1, -1}, {2, -1, -1}, {1, 2, 3},   {2, -1, -1},
                                {3, -1, -1}, {0, 1, 2},   {1, 2, -1},  {2, -1, -1}, {1, -1, -1}};

static int parse(const char* data, int* bench, int64_t* dims, int* stock, int64_t* instance) {
  const char* colon = strchr(data, ':');
  if (!colon) return -1;
  *bench = -1;
  for (int b = 0; b < 15; ++b)
    if ((size_t)(colon - data) == strlen(kNames[b]) && !strncmp(data, kNames[b], colon - data)) *bench = b;
  if (*bench < 0) return -1;
  for (int i = 0; i < 6; ++i) dims[i] = 0;
  const char* p = colon + 1;
  int nd = 0;
  while (*p && *p != '#') {
    const char* eq = strchr(p, '=');
    if (!eq || nd >= 6) return -1;
    char* end;
    dims[nd++] = strtoll(eq + 1, &end, 10);
    if (dims[nd - 1] < 1) return -1;
    p = (*end == ',') ? end + 1 : end;
  }
  *stock = 1;
  *instance = -1;
  if (*p == '#') {
    *stock = 0;
    *instance = strtoll(p + 1, NULL, 10);
  }
  return nd > 0 ? 0 : -1;
}

int main(int argc, char** argv) {
  if (argc != 4) {
    fprintf(stderr, "usage: %s <artifact> <data> <kind>\n", argv[0]);
    return 2;
  }
  FILE* art = fopen(argv[1], "rb");
  if (!art) {
    fprintf(stderr, "cannot open artifact %s\n", argv[1]);
    return 2;
  }
  fclose(art);
  int bench, stock;
  int64_t dims[6], instance;
  if (parse(argv[2], &bench, dims, &stock, &instance)) {
    fprintf(stderr, "bad data descriptor %s\n", argv[2]);
    return 2;
  }
  const int validation = !strcmp(argv[3], "validation");
  if (!validation && strcmp(argv[3], "measurement")) {
    fprintf(stderr, "bad kind %s\n", argv[3]);
    return 2;
  }
  const char* th = getenv("PF_RUNNER_THREADS");
  orc_set_threads(th ? atoi(th) : 0);
  float* x[8] = {0};
  for (int a = 0; a < kNArrays[bench]; ++a) {
    const int64_t n = orc_array_elems(bench, dims, a);
    x[a] = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
    if (!x[a] || orc_generate(bench, dims, a, stock, 1729, instance, x[a])) return 3;
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  if (orc_run(bench, dims, x)) return 3;
  clock_gettime(CLOCK_MONOTONIC, &t1);
  double secs = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
  if (secs <= 0) secs = 1e-9;
  int64_t nout = 0;
  if (validation)
    for (int k = 0; k < 3 && kOut[bench][k] >= 0; ++k) nout += orc_array_elems(bench, dims, kOut[bench][k]);
  printf("TIME %.9g\nOUT %lld\n", secs, (long long)nout);
  if (validation)
    for (int k = 0; k < 3 && kOut[bench][k] >= 0; ++k) {
      const int a = kOut[bench][k];
      const int64_t n = orc_array_elems(bench, dims, a);
      for (int64_t i = 0; i < n; ++i) printf("%.9g\n", x[a][i]);
    }
  return 0;
}
