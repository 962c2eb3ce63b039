/*
 * pfgpu.h -- C ABI of libpfgpu.so, the B200 (sm_100a) variant-evaluation
 * engine for the 15 PolyBench/GPU kernels of arXiv 1810.10496.
 *
 * This library replaces the process boundary of the reference's only real
 * execution backend.  In the reference, every candidate crosses two process
 * boundaries:
 *
 *   compile : ToolchainBackend.compile -> compile_kernel
 *             (/root/reference/pkg/src/phaseforge/backend/toolchain.py:122-175,
 *              4 x subprocess.run at :113-119)
 *   execute : ToolchainBackend.execute -> execute_artifact
 *             (toolchain.py:216-273; runner subprocess at :250-258; the runner
 *              prints the TIME/OUT report parsed by parse_report :178-213)
 *
 * and both sit behind the Backend ABC (backend/types.py:121-152).  Here the
 * compile step is a lookup of a precompiled variant (pf_variant_*), input data
 * is generated on the device (pf_ws_generate), and one "execute" is a
 * CUDA-event-timed run (pf_run) whose outputs are read back with
 * pf_ws_download.  Python binds these with ctypes
 * (paper_1810_10496_b200/_abi.py); INTEGRATION.md shows the binding.
 *
 * Conventions: plain pointers and sizes; every function returns 0 on success
 * or a negative PF_E* code, with a thread-local message in pf_last_error().
 * Times are milliseconds (float) as measured by cudaEventElapsedTime.
 */
#ifndef PFGPU_H_
#define PFGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFGPU_ABI_VERSION 2

/* error codes */
#define PF_OK 0
#define PF_EINVAL (-1)   /* bad arguments / configuration -> BackendError (types.py:19-20) */
#define PF_ECUDA (-2)    /* CUDA runtime failure; sticky errors need pf_device_reset -> CRASH (types.py:68-73) */
#define PF_ENOMEM (-3)   /* device allocation failed -> BackendError */
#define PF_ENOTBUILT (-4)/* benchmark module not compiled into this library */

/* roles of a benchmark's arrays */
#define PF_ROLE_IN 0     /* generated input, read-only */
#define PF_ROLE_INOUT 1  /* generated input modified in place (restored before each run) */
#define PF_ROLE_OUT 2    /* output / temporary, zeroed before each run */

#define PF_MAX_DIMS 6
#define PF_NKNOBS 5      /* stage, store, unroll, lsr, vec */

typedef struct pf_ws pf_ws; /* device workspace: one benchmark instance on one GPU */

/* ---- library / device ---------------------------------------------------- */
int pf_abi_version(void);
const char* pf_last_error(void);
int pf_device_count(int* count);
/* Releases every workspace-independent resource of `device` and resets it
 * after a sticky error (the reference kills the runner process instead,
 * toolchain.py:250-264). */
int pf_device_reset(int device);
int pf_device_info(int device, char* name, size_t len, int* sm_count, int64_t* l2_bytes,
                   int* cc_major, int* cc_minor);

/* ---- benchmark registry (the compile-side lookup tables) ---------------- */
/* Benchmarks are numbered in the PolyBench/GPU order of PAPER.md:114-124:
 * 2DCONV 3DCONV 2MM 3MM ATAX BICG CORR COVAR FDTD-2D GEMM GESUMMV GRAMSCHM
 * MVT SYR2K SYRK. */
int pf_bench_count(void);
int pf_bench_info(int bench, char* name, size_t len, int* ndims, int* narrays);
int pf_bench_dim_name(int bench, int dim, char* name, size_t len);
int pf_array_info(int bench, int array, char* name, size_t len, int* role, int* is_output);
int pf_array_elems(int bench, const int64_t* dims, int array, int64_t* elems);
/* Algorithmic (compulsory) bytes and flops of one run: the roofline basis
 * (SURVEY §8d). */
int pf_alg_work(int bench, const int64_t* dims, double* bytes, double* flops);

/* ---- variants: what compile() selects among ------------------------------ */
int pf_variant_count(int bench);
/* knobs[PF_NKNOBS] = {stage, store(0 rmw,1 reg,2 depot), unroll(0 = nvcc default), lsr, vec} */
int pf_variant_knobs(int bench, int variant, int* knobs);
/* Kernel launches one run of `variant` issues at `dims` (host-side count). */
int pf_variant_launches(int bench, int variant, const int64_t* dims, int64_t* launches);
/* 0 if the variant supports these dims (alignment / tile constraints). */
int pf_variant_supported(int bench, int variant, const int64_t* dims);

/* ---- workspaces ----------------------------------------------------------- */
int pf_ws_create(int device, int bench, const int64_t* dims, pf_ws** out);
int pf_ws_destroy(pf_ws* ws);
/* On-device input generation.  stock=1: the PolyBench/GPU initialisation
 * formulas; stock=0: the `instance`-th random input (U[0,1) from a counter
 * RNG keyed by (seed, bench, array, instance)), the analogue of the runner's
 * "<validation_input>#n" data descriptor (toolchain.py:231-233).  Also takes
 * the pristine snapshot used to restore in-place arrays. */
int pf_ws_generate(pf_ws* ws, int stock, uint64_t seed, int64_t instance);
/* Host <-> device copies of one array (plain float buffers of `n` elements).
 * Upload also refreshes the pristine snapshot.  Used by the end-to-end path
 * whose inputs live in (pinned) host memory. */
int pf_ws_upload(pf_ws* ws, int array, const float* host, int64_t n);
int pf_ws_download(pf_ws* ws, int array, float* host, int64_t n);
/* Asynchronous upload (host should be pinned: pf_host_alloc): enqueued on the
 * device's copy stream after the work already enqueued on the workspace, and
 * every later use of the workspace (any pf_* call, pf_eval_batch included)
 * is ordered after it.  Returns without waiting, so the copy engine streams
 * one workspace's inputs while another workspace's candidates run (the
 * runner's input load of toolchain.py:216-273, overlapped). */
int pf_ws_upload_async(pf_ws* ws, int array, const float* host, int64_t n);
/* Restore INOUT arrays and zero OUT arrays (enqueued, not timed). */
int pf_ws_restore(pf_ws* ws);
/* Device pointer of an array (for zero-copy interop; never freed by caller). */
int pf_ws_array_ptr(pf_ws* ws, int array, void** dptr);

/* ---- execution & timing ---------------------------------------------------
 * One sample = [restore] -> [L2 flush] -> event0 -> `batch` x variant run ->
 * event1.  ms[s] = elapsed / batch.  restore!=0 restores in-place state before
 * every sample (outputs of the last sample are then those of one run when
 * batch==1).  flush_l2!=0 writes a scratch buffer of 2 x L2 and reads it
 * back before each sample (L2 left clean: no write-backs inside the timed
 * run).  Synchronises the workspace stream. */
int pf_run(pf_ws* ws, int variant, int samples, int batch, int restore, int flush_l2, float* ms);
/* End-to-end: per sample, H2D of every generated input array from `host_in`
 * (array-indexed table of host pointers, NULL entries skipped), restore of
 * OUT arrays, one variant run, D2H of every output array into `host_out`;
 * all inside the timed region. */
int pf_run_e2e(pf_ws* ws, int variant, int samples, float* const* host_in, float* const* host_out,
               float* ms);

/* Batched evaluation: the candidate evaluations of an exploration round,
 * enqueued back to back on one stream (all workspaces on one device) with no
 * host synchronisation between candidates.  For evaluation i:
 *   [H2D of every non-NULL host_in[a] into ws (the runner's input upload)]
 *   [restore in-place state] [L2 flush] start_i -> `batch` x variant run -> end_i
 *   [D2H of every output array into non-NULL host_out[a]]
 * ms_each[i] = (end_i - start_i) / batch (one run's device time); *ms_total =
 * first recorded event to last (the whole batch, copies included).  The
 * upload of a workspace's first evaluation in the batch is issued up front on
 * a per-device copy stream (it overlaps earlier candidates; the evaluation
 * waits for it); later uploads into an already used workspace stay in order. */
typedef struct pf_eval {
  pf_ws* ws;
  int variant;
  float* const* host_in;  /* NULL or array-indexed host pointers */
  float* const* host_out; /* NULL or array-indexed host pointers */
  int batch;              /* runs between the events; 0 or 1 = one run (us-scale kernels use more) */
  int no_flush;           /* 1: no L2 flush before this evaluation (untimed validation runs) */
} pf_eval;
int pf_eval_batch(const pf_eval* evals, int n, int restore, int flush_l2, float* ms_each, float* ms_total);

/* ---- checking --------------------------------------------------------------
 * Device-side comparison of the output arrays of `test` against `ref`
 * (same bench and dims): element passes iff |t - r| <= max(atol, rtol*|r|)
 * with atol = atol_rel * max|r| over that array -- the comparator of
 * explorer.py:95-106 with a per-array absolute floor.  Returns the largest
 * |t - r| / max(|r|, atol) and the failing-element count. */
int pf_compare(pf_ws* test, pf_ws* ref, double rtol, double atol_rel, double* max_err, int64_t* nbad);
/* sum and sum of |x| of one array in fp64 (size-independent property checks) */
int pf_checksum(pf_ws* ws, int array, double* sum, double* abs_sum);

/* ---- pinned host memory for the end-to-end path -------------------------- */
int pf_host_alloc(size_t bytes, void** ptr);
int pf_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* PFGPU_H_ */
