"""``B200Backend``: the reference ``Backend`` contract on libpfgpu.so.

Drop-in for ``ToolchainBackend`` (`/root/reference/pkg/src/phaseforge/
backend/toolchain.py:276-307`) behind the ABC of `backend/types.py:121-152`:

* ``compile(kernel, order)``: the order is interpreted by ``passmodel`` into
  a transformation state, which selects one precompiled sm_100a variant; the
  artifact is that variant's SASS (normalised), so identical machine code
  yields identical digests.  Pure in (kernel, order).
* ``execute(..., VALIDATION)``: one untimed run on the small stock input,
  outputs read back (never timed, explorer.py:203).
* ``execute(..., MEASUREMENT)``: a CUDA-event-timed run on the measurement
  input (never validated, explorer.py:210-211); wall time in seconds.
* ``execute(..., random_input_index=n)``: the n-th random validation-size
  input, generated on the device (the ``<validation_input>#n`` descriptor of
  toolchain.py:231-233).
* ``measurement_lock``: one lock per backend, and one backend per device.
* ``prefetch(kernel, orders)`` / ``prefetch_many(jobs)``: the fresh
  evaluations ``explore`` is about to perform (the first order of every
  distinct digest, explorer.py:175-190) run as ONE device batch
  (``pf_eval_batch``): validation runs with their outputs copied back and
  the timed measurement samples, back to back on one stream.  ``execute``
  then serves those calls from the batch's results, so the engine's record
  stream is unchanged (same calls, same order) while the device never waits
  for the host between candidates.

Error mapping: a CUDA failure returns ``CRASH`` and resets the
device -- unless torch shares the CUDA context in this process (NCCL groups,
tensors), where a reset would destroy them: the backend is then marked
failed and later calls raise ``BackendError``; a run slower than ``set_timeout_override`` returns ``TIMEOUT``
(toolchain.py:250-258 kills the runner; an in-process kernel cannot be
killed, so every variant is bounded by construction); configuration errors
raise ``BackendError``.  There is no CPU path: without libpfgpu.so this module
does not import.
"""

from __future__ import annotations

import contextlib
import ctypes
import gzip
import json
import operator
import os
import statistics
import sys
from collections import OrderedDict
from ctypes import byref, c_double, c_float, c_int, c_int64, c_void_p
from pathlib import Path

from .. import _abi, passmodel, registry
from ..catalog import PhaseOrder, PassId
from . import types as _own_types
from .types import Artifact, Backend, BackendError, KernelCase

ARTIFACTS_PATH = Path(__file__).resolve().parent.parent / "artifacts.json.gz"
_NAME = operator.attrgetter("name")
ARTIFACT_MAGIC = "pfgpu-artifact/1"


class Workspace:
    """One benchmark instance resident on one GPU (owns a ``pf_ws``)."""

    def __init__(self, device: int, bench: str, dims: tuple[int, ...]):
        self.lib = _abi.lib()
        self.device = device
        self.bench = bench
        self.bench_id = registry.bench_index(bench)
        self.dims = tuple(int(d) for d in dims)
        self._dims_c = _abi.dims_array(self.dims)
        handle = c_void_p()
        _abi.check(self.lib.pf_ws_create(device, self.bench_id, self._dims_c, byref(handle)))
        self.handle = handle
        info = bench_arrays(bench)
        self.arrays = info
        self.elems = []
        for a in range(len(info)):
            n = c_int64()
            _abi.check(self.lib.pf_array_elems(self.bench_id, self._dims_c, a, byref(n)))
            self.elems.append(n.value)
        self.nbytes = 4 * sum(self.elems) + 4 * sum(
            n for (_, role, _), n in zip(info, self.elems) if role == _abi.ROLE_INOUT
        )
        self.input_tag = None
        self.warm: set[int] = set()

    def generate(self, stock: bool, seed: int, instance: int) -> None:
        tag = (bool(stock), int(seed), int(instance))
        if self.input_tag == tag:
            return
        _abi.check(self.lib.pf_ws_generate(self.handle, int(stock), seed, instance))
        self.input_tag = tag

    def run(self, variant: int, samples: int = 1, batch: int = 1, restore: bool = True,
            flush: bool = False) -> list[float]:
        ms = (c_float * samples)()
        _abi.check(self.lib.pf_run(self.handle, variant, samples, batch, int(restore), int(flush), ms))
        return list(ms)

    def run_e2e(self, variant: int, samples: int, host_in, host_out) -> list[float]:
        ms = (c_float * samples)()
        n = len(self.arrays)
        hin = (c_void_p * n)(*[host_in.get(a) for a in range(n)])
        hout = (c_void_p * n)(*[host_out.get(a) for a in range(n)])
        _abi.check(self.lib.pf_run_e2e(self.handle, variant, samples, hin, hout, ms))
        return list(ms)

    def restore(self) -> None:
        """Reset in-place (INOUT) arrays to the generated input (pf_ws_restore)."""
        _abi.check(self.lib.pf_ws_restore(self.handle))

    def download(self, array: int):
        import numpy as np

        out = np.empty(self.elems[array], dtype=np.float32)
        _abi.check(self.lib.pf_ws_download(self.handle, array, out.ctypes.data_as(c_void_p), out.size))
        return out

    def upload(self, array: int, data) -> None:
        import numpy as np

        buf = np.ascontiguousarray(data, dtype=np.float32).ravel()
        _abi.check(self.lib.pf_ws_upload(self.handle, array, buf.ctypes.data_as(c_void_p), buf.size))
        self.input_tag = None

    def outputs(self) -> list:
        return [self.download(a) for a, (_, _, is_out) in enumerate(self.arrays) if is_out]

    def checksum(self, array: int) -> tuple[float, float]:
        s, a = c_double(), c_double()
        _abi.check(self.lib.pf_checksum(self.handle, array, byref(s), byref(a)))
        return s.value, a.value

    def compare(self, ref: "Workspace", rtol: float, atol_rel: float) -> tuple[float, int]:
        err, bad = c_double(), c_int64()
        _abi.check(self.lib.pf_compare(self.handle, ref.handle, rtol, atol_rel, byref(err), byref(bad)))
        return err.value, bad.value

    def close(self) -> None:
        if self.handle:
            self.lib.pf_ws_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ARRAY_CACHE: dict[str, list[tuple[str, int, int]]] = {}


def bench_arrays(bench: str) -> list[tuple[str, int, int]]:
    """[(name, role, is_output)] of a benchmark's arrays, from the library."""
    if bench not in _ARRAY_CACHE:
        lib = _abi.lib()
        bid = registry.bench_index(bench)
        narr = c_int()
        _abi.check(lib.pf_bench_info(bid, None, 0, None, byref(narr)))
        rows = []
        for a in range(narr.value):
            name = ctypes.create_string_buffer(64)
            role, out = c_int(), c_int()
            _abi.check(lib.pf_array_info(bid, a, name, 64, byref(role), byref(out)))
            rows.append((name.value.decode(), role.value, out.value))
        _ARRAY_CACHE[bench] = rows
    return _ARRAY_CACHE[bench]


_FAMILIES: dict[str, passmodel.VariantFamily] = {}


def family(bench: str) -> passmodel.VariantFamily:
    if bench not in _FAMILIES:
        lib = _abi.lib()
        bid = registry.bench_index(bench)
        n = lib.pf_variant_count(bid)
        if n <= 0:
            raise BackendError(f"benchmark {bench!r} is not built into libpfgpu.so")
        knobs = []
        buf = (c_int * _abi.NKNOBS)()
        for v in range(n):
            _abi.check(lib.pf_variant_knobs(bid, v, buf))
            knobs.append(tuple(buf))
        _FAMILIES[bench] = passmodel.VariantFamily(bench, knobs)
    return _FAMILIES[bench]


_ARTIFACT_TEXT: dict | None = None


def _artifact_table() -> dict:
    global _ARTIFACT_TEXT
    if _ARTIFACT_TEXT is None:
        if not ARTIFACTS_PATH.exists():
            raise BackendError(f"{ARTIFACTS_PATH.name} missing: run tools/gen_artifacts.py (part of build())")
        _ARTIFACT_TEXT = json.loads(gzip.decompress(ARTIFACTS_PATH.read_bytes()))["benches"]
    return _ARTIFACT_TEXT


def variant_sass(bench: str, variant: int) -> str:
    try:
        return _artifact_table()[bench][str(variant)]
    except KeyError as exc:
        raise BackendError(f"no SASS recorded for {bench} variant {variant}") from exc


def artifact_content(bench: str, variant: int) -> bytes:
    """The artifact bytes of one variant: a header naming the benchmark and the
    launch stage, then the normalised SASS.  Variants with identical machine
    code have identical content, hence identical digests."""
    knobs = family(bench).knobs[variant]
    header = f"{ARTIFACT_MAGIC} bench={bench} launch=stage{knobs[0]}\n"
    return (header + variant_sass(bench, variant)).encode()


def variant_of_artifact(bench: str, content: bytes) -> int:
    """Inverse of ``artifact_content``: the first variant with these bytes."""
    for v in range(len(family(bench).knobs)):
        if artifact_content(bench, v) == content:
            return v
    raise BackendError(f"artifact is not a {bench} variant of this libpfgpu build")


def _supported_dims(bench: str, variant: int, dims) -> bool:
    rc = _abi.lib().pf_variant_supported(registry.bench_index(bench), variant, _abi.dims_array(dims))
    return rc == 0


def variant_launches(bench: str, variant: int, dims) -> int:
    n = c_int64()
    _abi.check(_abi.lib().pf_variant_launches(registry.bench_index(bench), variant, _abi.dims_array(dims), byref(n)))
    return n.value


def alg_work(bench: str, dims) -> tuple[float, float]:
    b, f = c_double(), c_double()
    _abi.check(_abi.lib().pf_alg_work(registry.bench_index(bench), _abi.dims_array(dims), byref(b), byref(f)))
    return b.value, f.value


def _eval_item(ws: Workspace, variant: int, batch: int = 1, no_flush: bool = True, host_out=None):
    it = _abi.PfEval()
    it.ws, it.variant, it.batch, it.no_flush = ws.handle, variant, batch, int(no_flush)
    it._keep = host_out  # the pointer table must outlive the batch
    if host_out is not None:
        it.host_out = ctypes.cast(host_out, c_void_p)
    return it


class _Staging:
    """A pinned host buffer (pf_host_alloc) reused across batches."""

    def __init__(self, lib, size: int):
        self.lib = lib
        p = c_void_p()
        _abi.check(lib.pf_host_alloc(size, byref(p)))
        self.ptr, self.size, self.busy = p.value, size, False

    def release(self) -> None:
        self.busy = False

    def free(self) -> None:
        if self.ptr:
            self.lib.pf_host_free(self.ptr)
            self.ptr = None


def _torch_shares_context() -> bool:
    """True when torch has initialised CUDA in this process (its tensors and
    NCCL communicators live in the same primary context as libpfgpu's)."""
    torch = sys.modules.get("torch")
    try:
        return bool(torch is not None and torch.cuda.is_initialized())
    except Exception:  # noqa: BLE001 -- a broken torch import means no shared context
        return False


def device_count() -> int:
    n = c_int()
    rc = _abi.lib().pf_device_count(byref(n))
    return n.value if rc == 0 else 0


class B200Backend(Backend):
    """compile = variant lookup; execute = device-timed run (see module doc)."""

    def __init__(
        self,
        device: int = 0,
        samples: int = 5,
        seed: int = 1729,
        flush_l2: bool = True,
        min_sample_ms: float = 0.05,
        max_batch: int = 64,
        slow_ms: float = 50.0,
        memory_budget: float = 100e9,
        types=None,
    ):
        """``types``: the module whose value types (Artifact, CompileOutcome,
        ExecutionOutcome, ExecutionStatus, BackendError) this backend returns.
        Defaults to this package's; pass ``phaseforge.backend.types`` to drive
        the reference's unmodified engine, which compares enums by identity."""
        super().__init__()
        self.T = types or _own_types
        self.lib = _abi.lib()
        self.device = device
        self.samples = samples
        self.seed = seed
        self.flush_l2 = flush_l2
        self.min_sample_ms = min_sample_ms
        self.max_batch = max_batch
        self.slow_ms = slow_ms
        self._first_ms: dict[tuple, float] = {}
        self.memory_budget = memory_budget
        self._ws: "OrderedDict[tuple, Workspace]" = OrderedDict()
        self._artifacts: dict[tuple[str, int], Artifact] = {}
        self._batch: dict[tuple, int] = {}
        self._timeouts: dict[str, float] = {}
        self.device_runs = 0
        self.kernel_launches = 0
        # Optional reuse of measurements by artifact digest ("identical machine
        # code -> identical performance", the premise of explorer.py:175-183);
        # off by default so final_reps averages independent runs.
        self.measurement_cache: dict | None = None
        # pure-function memos: compile is pure in (kernel, order)
        self._variant_memo: dict[tuple, int] = {}
        self._order_memo: dict[tuple, tuple] = {}  # (id(order), bench) -> (order, variant)
        self._use_order_memo = os.environ.get("PF_ORDER_MEMO", "1") != "0"
        self._supported_memo: dict[tuple, bool] = {}
        self._compile_memo: dict[tuple, object] = {}
        # results of the last prefetch, consumed by execute():
        # (digest, "validation"|"measurement", input descriptor) -> (ms, outputs | None)
        self._prefetched: dict[tuple, tuple] = {}
        self._pending: list = []        # [(future, keys, job)] in submission order
        self._pending_keys: dict = {}   # key -> future of the batch that will produce it
        self._staging_pool: list = []
        self._worker = None
        self.failed: str | None = None
        self.prefetch_batches = 0
        self.batch_ms = 0.0

    # ------------------------------------------------------------ helpers
    def set_timeout_override(self, kernel_id: str, timeout: float) -> None:
        """Runs slower than ``timeout`` seconds report TIMEOUT (cli.py:194-195)."""
        if timeout <= 0:
            raise ValueError(f"timeout must be positive, got {timeout}")
        self._timeouts[kernel_id] = timeout

    def variant_for(self, kernel: KernelCase, order) -> tuple[str, int]:
        bench = registry.bench_of(kernel)
        # the engine asks about the same order objects several times (the
        # prefetch walk, explore's compile, the record): an identity memo
        # skips re-keying up to 256 pass names per call (the order is kept
        # alive by the memo, so its id cannot be reused while it is there)
        hit = self._order_memo.get((id(order), bench))
        if hit is not None and hit[0] is order:
            return bench, hit[1]
        key = (bench, tuple(map(_NAME, order.passes)))
        v = self._variant_memo.get(key)
        if v is None:
            if isinstance(order, PhaseOrder):
                own = order
            else:  # a foreign (reference) PhaseOrder: same pass names
                own = PhaseOrder(tuple(PassId(p.name) for p in order.passes))
            v = family(bench).select(passmodel.interpret(own))
            self._variant_memo[key] = v
        if self._use_order_memo:
            if len(self._order_memo) >= 1 << 18:
                self._order_memo.clear()
            self._order_memo[(id(order), bench)] = (order, v)
        return bench, v

    def artifact(self, bench: str, variant: int):
        key = (bench, variant)
        art = self._artifacts.get(key)
        if art is None:
            art = self.T.Artifact.from_content(artifact_content(bench, variant))
            self._artifacts[key] = art
        return art

    def workspace(self, bench: str, dims: tuple[int, ...], stock: bool, instance: int) -> Workspace:
        key = (bench, tuple(dims), "stock" if stock else "random")
        ws = self._ws.get(key)
        if ws is None:
            ws = Workspace(self.device, bench, dims)
            self._ws[key] = ws
            self._evict(keep=key)
        else:
            self._ws.move_to_end(key)
        ws.generate(stock, self.seed, instance)
        return ws

    def _evict(self, keep) -> None:
        total = sum(w.nbytes for w in self._ws.values())
        for key in list(self._ws):
            if total <= self.memory_budget:
                break
            if key == keep:
                continue
            w = self._ws.pop(key)
            total -= w.nbytes
            w.close()

    def close(self) -> None:
        self._drain()
        if self._worker is not None:
            self._worker.shutdown()
            self._worker = None
        for w in self._ws.values():
            w.close()
        self._ws.clear()
        for st in self._staging_pool:
            st.free()
        self._staging_pool.clear()

    def _crash(self, exc: _abi.PfError):
        # A sticky CUDA error poisons the context: drop every workspace and reset
        # -- unless torch shares the primary context (a reset would destroy its
        # tensors and NCCL communicators): then the backend is marked failed.
        self._prefetched.clear()
        self._pending.clear()
        self._pending_keys.clear()
        if _torch_shares_context():
            self.failed = str(exc)
            return self.T.ExecutionOutcome(self.T.ExecutionStatus.CRASH, log=str(exc) + " (device left failed)")
        for w in self._ws.values():
            w.handle = None  # memory dies with the context
            w.warm.clear()
        self._ws.clear()
        for st in self._staging_pool:
            st.ptr = None  # pinned memory dies with the context
        self._staging_pool.clear()
        self.lib.pf_device_reset(self.device)
        return self.T.ExecutionOutcome(self.T.ExecutionStatus.CRASH, log=str(exc))

    def _supported(self, bench: str, variant: int, dims) -> bool:
        key = (bench, variant, tuple(dims))
        ok = self._supported_memo.get(key)
        if ok is None:
            ok = self._supported_memo[key] = _supported_dims(bench, variant, dims)
        return ok

    @contextlib.contextmanager
    def digest_timing(self):
        """Inside the block, measurements are keyed by artifact digest: an
        artifact measured once keeps that time (identical machine code ->
        identical performance, the premise of REUSED, explorer.py:175-183).
        Used around reduce_order, whose trials mostly re-measure the same
        artifact and would otherwise be rejected by run-to-run noise."""
        was = self.measurement_cache
        self.measurement_cache = {} if was is None else was
        try:
            yield
        finally:
            self.measurement_cache = was

    # ------------------------------------------------------------ Backend API
    def compile(self, kernel: KernelCase, order):
        bench, variant = self.variant_for(kernel, order)
        key = (bench, variant, kernel.validation_input, kernel.measurement_input)
        out = self._compile_memo.get(key)
        if out is not None:
            return out
        out = self.T.CompileOutcome.success(self.artifact(bench, variant))
        for text in (kernel.validation_input, kernel.measurement_input):
            _, dims = registry.parse_descriptor(text)
            if not self._supported(bench, variant, dims):
                out = self.T.CompileOutcome.codegen_failure(
                    f"{bench} variant {family(bench).key(variant)} does not support {text}"
                )
                break
        self._compile_memo[key] = out
        return out

    def execute(
        self,
        kernel: KernelCase,
        order,
        artifact,
        input_kind,
        random_input_index: int | None = None,
    ):
        bench, variant = self.variant_for(kernel, order)
        if self.artifact(bench, variant).digest != artifact.digest:
            raise self.T.BackendError(
                f"artifact {artifact.digest[:12]} was not compiled from this order for {kernel.id!r}"
            )
        return self.execute_variant(kernel, bench, variant, input_kind, random_input_index)

    def execute_variant(self, kernel: KernelCase, bench: str, variant: int, input_kind,
                        random_input_index: int | None = None):
        """``execute`` after the order -> variant lookup (also the entry of the
        process-level runner, ``pftool run``)."""
        if self.failed:
            raise self.T.BackendError(f"device {self.device} failed earlier: {self.failed}")
        artifact = self.artifact(bench, variant)
        if random_input_index is None and (self._prefetched or self._pending):
            kind = input_kind.value
            desc = kernel.validation_input if kind == "validation" else kernel.measurement_input
            key = (artifact.digest, kind, desc)
            if key in self._pending_keys:
                self._wait_for(key)
            else:
                self._drain()  # no device work of this backend may overlap a batch
            hit = self._prefetched.pop(key, None)
            if hit is not None:
                return self._finish(kernel, hit[0], hit[1])
        elif self._pending:
            self._drain()
        try:
            # compare by value: the caller may use the reference's InputKind enum
            if random_input_index is not None or input_kind.value == "validation":
                _, dims = registry.parse_descriptor(kernel.validation_input)
                stock = random_input_index is None
                ws = self.workspace(bench, dims, stock, -1 if stock else int(random_input_index))
                ms = ws.run(variant, samples=1, batch=1, restore=True, flush=False)
                self._count(bench, variant, dims, 1)
                outs = ws.outputs()
                values = tuple(float(x) for arr in outs for x in arr.tolist())
                return self._finish(kernel, ms[0], values)
            _, dims = registry.parse_descriptor(kernel.measurement_input)
            ckey = (kernel.measurement_input, artifact.digest)
            if self.measurement_cache is not None and ckey in self.measurement_cache:
                return self._finish(kernel, self.measurement_cache[ckey], None)
            ws = self.workspace(bench, dims, True, -1)
            ms = statistics.median(self._timed(ws, variant))
            if self.measurement_cache is not None:
                self.measurement_cache[ckey] = ms
            return self._finish(kernel, ms, None)
        except _abi.PfError as exc:
            if exc.code == _abi.PF_ECUDA:
                return self._crash(exc)
            raise self.T.BackendError(str(exc)) from exc

    def _finish(self, kernel: KernelCase, ms: float, outputs):
        seconds = max(ms, 1e-6) * 1e-3
        limit = self._timeouts.get(kernel.id)
        T = self.T
        if limit is not None and seconds > limit:
            return T.ExecutionOutcome(T.ExecutionStatus.TIMEOUT, log=f"{seconds:.6f}s > timeout {limit:.6f}s")
        return T.ExecutionOutcome(T.ExecutionStatus.VALID, wall_time=seconds, outputs=outputs)

    def _count(self, bench: str, variant: int, dims, runs: int) -> None:
        self.device_runs += runs
        self.kernel_launches += runs * variant_launches(bench, variant, dims)

    def _timed(self, ws: Workspace, variant: int) -> list[float]:
        """Median-of-``samples`` device time of one run (ms).  The first use of
        a (workspace, variant) does an untimed warm-up (module load, scratch,
        graph capture) and sizes the batch so a sample spans at least
        ``min_sample_ms`` (us-scale kernels); runs slower than ``slow_ms`` take
        a single sample (their relative jitter is already far below 1%)."""
        key = (ws.bench, ws.dims, variant)
        if variant not in ws.warm:
            first = ws.run(variant, samples=1, batch=1, restore=True, flush=False)[0]
            warmups = 1
            if first <= self.slow_ms:  # a slow run's one-time costs are below its jitter: one warm-up
                first = ws.run(variant, samples=1, batch=1, restore=True, flush=False)[0]
                warmups = 2
            self._count(ws.bench, variant, ws.dims, warmups)
            ws.warm.add(variant)
            self._first_ms[key] = first
            if key not in self._batch:
                batch = 1
                if first < self.min_sample_ms:
                    batch = min(self.max_batch, max(1, int(self.min_sample_ms / max(first, 1e-4)) + 1))
                self._batch[key] = batch
        batch = self._batch.get(key, 1)
        samples = 1 if self._first_ms.get(key, 0.0) > self.slow_ms else self.samples
        ms = ws.run(variant, samples=samples, batch=batch, restore=True, flush=self.flush_l2)
        self._count(ws.bench, variant, ws.dims, samples * batch)
        return ms

    def prewarm(self, kernel: KernelCase) -> int:
        """Give every variant of ``kernel``'s family its first-use warm-up
        (module load, scratch, graph capture, batch sizing: the untimed
        runs ``_timed`` / the prefetch do on first use) at the measurement
        size, so later measurements are steady-state.  Returns the number of
        variants warmed."""
        bench = registry.bench_of(kernel)
        _, mdims = registry.parse_descriptor(kernel.measurement_input)
        ws = self.workspace(bench, mdims, True, -1)
        n = 0
        for v in range(len(family(bench).knobs)):
            if v in ws.warm or not self._supported(bench, v, mdims):
                continue
            first = ws.run(v, samples=1, batch=1, restore=True, flush=False)[0]
            warmups = 1
            if first <= self.slow_ms:
                first = ws.run(v, samples=1, batch=1, restore=True, flush=False)[0]
                warmups = 2
            self._count(bench, v, mdims, warmups)
            ws.warm.add(v)
            key = (bench, ws.dims, v)
            self._first_ms[key] = first
            if key not in self._batch:
                self._batch[key] = (min(self.max_batch, max(1, int(self.min_sample_ms / max(first, 1e-4)) + 1))
                                    if first < self.min_sample_ms else 1)
            n += 1
        return n

    # ------------------------------------------------------------ batched evaluation
    def prefetch(self, kernel: KernelCase, orders) -> int:
        """``explore(..., prefetch=True)`` hook: batch the fresh evaluations of
        ``orders`` (see module doc).  Returns the number of candidates."""
        return self.prefetch_many([(kernel, orders)])

    def fresh_candidates(self, kernel: KernelCase, orders) -> list[tuple[str, int, str]]:
        """(bench, variant, digest) of the first order of every distinct
        digest in ``orders`` that compiles -- explore's fresh evaluations."""
        out, seen = [], set()
        for order in orders:
            c = self.compile(kernel, order)
            if not c.is_ok or c.artifact.digest in seen:
                continue
            seen.add(c.artifact.digest)
            bench, variant = self.variant_for(kernel, order)
            out.append((bench, variant, c.artifact.digest))
        return out

    def prefetch_many(self, jobs, host_inputs: dict | None = None) -> int:
        """Run the fresh evaluations of several (kernel, orders) jobs as
        device batches, one per job, issued by a worker thread so that the
        host prepares job k+1 (and the engine walks job k's records) while
        the device runs job k.  Per candidate: one validation run on the
        stock validation input (outputs copied back) and the measurement
        protocol of ``execute`` (first use: two warm-up runs -- one for a run
        slower than ``slow_ms`` -- that size the batch of us-scale kernels; then ``samples`` timed samples, each after
        an L2 flush; median).  ``host_inputs`` maps (kernel id, "validation"
        | "measurement") to {array index: pinned host pointer}: those inputs
        are uploaded first, asynchronously on the copy stream (the end-to-end
        path).  ``execute`` waits for a job's batch only when it asks for
        one of that job's results.  A CUDA failure inside a batch drops the
        remaining results (the engine then evaluates candidate by candidate,
        which isolates the failing one as a CRASH record).  Returns the
        number of candidates."""
        if self.failed:
            raise self.T.BackendError(f"device {self.device} failed earlier: {self.failed}")
        self._drain()
        host_inputs = host_inputs or {}
        total = 0
        try:
            for (kid, kind), table in host_inputs.items():
                kernel = next(k for k, _ in jobs if k.id == kid)
                _, dims = registry.parse_descriptor(
                    kernel.validation_input if kind == "validation" else kernel.measurement_input)
                ws = self.workspace(registry.bench_of(kernel), dims, True, -1)
                for a, ptr in sorted(table.items()):
                    _abi.check(self.lib.pf_ws_upload_async(ws.handle, a, ptr, ws.elems[a]))
                # the uploaded arrays ARE this descriptor's input (the runner's
                # data file); a later generate() for it is a no-op
                ws.input_tag = (True, int(self.seed), -1)
            # the jobs' streams are walked round-robin, chunk by chunk, so the
            # device has every kernel's first candidates early instead of
            # idling while the host draws one kernel's whole stream
            walkers = [self._submit_job(kernel, orders) for kernel, orders in jobs]
            while walkers:
                for w in list(walkers):
                    n = next(w, None)
                    if n is None:
                        walkers.remove(w)
                    else:
                        total += n
        except _abi.PfError as exc:
            return self._batch_failed(exc) or total
        return total

    def _submit_job(self, kernel: KernelCase, orders):
        """Walk ``orders`` (any iterable, e.g. a lazy draw) in geometrically
        growing chunks and submit each chunk's new fresh candidates as one
        batch: the device starts on the first candidates while the host is
        still compiling the rest of the stream.  A generator: yields the
        number of candidates submitted after each chunk."""
        seen, chunk, pending = set(), 16, []
        for i, order in enumerate(orders):
            c = self.compile(kernel, order)
            if c.is_ok and c.artifact.digest not in seen:
                seen.add(c.artifact.digest)
                bench, variant = self.variant_for(kernel, order)
                pending.append((bench, variant, c.artifact.digest))
            if i + 1 == chunk:
                yield self._submit_cands(kernel, pending) if pending else 0
                pending = []
                chunk *= 4
        yield self._submit_cands(kernel, pending) if pending else 0

    def _submit_cands(self, kernel: KernelCase, cands) -> int:
        _, vdims = registry.parse_descriptor(kernel.validation_input)
        _, mdims = registry.parse_descriptor(kernel.measurement_input)
        plan = [(bench, variant, digest, self.workspace(bench, vdims, True, -1),
                 self.workspace(bench, mdims, True, -1)) for bench, variant, digest in cands]
        # first use of a measurement variant: warm-up runs decide the batch size
        cold = []
        for bench, variant, digest, vws, mws in plan:
            if variant not in mws.warm and (mws, variant) not in cold:
                cold.append((mws, variant))
        if cold:
            # one warm-up each; a second one only for runs not slower than
            # slow_ms (a slow run's one-time costs are below its jitter)
            ms = self._worker_submit([_eval_item(ws, v) for ws, v in cold]).result()
            again = [i for i, t in enumerate(ms) if t <= self.slow_ms]
            if again:
                ms2 = self._worker_submit([_eval_item(*cold[i]) for i in again]).result()
                for i, t in zip(again, ms2):
                    ms[i] = t
            for i, (ws, variant) in enumerate(cold):
                key = (ws.bench, ws.dims, variant)
                first = ms[i]
                ws.warm.add(variant)
                self._first_ms[key] = first
                self._count(ws.bench, variant, ws.dims, 2 if i in again else 1)
                if key not in self._batch:
                    self._batch[key] = (min(self.max_batch, max(1, int(self.min_sample_ms / max(first, 1e-4)) + 1))
                                        if first < self.min_sample_ms else 1)
        out_n = [sum(n for (_, _, o), n in zip(vws.arrays, vws.elems) if o) for _, _, _, vws, _ in plan]
        staging = self._staging_buffer(4 * sum(out_n))
        items, layout, off = [], [], 0
        for (bench, variant, digest, vws, mws), nout in zip(plan, out_n):
            ptrs, o = [], off
            for (_, _, is_out), n in zip(vws.arrays, vws.elems):
                ptrs.append(staging.ptr + o if is_out else None)
                o += 4 * n if is_out else 0
            items.append(_eval_item(vws, variant, host_out=(c_void_p * len(vws.arrays))(*ptrs)))
            entry = {"v": len(items) - 1, "off": off // 4, "n": nout, "m": []}
            off = o
            if not (self.measurement_cache is not None and (kernel.measurement_input, digest) in self.measurement_cache):
                key = (bench, mws.dims, variant)
                samples = 1 if self._first_ms.get(key, 0.0) > self.slow_ms else self.samples
                for _ in range(samples):
                    items.append(_eval_item(mws, variant, batch=self._batch.get(key, 1), no_flush=not self.flush_l2))
                    entry["m"].append(len(items) - 1)
            layout.append(entry)
        future = self._worker_submit(items)
        keys = []
        for (bench, variant, digest, vws, mws) in plan:
            keys += [(digest, "validation", kernel.validation_input), (digest, "measurement", kernel.measurement_input)]
        self._pending.append((future, keys, (kernel, plan, layout, staging)))
        for k in keys:
            self._prefetched.pop(k, None)
            self._pending_keys[k] = future
        return len(plan)

    def _collect(self, future, job) -> None:
        """Turn one finished batch into prefetched execute() results."""
        kernel, plan, layout, staging = job
        ms = future.result()
        import numpy as np

        for (bench, variant, digest, vws, mws), entry in zip(plan, layout):
            values = tuple(np.ctypeslib.as_array(
                (ctypes.c_float * max(1, entry["n"])).from_address(staging.ptr + 4 * entry["off"]))[:entry["n"]].tolist())
            self._prefetched[(digest, "validation", kernel.validation_input)] = (ms[entry["v"]], values)
            self._count(bench, variant, vws.dims, 1)
            ckey = (kernel.measurement_input, digest)
            if entry["m"]:
                key = (bench, mws.dims, variant)
                t = statistics.median(ms[i] for i in entry["m"])
                self._count(bench, variant, mws.dims, len(entry["m"]) * self._batch.get(key, 1))
                if self.measurement_cache is not None:
                    self.measurement_cache[ckey] = t
            else:
                t = self.measurement_cache[ckey]
            self._prefetched[(digest, "measurement", kernel.measurement_input)] = (t, None)
        staging.release()
        self.prefetch_batches += 1

    def _wait_for(self, key) -> None:
        """Block until the batch holding ``key`` (and every earlier one) is done."""
        future = self._pending_keys.get(key)
        if future is None:
            return
        while self._pending:
            f, keys, job = self._pending.pop(0)
            for k in keys:
                self._pending_keys.pop(k, None)
            try:
                self._collect(f, job)
            except _abi.PfError as exc:
                self._batch_failed(exc)
                return
            if f is future:
                return

    def _drain(self) -> None:
        while self._pending:
            self._wait_for(self._pending[0][1][0])

    def _batch_failed(self, exc: "_abi.PfError") -> int:
        for f, _, _ in self._pending:
            try:
                f.result()
            except Exception:  # noqa: BLE001 -- the batch after a failed one is dropped too
                pass
        self._pending.clear()
        self._pending_keys.clear()
        self._prefetched.clear()
        if exc.code != _abi.PF_ECUDA:
            raise self.T.BackendError(str(exc)) from exc
        self._crash(exc)
        if self.failed:
            raise self.T.BackendError(f"device {self.device} failed: {exc}") from exc
        return 0

    def _worker_submit(self, items):
        """Enqueue one pf_eval_batch on the backend's device worker (a single
        thread: batches never overlap on the device; ctypes drops the GIL)."""
        if self._worker is None:
            from concurrent.futures import ThreadPoolExecutor

            self._worker = ThreadPoolExecutor(max_workers=1, thread_name_prefix=f"pfgpu-dev{self.device}")
        arr = (_abi.PfEval * len(items))(*items)
        keep = [it._keep for it in items]

        def run():
            n = len(items)
            ms = (c_float * n)()
            total = c_float()
            _abi.check(self.lib.pf_eval_batch(arr, n, 1, 1, ms, byref(total)))
            self.batch_ms += total.value
            return list(ms)

        return self._worker.submit(run)

    def _staging_buffer(self, nbytes: int) -> "_Staging":
        """Pinned host staging for one batch's validation outputs (pooled)."""
        for st in self._staging_pool:
            if not st.busy and st.size >= nbytes:
                st.busy = True
                return st
        st = _Staging(self.lib, max(nbytes, 1 << 20))
        st.busy = True
        self._staging_pool.append(st)
        return st

    # ------------------------------------------------------------ conveniences
    def baseline_outputs(self, kernel: KernelCase) -> tuple[float, ...]:
        """Validation-input outputs of the empty-order (baseline) variant."""
        compiled = self.compile(kernel, PhaseOrder())
        if not compiled.is_ok:
            raise self.T.BackendError(f"baseline compile failed for {kernel.id!r}")
        out = self.execute(kernel, PhaseOrder(), compiled.artifact, _own_types.InputKind.VALIDATION)
        if out.status.value != "valid" or out.outputs is None:
            raise self.T.BackendError(f"baseline validation run failed for {kernel.id!r}: {out.log}")
        return out.outputs

    def time_variant(self, bench: str, dims, variant: int, samples: int | None = None) -> float:
        """Median device time (s) of ``variant`` on the stock input at ``dims``."""
        ws = self.workspace(bench, tuple(dims), True, -1)
        old = self.samples
        if samples:
            self.samples = samples
        try:
            return statistics.median(self._timed(ws, variant)) * 1e-3
        finally:
            self.samples = old


__all__ = ["B200Backend", "Workspace", "alg_work", "bench_arrays", "device_count", "family", "variant_launches",
           "variant_sass"]
