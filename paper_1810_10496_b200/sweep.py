"""Batched candidate evaluation and the multi-GPU candidate scheduler.

The reference evaluates candidates one at a time: ``explore`` draws an
order, compiles it, and runs validation + one measurement per fresh digest
(`/root/reference/pkg/src/phaseforge/explorer.py:152-214`), each execution a
runner process (toolchain.py:216-273).  Here:

* ``candidate_set`` replays ``explore``'s order stream (same RNG use,
  catalog.py:138-145) through ``compile`` and keeps the first order of every
  distinct artifact digest -- exactly the set of fresh evaluations ``explore``
  performs; REUSED records never touch the device (explorer.py:175-183);
* ``evaluate_round`` runs a list of (workspace, variant) evaluations as one
  device batch (``pf_eval_batch``): back-to-back on one stream, one CUDA event
  pair per candidate, no host synchronisation in between;
* ``explore_suite`` runs ``explore`` for several kernels with their device
  work batched ahead (``B200Backend.prefetch_many``) -- the product path the
  bench times;
* ``shard`` splits work across GPUs for the one-process-per-GPU scheduler
  (independent evaluations, no collective; longest-processing-
  time-first by estimated cost).
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_float, c_void_p
from dataclasses import dataclass
from random import Random

from . import _abi, passmodel, registry
from .backend.b200 import B200Backend, Workspace, family, variant_launches
from .catalog import PassCatalog, PhaseOrder, random_phase_order
from .dist import shard
from .explorer import ExplorationConfig, draw_orders, explore, remember_orders, stream_key


@dataclass(frozen=True)
class Candidate:
    bench: str
    variant: int
    digest: str
    order: PhaseOrder
    first_index: int


def candidate_set(backend: B200Backend, bench: str, catalog: PassCatalog | None = None,
                  num_sequences: int = 1000, max_len: int = 256, seed: int = 1729,
                  include_baseline: bool = True) -> list[Candidate]:
    """Distinct-digest candidates of ``explore``'s stream, in first-seen order."""
    catalog = catalog or passmodel.default_catalog()
    cfg = ExplorationConfig(num_sequences=num_sequences, max_len=max_len, seed=seed)
    fam = family(bench)
    out: list[Candidate] = []
    seen: set[str] = set()
    if include_baseline:
        v0 = fam.select(passmodel.BASELINE_STATE)
        art = backend.artifact(bench, v0)
        out.append(Candidate(bench, v0, art.digest, PhaseOrder(), -1))
        seen.add(art.digest)
    for i, order in enumerate(draw_orders(catalog, cfg)):
        v = fam.select(passmodel.interpret(order))
        d = backend.artifact(bench, v).digest
        if d not in seen:
            seen.add(d)
            out.append(Candidate(bench, v, d, order, i))
    return out


def _ptr_table(ws: Workspace, table: dict | None):
    if table is None:
        return None
    arr = (c_void_p * len(ws.arrays))(*[table.get(a) for a in range(len(ws.arrays))])
    return arr


def evaluate_round(items: list[tuple[Workspace, int]], restore: bool = True, flush_l2: bool = False,
                   host_in: dict | None = None, host_out: dict | None = None) -> tuple[list[float], float]:
    """Run ``items`` as one batch; returns (per-evaluation ms, whole-batch ms).

    ``host_in`` / ``host_out`` map a Workspace to {array index: host pointer};
    inputs are uploaded before the first evaluation of that workspace only.
    """
    n = len(items)
    evals = (_abi.PfEval * n)()
    keep = []
    uploaded: set[int] = set()
    for i, (ws, v) in enumerate(items):
        evals[i].ws = ws.handle
        evals[i].variant = v
        hin = None
        if host_in is not None and id(ws) not in uploaded and ws in host_in:
            hin = _ptr_table(ws, host_in[ws])
            uploaded.add(id(ws))
            ws.input_tag = None  # device inputs (and the pristine copy) are now the uploaded data
        hout = _ptr_table(ws, host_out[ws]) if host_out is not None and ws in host_out else None
        keep += [hin, hout]
        evals[i].host_in = ctypes.cast(hin, c_void_p) if hin is not None else None
        evals[i].host_out = ctypes.cast(hout, c_void_p) if hout is not None else None
    ms_each = (c_float * n)()
    total = c_float()
    _abi.check(_abi.lib().pf_eval_batch(evals, n, int(restore), int(flush_l2), ms_each, byref(total)))
    return list(ms_each), total.value


def _lazy_orders(catalog: PassCatalog, config: ExplorationConfig):
    """``draw_orders(catalog, config)`` one order at a time (same RNG use,
    explorer.py:163-167), so batches can start before the stream is drawn;
    the finished stream is remembered for ``explore``'s own draw."""
    rng = Random(config.seed)
    drawn = []
    for _ in range(config.num_sequences):
        order = random_phase_order(catalog, config.max_len, rng)
        drawn.append(order)
        yield order
    remember_orders(stream_key(catalog, config), drawn)


def explore_suite(kernels, catalog: PassCatalog, configs, backend: B200Backend, host_inputs: dict | None = None):
    """The exploration step of ``cmd_explore`` (cli.py:168-218) for several
    kernels: ``explorer.explore`` per kernel, unchanged, with the device work
    of every kernel's fresh evaluations batched ahead of it
    (``B200Backend.prefetch_many``: one batch per kernel, issued by the
    device worker while the engine walks the previous kernel's records).
    Returns {kernel id: sorted records}, the same records ``explore`` gives
    without prefetching."""
    jobs = [(k, _lazy_orders(catalog, c)) for k, c in zip(kernels, configs)]
    backend.prefetch_many(jobs, host_inputs)
    return {k.id: explore(k, catalog, c, backend) for k, c in zip(kernels, configs)}


def launches_of(items: list[tuple[Workspace, int]]) -> int:
    return sum(variant_launches(ws.bench, v, ws.dims) for ws, v in items)


__all__ = ["Candidate", "candidate_set", "evaluate_round", "explore_suite", "launches_of", "shard"]
