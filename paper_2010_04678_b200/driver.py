"""Batch drivers -- the drop-in for the reference's ``cals.driver.run``.

``run(t, models, cfg, mode=ExecutionMode.CALS, r_star=...)`` keeps the
reference's signature, validation order, errors and result layout
(driver.py:73-121), and executes the fused CALS loop entirely on the GPU
(csrc/engine.cu).  SEQUENTIAL / PARALLEL are served by the same engine one
model at a time: the fused kernels are bitwise position-independent, so a
K=1 run reproduces that model's columns of a K>1 run exactly.
"""

from __future__ import annotations

import enum
import os
import threading
import time
import warnings
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

from .als import ConvergenceConfig, LineSearchConfig, NonConvergedNnlsWarning
from .engine import CalsEngine
from .model import STATUS_FROM_CODE, Model, ModelStatus
from .mttkrp import mttkrp_flops
from .multimatrix import DEFAULT_R_STAR, CapacityError
from .tensor import DenseTensor


# host-side phase timings of the most recent fused run (diagnostics / bench)
LAST_RUN_PROFILE: dict = {}


class ExecutionMode(enum.Enum):
    SEQUENTIAL = "sequential"
    PARALLEL = "parallel"
    CALS = "cals"


@dataclass
class SegmentTrace:
    """Timing/flop record for one measured segment (driver.py:46-53)."""

    label: str
    flops: int
    seconds: float
    meta: dict = field(default_factory=dict)


def run(t: DenseTensor, models: Iterable[Model], cfg: ConvergenceConfig, *,
        mode: ExecutionMode = ExecutionMode.CALS, r_star: int = DEFAULT_R_STAR,
        ls: LineSearchConfig | None = None, nonneg: bool = False, threads: int = 1,
        deterministic: bool = False, trace: list | None = None,
        variant_table=None) -> list[Model]:
    """Fit every queued model against the shared tensor and return the output
    queue (retirement order).  Inputs are read-only starting points; their
    ``status`` is set to ACTIVE once admitted, as in the reference.

    ``threads`` / ``deterministic`` / ``variant_table`` are accepted for API
    compatibility: the GPU path is always deterministic (fixed split-K order)
    and runs one fused kernel for every mode.
    """
    if ls is None:
        ls = LineSearchConfig()
    queue = list(models)
    for m in queue:
        if m.dims != t.dims:
            raise ValueError(f"model {m.id!r} dims {m.dims} != tensor {t.dims}")
    if mode is ExecutionMode.CALS:
        for m in queue:
            if m.rank > r_star:
                raise CapacityError(f"model {m.id!r} rank {m.rank} exceeds r_star {r_star}")
    if mode not in (ExecutionMode.SEQUENTIAL, ExecutionMode.PARALLEL, ExecutionMode.CALS):
        raise ValueError(f"unknown execution mode {mode!r}")
    if not queue:
        return []
    # (the ||T||^2 > 0 check runs in _run_fused, on the device copy, once
    # the uploads are queued -- still before any model is touched)
    if t._sqnorm is not None and t._sqnorm <= 0.0:
        raise ValueError("tensor squared norm must be positive")
    if mode is ExecutionMode.CALS:
        return _run_fused(t, queue, cfg, r_star, trace, label_per_model=False, ls=ls,
                          nonneg=nonneg)
    # SEQUENTIAL / PARALLEL: one instance at a time (driver.py:133-160); a
    # numerical failure retires it with the reference's _fit_or_fail record
    out = []
    for m in queue:
        out += _run_fused(t, [m], cfg, m.rank, trace, label_per_model=True, ls=ls,
                          nonneg=nonneg)
    return out


def _prebuild_results(eng: CalsEngine, queue: list[Model], pool: np.ndarray, shells: list) -> None:
    """Result Model objects whose factors are (Fortran) views into the result
    pool ``pool`` -- filled by the device later; scalars set by _run_fused.
    Runs on a helper thread while the caller sits in the device loop: the
    initial sleep hands the GIL back so the caller enters the C library
    (which releases it) before this loop takes it."""
    time.sleep(0.001)
    for k, src in enumerate(queue):
        shells[k] = Model._from_engine(id=src.id, rank=src.rank, factors=eng.unpack(pool, k),
                                       error=float("nan"), fit=float("nan"), iterations_done=0,
                                       status=ModelStatus.ACTIVE, seconds_active=0.0,
                                       meta=dict(src.meta))


def _failure_record(src: Model) -> Model:
    """_fit_or_fail's result for an instance whose update raised
    (driver.py:148-160): the starting factors, no iterations, error nan."""
    return Model(id=src.id, rank=src.rank, factors=src.copy_factors(), error=float("nan"),
                 fit=-np.inf, status=ModelStatus.FAILED, meta=dict(src.meta))


def _instance_flops(t: DenseTensor, rank: int, iterations: int) -> int:
    return iterations * t.order * mttkrp_flops(t.dims, rank)


class _EngineCache:
    """Device engines kept between ``run`` calls (keyed by shape, capacity and
    the rank sequence) so repeated sweeps reuse every device allocation and
    re-bind to the new tensor instead of re-allocating.  An engine is checked
    out while in use, so concurrent callers never share one."""

    def __init__(self, limit: int = 4):
        self.limit = limit
        self.free: list = []
        self.lock = threading.Lock()

    def acquire(self, dev, r_star: int, ranks, trace_capacity: int) -> CalsEngine:
        import torch

        key = (torch.cuda.current_device(), tuple(dev.dims), int(r_star), tuple(int(r) for r in ranks), int(trace_capacity),
               os.environ.get("CALS_TREE"), os.environ.get("CALS_SPLITS"))
        with self.lock:
            for i, (k, e) in enumerate(self.free):
                if k == key:
                    del self.free[i]
                    e.set_tensor(dev)
                    e._cache_key = key
                    return e
        e = CalsEngine(dev, r_star, ranks, trace_capacity=trace_capacity)
        e._cache_key = key
        return e

    def release(self, e: CalsEngine) -> None:
        with self.lock:
            self.free.append((e._cache_key, e))
            while len(self.free) > self.limit:
                self.free.pop(0)[1].close()

    def clear(self) -> None:
        with self.lock:
            for _, e in self.free:
                e.close()
            self.free.clear()


_ENGINES = _EngineCache()


def clear_engine_cache() -> None:
    """Free the device workspaces kept between ``run`` calls."""
    _ENGINES.clear()


def _run_fused(t: DenseTensor, queue: list[Model], cfg: ConvergenceConfig, r_star: int,
               trace: list | None, label_per_model: bool,
               ls: LineSearchConfig | None = None, nonneg: bool = False,
               raise_on_update_failure: bool = False) -> list[Model]:
    """``label_per_model``: the run is one SEQUENTIAL / PARALLEL instance --
    the input's status is left alone and an update failure returns the
    reference's failure record; ``raise_on_update_failure`` (run_single_als)
    raises ValueError instead, as update_factor does (als.py:84-85)."""
    import torch

    prof = LAST_RUN_PROFILE
    prof.clear()
    t0 = time.perf_counter()
    dev = t.device()  # queued: the tensor upload overlaps the host packing below
    t1 = time.perf_counter()
    ranks = [m.rank for m in queue]
    tcap = _trace_cap(queue, cfg) if trace is not None else 1
    eng = _ENGINES.acquire(dev, r_star, ranks, tcap)
    t2 = time.perf_counter()
    try:
        eng.prepare()  # tensor slicing overlaps the host packing below
        eng.set_line_search(bool(ls is not None and ls.enabled), None if ls is None else ls.alpha)
        eng.set_nonneg(nonneg)
        t2p = time.perf_counter()
        eng.load_pool(eng.pack([m.factors for m in queue], out=eng.staging()))
        t3 = time.perf_counter()
        sqnorm = t.device_sqnorm()  # waits for both uploads
        if sqnorm <= 0.0:
            raise _BadNorm()
        # the result pool lands in a fresh page-locked block (torch's caching
        # host allocator -> no cudaHostAlloc per run) that the returned
        # factors view directly: no host-side copy.  The result Model objects
        # (factor views into it) are built by a helper thread while the device
        # loop runs -- eng.run blocks inside the C library with the GIL
        # released -- and only get their scalars afterwards.
        pool_t = torch.empty(max(eng.pool_elems, 1), dtype=torch.float64, pin_memory=True)
        shells: list = [None] * len(queue)
        builder = threading.Thread(target=_prebuild_results, args=(eng, queue, pool_t.numpy(),
                                                                   shells), daemon=True)
        tic = time.perf_counter()
        builder.start()
        eng.run(cfg.tol, cfg.max_iterations, sqnorm)
        t4 = time.perf_counter()
        res = eng.results(with_pool=False)
        # the factor pool comes down while the Model objects are built below
        # (they are views into it); the stream is synchronised before return
        eng.pool_download(pool_t.numpy())
        warned = eng.nnls_warnings() if nonneg else None
        upd_failed = eng.update_failures() if label_per_model else None
        wall = time.perf_counter() - tic
        records = eng.trace() if (trace is not None and not label_per_model) else None
    except _BadNorm:
        _ENGINES.release(eng)  # nothing ran: the engine stays reusable
        raise ValueError("tensor squared norm must be positive") from None
    except BaseException:
        eng.close()
        raise
    if warned is not None and warned.any():
        warnings.warn("active-set search hit its iteration cap", NonConvergedNnlsWarning,
                      stacklevel=3)
    t5 = time.perf_counter()
    prof.update(tensor_upload_s=t1 - t0, engine_create_s=t2 - t1, prepare_s=t2p - t2,
                pool_upload_s=t3 - t2p,
                upload_wait_s=tic - t3, device_loop_s=t4 - tic, results_download_s=t5 - t4)
    if not label_per_model:
        for m in queue:
            m.status = ModelStatus.ACTIVE  # admitted (driver.py:202)
    builder.join()
    order = np.argsort(res.retire_seq, kind="stable").tolist()
    lam_off = np.concatenate([[0], np.cumsum(ranks)]).tolist()
    status, err, fit = res.status.tolist(), res.error.tolist(), res.fit.tolist()
    iters, secs = res.iterations.tolist(), res.seconds_active.tolist()
    if label_per_model:
        # one instance per call: its wall time is both its seconds_active and
        # its trace segment, as _run_sequential records them (driver.py:133-144)
        secs = [wall] * len(secs)
    lam = res.lambdas
    out = []
    try:
        for k in order:
            src = queue[k]
            if upd_failed is not None and upd_failed[k]:
                if raise_on_update_failure:
                    raise ValueError("non-finite values in the factor update of model "
                                     f"{src.id!r}")
                rec = _failure_record(src)
                rec.seconds_active = secs[k]
                out.append(rec)
                continue
            m = shells[k]
            m.error, m.fit, m.iterations_done = err[k], fit[k], iters[k]
            m.status, m.seconds_active = STATUS_FROM_CODE[status[k]], secs[k]
            m.meta["lambdas"] = lam[lam_off[k]:lam_off[k + 1]]
            out.append(m)
    finally:
        # the factor views are valid once the pool download has landed; only
        # then may another run reuse the engine (and its device pool)
        torch.cuda.current_stream().synchronize()
        _ENGINES.release(eng)
    prof["build_models_s"] = time.perf_counter() - t5
    if trace is not None:
        if label_per_model:
            for r in out:
                trace.append(SegmentTrace(
                    label=f"als:{r.id}", flops=_instance_flops(t, r.rank, r.iterations_done),
                    seconds=r.seconds_active, meta={"id": r.id, "rank": r.rank,
                                        "iterations": r.iterations_done}))
        else:
            for width, n_active, secs in records:
                trace.append(SegmentTrace(
                    label="cals-iteration", flops=t.order * mttkrp_flops(t.dims, width),
                    seconds=secs, meta={"width": width, "n_active": n_active}))
    return out


class _BadNorm(Exception):
    pass


def _trace_cap(queue, cfg) -> int:
    # every driver iteration retires or advances >= 1 model; bound generously
    return int(min(1 << 22, cfg.max_iterations * len(queue) + 2))
