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
import time
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

from .als import ConvergenceConfig, LineSearchConfig, _NEXT
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
    if nonneg:
        raise NotImplementedError(_NEXT)
    if not queue:
        return []
    if t.sqnorm <= 0.0:
        raise ValueError("tensor squared norm must be positive")
    if mode is ExecutionMode.CALS:
        return _run_fused(t, queue, cfg, r_star, trace, label_per_model=False, ls=ls)
    out = []
    for m in queue:
        out += _run_fused(t, [m], cfg, m.rank, trace, label_per_model=True, ls=ls)
    return out


def _instance_flops(t: DenseTensor, rank: int, iterations: int) -> int:
    return iterations * t.order * mttkrp_flops(t.dims, rank)


def _run_fused(t: DenseTensor, queue: list[Model], cfg: ConvergenceConfig, r_star: int,
               trace: list | None, label_per_model: bool,
               ls: LineSearchConfig | None = None) -> list[Model]:
    prof = LAST_RUN_PROFILE
    prof.clear()
    t0 = time.perf_counter()
    dev = t.device()
    t1 = time.perf_counter()
    eng = CalsEngine(dev, r_star, [m.rank for m in queue],
                     trace_capacity=_trace_cap(queue, cfg) if trace is not None else 1)
    t2 = time.perf_counter()
    try:
        if ls is not None and ls.enabled:
            eng.set_line_search(True, ls.alpha)
        eng.load_pool(eng.pack([m.factors for m in queue]))
        tic = time.perf_counter()
        eng.run(cfg.tol, cfg.max_iterations, t.sqnorm)
        t4 = time.perf_counter()
        res = eng.results()
        wall = time.perf_counter() - tic
        records = eng.trace() if (trace is not None and not label_per_model) else None
    finally:
        eng.close()
    t5 = time.perf_counter()
    prof.update(tensor_upload_s=t1 - t0, engine_create_s=t2 - t1, pool_upload_s=tic - t2,
                device_loop_s=t4 - tic, results_download_s=t5 - t4)
    for m in queue:
        m.status = ModelStatus.ACTIVE
    order = np.argsort(res.retire_seq, kind="stable")
    lam_off = np.concatenate([[0], np.cumsum([m.rank for m in queue])])
    out = []
    for k in order:
        src = queue[k]
        status = STATUS_FROM_CODE[int(res.status[k])]
        meta = dict(src.meta)
        meta["lambdas"] = res.lambdas[lam_off[k]:lam_off[k + 1]].copy()
        out.append(Model(id=src.id, rank=src.rank, factors=eng.unpack(res.pool, k),
                         error=float(res.error[k]), fit=float(res.fit[k]),
                         iterations_done=int(res.iterations[k]), status=status,
                         seconds_active=float(res.seconds_active[k]), meta=meta))
    prof["build_models_s"] = time.perf_counter() - t5
    if trace is not None:
        if label_per_model:
            for r in out:
                trace.append(SegmentTrace(
                    label=f"als:{r.id}", flops=_instance_flops(t, r.rank, r.iterations_done),
                    seconds=wall, meta={"id": r.id, "rank": r.rank,
                                        "iterations": r.iterations_done}))
        else:
            for width, n_active, secs in records:
                trace.append(SegmentTrace(
                    label="cals-iteration", flops=t.order * mttkrp_flops(t.dims, width),
                    seconds=secs, meta={"width": width, "n_active": n_active}))
    return out


def _trace_cap(queue, cfg) -> int:
    # every driver iteration retires or advances >= 1 model; bound generously
    return int(min(1 << 22, cfg.max_iterations * len(queue) + 2))
