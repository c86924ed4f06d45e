"""Single-instance ALS mathematics (API of the reference's ``cals.als``).

``update_factor`` runs the batched update kernel (csrc/update.cuh) for one
block on the GPU; ``run_single_als`` is the device-resident driver at K=1.
``fast_error`` / ``fit_from_error`` are the scalar formulas the engine
evaluates on the device (exposed for callers that hold host arrays).
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .tensor import hadamard_fold

# largest rank the GPU update kernels take (csrc/update.cuh kMaxRank; the R x R
# matrix moves from shared memory to global scratch above 128)
MAX_RANK = 512


@dataclass
class ConvergenceConfig:
    """Stop when the fit improves by less than ``tol`` or after
    ``max_iterations``; ``tol <= 0`` disables the fit test (als.py:24-37)."""

    tol: float = 1e-6
    max_iterations: int = 1000

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass
class LineSearchConfig:
    """Linear extrapolation between iterates (als.py:40-53); ``alpha=None``
    selects alpha = i^(1/3)."""

    enabled: bool = False
    alpha: float | None = None

    def __post_init__(self):
        if self.alpha is not None and self.alpha <= 1.0:
            raise ValueError(f"extrapolation alpha must be > 1, got {self.alpha}")


def alpha_for_iteration(cfg: LineSearchConfig, iteration: int) -> float:
    return cfg.alpha if cfg.alpha is not None else float(iteration) ** (1.0 / 3.0)


class NnlsState:
    """Per-mode, per-row active sets (True = pinned to zero)."""

    def __init__(self, dims: Sequence[int], rank: int):
        self.active = [np.zeros((int(d), rank), dtype=bool) for d in dims]


class NonConvergedNnlsWarning(RuntimeWarning):
    """Active-set search hit its iteration cap."""


def update_factor(m: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Solve ``A @ h = m`` on the GPU (replaces als.py:74-96): upper Cholesky
    + triangular solves, eigen-pinv fallback (cutoff 1e-12 * lambda_max).
    Raises ValueError for a non-square ``h`` or non-finite inputs."""
    import torch

    m = np.asarray(m, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError(f"h must be square, got {h.shape}")
    if m.ndim != 2 or m.shape[1] != h.shape[0]:
        raise ValueError(f"m has shape {m.shape}, expected (*, {h.shape[0]})")
    rows, r = m.shape
    if r > MAX_RANK:
        raise ValueError(f"update_factor supports rank <= {MAX_RANK} on the GPU")
    lib = _native.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    md = torch.from_numpy(np.ascontiguousarray(m)).to(dev)
    hd = torch.from_numpy(np.ascontiguousarray(h)).to(dev)
    ad = torch.empty((max(rows, 1), r), dtype=torch.float64, device=dev)
    scratch = torch.empty((lib.cals_update_scratch_bytes(r) + 7) // 8, dtype=torch.float64,
                          device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.call("cals_update_factor", rows, r, md.data_ptr(), r, hd.data_ptr(), ad.data_ptr(), r,
                 scratch.data_ptr(), status.data_ptr(), torch.cuda.current_stream().cuda_stream)
    if int(status.item()) != 0:
        raise ValueError("non-finite input to factor update")
    return np.asfortranarray(ad[:rows].cpu().numpy())


def fast_error(t_sqnorm: float, factors: Sequence[np.ndarray], last_mttkrp: np.ndarray,
               grams: Sequence[np.ndarray]) -> float:
    """||T||^2 + sum(hadamard of all Gramians) - 2 <A_last, M_last>, clamped
    with ``e if e > 0 else 0`` (als.py:99-115; NaN clamps to 0 as there)."""
    e = (t_sqnorm + float(hadamard_fold(grams).sum())
         - 2.0 * float(np.vdot(np.asarray(factors[-1]), np.asarray(last_mttkrp))))
    return e if e > 0.0 else 0.0


def fit_from_error(e: float, t_sqnorm: float) -> float:
    """1 - sqrt(e)/||T|| (als.py:118-124)."""
    if t_sqnorm <= 0.0:
        raise ValueError("tensor squared norm must be positive")
    if e < 0.0:
        raise ValueError(f"negative squared error {e}")
    return 1.0 - math.sqrt(e) / math.sqrt(t_sqnorm)


def extrapolate_factors(t, prev, curr, alpha: float, ws=None, variant_table=None):
    """Candidate ``prev + alpha * (curr - prev)``, its Gramians and exact
    error from a fresh last-mode MTTKRP on the GPU (als.py:127-144).  Inside
    ``run(..., ls=...)`` the engine evaluates every model's candidate with
    one fused MTTKRP instead."""
    from .mttkrp import mttkrp, select_variant
    from .tensor import gramian

    cand = [np.asfortranarray(p + alpha * (c - p)) for p, c in zip(prev, curr)]
    grams = [gramian(f) for f in cand]
    n_last = t.order - 1
    variant = select_variant(t.dims, n_last, cand[0].shape[1], variant_table)
    m_last = mttkrp(t, cand, n_last, variant=variant, ws=ws)
    return cand, grams, fast_error(t.sqnorm, cand, m_last, grams)


def line_search_step(prev, curr, cfg: LineSearchConfig, t, iteration: int | None = None,
                     ws=None):
    """Extrapolate from two consecutive iterates and keep whichever errs less
    (als.py:147-182)."""
    from .model import Model

    if not cfg.enabled:
        raise ValueError("line search disabled in config")
    if prev.rank != curr.rank or prev.dims != curr.dims:
        raise ValueError("prev/curr models do not conform")
    if iteration is None:
        iteration = max(curr.iterations_done, 2)
    cand, _, e_cand = extrapolate_factors(t, prev.factors, curr.factors,
                                          alpha_for_iteration(cfg, iteration), ws)
    if not (e_cand < curr.error):
        return curr
    return Model(id=curr.id, rank=curr.rank, factors=cand, error=e_cand,
                 fit=fit_from_error(e_cand, t.sqnorm), iterations_done=curr.iterations_done,
                 status=curr.status, meta=dict(curr.meta))


def _nnls_rows_gpu(m: np.ndarray, h: np.ndarray, active: np.ndarray, max_iter: int):
    """Run the warp-per-row Lawson-Hanson kernel (csrc/nnls.cuh) on a block."""
    import torch

    _native.load()
    m = np.ascontiguousarray(m, dtype=np.float64)
    rows, r = m.shape
    if r > 32:
        raise ValueError("the GPU NNLS kernel supports ranks up to 32")
    bits = (np.asarray(active, dtype=bool) * (1 << np.arange(r, dtype=np.uint64))).sum(
        axis=1).astype(np.uint32) if rows else np.zeros(0, np.uint32)
    dev = torch.device("cuda", torch.cuda.current_device())
    md = torch.from_numpy(m).to(dev)
    hd = torch.from_numpy(np.ascontiguousarray(h, dtype=np.float64)).to(dev)
    ad = torch.from_numpy(bits.view(np.int32).copy()).to(dev)
    xd = torch.empty((max(rows, 1), r), dtype=torch.float64, device=dev)
    cd = torch.empty(max(rows, 1), dtype=torch.int32, device=dev)
    _native.call("cals_nnls_rows", rows, r, md.data_ptr(), r, hd.data_ptr(), ad.data_ptr(),
                 xd.data_ptr(), r, cd.data_ptr(), int(max_iter),
                 torch.cuda.current_stream().cuda_stream)
    x = xd[:rows].cpu().numpy()
    newbits = ad.cpu().numpy().view(np.uint32)[:rows]
    act = ((newbits[:, None] >> np.arange(r, dtype=np.uint32)) & 1).astype(bool)
    return x, act, cd.cpu().numpy()[:rows].astype(bool)


def nnls_solve_row(h: np.ndarray, f: np.ndarray, active: np.ndarray | None = None,
                   max_iter: int | None = None):
    """min x^T h x - 2 f^T x s.t. x >= 0, warm-started (als.py:185-263);
    returns (x, active, converged)."""
    f = np.asarray(f, dtype=np.float64).ravel()
    r = f.size
    # no warm start = every variable pinned to zero, an empty passive set
    # (als.py:203: passive = zeros when active is None) -- unlike nnls_update,
    # whose NnlsState starts with nothing pinned
    act = np.ones((1, r), bool) if active is None else np.asarray(active, bool).reshape(1, r)
    x, a, conv = _nnls_rows_gpu(f[None, :], h, act, -1 if max_iter is None else max_iter)
    if not conv[0]:
        warnings.warn("active-set search hit its iteration cap", NonConvergedNnlsWarning,
                      stacklevel=2)
    return x[0], a[0], bool(conv[0])


def nnls_update(m: np.ndarray, h: np.ndarray, state: NnlsState, mode: int) -> np.ndarray:
    """Row-wise non-negative update warm-started from ``state`` (als.py:266-278)."""
    x, a, conv = _nnls_rows_gpu(np.asarray(m), h, state.active[mode], -1)
    state.active[mode][...] = a
    if not conv.all():
        warnings.warn("active-set search hit its iteration cap", NonConvergedNnlsWarning,
                      stacklevel=2)
    return np.asfortranarray(x)


def run_single_als(t, start, cfg: ConvergenceConfig, ls: LineSearchConfig | None = None,
                   nonneg: bool = False, ws=None, variant_table=None):
    """Fit one instance (als.py:281-356) -- the device-resident driver at K=1,
    which is bitwise identical to that model's columns in a fused run."""
    from .driver import _run_fused

    if start.dims != t.dims:
        raise ValueError(f"model dims {start.dims} != tensor dims {t.dims}")
    if ls is None:
        ls = LineSearchConfig()
    # the starting model is not mutated (status included); an update on
    # non-finite input raises ValueError as update_factor does (als.py:84-85)
    (out,) = _run_fused(t, [start], cfg, start.rank, None, label_per_model=True, ls=ls,
                        nonneg=nonneg, raise_on_update_failure=True)
    return out
