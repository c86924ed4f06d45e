"""CPU oracle for the CALS hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(arxiv/paper_2010_04678, package ``cals`` at ``pkg/src/cals``).  It is the
checker the CUDA path is compared against; it is never imported by the
product package (``paper_2010_04678_b200``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may use it.

Parity pinning: every function below is checked against golden vectors
produced by the real reference (``oracle/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and writes
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.

Citations are ``file:line`` into ``/root/reference/pkg/src/cals``.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import cho_factor, cho_solve

# --------------------------------------------------------------------------
# tensor helpers (tensor.py)
# --------------------------------------------------------------------------


def unfold(arr_flat: np.ndarray, dims, mode: int) -> np.ndarray:
    """Mode-n unfolding, remaining indices lower-mode-fastest.

    tensor.py:115-131 (``unfold``); the flat data is mode-0 fastest
    (tensor.py:1-5).
    """
    nd = np.asarray(arr_flat).reshape(dims, order="F")
    return np.reshape(np.moveaxis(nd, mode, 0), (dims[mode], -1), order="F")


def khatri_rao(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Column-wise Kronecker, ``b`` index fastest: row i*J+k = a[i]*b[k].

    tensor.py:134-157.
    """
    ia, r = a.shape
    jb = b.shape[0]
    return (a[:, None, :] * b[None, :, :]).reshape(ia * jb, r)


def krp_descending(factors, mode: int) -> np.ndarray:
    """KRP of every factor except ``mode`` in descending mode order.

    mttkrp.py:117-118 (``_descending_others``) + mttkrp.py:121-134.
    """
    parts = [factors[i] for i in range(len(factors) - 1, -1, -1) if i != mode]
    acc = parts[0]
    for p in parts[1:]:
        acc = khatri_rao(acc, p)
    return acc


def gramian(a: np.ndarray) -> np.ndarray:
    """A^T A with the lower triangle overwritten by the upper (tensor.py:183-188)."""
    g = a.T @ a
    iu = np.triu_indices(g.shape[0], k=1)
    g[iu[1], iu[0]] = g[iu]
    return g


def hadamard_fold(mats) -> np.ndarray:
    """Left-to-right elementwise product (tensor.py:169-180)."""
    mats = list(mats)
    acc = np.array(mats[0], dtype=np.float64, copy=True)
    for m in mats[1:]:
        acc *= m
    return acc


# --------------------------------------------------------------------------
# MTTKRP (mttkrp.py)
# --------------------------------------------------------------------------


def mttkrp(arr_flat: np.ndarray, dims, factors, mode: int) -> np.ndarray:
    """T_(n) @ KRP(others, descending)  (mttkrp.py:3-8, 157-209).

    The reference picks FIRST/MIDDLE/LAST/EXPLICIT variants that only differ
    in summation order; the oracle uses the explicit unfolding, which is the
    definition every variant is tested against (tests/oracles.py:30-33).
    """
    return unfold(arr_flat, dims, mode) @ krp_descending(factors, mode)


def mttkrp_flops(dims, width: int) -> int:
    """2 * W * prod(dims) (mttkrp.py:72-76)."""
    return 2 * int(width) * int(math.prod(int(d) for d in dims))


# --------------------------------------------------------------------------
# ALS maths (als.py)
# --------------------------------------------------------------------------


def update_factor(m: np.ndarray, h: np.ndarray) -> np.ndarray:
    """A = M H^{-1} via upper Cholesky, eigen-pinv fallback (als.py:74-96)."""
    m = np.asarray(m, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError("h must be square")
    if not (np.all(np.isfinite(m)) and np.all(np.isfinite(h))):
        raise ValueError("non-finite input to factor update")
    try:
        c = cho_factor(h, lower=False, check_finite=False)
        a = cho_solve(c, m.T, check_finite=False).T
        if np.all(np.isfinite(a)):
            return np.asfortranarray(a)
    except np.linalg.LinAlgError:
        pass
    lam, vec = np.linalg.eigh(h)
    cut = 1e-12 * max(float(lam[-1]), 0.0)
    keep = lam > cut
    inv = np.zeros_like(lam)
    inv[keep] = 1.0 / lam[keep]
    return np.asfortranarray(m @ ((vec * inv) @ vec.T))


def fast_error(t_sqnorm: float, last_factor, last_mttkrp, grams) -> float:
    """||T||^2 + sum(*grams) - 2<A_last, M_last>, clamped at 0 (als.py:99-115).

    NB: the clamp is written ``e if e > 0 else 0`` so a NaN error clamps to
    0.0 exactly like the reference.
    """
    model_sq = float(hadamard_fold(grams).sum())
    inner = float(np.einsum("ir,ir->", last_factor, last_mttkrp))
    e = t_sqnorm + model_sq - 2.0 * inner
    return e if e > 0.0 else 0.0


def fit_from_error(e: float, t_sqnorm: float) -> float:
    """1 - sqrt(e)/||T|| (als.py:118-124)."""
    if t_sqnorm <= 0.0:
        raise ValueError("tensor squared norm must be positive")
    if e < 0.0:
        raise ValueError("negative squared error")
    return 1.0 - math.sqrt(e) / math.sqrt(t_sqnorm)


# --------------------------------------------------------------------------
# input builders (io.py, model.py) -- reproduced bit-for-bit
# --------------------------------------------------------------------------


def generate_synthetic(dims, true_rank: int, noise_level: float = 0.0, seed=None):
    """Flat mode-0-fastest data of a random low-rank tensor + noise (io.py:114-136)."""
    dims = tuple(int(d) for d in dims)
    rng = np.random.default_rng(seed)
    fac = [rng.random((d, true_rank)) for d in dims]
    letters = "abcdefghijklmnopqrstuvwxyz"[: len(dims)]
    signal = np.einsum(",".join(c + "z" for c in letters) + "->" + letters, *fac)
    if noise_level > 0.0:
        g = rng.standard_normal(dims)
        signal = signal + noise_level * (np.linalg.norm(signal) / np.linalg.norm(g)) * g
    return dims, signal.ravel(order="F")


def build_models(dims, ranks, per_rank: int, seed: int):
    """[(id, rank, factors)] in ascending rank/replicate order (io.py:154-170,
    model.py:59-73: uniform(0,1) Fortran factors from SeedSequence children)."""
    ss = np.random.SeedSequence(seed)
    kids = iter(ss.spawn(len(ranks) * per_rank))
    out, seen = [], {}
    for rank in ranks:
        for _ in range(per_rank):
            rng = np.random.default_rng(next(kids))
            j = seen.get(rank, 0)
            seen[rank] = j + 1
            fac = [np.asfortranarray(rng.random((int(d), rank))) for d in dims]
            out.append((f"r{rank:02d}-{j:02d}", rank, fac))
    return out


# --------------------------------------------------------------------------
# the fused CALS driver (driver.py:185-307)
# --------------------------------------------------------------------------

CONVERGED, ITERATION_CAP, FAILED = "converged", "iteration_cap", "failed"


@dataclass
class OracleResult:
    id: str
    rank: int
    factors: list
    error: float
    fit: float
    iterations: int
    status: str


@dataclass
class _Inst:
    id: str
    rank: int
    off: int
    iteration: int = 0
    f_prev: float = -np.inf
    error: float = np.inf
    fit: float = -np.inf
    grams: list = field(default_factory=list)
    snapshot: list | None = None
    failed: bool = False


def extrapolate(arr_flat, dims, sq, prev, curr, alpha):
    """Candidate prev + alpha (curr - prev), its Gramians and exact error
    (als.py:127-144)."""
    cand = [np.asfortranarray(p + alpha * (c - p)) for p, c in zip(prev, curr)]
    grams = [gramian(f) for f in cand]
    m_last = mttkrp(arr_flat, dims, cand, len(dims) - 1)
    return cand, grams, fast_error(sq, cand[-1], m_last, grams)


def run_cals(arr_flat, dims, models, tol: float, max_iterations: int, r_star: int,
             trace: list | None = None, ls: bool = False, ls_alpha: float | None = None):
    """Algorithm 4 of the paper as the reference driver executes it.

    ``models`` is ``[(id, rank, factors)]``.  Semantics restated from
    driver.py:185-285: strict-FIFO admission with head-of-line blocking
    (:199-208, multimatrix.py:143-158), per mode one wide MTTKRP over the
    packed columns then per-model Hadamard/solve/Gram refresh in registry
    order (:213-235), then per-model iteration++, fast error, fit and the
    FAILED/CONVERGED/ITERATION_CAP decision (:241-273), retirement in
    registry order (:274-275), compression (:276) and one trace record per
    driver iteration (:278-284).  Returns results in retirement order.
    """
    dims = tuple(int(d) for d in dims)
    n_modes = len(dims)
    arr_flat = np.asarray(arr_flat, dtype=np.float64)
    sq = float(np.dot(arr_flat, arr_flat))
    queue = deque((mid, r, [np.array(f, dtype=np.float64, order="F") for f in fac])
                  for mid, r, fac in models)
    for _, r, _ in queue:
        if r > r_star:
            raise ValueError("rank exceeds r_star")
    bufs = [np.zeros((d, r_star), order="F") for d in dims]
    reg: list[_Inst] = []
    out: list[OracleResult] = []

    def end():
        return reg[-1].off + reg[-1].rank if reg else 0

    while queue or reg:
        while queue and end() + queue[0][1] <= r_star:
            mid, r, fac = queue.popleft()
            off = end()
            for n in range(n_modes):
                bufs[n][:, off:off + r] = fac[n]
            reg.append(_Inst(mid, r, off,
                             grams=[gramian(bufs[n][:, off:off + r]) for n in range(n_modes)]))
        width = end()
        m_fused = None
        for n in range(n_modes):
            m_fused = mttkrp(arr_flat, dims, [b[:, :width] for b in bufs], n)
            for inst in reg:
                if inst.failed:
                    continue
                sl = slice(inst.off, inst.off + inst.rank)
                h = hadamard_fold([inst.grams[i] for i in range(n_modes) if i != n])
                try:
                    a_new = update_factor(m_fused[:, sl], h)
                except (ValueError, ArithmeticError, np.linalg.LinAlgError):
                    inst.failed = True
                    continue
                bufs[n][:, sl] = a_new
                inst.grams[n] = gramian(bufs[n][:, sl])
        retiring = []
        for inst in reg:
            inst.iteration += 1
            if inst.failed:
                inst.error, inst.fit = float("nan"), -np.inf
                retiring.append((inst, FAILED))
                continue
            sl = slice(inst.off, inst.off + inst.rank)
            e = fast_error(sq, bufs[-1][:, sl], m_fused[:, sl], inst.grams)
            if ls and inst.snapshot is not None and np.isfinite(e):
                # driver.py:250-259
                alpha = ls_alpha if ls_alpha is not None else float(inst.iteration) ** (1.0 / 3.0)
                cand, cgrams, ec = extrapolate(arr_flat, dims, sq, inst.snapshot,
                                               [b[:, sl] for b in bufs], alpha)
                if ec < e:
                    for b, c in zip(bufs, cand):
                        b[:, sl] = c
                    inst.grams = cgrams
                    e = ec
            if not np.isfinite(e):
                inst.error, inst.fit = float(e), -np.inf
                retiring.append((inst, FAILED))
                continue
            fit = fit_from_error(e, sq)
            inst.error, inst.fit = float(e), float(fit)
            if tol > 0 and fit - inst.f_prev < tol:
                retiring.append((inst, CONVERGED))
            elif inst.iteration >= max_iterations:
                retiring.append((inst, ITERATION_CAP))
            else:
                inst.f_prev = fit
                if ls:  # driver.py:272-273
                    inst.snapshot = [np.array(b[:, sl], order="F") for b in bufs]
        n_active = len(reg)
        for inst, status in retiring:
            sl = slice(inst.off, inst.off + inst.rank)
            out.append(OracleResult(inst.id, inst.rank,
                                    [np.array(b[:, sl], order="F") for b in bufs],
                                    inst.error, inst.fit, inst.iteration, status))
            reg.remove(inst)
        # compress: pack survivors left in registry order (multimatrix.py:103-114)
        off = 0
        for inst in reg:
            if inst.off != off:
                for b in bufs:
                    b[:, off:off + inst.rank] = b[:, inst.off:inst.off + inst.rank]
                inst.off = off
            off += inst.rank
        if trace is not None:
            trace.append({"width": width, "n_active": n_active,
                          "flops": n_modes * mttkrp_flops(dims, width)})
    return out
