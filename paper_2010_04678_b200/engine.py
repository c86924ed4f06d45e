"""Python handle of the device-resident CALS engine (csrc/engine.cu).

The engine owns, in HBM: the per-mode factor multi-matrices, Gramians,
per-model status / fit bookkeeping, the FIFO queue and a model pool holding
every model's starting (and finally its fitted) factors.  ``run`` replays a
CUDA graph of one driver iteration until the device reports that every
model has retired.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native


class _CudaBuffer:
    """Minimal ``__cuda_array_interface__`` exporter for engine-owned memory."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


@dataclass
class EngineResults:
    pool: np.ndarray
    status: np.ndarray
    iterations: np.ndarray
    error: np.ndarray
    fit: np.ndarray
    retire_seq: np.ndarray
    seconds_active: np.ndarray
    lambdas: np.ndarray


class CalsEngine:
    def __init__(self, dev_tensor, r_star: int, ranks: Sequence[int], trace_capacity: int = 4096):
        _native.load()
        self.dims = tuple(dev_tensor.dims)
        self.order = len(self.dims)
        self.ranks = np.asarray(ranks, dtype=np.int32)
        self.r_star = int(r_star)
        self.trace_capacity = int(trace_capacity)
        self._tensor = dev_tensor  # keep alive
        h = C.c_void_p()
        _native.call("cals_engine_create", dev_tensor.handle, self.r_star, len(self.ranks),
                     self.ranks.ctypes.data_as(C.POINTER(C.c_int32)), self.trace_capacity,
                     C.byref(h))
        self.handle = h
        ptr, n = C.c_void_p(), C.c_int64()
        _native.call("cals_engine_pool", h, C.byref(ptr), C.byref(n))
        self.pool_ptr = ptr.value
        self.pool_elems = n.value
        # pool offsets (must match engine_create): model-major, modes ascending
        self.offsets = np.zeros((len(self.ranks), self.order), dtype=np.int64)
        at = 0
        for k, r in enumerate(self.ranks):
            for n_ in range(self.order):
                self.offsets[k, n_] = at
                at += self.dims[n_] * int(r)
        assert at == self.pool_elems or (at == 0 and self.pool_elems == 0)

    # -------------------------------------------------------------- pool
    def staging(self) -> np.ndarray:
        """Page-locked host buffer of the pool's size (allocated once)."""
        if getattr(self, "_staging", None) is None:
            import torch

            self._staging_t = torch.empty(max(self.pool_elems, 1), dtype=torch.float64,
                                          pin_memory=True)
            self._staging = self._staging_t.numpy()
        return self._staging

    def prepare(self, stream=None):
        """Enqueue the tensor slicing of the INT8 tensor-core views without
        waiting (finished and checked by ``run``)."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_prepare", self.handle, s)

    def set_tensor(self, dev_tensor):
        """Re-bind to another device tensor of the same shape."""
        _native.call("cals_engine_set_tensor", self.handle, dev_tensor.handle)
        self._tensor = dev_tensor

    def pack(self, factor_lists, out: np.ndarray | None = None) -> np.ndarray:
        """Host pool: per model, per mode, the Fortran (I_n, R_k) factor's
        bytes (column-major) -- one concatenation, no per-element work."""
        pool = np.empty(max(self.pool_elems, 1)) if out is None else out
        parts = [np.asarray(f, dtype=np.float64).ravel(order="F")
                 for facs in factor_lists for f in facs]
        if parts:
            np.concatenate(parts, out=pool[:self.pool_elems])
        return pool[:self.pool_elems]

    def unpack(self, pool: np.ndarray, k: int) -> list[np.ndarray]:
        """Fortran (I_n, R_k) views of model k's blocks in ``pool`` (no copy)."""
        if getattr(self, "_blocks", None) is None:  # plain-int (offset, shape) per block
            self._blocks = [[(int(self.offsets[j, n_]), int(self.dims[n_]) * int(r),
                              (int(self.dims[n_]), int(r))) for n_ in range(self.order)]
                            for j, r in enumerate(self.ranks)]
        return [pool[o:o + size].reshape(shape, order="F") for o, size, shape in self._blocks[k]]

    def load_pool(self, pool, stream=None):
        """``pool`` is a host ndarray or a CUDA tensor (device-to-device copy)."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        if isinstance(pool, np.ndarray):
            # stream-ordered (async from pinned memory); ``run`` synchronises
            # before returning, so the buffer may be reused after it
            pool = np.ascontiguousarray(pool, dtype=np.float64)
            _native.call("cals_engine_load_pool", self.handle, pool.ctypes.data, 0, s)
            self._pool_src = pool
        else:
            _native.call("cals_engine_load_pool", self.handle, C.c_void_p(pool.data_ptr()), 1, s)

    # --------------------------------------------------------------- run
    def run(self, tol: float, max_iterations: int, sqnorm: float, use_graph: bool = True,
            stream=None) -> int:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        it = C.c_int()
        _native.call("cals_engine_run", self.handle, float(tol), int(max_iterations),
                     float(sqnorm), 1 if use_graph else 0, s, C.byref(it))
        return it.value

    def results(self, with_pool: bool = True, stream=None, pool_out: np.ndarray | None = None
                ) -> EngineResults:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        k = len(self.ranks)
        pool = None
        if with_pool:
            pool = pool_out if pool_out is not None else np.empty(max(self.pool_elems, 1))
        status = np.empty(k, np.int32)
        iters = np.empty(k, np.int32)
        err = np.empty(k)
        fit = np.empty(k)
        seq = np.empty(k, np.int32)
        secs = np.empty(k)
        lam = np.empty(max(int(self.ranks.sum()), 1))
        ptr = (lambda a: None if a is None else a.ctypes.data)
        _native.call("cals_engine_results", self.handle, ptr(pool), ptr(status), ptr(iters),
                     ptr(err), ptr(fit), ptr(seq), ptr(secs), ptr(lam), s)
        return EngineResults(pool, status, iters, err, fit, seq, secs, lam)

    def last_launches(self) -> int:
        """Kernel launches of the last ``run`` (graph kernel nodes x graph
        launches + the direct ones), counted by the library."""
        n = C.c_longlong()
        _native.call("cals_engine_last_launches", self.handle, C.byref(n))
        return int(n.value)

    def pool_download(self, pool_out: np.ndarray, stream=None) -> None:
        """Enqueue the pool's device-to-host copy into ``pool_out`` (page-locked)
        without waiting; synchronise the stream before reading it."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_pool_download", self.handle, pool_out.ctypes.data, s)

    def trace(self):
        cap = self.trace_capacity
        w = np.empty(cap, np.int32)
        a = np.empty(cap, np.int32)
        sec = np.empty(cap)
        cnt = C.c_int()
        _native.call("cals_engine_trace", self.handle, w.ctypes.data, a.ctypes.data,
                     sec.ctypes.data, cap, C.byref(cnt))
        n = min(cnt.value, cap)
        return [(int(w[i]), int(a[i]), float(sec[i])) for i in range(n)]

    def set_line_search(self, enabled: bool, alpha: float | None = None):
        """Line search after every iteration (alpha None -> iteration^(1/3))."""
        _native.call("cals_engine_set_line_search", self.handle, 1 if enabled else 0,
                     0.0 if alpha is None else float(alpha))

    def set_nonneg(self, enabled: bool):
        """Non-negative (NNLS) factor updates, ranks <= 32."""
        _native.call("cals_engine_set_nonneg", self.handle, 1 if enabled else 0)

    def nnls_warnings(self) -> np.ndarray:
        flags = np.zeros(max(len(self.ranks), 1), np.int32)
        _native.call("cals_engine_nnls_warnings", self.handle, flags.ctypes.data)
        return flags[:len(self.ranks)]

    def update_failures(self) -> np.ndarray:
        """Per model: a factor update saw non-finite input (the reference's
        ValueError, als.py:84-85)."""
        flags = np.zeros(max(len(self.ranks), 1), np.int32)
        _native.call("cals_engine_update_failures", self.handle, flags.ctypes.data)
        return flags[:len(self.ranks)].astype(bool)

    # ------------------------------------------------------- step-wise
    def begin(self, tol: float, max_iterations: int, sqnorm: float, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_begin", self.handle, float(tol), int(max_iterations),
                     float(sqnorm), s)

    def enqueue_mttkrp(self, mode: int, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_enqueue_mttkrp", self.handle, mode, s)

    def enqueue_update(self, mode: int, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_enqueue_update", self.handle, mode, s)

    def enqueue_plan(self, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _native.call("cals_engine_enqueue_plan", self.handle, s)

    def done(self) -> bool:
        d = C.c_int()
        _native.call("cals_engine_done", self.handle, C.byref(d))
        return bool(d.value)

    def buffers(self) -> dict:
        """Zero-copy torch views of the device buffers (``__cuda_array_interface__``)."""
        import torch

        mo, gr = C.c_void_p(), C.c_void_p()
        ld, gs = C.c_int64(), C.c_int64()
        fac = (C.c_void_p * self.order)()
        _native.call("cals_engine_buffers", self.handle, C.byref(mo), C.byref(gr), C.byref(ld),
                     C.byref(gs), fac)

        def view(ptr, shape):
            return torch.as_tensor(_CudaBuffer(ptr, shape), device="cuda")

        return {"mttkrp": view(mo.value, (max(self.dims), ld.value)),
                "grams": view(gr.value, (self.order, gs.value)),
                "factors": [view(fac[n], (self.dims[n], ld.value)) for n in range(self.order)],
                "ld": ld.value, "gram_stride": gs.value}

    def variant(self, mode: int) -> dict:
        v, bm, bn, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _native.call("cals_engine_variant", self.handle, mode, C.byref(v), C.byref(bm),
                     C.byref(bn), C.byref(s))
        return {"variant": v.value, "BM": bm.value, "BN": bn.value, "splits": s.value}

    def close(self):
        if getattr(self, "handle", None):
            _native.load(require_cuda=False).cals_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
