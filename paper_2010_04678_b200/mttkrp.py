"""MTTKRP operator API on the B200 fused kernel.

Same surface as the reference's ``cals.mttkrp`` (pkg/src/cals/mttkrp.py):
``MttkrpVariant`` / ``DEFAULT_VARIANT_TABLE`` / ``validate_variant`` /
``select_variant`` / ``mttkrp_flops`` / ``MttkrpWorkspace`` / ``mttkrp`` /
``fused_mttkrp``.  Every call runs ``cals_mttkrp`` (csrc/mttkrp.cuh) on the
GPU: the reference's variants differ only in summation structure, and the
single fused DMMA kernel handles every (order, mode) pair, so the variant
argument is validated for API compatibility and otherwise does not change the
computation.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
from typing import Sequence

import numpy as np

from . import _native
from .tensor import DenseTensor


class MttkrpVariant(enum.Enum):
    EXPLICIT_KRP_GEMM = "explicit"
    FIRST_MODE_GEMM = "first"
    LAST_MODE_GEMM = "last"
    MIDDLE_MODE_SLICE_GEMM = "middle"


DEFAULT_VARIANT_TABLE: dict[tuple[int, int], MttkrpVariant] = {
    (2, 0): MttkrpVariant.FIRST_MODE_GEMM,
    (2, 1): MttkrpVariant.LAST_MODE_GEMM,
    (3, 0): MttkrpVariant.FIRST_MODE_GEMM,
    (3, 1): MttkrpVariant.MIDDLE_MODE_SLICE_GEMM,
    (3, 2): MttkrpVariant.LAST_MODE_GEMM,
}


def validate_variant(variant: MttkrpVariant, order: int, mode: int) -> None:
    """Reject variant/mode pairings outside the variant's domain (mttkrp.py:40-54)."""
    if not 0 <= mode < order:
        raise ValueError(f"mode {mode} out of range for order {order}")
    allowed = {
        MttkrpVariant.EXPLICIT_KRP_GEMM: True,
        MttkrpVariant.FIRST_MODE_GEMM: mode == 0,
        MttkrpVariant.LAST_MODE_GEMM: mode == order - 1,
        MttkrpVariant.MIDDLE_MODE_SLICE_GEMM: order == 3 and mode == 1,
    }
    if not allowed[variant]:
        raise ValueError(f"variant {variant.value} invalid for mode {mode} of an order-{order} tensor")


def select_variant(dims: Sequence[int], mode: int, width: int, table=None) -> MttkrpVariant:
    """Deterministic (order, mode) -> variant lookup (mttkrp.py:57-69)."""
    order = len(dims)
    if not 0 <= mode < order:
        raise ValueError(f"mode {mode} out of range for order {order}")
    return (DEFAULT_VARIANT_TABLE if table is None else table).get(
        (order, mode), MttkrpVariant.EXPLICIT_KRP_GEMM)


def mttkrp_flops(dims: Sequence[int], width: int) -> int:
    """2 * W * prod(dims) -- the reference flop model (mttkrp.py:72-76)."""
    if width < 0:
        raise ValueError("width must be >= 0")
    return 2 * int(width) * math.prod(int(d) for d in dims)


def _round8(x: int) -> int:
    return (int(x) + 7) // 8 * 8


class MttkrpWorkspace:
    """Device buffers for one caller: row-major factor staging ``[I_n][ld]``,
    the ``[max I][ld]`` output and the split-K / KRP workspace, sized once
    for a shape and a maximum width (the reference's "no per-iteration
    allocation").  Results are returned as a Fortran ``(I_n, W)``
    view into a host buffer overwritten by the next call (mttkrp.py:221-223).
    """

    def __init__(self, dims: Sequence[int], capacity: int):
        dims = tuple(int(d) for d in dims)
        if capacity < 1:
            raise ValueError("workspace capacity must be >= 1")
        self.dims = dims
        self.capacity = int(capacity)
        self.ld = _round8(self.capacity)
        self._out_host = np.empty(max(dims) * self.capacity)
        self._dev = None  # lazily allocated on first GPU use

    def _device(self, t: DenseTensor):
        import torch

        if self._dev is None:
            dev = torch.device("cuda", torch.cuda.current_device())
            fac = [torch.zeros((d, self.ld), dtype=torch.float64, device=dev) for d in self.dims]
            out = torch.empty((max(self.dims), self.ld), dtype=torch.float64, device=dev)
            need = 0
            h = t.device().handle
            for n in range(len(self.dims)):
                b = C.c_size_t()
                _native.call("cals_mttkrp_workspace_bytes", h, n, self.ld, C.byref(b))
                need = max(need, b.value)
            work = torch.empty((need + 7) // 8, dtype=torch.float64, device=dev)
            self._dev = (fac, out, work, need)
        return self._dev

    def out_view(self, rows: int, width: int) -> np.ndarray:
        if rows * width > self._out_host.size or width > self.capacity:
            raise ValueError(f"width {width} exceeds workspace capacity {self.capacity}")
        return self._out_host[:rows * width].reshape((rows, width), order="F")


def _check_factors(t: DenseTensor, factors: Sequence[np.ndarray], mode: int) -> int:
    if len(factors) != t.order:
        raise ValueError(f"expected {t.order} factors, got {len(factors)}")
    width = None
    for i, f in enumerate(factors):
        if i == mode:
            continue
        if np.ndim(f) != 2 or np.shape(f)[0] != t.dims[i]:
            raise ValueError(f"factor {i} has shape {np.shape(f)}, expected ({t.dims[i]}, W)")
        if width is None:
            width = int(np.shape(f)[1])
        elif np.shape(f)[1] != width:
            raise ValueError("factors disagree on column count")
    return width


def _gpu_mttkrp(t: DenseTensor, factors, mode: int, ws: MttkrpWorkspace) -> np.ndarray:
    import torch

    _native.load()  # raises NativeUnavailable without a GPU: no CPU fallback
    width = _check_factors(t, factors, mode)
    if width > ws.capacity:
        raise ValueError(f"width {width} exceeds workspace capacity {ws.capacity}")
    if tuple(ws.dims) != tuple(t.dims):
        raise ValueError("workspace was sized for another tensor shape")
    out_view = ws.out_view(t.dims[mode], width)
    if width == 0:
        return out_view
    fac, out, work, need = ws._device(t)
    ptrs = (C.c_void_p * t.order)()
    for i, f in enumerate(factors):
        if i == mode:
            ptrs[i] = fac[i].data_ptr()
            continue
        fac[i][:, :width].copy_(torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)))
        ptrs[i] = fac[i].data_ptr()
    stream = torch.cuda.current_stream()
    _native.call("cals_mttkrp", t.device().handle, mode, width, ptrs, ws.ld, out.data_ptr(),
                 ws.ld, work.data_ptr(), need, -1, stream.cuda_stream)
    host = out[:t.dims[mode], :width].cpu().numpy()
    out_view[...] = host
    return out_view


def mttkrp(t: DenseTensor, factors: Sequence[np.ndarray], mode: int,
           variant: MttkrpVariant | None = None, ws: MttkrpWorkspace | None = None) -> np.ndarray:
    """Mode-n MTTKRP ``T_(n) @ KRP(factors[i != mode], descending)``, shape
    (I_n, W), on the GPU (replaces mttkrp.py:212-231)."""
    if variant is None:
        width = np.shape(factors[(mode + 1) % len(factors)])[1]
        variant = select_variant(t.dims, mode, width)
    validate_variant(variant, t.order, mode)
    if ws is None:
        ws = MttkrpWorkspace(t.dims, max(1, _check_factors(t, factors, mode)))
    return _gpu_mttkrp(t, factors, mode, ws)


def fused_mttkrp(t: DenseTensor, multis: Sequence, mode: int, ws: MttkrpWorkspace,
                 variant: MttkrpVariant | None = None) -> np.ndarray:
    """One wide MTTKRP over the packed active columns of every multi-matrix
    (replaces mttkrp.py:234-256)."""
    widths = {mm.active_width for mm in multis}
    if len(widths) != 1:
        raise ValueError(f"multi-matrices disagree on active width: {widths}")
    (width,) = widths
    if width == 0:
        raise ValueError("no active instances")
    views = [mm.packed_view() for mm in multis]
    if variant is None:
        variant = select_variant(t.dims, mode, width)
    validate_variant(variant, t.order, mode)
    return _gpu_mttkrp(t, views, mode, ws)
