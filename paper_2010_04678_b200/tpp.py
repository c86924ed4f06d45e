"""Peak-performance model and efficiency records (API of the reference's
``cals.bench`` TPP helpers, bench.py:35-76).

On the B200 the denominator of an efficiency is the *measured* FP64
tensor-core peak (profiles/r01_fp64_peak_probe.txt: DMMA.8x8x4 at
37.1 TFLOP/s), exposed as ``B200_FP64_DMMA_TFLOPS``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

B200_FP64_DMMA_TFLOPS = 37.1   # measured, 148 SMs, 4+ warps/SM, 1965 MHz
B200_DGEMM_TFLOPS = 35.4       # cuBLAS DGEMM 8192^3 (torch.matmul float64), measured


@dataclass(frozen=True)
class TppModel:
    """Theoretical peak 2 * freq * threads * doubles-per-vector * FMA units (GF/s)."""

    freq_ghz: float
    nt: int
    nd: int = 8
    nv: int = 2

    def __post_init__(self):
        for name in ("freq_ghz", "nt", "nd", "nv"):
            if getattr(self, name) <= 0:
                raise ValueError(f"TPP parameter {name} must be positive")

    def gflops(self) -> float:
        return 2.0 * self.freq_ghz * self.nt * self.nd * self.nv


def tpp(model: TppModel) -> float:
    return model.gflops()


@dataclass
class BenchRecord:
    label: str
    flops: int
    seconds: float
    efficiency: float
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if not 0.0 < self.efficiency < 1.5:
            raise ValueError(f"efficiency {self.efficiency:.3f} outside sanity band (0, 1.5) "
                             f"for {self.label!r}; check the peak parameters")


def efficiency(flops: int, seconds: float, peak_gflops: float) -> float:
    return flops / seconds / 1e9 / peak_gflops
