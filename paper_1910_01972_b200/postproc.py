"""Post-processing specs (reference: olsconv/postproc.py:12-38).

All four kinds are fused into the engine's writeback (C-ABI pp_kind 0-3):
``none`` and ``scale`` (_store kinds 0/1, _kernels_nb.py:218-226),
``magnitude_squared`` (|y|^2 real rows, olsb_fused_c2c_abs2 / fused_r2r
pp_kind 2, _kernels_nb.py:288-337) and ``derivative`` (the non-local
epilogue with the halo geometry, _kernels_nb.py:224-262; tap length 1 runs
through the range entries, whose geometry always has a halo).
Every entry (device, host streaming, range, shard) takes every kind; the
derivative's range geometry is t0 = M, L = N - M - 1 (olsb_input_extent_pp).
"""

from __future__ import annotations

from dataclasses import dataclass

KINDS = ("none", "scale", "magnitude_squared", "derivative")
_CODES = {k: i for i, k in enumerate(KINDS)}


@dataclass(frozen=True)
class PostProcSpec:
    kind: str = "none"
    scale: float = 1.0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown postproc kind {self.kind!r}")

    @property
    def code(self) -> int:
        return _CODES[self.kind]

    @property
    def halo(self) -> int:
        """Valid neighbor samples needed on each side of the output span."""
        return 1 if self.kind == "derivative" else 0

    @property
    def real_output(self) -> bool:
        return self.kind == "magnitude_squared"


NONE = PostProcSpec()
