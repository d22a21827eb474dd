"""Post-processing specs (reference: olsconv/postproc.py:12-38).

``none`` and ``scale`` are fused into the engine's writeback (C-ABI pp_kind
0/1).  ``magnitude_squared`` and ``derivative`` (the reference's non-local
epilogues, postproc.py:44-85 / _kernels_nb.py:224-262) are SURVEY §8(f)3
"next" rows; the engine rejects them with EngineError until they land.
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
