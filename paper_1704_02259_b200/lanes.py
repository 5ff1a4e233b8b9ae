"""VecConfig — the reference's vector-kernel knobs (lanes.py:30-41).

On the GPU a warp covers 32 vertices and probes rows with uint4 loads; the
reference's 16-lane emulation has no device counterpart.  ``max_pos`` is kept
because it defines the trace counters (gathers / fallbacks) the reference
reports, which the device reproduces exactly; ``backend`` is
accepted for API compatibility and must be one of the reference's values.
"""

from __future__ import annotations

from dataclasses import dataclass

LANES = 16
BACKENDS = ("simd", "emulate")


@dataclass
class VecConfig:
    max_pos: int = 8
    backend: str = "simd"

    def __post_init__(self):
        if self.max_pos < 1:
            raise ValueError("max_pos must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}")
