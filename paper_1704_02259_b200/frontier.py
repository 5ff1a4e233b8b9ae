"""Data contract shared with the reference (frontier.py:16-121).

Sentinels and the tree container keep the reference's layouts bit-for-bit:
parent uint32 with NIL = 0xFFFFFFFF and parent[source] = source; levels int32
with UNREACHED = -1.  Bitmaps on the device are the same LSB-first 32-bit
words (bit v in word v >> 5 at position v & 31).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NIL = 0xFFFFFFFF
UNREACHED = -1
WORD_BITS = 32


@dataclass
class BfsTree:
    """Predecessor array (frontier.py:94-110)."""

    parent: np.ndarray  # uint32, length n
    source: int

    @classmethod
    def fresh(cls, n: int, source: int) -> "BfsTree":
        if not 0 <= source < n:
            raise IndexError(f"source {source} out of range [0, {n})")
        parent = np.full(n, NIL, dtype=np.uint32)
        parent[source] = source
        return cls(parent=parent, source=source)

    def visited_mask(self) -> np.ndarray:
        return self.parent != np.uint32(NIL)


@dataclass
class LayerCounters:
    """Heuristic inputs per layer (frontier.py:113-121)."""

    e_f: int = 0
    v_f: int = 0
    e_u: int = 0
