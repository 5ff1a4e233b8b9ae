"""Engine selection (engine.py:26, :64-78 in the reference).

The reference routes each layer to a compiled CPU core or a Python engine.
This package has exactly one engine, ``"cuda"``: the whole traversal runs in
libhbfs on the GPU.  ``"auto"`` resolves to it; the reference's CPU engine
names are rejected rather than silently served by a CPU path.
"""

from __future__ import annotations

ENGINES = ("auto", "cuda")
REFERENCE_ONLY = ("native", "python")


def native_available() -> bool:
    """True when libhbfs.so is built and loadable (engine.py:60-61 analogue)."""
    from . import _lib

    try:
        _lib.load()
        return True
    except (ImportError, OSError):
        return False


def resolve_engine(engine: str = "auto", backend: str = "simd") -> str:
    if engine in REFERENCE_ONLY:
        raise RuntimeError(
            f"engine {engine!r} is a CPU engine of the reference package; this package "
            "runs only on the GPU (engine='cuda')"
        )
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}")
    return "cuda"


def bfs_reference(g, source: int, engine: str = "auto"):
    """Oracle traversal (engine.py:158-170): the FIFO-queue BFS of
    _native.bfs_reference on the GPU -> (BfsTree, levels int32[n]).  Parents
    follow the queue's first-discoverer rule, not the min-id rule."""
    from . import native
    from .frontier import BfsTree

    resolve_engine(engine)
    n = g.num_vertices
    if not 0 <= source < n:
        raise IndexError(f"source {source} out of range [0, {n})")
    parent, levels = native.bfs_reference(g.row_starts, g.adjacency, n, source)
    return BfsTree(parent=parent, source=int(source)), levels
