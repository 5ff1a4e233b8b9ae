"""TEST/BASELINE INFRASTRUCTURE — import the reference's STOCK package ``hybfs``.

``oracle/build_ref.py`` compiles the reference's ``_native`` and ships the
unmodified ``hybfs/*.py`` next to it in ``oracle/_ref/<variant>/hybfs/``
(git-ignored, travels to the GPU box).  ``load()`` puts that directory on
``sys.path`` and imports the package, so callers get the reference's own
controller (``hybfs.hybrid.hybrid_bfs``, hybrid.py:83-175), engine dispatch
(``hybfs.engine``, engine.py:64-155) and harness (``hybfs.harness``) running
on its own compiled kernels — nothing restated.

Only tests, bench.py's reference arm / cpu_baseline and golden generation
import this; the product never does.
"""

from __future__ import annotations

import os
import sys

from . import build_ref, refnative


def package_dir():
    """oracle/_ref/<variant> holding the stock package for this CPU, or None."""
    order = ["avx512", "scalar"] if refnative.cpu_has_avx512f() else ["scalar"]
    for variant in order:
        d = os.path.join(build_ref.OUT_ROOT, variant)
        if os.path.exists(os.path.join(d, "hybfs", "__init__.py")) and \
                os.path.exists(build_ref.built_paths()[variant]):
            return d
    return None


def load():
    """The stock ``hybfs`` package (with its compiled engine), or None if absent."""
    mod = sys.modules.get("hybfs")
    if mod is not None:
        return mod
    d = package_dir()
    if d is None:
        return None
    if d not in sys.path:
        sys.path.insert(0, d)
    import hybfs  # noqa: F401  (the reference's own __init__)
    import hybfs.engine as eng

    if not eng.native_available():
        raise RuntimeError(f"stock hybfs imported from {d} but its _native did not load")
    return sys.modules["hybfs"]
