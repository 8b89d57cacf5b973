"""Import helper for the UNMODIFIED reference package (TEST INFRASTRUCTURE).

Only usable in the build container, where ``/root/reference`` exists; the GPU
box has no reference tree, so nothing in ``-m gpu`` tests, ``smoke()`` or
``bench.py`` calls this. It is used by ``tests/golden/gen_golden.py`` to
produce the committed golden fixtures and by the CPU tests that cross-check
the numpy restatement (``oracle/collectives.py``) against the reference.
"""

from __future__ import annotations

import os
import sys

REFERENCE_SRC = "/root/reference/pkg/src"
_SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "refshim")


def available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "collectium"))


def load():
    """Return the reference ``collectium`` module (greenlet shim first)."""
    if not available():
        raise RuntimeError("reference tree not present (GPU box?)")
    for path in (REFERENCE_SRC, _SHIM):
        if path not in sys.path:
            sys.path.insert(0, path)
    import collectium  # noqa: F401  (reference package)
    return collectium


def run_group(p: int, fn):
    """Run ``fn(rank, endpoint)`` on the reference's simulated network
    (``transport/sim.py:234-239``); returns the per-rank results."""
    ref = load()
    return ref.SimNetwork(p).run(fn)
