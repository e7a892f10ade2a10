"""Locate the reference host-side package (ragsim).

The product keeps the reference's Python decision logic unchanged (north
star): ragsim must be importable.  Search order: an installed ``ragsim``,
the offline install at ``baseline/_ref`` (travels to the GPU box), then the
read-only reference checkout (this container only).
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = (
    os.path.join(_ROOT, "baseline", "_ref"),
    "/root/reference/pkg/src",
)


def import_ragsim():
    try:
        return importlib.import_module("ragsim")
    except ImportError:
        pass
    for cand in _CANDIDATES:
        if os.path.isdir(os.path.join(cand, "ragsim")):
            if cand not in sys.path:
                sys.path.append(cand)
            return importlib.import_module("ragsim")
    raise ImportError(
        "ragsim (the reference host-side API) is not importable; install it with "
        "`pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of reference>/pkg`"
    )


def ragsim_available() -> bool:
    try:
        import_ragsim()
        return True
    except ImportError:
        return False
