"""Locate the reference package (`loomtune`) that this package plugs into.

The host data model (expressions, ComputeDAG, loop-nest State, rewrite steps,
`validate`, the JSON codec) and the search loop that calls the GPU path are the
reference's own code, imported unchanged — this package replaces only the hot
path (measurement and population scoring) behind its API.

Search order: an already importable `loomtune`; the in-tree offline install
`baseline/_ref` (`pip install --target baseline/_ref`, travels with the repo to
the GPU box); the reference source tree `/root/reference/pkg/src`.  Missing
everywhere is an ImportError, never a fallback.
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def locate() -> str | None:
    for cand in CANDIDATES:
        if os.path.isdir(os.path.join(cand, "loomtune")):
            return cand
    return None


def load():
    """Import and return the `loomtune` package (adding its install dir to sys.path)."""
    try:
        return importlib.import_module("loomtune")
    except ImportError:
        pass
    cand = locate()
    if cand is None:
        raise ImportError("the reference package `loomtune` is not importable: install it with "
                          "`pip install --no-deps --target baseline/_ref <reference>/pkg`")
    if cand not in sys.path:
        sys.path.insert(0, cand)
    return importlib.import_module("loomtune")


loomtune = load()
