"""Locate the reference ``prefillsim`` package (the scheduler/engine API, imported unchanged).

FlowPrefill's scheduler, workload model and metrics are the CALLER of the hot path and stay the
reference's own Python code (BASELINE.json north_star: "The reference's Python scheduler/engine
API stays unchanged"). They are loaded, unmodified, from the offline install under
``baseline/_ref`` (travels to the GPU box) or from the read-only source tree when present.
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (
    os.environ.get("PREFILLSIM_PATH", ""),
    os.path.join(_ROOT, "baseline", "_ref"),
    "/root/reference/pkg/src",
)


def available() -> bool:
    try:
        load()
        return True
    except ImportError:
        return False


def load():
    """Return the ``prefillsim`` module; raises ImportError if no copy is reachable."""
    if "prefillsim" in sys.modules:
        return sys.modules["prefillsim"]
    for p in CANDIDATES:
        if p and os.path.isdir(os.path.join(p, "prefillsim")):
            if p not in sys.path:
                sys.path.append(p)
            return importlib.import_module("prefillsim")
    raise ImportError(
        "prefillsim (reference scheduler) not found; install it with "
        "`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`"
    )
