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
INSTALL_DIR = os.path.join(_ROOT, "baseline", "_ref")
REFERENCE_SRC = "/root/reference/pkg"


def candidates() -> tuple:
    """Search order: $PREFILLSIM_PATH, the offline install under baseline/_ref (what travels to
    the GPU box), then the read-only source tree (build container only; FP_REFSIM_NO_SRC=1
    disables it so tests can prove the GPU-box configuration works without it)."""
    c = [os.environ.get("PREFILLSIM_PATH", ""), INSTALL_DIR]
    if os.environ.get("FP_REFSIM_NO_SRC", "") != "1":
        c.append(os.path.join(REFERENCE_SRC, "src"))
    return tuple(p for p in c if p)


def install(force: bool = False) -> bool:
    """Install the UNMODIFIED reference package into baseline/_ref (offline, no deps: numpy is
    already in the image), from a /tmp copy because the source tree is read-only. Returns True
    when baseline/_ref holds prefillsim afterwards. Called by __graft_entry__.build()."""
    import shutil
    import subprocess
    import tempfile

    if not force and os.path.isdir(os.path.join(INSTALL_DIR, "prefillsim")):
        return True
    if not os.path.isdir(REFERENCE_SRC):
        return os.path.isdir(os.path.join(INSTALL_DIR, "prefillsim"))
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REFERENCE_SRC, src)
        shutil.rmtree(INSTALL_DIR, ignore_errors=True)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", INSTALL_DIR, src]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError("reference install failed:\n" + proc.stdout[-2000:] + proc.stderr[-2000:])
    return os.path.isdir(os.path.join(INSTALL_DIR, "prefillsim"))


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
    for p in candidates():
        if os.path.isdir(os.path.join(p, "prefillsim")):
            if p not in sys.path:
                sys.path.append(p)
            return importlib.import_module("prefillsim")
    raise ImportError(
        "prefillsim (reference scheduler) not found; install it with "
        "`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`"
    )
