"""BASELINE INFRASTRUCTURE ONLY -- the unmodified reference package, staged.

``stage()`` installs the reference (``/root/reference/pkg``, the ``hhsar``
package: Python + Numba) into ``oracle/_ref/`` with the reference's own
packaging (``pip install --no-index --no-build-isolation --no-deps
--target``, from a copy in a temporary directory because the reference tree
is read-only).  ``oracle/_ref/`` is git-ignored -- no reference source enters
the repository history -- but it is not gpurun-ignored, so the staged copy
travels to the GPU box next to the built libraries and bench.py can time the
reference's own CPU path there (``load()``).  numba is in the image, so the
staged package runs its Numba kernels (_kernels.py:18-31, HAVE_NUMBA).

Only bench.py's reference arm / CPU baseline legs and tests import it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
SOURCE = Path("/root/reference/pkg")


def staged() -> bool:
    return (REF_DIR / "hhsar" / "__init__.py").exists()


def stage(source: Path = SOURCE, force: bool = False) -> bool:
    """Install the reference package into oracle/_ref (no-op when staged or
    when the reference tree is absent, e.g. on the GPU box)."""
    if staged() and not force:
        return True
    if not (Path(source) / "pyproject.toml").exists():
        return False
    with tempfile.TemporaryDirectory() as tmp:
        copy = Path(tmp) / "pkg"
        shutil.copytree(source, copy, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        out = Path(tmp) / "out"
        subprocess.check_call([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                               "--no-build-isolation", "--no-deps", "--target", str(out),
                               str(copy)])
        if REF_DIR.exists():
            shutil.rmtree(REF_DIR)
        REF_DIR.mkdir(parents=True)
        shutil.copytree(out / "hhsar", REF_DIR / "hhsar")
    return staged()


def load():
    """Import the staged reference package (``hhsar``) with its Numba JIT
    cache redirected to /tmp; raises ImportError if it is not staged."""
    if not staged():
        raise ImportError(f"reference not staged in {REF_DIR} (oracle.reference.stage())")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hhsar_numba_cache")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import hhsar
    if not str(Path(hhsar.__file__).resolve()).startswith(str(REF_DIR)):
        raise ImportError(f"hhsar imported from {hhsar.__file__}, not the staged copy")
    return hhsar


def load_or_port():
    """(module, kind): the staged reference package ("reference") or, where
    it is missing, the oracle port behind the same API (oracle/port_api.py,
    "port")."""
    try:
        return load(), "reference"
    except ImportError:
        from . import pipeline, port_api
        pipeline.build_library()
        return port_api, "port"


def threads() -> int:
    """Numba's thread count (default: every host core); the port's OpenMP
    loops use the same."""
    try:
        import numba
        return int(numba.get_num_threads())
    except Exception:
        return os.cpu_count() or 1
