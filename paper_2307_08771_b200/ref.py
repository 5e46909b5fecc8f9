"""Import the UNMODIFIED reference package `reslice` (pkg/src/reslice).

The reference's IR, plan value types, planner and the graph half of
`apply_plan` are consumed as they are (rows marked *C), never
re-typed here.  Where the package comes from, first hit wins:

  1. an importable `reslice` (e.g. pip-installed),
  2. `$UB_RESLICE_PATH`,
  3. `<repo>/baseline/_ref` -- the offline install made by `install()` below
     (`pip install --no-index --target baseline/_ref <copy of /root/reference/pkg>`);
     git-ignored but shipped to the GPU hosts with the tree,
  4. `/root/reference/pkg/src` (the build container).

`install()` is called by `__graft_entry__.build()`; nothing is copied from the
reference into this package.
"""

from __future__ import annotations

import importlib
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_INSTALL = ROOT / "baseline" / "_ref"
REF_SOURCE = Path("/root/reference/pkg")


class ReferenceMissingError(ImportError):
    """The reference package `reslice` cannot be located."""


def _candidates() -> list[Path]:
    out = []
    if os.environ.get("UB_RESLICE_PATH"):
        out.append(Path(os.environ["UB_RESLICE_PATH"]))
    out += [REF_INSTALL, REF_SOURCE / "src"]
    return out


def load():
    """Return the imported `reslice` module."""
    try:
        return importlib.import_module("reslice")
    except ImportError:
        pass
    for p in _candidates():
        if (p / "reslice" / "__init__.py").exists():
            sys.path.insert(0, str(p))
            return importlib.import_module("reslice")
    raise ReferenceMissingError(
        "the reference package `reslice` is not importable; run "
        "`python -c 'from paper_2307_08771_b200 import ref; ref.install()'` in a tree with "
        f"{REF_SOURCE} present, or set UB_RESLICE_PATH")


def install(force: bool = False) -> Path | None:
    """Offline install of the reference into baseline/_ref (the task's one sanctioned
    install).  The build copies the read-only source tree to /tmp first, since a
    setuptools build writes next to pyproject.toml.  No-op when already installed or
    when the reference sources are absent (GPU hosts get the installed copy)."""
    if (REF_INSTALL / "reslice" / "__init__.py").exists() and not force:
        return REF_INSTALL
    if not (REF_SOURCE / "pyproject.toml").exists():
        return None
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_SOURCE, src, ignore=shutil.ignore_patterns("tests", "demos", "__pycache__"))
        if REF_INSTALL.exists():
            shutil.rmtree(REF_INSTALL)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", str(REF_INSTALL), str(src)]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
    return REF_INSTALL


reslice = load()
