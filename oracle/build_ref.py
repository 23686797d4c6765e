"""Recipe for oracle/_ref: the reference package itself, for the CPU baseline.

TEST / MEASUREMENT INFRASTRUCTURE -- never imported by the product path.

The reference (`commviz`, /root/reference/pkg/src/commviz) is pure Python +
numba, so "building" it is packaging the unmodified sources:
`build()` (run by __graft_entry__.build() in the build container, where
/root/reference exists) zips the package into oracle/_ref/commviz.zip.
oracle/_ref/ is git-ignored (no reference source enters the history) but not
gpurun-ignored, so the archive travels to the GPU box, where `load()`
extracts it into a private temporary directory (numba's cache=True needs a
real source file next to a writable __pycache__) and imports it.
bench.py's reference arm times it beside the C/numpy port (oracle.py).
"""

from __future__ import annotations

import importlib
import os
import sys
import tempfile
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ZIP = os.path.join(REF_DIR, "commviz.zip")
SRC = "/root/reference/pkg/src/commviz"


def build() -> str | None:
    """Package the reference sources (no-op where /root/reference is absent)."""
    if not os.path.isdir(SRC):
        return None
    os.makedirs(REF_DIR, exist_ok=True)
    names = sorted(f for f in os.listdir(SRC) if f.endswith(".py"))
    tmp = ZIP + ".tmp"
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as z:
        for f in names:
            # fixed timestamps: the archive is byte-stable across builds
            info = zipfile.ZipInfo(f"commviz/{f}", date_time=(2020, 1, 1, 0, 0, 0))
            with open(os.path.join(SRC, f), "rb") as fh:
                z.writestr(info, fh.read())
    os.replace(tmp, ZIP)
    return ZIP


_mod = None


def load():
    """Import the packaged reference (raises ImportError if not packaged or
    numba is missing)."""
    global _mod
    if _mod is not None:
        return _mod
    if not os.path.exists(ZIP):
        raise ImportError(f"{ZIP} missing (run oracle.build_ref.build() where "
                          "/root/reference exists)")
    importlib.import_module("numba")
    d = tempfile.mkdtemp(prefix="commviz_ref_")
    with zipfile.ZipFile(ZIP) as z:
        z.extractall(d)
    sys.path.insert(0, d)
    try:
        _mod = importlib.import_module("commviz")
    finally:
        sys.path.remove(d)
    return _mod


if __name__ == "__main__":
    print(build())
