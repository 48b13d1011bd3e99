"""Locate the UNMODIFIED reference package `fpmat` for the drop-in tests.

Resolution order: $FPMAT_REF, then
/root/reference/pkg/src (the build container), then baseline/_ref (the
offline pip install of /root/reference, git-ignored but shipped to the GPU
box with the snapshot).  Test infrastructure only.
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.environ.get("FPMAT_REF"), "/root/reference/pkg/src",
              os.path.join(ROOT, "baseline", "_ref")]


def reference_root():
    for c in CANDIDATES:
        if c and os.path.isfile(os.path.join(c, "fpmat", "polmat.py")):
            return c
    return None


def import_reference():
    """The reference `fpmat` package, or None when no copy is present."""
    root = reference_root()
    if root is None:
        return None
    sys.dont_write_bytecode = True  # /root/reference is read-only
    if root not in sys.path:
        sys.path.insert(0, root)
    return importlib.import_module("fpmat")
