"""Import the LIVE reference package (this container only).

``/root/reference/pkg/src`` is put on ``sys.path`` and the reference's own
compiled kernel, built into ``oracle/_ref`` by ``oracle/Makefile``, is
registered as ``elastik._speedups`` so ``backend="compiled"`` works without
building inside the read-only tree.  Returns None when the reference is absent
(e.g. on the GPU box), so callers can skip.
"""

from __future__ import annotations

import importlib.machinery
import importlib.util
import os
import sys

REF_SRC = "/root/reference/pkg/src"
_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def load():
    if not os.path.isdir(os.path.join(REF_SRC, "elastik")):
        return None
    if "elastik" in sys.modules:
        return sys.modules["elastik"]
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, _REPO)
    from oracle import refdrive

    path = refdrive.ref_path()
    if path is not None:
        loader = importlib.machinery.ExtensionFileLoader("elastik._speedups", path)
        spec = importlib.util.spec_from_loader("elastik._speedups", loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        sys.modules["elastik._speedups"] = mod
    import elastik

    return elastik
