import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native kernels")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_sessionfinish(session, exitstatus):
    """Tie-swap counts of every selection comparison (evidence for the
    bounded tie rule) -> gpurun_out/tie_swaps.json when that
    directory exists (GPU runs)."""
    import json

    from tests.helpers import TIE_LOG

    out = os.path.join(ROOT, "gpurun_out")
    if TIE_LOG and os.path.isdir(out):
        rows = [{"test": t, "k": k, "swaps": s} for t, k, s in TIE_LOG]
        with open(os.path.join(out, "tie_swaps.json"), "w") as f:
            json.dump({"checks": len(rows), "max_swaps": max(r["swaps"] for r in rows), "rows": rows}, f, indent=1)
