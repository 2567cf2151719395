import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (skipped unless GO_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("GO_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow test; set GO_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = dict(np.load(GOLDEN / f"golden_{name}.npz", allow_pickle=False))
    return _cache[name]


def oracle_graph(z, prefix):
    from oracle import graph as og
    g = og.make(int(z[prefix + "n"]), z[prefix + "op"], z[prefix + "flops"],
                z[prefix + "out_bytes"], z[prefix + "src"], z[prefix + "dst"],
                z[prefix + "ebytes"], z[prefix + "coloc"])
    return g


def forward_meta():
    return json.loads(str(golden("forward")["meta"]))


def rel_err(a, b):
    """Normwise relative error max|a-b| / max|b| (the 1e-4 parity metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(b).max(initial=0.0), 1e-30)
    return float(np.abs(a - b).max(initial=0.0) / den)
