import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def golden_cases(pattern="*.npz", exclude=("proxy_kat", "lod", "train", "vertex", "vertex_f64", "kl",
                                            "f64_inputs")):
    names = sorted(os.path.splitext(os.path.basename(p))[0]
                   for p in glob.glob(os.path.join(GOLDEN, pattern)))
    return [n for n in names if n not in exclude]


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def golden_config(g):
    return json.loads(str(g["config"]))


def golden_levels(g):
    levels = []
    i = 0
    while f"lat{i}" in g:
        levels.append(g[f"lat{i}"])
        i += 1
    return levels


def golden_nets(g, prefix):
    n = int(g[prefix + "_n"])
    return [(g[f"{prefix}_w{i}"], g[f"{prefix}_b{i}"],
             "linear" if int(g[f"{prefix}_a{i}"]) == 0 else "leaky_relu") for i in range(n)]


def rel_err(a, b):
    """The reference's own agreement metric |a-b| / (|b| + 1e-2) (cli.py:213)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / (np.abs(b) + 1e-2)
