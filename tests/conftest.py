import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def cases(d, prefix):
    """Sorted case indices i for keys '<prefix><i>_...'."""
    out = set()
    for k in d.files:
        if k.startswith(prefix) and k[len(prefix)].isdigit():
            out.add(int(k[len(prefix):].split("_")[0]))
    return sorted(out)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ---- fixtures mirroring /root/reference/pkg/tests/conftest.py:23-75 ----
def planted_edges(seed, cliques=8, size=16, bridges=8):
    rng = np.random.default_rng(seed)
    edges = []
    for c in range(cliques):
        base = c * size
        for i in range(size):
            for j in range(i + 1, size):
                edges.append((base + i, base + j))
    for _ in range(bridges):
        a, b = rng.choice(cliques, size=2, replace=False)
        edges.append((int(a * size + rng.integers(size)), int(b * size + rng.integers(size))))
    return np.array(edges, dtype=np.int64)


def exact_recovered(labels, cliques=8, size=16):
    n = 0
    for c in range(cliques):
        member = labels[c * size:(c + 1) * size]
        if len(np.unique(member)) == 1 and np.sum(labels == member[0]) == size:
            n += 1
    return n
