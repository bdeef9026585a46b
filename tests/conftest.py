"""Shared pytest setup: `gpu` marker, repo root on sys.path, golden loader."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def unragged(counts, rows, stride=None):
    """Inverse of make_golden.ragged: (n, stride) int32 zero-padded rows."""
    counts = np.asarray(counts)
    width = int(stride if stride is not None else max(int(counts.max()), 1))
    out = np.zeros((counts.size, width), dtype=np.int32)
    at = 0
    for i, c in enumerate(counts):
        out[i, :c] = rows[at:at + c]
        at += c
    return out
