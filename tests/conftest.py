"""Shared fixtures.  `gpu` tests need a CUDA device and libkfb200.so; the rest
run on CPU (oracle vs golden vectors, host setup, ABI symbol table, gloo)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkfb200.so")


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def make_system(seq, solvation=False, samples=1024, dielectric=None, pkg=None):
    """Chain + params + weights + Field built with this package's host setup."""
    import paper_1712_05012_b200 as P
    pkg = pkg or P
    ch = pkg.build_chain(list(seq))
    ps = pkg.load_params()
    params = ps.resolve(ch)
    w = pkg.TreeWeights(pkg.build_tree(ch), ps.weights)
    kw = dict(solvation=solvation, solvation_cfg=pkg.SolvationConfig(samples=samples))
    if dielectric is not None:
        kw["dielectric"] = dielectric
    return ch, params, w, pkg.Field(params, w, pkg.FieldConfig(**kw))


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
