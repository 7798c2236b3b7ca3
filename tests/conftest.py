"""Shared fixtures. `gpu`-marked tests need a B200 (run with -m gpu); the
rest run on CPU. The oracle (oracle/) is test infrastructure only."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "expected.json")) as f:
        exp = json.load(f)
    grids = dict(np.load(os.path.join(GOLDEN, "grids.npz")))
    return exp, grids


@pytest.fixture(scope="session")
def oracle():
    import pyoracle as po
    return po.Oracle()


@pytest.fixture(scope="session")
def ref():
    import pyoracle as po
    if not po.Ref.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return po.Ref()


def corpus(golden, name):
    exp, grids = golden
    return [(uid, grids[f"{name}/{uid}"]) for uid in exp["corpora"][name]]


def same_result(got, want, tol=1e-9):
    """Field-by-field, like test_batched.cpp:27-31 (joint within tol)."""
    return (got.tokens == want["tokens"] and got.label_times == want["label_times"]
            and got.steps_taken == want["steps"] and got.eos_trigger == want["eos_trigger"]
            and abs(got.joint_logp - want["joint_logp"]) <= tol)
