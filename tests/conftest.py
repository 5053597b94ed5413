"""Test configuration.

Markers:
  gpu  needs a CUDA device (B200); these are the parity tests proper and call
       the product through the C-ABI (libbbs_b200.so).
Everything unmarked runs on CPU: the oracle restatement against the golden
fixtures and the reference, host-side logic, the C-ABI surface (symbols,
struct layouts, error mapping) and the multi-rank host protocol over gloo.
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import harness as H  # noqa: E402  (synthetic inputs)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def B():
    import paper_2310_10023_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Reference, REFERENCE_SO
    if not os.path.exists(REFERENCE_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def orc():
    from pyoracle import Restated
    return Restated()


@pytest.fixture(scope="session")
def golden_scenes():
    with open(os.path.join(GOLDEN, "scenes.json")) as f:
        return json.load(f)


def load_case(B, scenes, name):
    """Regenerate a golden case's inputs with the product's scene restatement
    (bit-identity against the reference's gen_scene is tested separately)."""
    sc = scenes[name]
    spec = H.SceneSpec.default(**sc["spec"])
    m, s, gt = H.gen_scene(spec, sc["seed"])
    if sc["K"] is not None:
        s = H.cut_scan(s, min(sc["K"], s.shape[0]), sc["cut_seed"])
    return m, s, gt, sc


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name))
