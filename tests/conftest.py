"""Shared fixtures. ``-m gpu`` tests need a B200 (run through gpurun); every
other test runs on CPU. Golden vectors from the reference live in
tests/golden/reference_golden.json (see tests/golden/make_golden.py)."""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.json"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


@pytest.fixture(scope="session")
def spec_file(golden, tmp_path_factory):
    """Write one of the reference's simulated device specs to a temp file."""
    root = tmp_path_factory.mktemp("specs")

    def make(name):
        path = root / f"{name}.json"
        if not path.exists():
            path.write_text(json.dumps(golden["specs"][name]))
        return path

    return make


@pytest.fixture(scope="session")
def reference():
    """The live reference package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference package not present")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import jouletune

    return jouletune


FULL_PIN = ROOT / "tests" / "golden" / "pnpoly_full_pin.json"


def assert_full_size_pin(bitmap) -> None:
    """A full-size (BASELINE) PnPoly bitmap against tests/golden/pnpoly_full_pin.json: it must be the
    formula-2 bitmap bit for bit, which differs from the paper's Kernel-Tuner op order (formula 0)
    at exactly the recorded points."""
    import hashlib

    import numpy as np

    pin = json.loads(FULL_PIN.read_text())
    got = np.ascontiguousarray(bitmap, dtype=np.int32)
    assert got.size == pin["n_points"]
    assert hashlib.sha256(got.tobytes()).hexdigest() == pin["sha256"]["formula2"]
    for d in pin["formula0_vs_formula2_differ"]:
        assert got[d["index"]] == d["formula2"] != d["formula0"]
