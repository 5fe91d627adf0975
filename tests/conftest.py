import json
import os
import random
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))   # test infrastructure: the CPU oracle
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and libtnc.so")


def pytest_collection_modifyitems(config, items):
    # -m "not gpu" never needs a device; -m gpu fails loudly (no skip) when
    # the device or the native library is missing.
    pass


@pytest.fixture(scope="session")
def golden_amplitudes():
    return json.loads((GOLDEN / "amplitudes.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_paths():
    return json.loads((GOLDEN / "paths.json").read_text())


@pytest.fixture
def rnd():
    return random.Random(1234)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_bits(rng, n):
    return "".join(rng.choice(["0", "1"], n))
