import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = os.path.join(HERE, "golden")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


MODEL_TAGS = ("case14", "case118", "C1", "T4", "C2")
TILES = {"C1": 1, "T4": 4, "C2": 143}


@pytest.fixture(scope="session")
def golden_models():
    return {t: dict(np.load(os.path.join(GOLDEN, f"{t}.npz"))) for t in MODEL_TAGS}


@pytest.fixture(scope="session")
def end_to_end():
    with open(os.path.join(GOLDEN, "end_to_end.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def networks_json():
    with open(os.path.join(GOLDEN, "networks.json")) as fh:
        return json.load(fh)


def golden_x(tag, tol):
    return np.load(os.path.join(GOLDEN, f"{tag}_{tol:g}_x.npz"))["x"]
