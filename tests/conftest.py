import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.setrecursionlimit(200000)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_kernel(name):
    with open(os.path.join(GOLD, "kernels", name + ".json")) as f:
        return json.load(f)


def load_model(name):
    with open(os.path.join(GOLD, "models", name + ".json")) as f:
        return json.load(f)


def load_cases():
    with open(os.path.join(GOLD, "cases.json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="session")
def cases():
    return load_cases()
