"""Shared fixtures. `-m gpu` tests need a B200 (run through gpurun); everything else runs
on CPU. Golden fixtures come from the unmodified reference (tests/golden/make_golden.py)."""
import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
KERNELS = os.path.join(ROOT, "paper_2007_01277_b200", "kernels")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

STEMS = ["vector_add", "strided_sum", "histogram", "batchnorm", "shuffle_reduce", "streamer", "hasher", "empty"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run via gpurun")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def corpus():
    return golden("corpus_sources.json")


@pytest.fixture(scope="session")
def hf():
    from paper_2007_01277_b200 import hfuse
    return hfuse


@pytest.fixture(scope="session")
def gpu(hf):
    if hf.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on a B200 (gpurun)")
    return hf


def read_kernel(form, stem):
    with open(os.path.join(KERNELS, form, stem + ".mk")) as f:
        return f.read()
