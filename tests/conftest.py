"""Shared test plumbing: the `gpu` marker and golden-fixture loading."""

import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA library")


def pytest_collection_modifyitems(config, items):
    # A `-m gpu` run on a box without CUDA must fail loudly, not skip.
    pass
