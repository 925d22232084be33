"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box with -m gpu).
Everything unmarked runs on a CPU-only machine.
"""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (paper-scale parameters)")


@pytest.fixture(scope="session")
def restated():
    from oracle_lib import RESTATED_SO, Restated

    if not RESTATED_SO.exists():
        pytest.fail("oracle/liboracle.so missing: run `make -C oracle restate`")
    return Restated()


@pytest.fixture(scope="session")
def reference():
    from oracle_lib import REFERENCE_SO, Reference

    if not REFERENCE_SO.exists():
        pytest.skip("oracle/_ref/libhemul_ref.so not built (needs /root/reference at build time)")
    return Reference()
