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
def reference(request):
    """The reference library itself (oracle/_ref, built from /root/reference by
    oracle/Makefile; prebuilt .so travels to the GPU box). Missing it is a
    failure, never a skip: the paper-scale parity tests depend on it."""
    from oracle_lib import REFERENCE_SO, Reference

    if not REFERENCE_SO.exists() and Path("/root/reference").exists():
        import subprocess

        subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], capture_output=True)
    if not REFERENCE_SO.exists():
        pytest.fail("oracle/_ref/libhemul_ref.so not built: run `python -c 'import "
                    "__graft_entry__ as g; g.build()'` where /root/reference exists")
    return Reference()
