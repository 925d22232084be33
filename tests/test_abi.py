"""CPU tests of the drop-in boundary: libhemul_gpu.so loads, exports exactly
the C-ABI that include/hemul_gpu.h declares, and behaves correctly without
a GPU (no CPU fallback: computing calls fail loudly)."""
from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hemul_gpu.h"


def _declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hemul_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("hemul_gpu_create", "hemul_gpu_he_mul", "hemul_gpu_rescale",
                     "hemul_gpu_set_evk", "hemul_gpu_set_level", "hemul_gpu_ntt",
                     "hemul_gpu_crt", "hemul_gpu_icrt", "hemul_gpu_pointwise",
                     "hemul_gpu_destroy", "hemul_gpu_last_error", "hemul_ciphertext_digest"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2003_04510_b200.hemul import LIB_PATH

    assert LIB_PATH.exists(), "run python -m paper_2003_04510_b200.build"
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hemul_\w+)", out))
    missing = [f for f in _declared_functions() if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(str(LIB_PATH))
    for f in _declared_functions():
        assert getattr(lib, f) is not None


def test_header_compiles_as_c():
    src = f'#include "{HEADER}"\nint main(void) {{ hemul_gpu_ctx *c = 0; (void)c; return 0; }}\n'
    res = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-x", "c", "-", "-o", "/dev/null"],
                         input=src, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_create_without_gpu_fails_loudly_or_succeeds_on_gpu():
    from paper_2003_04510_b200.hemul import (HEMUL_E_CUDA, HEMUL_OK, Context, HemulGpuError,
                                             load_library, make_params)

    lib = load_library()
    h = ctypes.c_void_p()
    st = lib.hemul_gpu_create(0, 30, 4, 10, ctypes.byref(h))
    assert st in (HEMUL_OK, HEMUL_E_CUDA)
    if st == HEMUL_OK:
        lib.hemul_gpu_destroy(h)
    else:
        with pytest.raises(HemulGpuError):
            Context(make_params(30, 4, 10))


def test_create_rejects_bad_arguments():
    from paper_2003_04510_b200.hemul import HEMUL_OK, load_library

    lib = load_library()
    h = ctypes.c_void_p()
    assert lib.hemul_gpu_create(0, 0, 4, 10, ctypes.byref(h)) != HEMUL_OK
    assert lib.hemul_gpu_create(0, 30, 0, 10, ctypes.byref(h)) != HEMUL_OK
    assert lib.hemul_gpu_create(0, 30, 100, 0, ctypes.byref(h)) != HEMUL_OK  # logQ > 2400
    assert lib.hemul_gpu_create(0, 30, 4, 10, None) != HEMUL_OK


def test_null_context_is_rejected():
    from paper_2003_04510_b200.hemul import HEMUL_E_ARG, load_library

    lib = load_library()
    assert lib.hemul_gpu_set_level(None, 120) == HEMUL_E_ARG
    assert lib.hemul_gpu_synchronize(None) == HEMUL_E_ARG
    assert lib.hemul_gpu_launch_count(None) == 0


def test_digest_matches_restated_oracle(restated):
    """ciphertext_digest (bench.cpp:35-47) is host code in the library."""
    from paper_2003_04510_b200.hemul import ciphertext_digest

    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**63, size=(64, 3), dtype=np.uint64)
    b = rng.integers(0, 2**63, size=(64, 3), dtype=np.uint64)
    assert ciphertext_digest(150, a, b) == restated.digest(150, 64, a, b)


def test_params_match_reference(reference):
    """make_params / the security table (params.cpp:56-74)."""
    from paper_2003_04510_b200.hemul import make_params

    for cfg in [(30, 4, 13), (30, 10, 0), (30, 20, 0), (30, 40, 0), (30, 80, 0), (25, 7, 0)]:
        p = make_params(*cfg)
        log_n, n, qmax = reference.make_params(*cfg)
        assert (p.log_n, p.n, p.log_q_max) == (log_n, n, qmax)
