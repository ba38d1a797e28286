"""The C-ABI library builds/loads on CPU and exports every symbol include/mgnn.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2410_22697_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mgnn.h")).read()
    return sorted(set(re.findall(r"MGNN_API[^;(]*?\b(mgnn_\w+)\s*\(", src)))


def test_header_lists_match_binding():
    assert _declared() == sorted(_lib.SYMBOLS)


def test_library_loads_and_exports():
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mgnn_\w+)", out))
    assert set(_declared()) <= exported
    assert not any(s.startswith("_ZN4mgnn") for s in re.findall(r"\bT (\S+)", out))   # internals hidden


def test_alpha_default_host_function():
    L = _lib.load()
    assert L.mgnn_alpha_default(0.5, 10) == 2.0 ** -10
    assert L.mgnn_alpha_default(1.0, 100) == 1.0


def test_ctx_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.load()
    h = ctypes.c_void_p()
    import numpy as np
    b = np.array([0, 10], dtype=np.int64)
    st = L.mgnn_ctx_create(0, 1, 10, b.ctypes.data_as(ctypes.c_void_p), 4, 1, ctypes.byref(h))
    assert st == 3 and not h.value          # MGNN_ECUDA, no context


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
