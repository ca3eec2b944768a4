"""CPU checks of the drop-in boundary: librk.so loads without a GPU and
exports every entry point declared in include/roundkv_b200.h; the Python
mirror exposes the reference's module API (names and error classes)."""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import REPO

HEADER = REPO / "include" / "roundkv_b200.h"
LIB = REPO / "paper_2502_15294_b200" / "librk.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|size_t|const char\*)\s+(rk_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for name in ("rk_attention_forward", "rk_decode_attention", "rk_round_scores", "rk_select",
                 "rk_h2d_gather", "rk_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        from paper_2502_15294_b200.build import build
        build()
    lib = ctypes.CDLL(str(LIB))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.rk_abi_version.restype = ctypes.c_int
    assert lib.rk_abi_version() == 1


def test_python_binding_matches_header():
    from paper_2502_15294_b200 import _lib
    assert sorted(_lib.symbols()) == declared_symbols()


def test_error_mapping_is_reference_hierarchy():
    from paper_2502_15294_b200 import errors as e
    assert issubclass(e.DomainError, e.InputError) and issubclass(e.InputError, e.RoundKVError)
    assert issubclass(e.CapacityError, e.RoundKVError)
    assert isinstance(e.from_status(-1, "x"), e.DomainError)
    assert isinstance(e.from_status(-2, "x"), e.CapacityError)
    assert isinstance(e.from_status(-3, "x"), e.ConsistencyError)
    assert isinstance(e.from_status(-4, "x"), e.InvariantError)


def test_status_codes_without_gpu():
    """Argument validation happens on the host and needs no device."""
    from paper_2502_15294_b200 import _lib
    from paper_2502_15294_b200.errors import DomainError
    st = _lib.lib.rk_select(None, -1, 1, 1, 0.1, 1, 1.0, None, None, None, None, None, None)
    assert st == -1 and "rounds" in _lib.last_error()
    with pytest.raises(DomainError):
        _lib.check(st, "rk_select")
    st = _lib.lib.rk_attention_forward(None, 1, 3, 8, None, None, 0, 4, 2, None, None, None, None, None,
                                       None, None, 0, None)
    assert st == -1 and "multiple" in _lib.last_error()


def test_cpu_only_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import numpy as np
    from paper_2502_15294_b200 import backend
    from paper_2502_15294_b200.errors import DeviceError
    q = np.zeros((1, 1, 2), np.float32)
    with pytest.raises(DeviceError):
        backend.attention_forward(q, q, q, [0], [0])


def test_backend_env_rejects_cpu_backends(monkeypatch):
    import importlib
    import paper_2502_15294_b200.backend as b
    monkeypatch.setenv("ROUNDKV_BACKEND", "numpy")
    with pytest.raises(ImportError):
        importlib.reload(b)
    monkeypatch.setenv("ROUNDKV_BACKEND", "auto")
    importlib.reload(b)
