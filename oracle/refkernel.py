"""ORACLE (test infrastructure only): load the reference's OWN compiled
attention kernel (Cython, /root/reference/pkg/src/roundkv/_attn_ext.pyx),
built by `make -C oracle ref` into oracle/_ref/roundkv/.

The compiled module imports two siblings of the reference package
(`from ._attn_np import check_attention_inputs`, `from .errors import
InvariantError`, _attn_ext.pyx:14-15).  The reference sources are not copied:
a synthetic package `roundkv` is registered whose `_attn_np` / `errors`
submodules are the oracle's restatements (oracle/attention.py:check_inputs,
paper_2502_15294_b200/errors.py), and whose __path__ is oracle/_ref/roundkv.
Use it only in processes that do not import another `roundkv`.
"""

from __future__ import annotations

import importlib
import sys
import types
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref" / "roundkv"


def available() -> bool:
    return any(REF_DIR.glob("_attn_ext*.so"))


def load():
    """Return the reference `_attn_ext` module (attention_forward, BACKEND_NAME)."""
    if "roundkv._attn_ext" in sys.modules:
        return sys.modules["roundkv._attn_ext"]
    if not available():
        raise ImportError("reference kernel not built (make -C oracle ref)")
    from paper_2502_15294_b200 import errors as rk_errors

    from . import attention as oatt
    pkg = types.ModuleType("roundkv")
    pkg.__path__ = [str(REF_DIR)]
    attn_np = types.ModuleType("roundkv._attn_np")
    attn_np.check_attention_inputs = oatt.check_inputs
    sys.modules["roundkv"] = pkg
    sys.modules["roundkv._attn_np"] = attn_np
    sys.modules["roundkv.errors"] = rk_errors
    return importlib.import_module("roundkv._attn_ext")
