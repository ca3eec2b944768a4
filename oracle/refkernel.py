"""ORACLE (test infrastructure only): load the reference package itself —
its unmodified Python modules and its OWN compiled attention kernel (Cython,
/root/reference/pkg/src/roundkv/_attn_ext.pyx) — staged by `make -C oracle ref`
into oracle/_ref/roundkv/ (git-ignored; travels to the GPU box, where
/root/reference does not exist).

`load_package()` imports it under its own name `roundkv` (the product package
is `paper_2502_15294_b200`, so the names never collide) and checks that its
backend selection (backend.py:31-44) picked the compiled kernel ("ext").
Nothing here imports the product package: a process that only runs the
reference (bench.py --impl reference) never maps librk.so.
"""

from __future__ import annotations

import hashlib
import importlib
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_ROOT = HERE / "_ref"
REF_DIR = REF_ROOT / "roundkv"


def available() -> bool:
    return any(REF_DIR.glob("_attn_ext*.so")) and (REF_DIR / "__init__.py").exists()


def load_package():
    """The reference package `roundkv` from oracle/_ref (BACKEND_NAME == "ext")."""
    mod = sys.modules.get("roundkv")
    if mod is not None:
        if not str(getattr(mod, "__file__", "")).startswith(str(REF_DIR)):
            raise ImportError(f"another `roundkv` is already imported: {getattr(mod, '__file__', mod)}")
        return mod
    if not available():
        raise ImportError("reference package not staged (make -C oracle ref)")
    sys.path.insert(0, str(REF_ROOT))
    try:
        mod = importlib.import_module("roundkv")
    finally:
        sys.path.remove(str(REF_ROOT))
    if mod.BACKEND_NAME != "ext":
        raise ImportError(f"reference backend is {mod.BACKEND_NAME!r}, expected the compiled 'ext' kernel")
    return mod


def load():
    """The reference `_attn_ext` module (attention_forward, BACKEND_NAME)."""
    load_package()
    return importlib.import_module("roundkv._attn_ext")


def kernel_identity() -> dict:
    """Path and sha256 of the compiled reference kernel this process loaded."""
    ext = load()
    p = Path(ext.__file__)
    return {"path": str(p.relative_to(HERE.parent)) if p.is_relative_to(HERE.parent) else str(p),
            "sha256": hashlib.sha256(p.read_bytes()).hexdigest()[:16]}
