"""libvsdock.so loads on a CPU-only box and exports every entry point the
C headers declare; without a device the GPU entry points fail loudly."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

from paper_2110_11644_b200 import abi, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in ("vs_dock.h", "vs_prep.h", "vs_codec.h", "vs_rank.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(vs_[a-z0-9_]+)\s*\(", text))
    return sorted(syms)


def test_library_loads_and_exports_every_declared_symbol():
    lib = native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(native.SIGNATURES), set(syms) - set(native.SIGNATURES)


def test_abi_version_and_struct_sizes():
    lib = native.lib()
    assert lib.vs_abi_version() == 1
    assert C.sizeof(abi.DockResult) == 104
    cfg = abi.ScoringConfig()
    ref = abi.ScoringConfig(restarts=0)
    lib.vs_scoring_config_default(C.byref(ref))
    for f, _ in abi.ScoringConfig._fields_:
        assert getattr(cfg, f) == getattr(ref, f), f


def test_no_device_fails_loudly():
    lib = native.lib()
    if lib.vs_device_count() > 0:
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    assert lib.vs_context_create(0, C.byref(h)) == abi.VS_ERR_NO_DEVICE
    from paper_2110_11644_b200 import api
    with pytest.raises(native.NativeError):
        api.Context(0)
