"""C-ABI library: loads without a GPU and exports every symbol include/rootbox_b200.h declares."""
import os
import re

from conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "rootbox_b200.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(rb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    from paper_1802_00330_b200 import _native
    L = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_native.EXPORTED)


def test_version_string_without_gpu():
    from paper_1802_00330_b200 import _native
    assert "sm_100a" in _native.version()
    assert _native.device_count() >= 0


def test_create_fails_loudly_without_device():
    """No CPU fallback: without a B200 rb_create must raise, not compute."""
    import pytest
    from paper_1802_00330_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("GPU present")
    from paper_1802_00330_b200.system import compile_tables
    from conftest import golden_spec
    with pytest.raises(Exception):
        _native.Engine(compile_tables(golden_spec("circle_line")), 0)
