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


def test_codegen_prepare_without_gpu(tmp_path, monkeypatch):
    """The system-specialised kernels compile with NVRTC on a machine without a
    GPU (build time); the cache key depends only on the system and the kernel
    headers, so two compilations of the same system share one entry."""
    from paper_1802_00330_b200 import _native
    from paper_1802_00330_b200.system import compile_tables
    from conftest import golden_spec
    monkeypatch.setenv("RB_KCACHE", str(tmp_path))
    k1 = _native.codegen_prepare(compile_tables(golden_spec("circle_line")))
    k2 = _native.codegen_prepare(compile_tables(golden_spec("circle_line")))
    k3 = _native.codegen_prepare(compile_tables(golden_spec("broyden_tri4")))
    assert re.fullmatch(r"[0-9a-f]{16}", k1) and k1 == k2 and k1 != k3
    files = sorted(os.listdir(tmp_path))
    assert files == sorted([f"{k1}.cubin", f"{k1}.names", f"{k3}.cubin", f"{k3}.names"])
    names = (tmp_path / f"{k1}.names").read_text().split()
    assert len(names) == 7 and all("GenEval" in n or "rbg" in n for n in names)
