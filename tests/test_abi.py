"""The C ABI library loads and exports every symbol include/rapp_b200.h declares (CPU only;
no compute calls)."""

import os
import re

from paper_2505_01968_b200 import _lib

from .conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "rapp_b200.h"), encoding="utf-8").read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rapp_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    from paper_2505_01968_b200 import _build
    _build.build()
    lib = _lib.load()
    assert b"sm_100a" in lib.rapp_version()


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 15
    bound = {name for name, _, _ in _lib.SIGNATURES}
    for name in declared:
        assert hasattr(lib, name), name
        assert name in bound, f"{name} declared in the header but not bound in _lib"


def test_error_mapping_uses_reference_exception_types():
    import pytest
    from paper_2505_01968_b200.errors import PlacementError, TableFormatError
    with pytest.raises(ValueError):
        _lib.check(_lib.RAPP_E_VALUE)
    with pytest.raises(TableFormatError):
        _lib.check(_lib.RAPP_E_TABLE)
    with pytest.raises(PlacementError):
        _lib.check(_lib.RAPP_E_PLACEMENT)


def test_no_cpu_fallback_without_device():
    """On a box without a GPU, creating a context must fail loudly, not fall back."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(_lib.DeviceError if hasattr(_lib, "DeviceError") else Exception):
        _lib.Context(0)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2505_01968_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f), encoding="utf-8").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f
