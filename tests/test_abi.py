"""The C-ABI library loads and exports every symbol include/*.h declares (CPU, no compute)."""

import glob
import os
import re

from conftest import REPO


def _declared():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(ckb_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    from paper_1201_1548_b200 import _lib
    lib = _lib.load()
    declared = _declared()
    assert declared, "no declarations found"
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == declared


def test_abi_version():
    from paper_1201_1548_b200 import _lib
    assert _lib.load().ckb_abi_version() == 6


def test_no_cpu_fallback_without_library(tmp_path):
    """A missing library raises loudly instead of falling back to the CPU."""
    import pytest
    from paper_1201_1548_b200 import _lib
    saved = _lib._lib
    _lib._lib = None
    try:
        with pytest.raises(_lib.CkbError):
            _lib.load(str(tmp_path / "missing.so"))
    finally:
        _lib._lib = saved


def test_product_package_never_imports_the_oracle():
    for path in glob.glob(os.path.join(REPO, "paper_1201_1548_b200", "**", "*.py"), recursive=True):
        src = open(path).read()
        assert "oracle" not in re.sub(r"#.*", "", src).replace("oracle/", ""), path


def test_ctypes_signatures_match_header_arity():
    """Every export has a ctypes signature whose arity equals the header's."""
    from paper_1201_1548_b200 import _lib
    src = ""
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src += re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
    assert set(_lib._SIGS) == set(_lib.EXPORTS)
    for name, (_, args) in _lib._SIGS.items():
        m = re.search(r"\b" + name + r"\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name
