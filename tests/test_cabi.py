"""The C-ABI library loads without a GPU and exports every declared symbol."""
from __future__ import annotations

import os
import re

from conftest import ROOT


def test_library_exports_header_symbols():
    from paper_1702_04739_b200 import _lib
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "isoclust_b200.h")).read()
    names = re.findall(r"^(?:int|void|const char \*)\s*\*?\s*(isoc_\w+)\(", header, re.M)
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert lib.isoc_version() == 1


def test_fold_stack_size_matches_header():
    from paper_1702_04739_b200 import _lib
    header = open(os.path.join(ROOT, "include", "isoclust_b200.h")).read()
    m = re.search(r"#define ISOC_FOLD_STACK_BYTES (\d+)", header)
    assert int(m.group(1)) == _lib.FOLD_STACK_BYTES


def test_status_mapping():
    import pytest
    from paper_1702_04739_b200 import _lib
    _lib.check(_lib.ISOC_OK)
    for code, exc in [(_lib.ISOC_EINVAL, ValueError), (_lib.ISOC_ETYPE, TypeError),
                      (_lib.ISOC_EINFEASIBLE, _lib.InfeasibleSubpartitionError),
                      (_lib.ISOC_ENOMEM, MemoryError), (_lib.ISOC_ECUDA, RuntimeError)]:
        with pytest.raises(exc):
            _lib.check(code)
