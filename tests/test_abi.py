"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; status codes match the Python exception mapping.  No
compute call is made here (no GPU)."""

from __future__ import annotations

import os
import re

from conftest import ROOT
from paper_2202_12429_b200 import _lib, errors

HEADER = os.path.join(ROOT, "include", "bagpipe_b200.h")


def _declared() -> set:
    text = open(HEADER).read()
    names = set(re.findall(r"^(?:int|int64_t|float\*|uint8_t\*|const char\*)\s+(bp_[a-z0-9_]+)\(", text, re.M))
    return names


def test_header_declares_the_bound_symbols():
    declared = _declared()
    assert declared, "no declarations parsed"
    assert set(_lib.exported_symbols()) <= declared | {"bp_version", "bp_last_error_message"}


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()  # dlopen only
    missing = [name for name in sorted(_declared()) if not hasattr(lib, name)]
    assert missing == []
    assert lib.bp_version().startswith(b"bagpipe_b200")


def test_status_codes_match_header():
    text = open(HEADER).read()
    codes = {int(v): k for k, v in re.findall(r"#define (BP_ERR_[A-Z_]+) (\d+)", text)}
    expect = {1: errors.ConfigurationError, 2: errors.CacheMissError, 3: errors.CacheCapacityError,
              4: errors.CacheOrderingError, 5: errors.StoreKeyError, 6: errors.StoreError, 7: errors.EngineError}
    for code, cls in expect.items():
        assert code in codes and errors.STATUS_TO_ERROR[code] is cls
    assert set(codes) == set(errors.STATUS_TO_ERROR)


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _lib._lib = None
    with pytest.raises(_lib.NativeUnavailable):
        _lib.lib()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2202_12429_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
