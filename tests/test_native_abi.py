"""The C-ABI library loads and exports every symbol include/chebm2l.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "chebm2l.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(cfm_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_table():
    from paper_1210_7292_b200 import _native

    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_all_symbols():
    from paper_1210_7292_b200 import _native

    if not _native.LIB_PATH.exists():
        pytest.fail("libchebm2l.so not built (run `make` or __graft_entry__.build())")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib2 = _native.load()
    assert lib2.cfm_abi_version() == 1
    assert lib2.cfm_last_error() == b""


def test_handler_create_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1210_7292_b200 import B200M2LHandler, ChebyshevGrid, laplace_kernel

    with pytest.raises(Exception):
        B200M2LHandler("nablk", laplace_kernel(), ChebyshevGrid(4), 1e-5)


def test_no_oracle_import_in_product():
    for p in (ROOT / "paper_1210_7292_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
