"""The C ABI library loads and exports every symbol include/ttn_cbc.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttn_cbc.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^TTN_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_19650_b200 import _build
    path = _build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("ttn_create", "cbc_apply", "ttn_overlap", "ttn_norm"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_lists_match_header():
    from paper_2601_19650_b200 import _lib
    assert sorted(_lib.SYMBOLS) == declared_symbols()


def test_version_and_no_device_is_an_error(lib):
    import paper_2601_19650_b200 as P
    assert "sm_100a" in P.ttn_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.TTNError):
        P.Context(0)
