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


def test_binding_checks_tensor_sizes_before_the_call():
    """ttn_create refuses tensors whose size does not match the ABI shape from (parent, phys,
    bond), before anything reaches the C side (no read past a short buffer)."""
    import numpy as np
    import paper_2601_19650_b200 as P
    parent, phys, bond = [-1, 0, 0], [2, 2, 2], [1, 3, 4]
    assert P.node_sizes(P.TTN_STATE, parent, phys, bond) == [2 * 1 * 3 * 4, 2 * 3, 2 * 4]
    assert P.node_sizes(P.TTN_OPERATOR, parent, phys, bond) == [4 * 12, 4 * 3, 4 * 4]
    good = [np.zeros((2, 1, 3, 4), complex), np.zeros((2, 3), complex), np.zeros((2, 4), complex)]
    bad = good[:2] + [np.zeros((2, 3), complex)]
    with pytest.raises(ValueError, match="node 2"):
        P.ttn_create(None, P.TTN_STATE, parent, phys, bond, bad)
    with pytest.raises(ValueError):
        P.ttn_create(None, P.TTN_STATE, parent, phys, bond, good[:2])
