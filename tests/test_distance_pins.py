"""Pins of the A18 distance used by every parity test (tests/_helpers.stable_distances):
checked against dense vectors (Eq. 2 contracted in full), including distances far below the
~1e-8 floor of the overlap formula, and bond-gauge invariance."""
import numpy as np
import pytest

import workloads as W
from oracle import TTN, to_dense_state

from ._helpers import overlap_distances, stable_distances


def _state(parent, chi, seed, d=2):
    inst = W.configs.random_instance(parent, [d] * len(parent), chi, 1, 4, seed=seed)
    return TTN(parent, inst.state)


def _dense_pair(a, b):
    va, vb = to_dense_state(a), to_dense_state(b)
    na, nb = np.linalg.norm(va), np.linalg.norm(vb)
    return 1 - np.vdot(va, vb).real / (na * nb), np.linalg.norm(va - vb) / nb


@pytest.mark.parametrize("parent", [W.chain(5), W.complete_binary(7), [-1, 0, 0, 0, 1]])
def test_stable_distance_matches_dense(parent):
    a, b = _state(parent, 3, 1), _state(parent, 2, 2)       # different bonds on purpose
    got = stable_distances(a, b)
    ref = _dense_pair(a, b)
    assert abs(got[0] - ref[0]) <= 1e-13 and abs(got[1] - ref[1]) <= 1e-13 * ref[1]


@pytest.mark.parametrize("eps", [1e-6, 1e-10, 1e-13])
def test_stable_distance_resolves_tiny_differences(eps):
    """b = a with one tensor perturbed by eps: ||a - b|| / ||b|| is exactly eps * ||delta psi||,
    resolved to a few digits even where the overlap formula returns noise (A18)."""
    parent = W.complete_binary(7)
    a = _state(parent, 3, 5)
    rng = np.random.default_rng(9)
    delta = W.complex_gaussian(rng, a.tensors[3].shape)
    b = a.copy()
    b.tensors[3] = b.tensors[3] + eps * delta
    dpsi = a.copy()
    dpsi.tensors[3] = delta
    ref = eps * np.linalg.norm(to_dense_state(dpsi)) / np.linalg.norm(to_dense_state(b))
    got = stable_distances(b, a)[1]
    assert abs(got - ref) <= 1e-3 * ref, (got, ref)
    if eps <= 1e-10:   # the overlap formula cannot see it (documents why A18 is needed)
        assert abs(overlap_distances(b, a)[1] - ref) > 1e-3 * ref


def test_stable_distance_gauge_invariant_and_zero():
    parent = W.chain(6)
    a = _state(parent, 4, 3)
    rng = np.random.default_rng(4)
    b = a.copy()
    z = W.complex_gaussian(rng, (4, 4))
    g, _ = np.linalg.qr(z)
    # insert g g^H on edge (2, parent 1): state unchanged
    b.tensors[2] = np.tensordot(g.conj().T, b.tensors[2], axes=([1], [1])).transpose(1, 0, 2)
    b.tensors[1] = np.tensordot(b.tensors[1], g, axes=([2], [0]))
    d_cos, d_rel = stable_distances(a, b)
    assert d_cos <= 1e-15 and d_rel <= 1e-14
