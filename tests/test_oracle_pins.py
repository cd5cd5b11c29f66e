"""Pins for the CPU oracle (P1-P13): checks against the paper's definitions,
brute force, closed forms and invariants — never against the oracle's own formulas."""
import itertools
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import (TTN, cbc_apply, cbc_apply_tt, direct_apply, exact_apply, gram_compress, norm,
                    overlap, sandwich, to_dense_operator, to_dense_state)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _inst(parent, d=2, chi=3, D=2, seed=0, phys=None):
    phys = phys or [d] * len(parent)
    inst = W.configs.random_instance(parent, phys, chi, D, 10**6, seed=seed)
    psi = TTN(inst.parent, inst.state)
    psi.tensors[psi.root] = psi.tensors[psi.root] / norm(psi)
    return TTN(inst.parent, inst.op, "operator"), psi


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- dense brute force
def _brute_state(parent, tensors):
    """Eq. 2 by explicit loops over every index assignment."""
    n = len(parent)
    ch = W.children_of(parent)
    d = [t.shape[0] for t in tensors]
    bond = [1 if parent[i] < 0 else tensors[i].shape[1] for i in range(n)]
    out = np.zeros(int(np.prod(d)), dtype=complex)
    for sig in itertools.product(*[range(x) for x in d]):
        acc = 0j
        for al in itertools.product(*[range(b) for b in bond]):
            prod = 1 + 0j
            for i in range(n):
                idx = (sig[i], al[i] if parent[i] >= 0 else 0) + tuple(al[c] for c in ch[i])
                prod *= tensors[i][idx]
            acc += prod
        out[np.ravel_multi_index(sig, d)] = acc
    return out


TINY_TREES = [W.chain(3), [-1, 0, 0], [-1, 0, 1, 1], W.complete_binary(5)]


@pytest.mark.parametrize("parent", TINY_TREES)
def test_dense_state_matches_definition(parent):
    _, psi = _inst(parent, chi=2, D=2, seed=3)
    assert _rel(to_dense_state(psi), _brute_state(parent, psi.tensors)) < 1e-13


@pytest.mark.parametrize("parent", TINY_TREES)
def test_dense_operator_matches_definition(parent):
    op, psi = _inst(parent, chi=2, D=2, seed=4)
    # operator element <s'|O|s> from Eq. 4: treat (s', s) as one physical index with the loop oracle
    d = [t.shape[0] for t in op.tensors]
    flat = [t.reshape((t.shape[0] * t.shape[1],) + t.shape[2:]) for t in op.tensors]
    vec = _brute_state(parent, flat).reshape(sum(([x, x] for x in d), []))
    n = len(parent)
    mat = vec.transpose([2 * i for i in range(n)] + [2 * i + 1 for i in range(n)]).reshape(int(np.prod(d)), -1)
    assert _rel(to_dense_operator(op), mat) < 1e-13


def test_overlap_and_exact_apply_match_dense():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=5)
    _, psi2 = _inst(W.complete_binary(7), chi=2, D=2, seed=6)
    v, v2, M = to_dense_state(psi), to_dense_state(psi2), to_dense_operator(op)
    assert abs(overlap(psi2, psi) - np.vdot(v2, v)) < 1e-13 * np.linalg.norm(v) * np.linalg.norm(v2)
    assert _rel(to_dense_state(exact_apply(op, psi)), M @ v) < 1e-13
    assert abs(sandwich(psi2, op, psi) - np.vdot(v2, M @ v)) < 1e-12 * np.linalg.norm(M @ v)


# ---------------------------------------------------------------- P1 untruncated exactness
P1_TREES = [
    ("cfg1", W.chain(6), 4, 3, 12),
    ("binary7", W.complete_binary(7), 3, 2, 64),
    ("star7", W.star_of_chains_literal(6, 1), 2, 2, 64),
    ("ttree", W.t_tree(2), 3, 2, 64),
    ("ftps", W.ftps(2), 2, 2, 64),
]


@pytest.mark.parametrize("name,parent,chi,D,mb", P1_TREES)
def test_P1_untruncated_equals_dense(name, parent, chi, D, mb):
    op, psi = _inst(parent, chi=chi, D=D, seed=11)
    phi = cbc_apply(op, psi, mb)
    ex = to_dense_operator(op) @ to_dense_state(psi)
    assert _rel(to_dense_state(phi), ex) < 1e-12


def test_P1_config1_exact_bonds():
    inst = W.make_config(1)
    psi = TTN(inst.parent, inst.state)
    psi.tensors[0] /= norm(psi)
    op = TTN(inst.parent, inst.op, "operator")
    phi = cbc_apply(op, psi, 12)
    assert phi.bonds() == [1, 2, 4, 8, 4, 2]
    assert _rel(to_dense_state(phi), to_dense_operator(op) @ to_dense_state(psi)) < 1e-12


# ---------------------------------------------------------------- P2 / P3 / P4 invariants
TRUNC = [("cfg1_mb6", W.chain(6), 4, 3, 6), ("binary15", W.complete_binary(15), 4, 3, 5),
         ("ttree", W.t_tree(3), 4, 3, 4), ("chain12", W.chain(12), 8, 4, 10)]


@pytest.mark.parametrize("name,parent,chi,D,mb", TRUNC)
def test_P2_projection_identity(name, parent, chi, D, mb):
    op, psi = _inst(parent, chi=chi, D=D, seed=21)
    phi = cbc_apply(op, psi, mb)
    n2 = norm(phi) ** 2
    val = sandwich(phi, op, psi)
    assert abs(val - n2) <= 1e-12 * n2


@pytest.mark.parametrize("name,parent,chi,D,mb", TRUNC)
def test_P3_isometry(name, parent, chi, D, mb):
    op, psi = _inst(parent, chi=chi, D=D, seed=22)
    phi = cbc_apply(op, psi, mb)
    for i, t in enumerate(phi.tensors):
        if i == phi.root:
            continue
        q = np.moveaxis(t, 1, -1).reshape(-1, t.shape[1])
        assert np.linalg.norm(q.conj().T @ q - np.eye(q.shape[1])) <= 1e-12
    assert max(phi.bonds()) <= mb
    assert abs(np.linalg.norm(phi.tensors[phi.root]) - norm(phi)) < 1e-12 * norm(phi)


def test_P4_factor_reconstructs_gram_untruncated():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=23)
    rec = {}
    cbc_apply(op, psi, 64, record=rec)
    assert rec["compress"]
    for c in rec["compress"]:
        x, f = c["x"], c["f"]
        g = x.conj().T @ x
        assert np.linalg.norm(f.conj().T @ f - g) <= 1e-12 * np.linalg.norm(g)
        assert c["w"] <= 1e-24 * np.linalg.norm(g)


# ---------------------------------------------------------------- P5 Eckart-Young bound
def _bipartition_sv(vec, parent, c):
    """Singular values of the dense vector split into subtree(c) vs the rest."""
    n = len(parent)
    sub = {c}
    changed = True
    while changed:
        changed = False
        for i in range(n):
            if parent[i] in sub and i not in sub:
                sub.add(i)
                changed = True
    a = sorted(sub)
    b = [i for i in range(n) if i not in sub]
    t = vec.reshape([2] * n).transpose(a + b).reshape(2 ** len(a), -1)
    return np.linalg.svd(t, compute_uv=False)


@pytest.mark.parametrize("seed", range(6))
def test_P5_eckart_young_lower_bound(seed):
    parent = W.chain(6) if seed % 2 == 0 else W.complete_binary(7)
    mb = 6 if seed % 2 == 0 else 3
    op, psi = _inst(parent, chi=4, D=3, seed=100 + seed)
    ex = to_dense_operator(op) @ to_dense_state(psi)
    phi = cbc_apply(op, psi, mb)
    eps = np.linalg.norm(to_dense_state(phi) - ex) / np.linalg.norm(ex)
    ey = 0.0
    for c in range(1, len(parent)):
        s = _bipartition_sv(ex, parent, c)
        ey = max(ey, np.sqrt(np.sum(s[mb:] ** 2)) / np.linalg.norm(ex))
    assert eps >= ey * (1 - 1e-12)
    assert eps > 0


# ---------------------------------------------------------------- P6 exact truncated special case
def _root_canonical(psi):
    T = [t.copy() for t in psi.tensors]
    ch = psi.children
    for i in psi.post_order():
        p = psi.parent[i]
        if p < 0:
            continue
        m = np.moveaxis(T[i], 1, -1)
        shp = m.shape
        q, r = np.linalg.qr(m.reshape(-1, shp[-1]))
        T[i] = np.moveaxis(q.reshape(shp[:-1] + (q.shape[1],)), -1, 1)
        leg = 2 + ch[p].index(i)
        T[p] = np.moveaxis(np.tensordot(r, T[p], axes=([1], [leg])), 0, leg)
    return TTN(psi.parent, T)


def test_P6_identity_op_single_overbudget_bond():
    parent = W.chain(4)
    _, psi = _inst(parent, chi=4, D=1, seed=31)
    psi = _root_canonical(psi)
    op = TTN(parent, W.identity_operator(parent, [2] * 4), "operator")
    v = to_dense_state(psi)
    phi = cbc_apply(op, psi, 3)
    eps2 = np.linalg.norm(to_dense_state(phi) - v) ** 2 / np.linalg.norm(v) ** 2
    s = _bipartition_sv(v, parent, 2)          # the middle bond (rank 4 > 3)
    ey2 = np.sum(s[3:] ** 2) / np.sum(s ** 2)
    assert ey2 > 1e-6
    assert abs(eps2 - ey2) <= 1e-12


# ---------------------------------------------------------------- P7 / P8 gauge invariances
def _haar(rng, n):
    z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def test_P7_bond_gauge_invariance():
    parent = W.complete_binary(7)
    op, psi = _inst(parent, chi=3, D=2, seed=41)
    rng = np.random.default_rng(7)
    T = [t.copy() for t in psi.tensors]
    O = [t.copy() for t in op.tensors]
    ch = psi.children
    for c in range(1, 7):
        p = parent[c]
        for arrs, off in ((T, 1), (O, 2)):
            u = _haar(rng, arrs[c].shape[off])
            arrs[c] = np.moveaxis(np.tensordot(arrs[c], u, axes=([off], [0])), -1, off)
            leg = off + 1 + ch[p].index(c)
            arrs[p] = np.moveaxis(np.tensordot(arrs[p], u.conj(), axes=([leg], [0])), -1, leg)
    for mb in (64, 3):
        a = to_dense_state(cbc_apply(op, psi, mb))
        b = to_dense_state(cbc_apply(TTN(parent, O, "operator"), TTN(parent, T), mb))
        assert _rel(b, a) < 1e-12


def test_P8_factor_gauge_invariance():
    parent = W.complete_binary(7)
    op, psi = _inst(parent, chi=3, D=2, seed=42)
    rng = np.random.default_rng(8)

    def hook(kind, node, f):
        return np.tensordot(_haar(rng, f.shape[0]), f, axes=([1], [0]))

    for mb in (64, 3):
        a = to_dense_state(cbc_apply(op, psi, mb))
        b = to_dense_state(cbc_apply(op, psi, mb, factor_hook=hook))
        assert _rel(b, a) < 1e-12


def test_P8_zero_padding_of_factors_is_exact():
    parent = W.complete_binary(7)
    op, psi = _inst(parent, chi=3, D=2, seed=43)

    def pad(kind, node, f):   # up-factors only: a padded DOWN factor widens the Eq. 13 QR
        if kind != "up":
            return f
        return np.concatenate([f, np.zeros((2,) + f.shape[1:], dtype=f.dtype)], axis=0)

    a = to_dense_state(cbc_apply(op, psi, 3))
    b = to_dense_state(cbc_apply(op, psi, 3, factor_hook=pad))
    assert _rel(b, a) < 1e-12


# ---------------------------------------------------------------- P9 compress routes
@pytest.mark.parametrize("mb", [64, 4])
def test_P9_gram_route_equals_svd_route(mb):
    op, psi = _inst(W.complete_binary(15), chi=4, D=3, seed=51)
    a = cbc_apply(op, psi, mb)
    b = cbc_apply(op, psi, mb, compress=gram_compress)
    assert a.bonds() == b.bonds()
    assert _rel(to_dense_state(b), to_dense_state(a)) < 1e-10


# ---------------------------------------------------------------- P10 direct method
def test_P10_direct_untruncated_agrees():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=61)
    a = to_dense_state(cbc_apply(op, psi, 64))
    b = to_dense_state(direct_apply(op, psi, 64))
    assert _rel(a, b) < 1e-12


def test_P10_direct_truncated_ratio():
    ratios = []
    for seed in range(10):
        parent = W.chain(6) if seed % 2 else W.complete_binary(7)
        mb = 5 if seed % 2 else 3
        op, psi = _inst(parent, chi=4, D=3, seed=200 + seed)
        ex = to_dense_operator(op) @ to_dense_state(psi)
        ec = _rel(to_dense_state(cbc_apply(op, psi, mb)), ex)
        ed = _rel(to_dense_state(direct_apply(op, psi, mb)), ex)
        ratios.append(ec / ed)
        assert ec / ed <= 3.0
    assert 1.0 <= np.mean(ratios) <= 3.0


# ---------------------------------------------------------------- P11 appendix A, chain reduction
def test_P11_appendix_a_shapes():
    g = json.load(open(os.path.join(GOLD, "appendix_a_l4.json")))
    op, psi = _inst(W.chain(g["L"]), d=g["d"], chi=g["chi"], D=g["D"], seed=71)
    rec = {}
    tt = cbc_apply_tt(op, psi, g["max_bond"], record=rec)
    assert [k for (_, k) in rec["left"]] == g["left_k"]
    assert [list(s[0]) for s in rec["right"]] == g["right_S_shapes"]
    assert [s[1] for s in rec["right"] if len(s) > 1] == g["right_r"]
    assert tt.bonds() == g["bonds"]
    tree = cbc_apply(op, psi, g["max_bond"])
    assert tree.bonds() == g["bonds"]


@pytest.mark.parametrize("n,chi,D,mb", [(6, 4, 3, 6), (8, 6, 3, 9), (5, 3, 2, 64)])
def test_P11_chain_reduction_tree_equals_tt(n, chi, D, mb):
    op, psi = _inst(W.chain(n), chi=chi, D=D, seed=72)
    a = cbc_apply(op, psi, mb)
    b = cbc_apply_tt(op, psi, mb)
    assert a.bonds() == b.bonds()
    assert _rel(to_dense_state(a), to_dense_state(b)) < 1e-12


# ---------------------------------------------------------------- P12 scale covariance, identity
def test_P12_scale_covariance():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=81)
    a = to_dense_state(cbc_apply(op, psi, 3))
    op2 = TTN(op.parent, [t * (2.0 ** 3) if i == 2 else t for i, t in enumerate(op.tensors)], "operator")
    psi2 = TTN(psi.parent, [t * (2.0 ** -5) if i == 4 else t for i, t in enumerate(psi.tensors)])
    b = to_dense_state(cbc_apply(op2, psi2, 3))
    assert _rel(b, a * 2.0 ** -2) < 1e-13


def test_P12_identity_operator_returns_state():
    parent = W.complete_binary(15)
    _, psi = _inst(parent, chi=3, D=1, seed=82)
    op = TTN(parent, W.identity_operator(parent, [2] * 15), "operator")
    phi = cbc_apply(op, psi, 64)
    assert _rel(to_dense_state(phi), to_dense_state(psi)) < 1e-12


# ---------------------------------------------------------------- A20 zero input, errors
def test_A20_zero_state_gives_zero_bond_one():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=91)
    z = TTN(psi.parent, [t * 0 for t in psi.tensors])
    phi = cbc_apply(op, z, 4)
    assert phi.bonds() == [1] * 7
    assert np.linalg.norm(phi.tensors[0]) == 0.0


def test_errors():
    op, psi = _inst(W.complete_binary(7), chi=3, D=2, seed=92)
    with pytest.raises(ValueError):
        cbc_apply(TTN(W.chain(7), [np.zeros((2, 2, 1, 1))] + [np.zeros((2, 2, 1, 1))] * 5
                      + [np.zeros((2, 2, 1))], "operator"), psi, 4)
    with pytest.raises(ValueError):
        cbc_apply(op, psi, 0)
    with pytest.raises(ValueError):
        TTN([-1, 0], [np.zeros((2, 1, 3)), np.zeros((2, 2))])


# ---------------------------------------------------------------- P13 unitary circuit layers
def _apply_gate_dense(v, n, c, p, g):
    t = v.reshape([2] * n)
    t = np.moveaxis(t, [c, p], [0, 1])
    sh = t.shape
    t = (g @ t.reshape(4, -1)).reshape(sh)
    return np.moveaxis(t, [0, 1], [c, p]).reshape(-1)


def test_P13_circuit_layers_match_statevector():
    parent = W.complete_binary(15)
    n = 15
    psi = TTN(parent, W.product_zero_state(parent, [2] * n))
    v = to_dense_state(psi)
    assert v[0] == 1.0
    for layer in range(4):
        ops, bond, gates = W.circuit_layer_operator(parent, seed=3, layer=layer)
        opn = TTN(parent, ops, "operator")
        for c, p, g in gates:
            assert np.linalg.norm(g.conj().T @ g - np.eye(4)) < 1e-12
            v = _apply_gate_dense(v, n, c, p, g)
        # A15: the SVD-split layer TTNO equals dense gate application
        assert _rel(to_dense_state(exact_apply(opn, psi)), _apply_gate_dense_all(to_dense_state(psi), n, gates)) < 1e-12
        psi = cbc_apply(opn, psi, 256)
        assert abs(norm(psi) - 1.0) < 1e-12
        assert _rel(to_dense_state(psi), v) < 1e-12


def _apply_gate_dense_all(v, n, gates):
    for c, p, g in gates:
        v = _apply_gate_dense(v, n, c, p, g)
    return v


def test_A15_layer_operator_dense_matrix():
    parent = W.complete_binary(7)
    for layer in range(3):
        ops, bond, gates = W.circuit_layer_operator(parent, seed=5, layer=layer)
        m = to_dense_operator(TTN(parent, ops, "operator"))
        ref = np.eye(128, dtype=complex)
        for j in range(128):
            ref[:, j] = _apply_gate_dense_all(ref[:, j].copy(), 7, gates)
        assert len(gates) >= 1
        assert np.linalg.norm(m - ref) < 1e-12 * np.linalg.norm(ref)


# ---------------------------------------------------------------- A3 tol branch (reading A3)
def _schmidt_pair(s, seed):
    """Two-site chain (d = 4 each, root = site 0) whose only bond has Schmidt values s:
    root T0[sigma, 1, a] = (U diag(s))[sigma, a], leaf T1[sigma, a] = V[sigma, a]^T with U, V
    unitary, so the leaf is already an isometry toward the root (root-canonical form)."""
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(W.complex_gaussian(rng, (4, 4)))
    v, _ = np.linalg.qr(W.complex_gaussian(rng, (4, 4)))
    t0 = (u * np.asarray(s)[None, :])[:, None, :]
    t1 = np.ascontiguousarray(v.T)
    return TTN([-1, 0], [t0, t1])


@pytest.mark.parametrize("tol,max_bond,k", [(0.45, 4, 2), (0.25, 4, 3), (0.05, 4, 4), (0.25, 2, 2),
                                            (0.95, 4, 1), (0.0, 3, 3)])
def test_A3_tol_keeps_sigma_above_tol_sigma1(tol, max_bond, k):
    """Reading A3 ("setting a tolerance for the SVD"): keep min(max_bond, #{sigma_j >
    tol sigma_1}).  The spectrum s = (1, .6, .3, .1) separates the readings: sigma > tol sigma_1
    (A3), sigma^2 > tol sigma_1^2 and sigma > tol^2 sigma_1 give different bonds at tol = 0.45
    (2, 1, 3) and 0.25 (3, 2, 3).  Identity TTNO on a root-canonical state: the result is the
    dense truncated SVD, so the bond and eps^2 = dropped tail / total are fixed by the
    spectrum alone (Eckart-Young, as in P6)."""
    s = np.array([1.0, 0.6, 0.3, 0.1])
    psi = _schmidt_pair(s, seed=17)
    op = TTN([-1, 0], W.identity_operator([-1, 0], [4, 4]), "operator")
    rec = {}
    phi = cbc_apply(op, psi, max_bond, tol, record=rec)
    assert phi.bonds() == [1, k]
    v, w = to_dense_state(psi), to_dense_state(phi)
    eps2 = np.linalg.norm(w - v) ** 2 / np.linalg.norm(v) ** 2
    tail = np.sum(s[k:] ** 2) / np.sum(s ** 2)
    assert abs(eps2 - tail) <= 1e-13
    # the one compress (down factor of the leaf) reports the dropped weight sum_{j>k} s_j^2
    assert len(rec["discarded"]) == 1
    assert abs(rec["discarded"][0] - np.sum(s[k:] ** 2)) <= 1e-13
    # the tensor-train oracle (Eqs. 5-9, written separately) takes the same decision
    phi_tt = cbc_apply_tt(op, psi, max_bond, tol)
    assert phi_tt.bonds() == [1, k]
    assert np.linalg.norm(to_dense_state(phi_tt) - w) <= 1e-13


def test_A3_tol_on_a_tree_matches_per_bond_dense_svd():
    """tol on a 3-node star whose two bonds have prescribed spectra (root-canonical leaves):
    each bond keeps #{sigma > tol sigma_1} of ITS spectrum, eps^2 is the dense projection error."""
    rng = np.random.default_rng(23)
    s1, s2 = np.array([1.0, 0.5, 0.2, 0.05]), np.array([1.0, 0.8, 0.08, 0.01])
    # root core T0[s, 1, a, b] = u[s, (a, b)] s1[a] s2[b] with u unitary: the spectrum of
    # bond a is s1 (times a constant), of bond b is s2
    core = np.zeros((16, 4, 4), dtype=np.complex128)
    u, _ = np.linalg.qr(W.complex_gaussian(rng, (16, 16)))
    for a in range(4):
        for b in range(4):
            core[:, a, b] = u[:, 4 * a + b] * s1[a] * s2[b]
    va, _ = np.linalg.qr(W.complex_gaussian(rng, (4, 4)))
    vb, _ = np.linalg.qr(W.complex_gaussian(rng, (4, 4)))
    psi = TTN([-1, 0, 0], [core[:, None], np.ascontiguousarray(va.T), np.ascontiguousarray(vb.T)])
    op = TTN([-1, 0, 0], W.identity_operator([-1, 0, 0], [16, 4, 4]), "operator")
    tol = 0.3
    phi = cbc_apply(op, psi, 16, tol)
    k1, k2 = int(np.sum(s1 > tol)), int(np.sum(s2 > tol))
    assert phi.bonds() == [1, k1, k2] == [1, 2, 2]
    v, w = to_dense_state(psi), to_dense_state(phi)
    # product spectrum: the kept state is the (k1 x k2) block of s1 s2^T
    kept = np.sum(np.outer(s1[:k1] ** 2, s2[:k2] ** 2))
    assert abs(np.linalg.norm(w - v) ** 2 / np.linalg.norm(v) ** 2 - (1 - kept / np.sum(np.outer(s1 ** 2, s2 ** 2)))) <= 1e-13
