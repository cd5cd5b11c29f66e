"""Shared test plumbing: build the same seeded instance for the oracle and the CUDA path,
and compare results gauge-invariantly (B:5: 1 - Re<a|b>/(|a||b|) <= 1e-10, eps^2 within 1e-10)."""
import numpy as np

import workloads as W
from oracle import TTN, cbc_apply as oracle_cbc, exact_apply, norm, overlap


def oracle_pair(inst):
    psi = TTN(inst.parent, [t.copy() for t in inst.state])
    r = psi.root
    psi.tensors[r] = psi.tensors[r] / norm(psi)
    return TTN(inst.parent, inst.op, "operator"), psi


def gpu_pair(P, ctx, inst, normalize=True):
    """Create (op, state) handles through the C ABI; the state is normalised with ttn_norm (A16)."""
    st = P.ttn_create(ctx, P.TTN_STATE, inst.parent, inst.phys, inst.state_bond, inst.state)
    if normalize:
        nrm = P.ttn_norm(ctx, st)
        tens = [t.copy() for t in inst.state]
        r = inst.parent.index(-1)
        tens[r] = tens[r] / nrm
        st.destroy()
        st = P.ttn_create(ctx, P.TTN_STATE, inst.parent, inst.phys, inst.state_bond, tens)
    op = P.ttn_create(ctx, P.TTN_OPERATOR, inst.parent, inst.phys, inst.op_bond, inst.op)
    return op, st


def to_oracle(P, h, parent):
    return TTN(list(parent), h.tensors(), "state")


def overlap_distances(a: TTN, b: TTN):
    """(1 - Re<a|b>/(|a||b|), ||a-b||/||b||) via overlaps: ||a-b|| floors near 1e-8 (A18);
    kept only to document that floor (tests/test_distance_pins.py)."""
    ab = overlap(a, b)
    na, nb = norm(a), norm(b)
    cos = ab.real / (na * nb)
    d2 = max(na * na + nb * nb - 2 * ab.real, 0.0)
    return 1.0 - cos, np.sqrt(d2) / nb


def eps2(phi: TTN, op: TTN, psi: TTN, opsi_norm2=None):
    if opsi_norm2 is None:
        opsi_norm2 = norm(exact_apply(op, psi)) ** 2
    return 1.0 - norm(phi) ** 2 / opsi_norm2, opsi_norm2


# ---------------------------------------------------------------- A18 stable distance
def _direct_sum_difference(a: TTN, b: TTN) -> TTN:
    """The TTN of a - b: every bond is the direct sum (a's block, then b's), each node tensor
    block-diagonal over (parent, children) legs; the root's extent-1 parent leg is shared, its
    b block enters with a minus sign."""
    n, root, ch = a.n, a.root, a.children
    out = []
    for i in range(n):
        ta, tb = a.tensors[i], b.tensors[i]
        if ta.shape[0] != tb.shape[0]:
            raise ValueError("physical dimensions differ")
        pa = 1 if i == root else ta.shape[1]
        pb = 0 if i == root else tb.shape[1]
        shape = (ta.shape[0], pa + pb) + tuple(ta.shape[2 + l] + tb.shape[2 + l] for l in range(len(ch[i])))
        t = np.zeros(shape, dtype=np.complex128)
        sa = (slice(None), slice(0, pa)) + tuple(slice(0, ta.shape[2 + l]) for l in range(len(ch[i])))
        sb = (slice(None), slice(0, 1) if i == root else slice(pa, pa + pb)) + \
            tuple(slice(ta.shape[2 + l], None) for l in range(len(ch[i])))
        t[sa] = ta
        t[sb] += -tb if i == root else tb
        out.append(t)
    return TTN(list(a.parent), out)


def canonical_norm(x: TTN) -> float:
    """||x|| by Householder QR toward the root (leaves first; each R is absorbed into the
    parent), then the Frobenius norm of the root: backward stable, absolute error ~1e-16 ||x||
    (the overlap formula loses half the digits of a small distance, A18)."""
    T = [t.copy() for t in x.tensors]
    for i in x.post_order():
        p = x.parent[i]
        if p < 0:
            continue
        m = np.moveaxis(T[i], 1, -1)
        shp = m.shape
        q, r = np.linalg.qr(m.reshape(-1, shp[-1]), mode="reduced")
        T[i] = None
        leg = 2 + x.children[p].index(i)
        T[p] = np.moveaxis(np.tensordot(r, T[p], axes=([1], [leg])), 0, leg)
    return float(np.linalg.norm(T[x.root]))


def stable_distances(a: TTN, b: TTN):
    """A18: (1 - Re<a|b>/(|a||b|), ||a - b|| / ||b||) from the QR-canonicalised
    direct-sum difference TTN, so distances far below 1e-8 are resolved."""
    na, nb = canonical_norm(a), canonical_norm(b)
    dn = canonical_norm(_direct_sum_difference(a, b))
    d_cos = max(dn * dn - (na - nb) ** 2, 0.0) / (2.0 * na * nb)
    return d_cos, dn / nb


# every parity test uses the stable form (A18)
distances = stable_distances
