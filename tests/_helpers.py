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


def distances(a: TTN, b: TTN):
    """(1 - Re<a|b>/(|a||b|), ||a-b||/||b||) via overlaps (A18)."""
    ab = overlap(a, b)
    na, nb = norm(a), norm(b)
    cos = ab.real / (na * nb)
    d2 = max(na * na + nb * nb - 2 * ab.real, 0.0)
    return 1.0 - cos, np.sqrt(d2) / nb


def eps2(phi: TTN, op: TTN, psi: TTN, opsi_norm2=None):
    if opsi_norm2 is None:
        opsi_norm2 = norm(exact_apply(op, psi)) ** 2
    return 1.0 - norm(phi) ** 2 / opsi_norm2, opsi_norm2
