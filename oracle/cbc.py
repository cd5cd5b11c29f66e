"""Tree CBC, step by step in the paper's order (oracle; test infrastructure only).

PAPER.md §III.B, P:163-200:
  1. up-sweep   (Eq. 10): for every non-root site i, leaves to root,
       L'^{[i]}[sigma', chi_c..., a0, b0] = sum T^{[i]} O^{[i]} prod_{c in C_i} L^{[c]}
     join (sigma', chi_c...) and compress it -> L^{[i]}[chi_i, a0, b0]
  2. down-sweep (Eq. 11): root to leaves, for every k in C_i,
       L'^{[(i,k)]} = sum T O L^{[(p_i,i)]} prod_{c in C_i \\ k} L^{[c]}, compress
     (the root uses the trivial factor L^{[(-,r)]} = 1, extent-1 legs).
  3. final sweep, leaves to root (Eqs. 12-14):
       S^{[i]} = sum T O L^{[(p_i,i)]} prod_c R^{[c]}                        Eq. 12
       root: T'^{[r]} = S^{[r]}; else S = Q R on the parent leg, T'^{[i]} = Q  Eq. 13
       R^{[i]} = sum T O Q* prod_c R^{[c]}                                   Eq. 14
  4. assembly.

Readings: compress = truncated SVD, factor = Sigma_k V_k^H (A2);
k = min(max_bond, #{s_j > tol*s_1}, #{s_j > 1e-14*s_1}), k >= 1 (A3, A4); Eq. 13's QR
splits off the parent leg and keeps r = min(m_S, kd) columns, diag(R) >= 0 (A5); Eq. 14
uses Q* like Eq. 8 (A6); up-factors that are never read are skipped (A9).  Eq. 12 and
Eq. 14 are evaluated through Z_i = sum T O prod_c R^{[c]} (the partial result the
appendix says to reuse): S = Z L^{[(p_i,i)]T}, R^{[i]} = Q^H Z.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional

import numpy as np

from .ttn import TTN

SV_FLOOR = 1e-14   # A4: numerical-rank floor relative to the largest singular value


def phi(t: np.ndarray, o: np.ndarray, factors: Dict[int, np.ndarray], open_leg: int) -> np.ndarray:
    """Contract a site's state and operator tensor with one factor F[f, a_l, b_l] on every
    virtual leg l in `factors`; the remaining leg `open_leg` stays open.

    Returns the matrix with rows (sigma', f_l for l ascending) and columns (a_o, b_o).
    Fixed order: T absorbs each factor in leg order, then the operator (tensordot only).
    """
    nv = t.ndim - 1
    assert set(factors) | {open_leg} == set(range(nv)) and open_leg not in factors
    a = t
    labels = ["s"] + [("a", l) for l in range(nv)]
    for l in sorted(factors):
        f = factors[l]
        ax = labels.index(("a", l))
        a = np.tensordot(a, f, axes=([ax], [1]))            # appends f_l, b_l
        labels = labels[:ax] + labels[ax + 1:] + [("f", l), ("b", l)]
    olabels = ["sp", "s"] + [("b", l) for l in range(nv)]
    cl = ["s"] + [("b", l) for l in sorted(factors)]
    a = np.tensordot(a, o, axes=([labels.index(x) for x in cl], [olabels.index(x) for x in cl]))
    labels = [x for x in labels if x not in cl] + [x for x in olabels if x not in cl]
    want = ["sp"] + [("f", l) for l in sorted(factors)] + [("a", open_leg), ("b", open_leg)]
    a = a.transpose([labels.index(x) for x in want])
    m = int(np.prod(a.shape[: 1 + len(factors)]))
    return a.reshape(m, -1)


def _keep(s: np.ndarray, max_bond: int, tol: float, floor: float) -> int:
    if s.size == 0 or s[0] <= 0.0:
        return 1
    k = min(max_bond, int(np.sum(s > tol * s[0])), int(np.sum(s > floor * s[0])))
    return max(k, 1)


def svd_compress(x: np.ndarray, max_bond: int, tol: float):
    """Truncated SVD: X = U S V^H; keep k; factor F = S_k V_k^H (k x n).
    The isometry U is dropped, as the paper says it cancels later."""
    u, s, vh = np.linalg.svd(x, full_matrices=False)
    k = _keep(s, max_bond, tol, SV_FLOOR)
    if s.size == 0 or s[0] <= 0.0:
        return np.zeros((1, x.shape[1]), dtype=np.complex128), {"k": 1, "w": 0.0, "s": s}
    f = s[:k, None] * vh[:k]
    return f, {"k": k, "w": float(np.sum(s[k:] ** 2)), "s": s}


def gram_compress(x: np.ndarray, max_bond: int, tol: float, floor: float = 1e-13):
    """Gram-route compress (used only by pin P9): eigendecomposition of X^H X (m >= n)
    or X X^H (m < n); same kept subspace as svd_compress, factor equal up to a unitary."""
    m, n = x.shape
    if m >= n:
        lam, v = np.linalg.eigh(x.conj().T @ x)
    else:
        lam, v = np.linalg.eigh(x @ x.conj().T)
    lam, v = lam[::-1], v[:, ::-1]
    lam = np.maximum(lam, 0.0)
    if lam.size == 0 or lam[0] <= 0.0:
        return np.zeros((1, n), dtype=np.complex128), {"k": 1, "w": 0.0, "s": np.sqrt(lam)}
    k = min(max_bond, int(np.sum(lam > tol * tol * lam[0])), int(np.sum(lam > floor * lam[0])))
    k = max(k, 1)
    if m >= n:
        f = np.sqrt(lam[:k])[:, None] * v[:, :k].conj().T
    else:
        f = v[:, :k].conj().T @ x
    return f, {"k": k, "w": float(np.sum(lam[k:])), "s": np.sqrt(lam)}


def qr_pos(s: np.ndarray):
    """Reduced Householder QR with a real non-negative diagonal of R."""
    q, r = np.linalg.qr(s, mode="reduced")
    d = np.diag(r)
    ph = np.where(np.abs(d) > 0, d / np.where(np.abs(d) > 0, np.abs(d), 1.0), 1.0)
    return q * ph[None, :], np.conj(ph)[:, None] * r


def used_up_factors(psi: TTN) -> List[bool]:
    """A9: L^{[c]} is read by the parent's down-sweep when c has a sibling, or by the
    parent's own up-sweep when that one is read.  Others are skipped."""
    used = [False] * psi.n
    for i in psi.pre_order():
        p = psi.parent[i]
        if p < 0:
            continue
        used[i] = len(psi.children[p]) >= 2 or used[p]
    return used


def cbc_apply(op: TTN, psi: TTN, max_bond: int, tol: float = 0.0, *,
              compress: Callable = svd_compress,
              factor_hook: Optional[Callable] = None,
              record: Optional[dict] = None) -> TTN:
    """CBC of O|psi>.  `factor_hook(kind, node, F) -> F'` may replace an
    environment factor (pin P8); `record` collects per-step data for the pins."""
    if op.parent != psi.parent:
        raise ValueError("topology mismatch")
    if op.phys() != psi.phys() or [t.shape[1] for t in op.tensors] != psi.phys():
        raise ValueError("leg mismatch: physical dimensions")
    if max_bond < 1 or not (0.0 <= tol < 1.0):
        raise ValueError("bad truncation arguments")
    n, root, ch, par = psi.n, psi.root, psi.children, psi.parent
    T, O = psi.tensors, op.tensors
    rec = record if record is not None else {}
    rec.setdefault("compress", [])
    rec.setdefault("qr", [])
    used = used_up_factors(psi)
    hook = factor_hook or (lambda kind, node, f: f)

    # 1. up-sweep, Eq. 10
    up: Dict[int, np.ndarray] = {}
    for i in psi.post_order():
        if i == root or not used[i]:
            continue
        x = phi(T[i], O[i], {1 + l: up[c] for l, c in enumerate(ch[i])}, 0)
        f, info = compress(x, max_bond, tol)
        a0, b0 = T[i].shape[1], O[i].shape[2]
        up[i] = hook("up", i, f.reshape(f.shape[0], a0, b0))
        rec["compress"].append(dict(kind="up", node=i, x=x if record is not None else None, f=f, **info))

    # 2. down-sweep, Eq. 11
    down: Dict[int, np.ndarray] = {root: np.ones((1, 1, 1), dtype=np.complex128)}
    for i in psi.pre_order():
        for lk, k in enumerate(ch[i]):
            facs = {0: down[i]}
            for l, c in enumerate(ch[i]):
                if c != k:
                    facs[1 + l] = up[c]
            y = phi(T[i], O[i], facs, 1 + lk)
            f, info = compress(y, max_bond, tol)
            down[k] = hook("down", k, f.reshape(f.shape[0], T[k].shape[1], O[k].shape[2]))
            rec["compress"].append(dict(kind="down", node=k, x=y if record is not None else None, f=f, **info))

    # 3. final sweep, Eqs. 12-14, and 4. assembly
    R: Dict[int, np.ndarray] = {}
    new: List[Optional[np.ndarray]] = [None] * n
    for i in psi.post_order():
        z = phi(T[i], O[i], {1 + l: R[c] for l, c in enumerate(ch[i])}, 0)
        d = O[i].shape[0]
        rc = tuple(R[c].shape[0] for c in ch[i])
        if i == root:
            new[i] = np.ascontiguousarray(z.reshape((d,) + rc)[:, None, ...])
            rec["root_z"] = z
            continue
        fd = down[i]
        s = z @ fd.reshape(fd.shape[0], -1).T                  # Eq. 12 via Z
        q, r = qr_pos(s)                                        # Eq. 13, parent leg split off
        ri = q.shape[1]
        new[i] = np.ascontiguousarray(np.moveaxis(q.reshape((d,) + rc + (ri,)), -1, 1))
        R[i] = (q.conj().T @ z).reshape(ri, T[i].shape[1], O[i].shape[2])   # Eq. 14 with Q*
        if record is not None:
            rec["qr"].append(dict(node=i, s=s, q=q, r=r))
    out = TTN(list(psi.parent), new, "state")
    rec["bonds"] = out.bonds()
    rec["discarded"] = [c["w"] for c in rec["compress"]]
    rec["norm"] = float(np.linalg.norm(new[root]))
    return out
