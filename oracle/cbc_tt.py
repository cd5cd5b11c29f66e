"""Tensor-train CBC, Eqs. 5-9 of PAPER.md §III.A — oracle, test infrastructure.

Written directly in the MPS notation of Eq. 3: site i = 1..L carries
T^{[i]}[sigma, alpha_{i-1}, alpha_i] and W^{[i]}[sigma', sigma, beta_{i-1}, beta_i] with
trivial boundary legs alpha_0 = alpha_L = 1 (legs are named, not positional: A7).
  left sweep  (Eq. 5):  L'^{[i]}[chi_{i-1}, sigma', alpha_i, beta_i]
                           = sum L^{[i-1]} W^{[i]} T^{[i]},  L^{[0]} = 1;
                        fuse (chi_{i-1}, sigma'), compress -> L^{[i]}, for i = 1..L-1
  right sweep (Eq. 6):  S^{[i]}[sigma', chi_{i-1}, chi_i] = sum L^{[i-1]} W T R^{[i]}, R^{[L]} = 1
              (Eq. 7):  S = R Q on leg chi_{i-1}; T'^{[i]} = Q   (i > 1)
              (Eq. 8):  R^{[i-1]} = sum Q* T W R^{[i]}
              (Eq. 9):  T'^{[1]} = S^{[1]}  ("if i = 0" read as the first site, A7)
This is an implementation independent of oracle.cbc (used by pin P11: chain reduction).
"""
from __future__ import annotations

import numpy as np

from .cbc import qr_pos, svd_compress
from .ttn import TTN


def cbc_apply_tt(op: TTN, psi: TTN, max_bond: int, tol: float = 0.0, record=None) -> TTN:
    L = psi.n
    assert psi.parent == [-1] + list(range(L - 1)), "chain rooted at site 0 expected"
    # ABI chain tensors -> MPS site tensors with explicit trivial right boundary leg
    T = [t if t.ndim == 3 else t[:, :, None] for t in psi.tensors]
    W = [w if w.ndim == 4 else w[:, :, :, None] for w in op.tensors]
    Ls = [np.ones((1, 1, 1), dtype=np.complex128)]                     # L^{[0]} = 1
    shapes = {"left": [], "right": []}
    for i in range(L - 1):
        # Eq. 5: sum_{sigma, alpha_{i-1}, beta_{i-1}} L[chi, a', b'] W[s', s, b', b] T[s, a', a]
        lw = np.tensordot(Ls[-1], W[i], axes=([2], [2]))                # [chi, a', s', s, b]
        lwt = np.tensordot(lw, T[i], axes=([1, 3], [1, 0]))             # [chi, s', b, a]
        lp = lwt.transpose(0, 1, 3, 2)                                   # [chi, s', a_i, b_i]
        x = lp.reshape(lp.shape[0] * lp.shape[1], -1)                    # fuse (chi_{i-1}, s')
        f, info = svd_compress(x, max_bond, tol)
        Ls.append(f.reshape(f.shape[0], lp.shape[2], lp.shape[3]))
        shapes["left"].append((x.shape, f.shape[0]))
    R = np.ones((1, 1, 1), dtype=np.complex128)                          # R^{[L]} = 1
    new = [None] * L
    for i in range(L - 1, -1, -1):
        # Eq. 6: S[s', chi_{i-1}, chi_i] = sum L[chi_{i-1}, a', b'] W[s', s, b', b] T[s, a', a] R[chi_i, a, b]
        lw = np.tensordot(Ls[i], W[i], axes=([2], [2]))                 # [chi', a', s', s, b]
        lwt = np.tensordot(lw, T[i], axes=([1, 3], [1, 0]))             # [chi', s', b, a]
        s = np.tensordot(lwt, R, axes=([3, 2], [1, 2]))                 # [chi', s', chi]
        s = s.transpose(1, 0, 2)                                         # [s', chi_{i-1}, chi_i]
        if i == 0:
            new[0] = s                                                   # Eq. 9
            shapes["right"].append((s.shape,))
            break
        # Eq. 7: S_{s' chi_{i-1} chi_i} = sum R_{chi_{i-1} chi'} Q_{s' chi' chi_i}
        mt = s.transpose(0, 2, 1).reshape(-1, s.shape[1])                # [(s', chi_i), chi_{i-1}] = Q~ R~
        qt, _ = qr_pos(mt)
        q = qt.reshape(s.shape[0], s.shape[2], -1).transpose(0, 2, 1)    # Q[s', chi', chi_i]
        new[i] = q
        shapes["right"].append((s.shape, q.shape[1]))
        # Eq. 8: R^{[i-1]}[chi', a', b'] = sum Q*[s', chi', chi] T[s, a', a] W[s', s, b', b] R[chi, a, b]
        qr_ = np.tensordot(np.conj(q), R, axes=([2], [0]))               # [s', chi', a, b]
        qrw = np.tensordot(qr_, W[i], axes=([0, 3], [0, 3]))             # [chi', a, s, b']
        R = np.tensordot(qrw, T[i], axes=([2, 1], [0, 2]))               # [chi', b', a']
        R = R.transpose(0, 2, 1)                                         # [chi', a', b']
    out = [new[0]] + [new[i] if i < L - 1 else new[i][:, :, 0] for i in range(1, L)]
    if L == 1:
        out = [new[0][:, :, 0]]
    if record is not None:
        record.update(shapes)
    return TTN(list(psi.parent), [np.ascontiguousarray(t) for t in out], "state")
