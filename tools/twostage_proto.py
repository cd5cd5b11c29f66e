"""Design prototype (NumPy) of the two-stage Hermitian tridiagonalisation used by
csrc/heev2s.cu -- NOT the oracle and not used by any test of the product; it checks the
algebra of the kernels (panel QR + compact WY two-sided update, bulge chasing with the
lag-3 lockstep schedule, and the back-transform order) against numpy.linalg.eigh.

  python tools/twostage_proto.py
"""
import numpy as np


def zlarfg(x):
    """H^H x = beta e1 with H = I - tau v v^H, v[0] = 1, beta real (LAPACK zlarfg)."""
    alpha = x[0]
    xn2 = float(np.vdot(x[1:], x[1:]).real)
    v = np.zeros_like(x)
    v[0] = 1.0
    if xn2 == 0.0 and alpha.imag == 0.0:
        return alpha.real, 0.0 + 0.0j, v
    beta = -np.copysign(np.sqrt(abs(alpha) ** 2 + xn2), alpha.real)
    tau = (beta - alpha.real) / beta - 1j * alpha.imag / beta
    v[1:] = x[1:] / (alpha - beta)
    return beta, tau, v


def he2hb(A, b):
    """Stage 1: A (full Hermitian) -> band of lower bandwidth b.  Returns the band matrix,
    the panel reflectors [(r0, V, T)] with Q1 = Q_0 Q_1 ... , Q_p = I - V T V^H on rows r0:."""
    A = A.copy()
    n = A.shape[0]
    panels = []
    p = 0
    while True:
        c0 = p * b
        r0 = c0 + b
        m = n - r0
        if m < 2:
            break
        P = A[r0:, c0:c0 + b].copy()
        kq = min(m, b)
        V = np.zeros((m, b), complex)
        taus = np.zeros(b, complex)
        for j in range(kq):
            beta, tau, v = zlarfg(P[j:, j])
            V[j:, j] = v
            taus[j] = tau
            P[j:, j] = 0
            P[j, j] = beta
            # H^H on the remaining columns
            u = v.conj() @ P[j:, j + 1:]
            P[j:, j + 1:] -= np.conj(tau) * np.outer(v, u)
        # compact WY (zlarft, forward columnwise): Q = I - V T V^H
        G = V.conj().T @ V
        T = np.zeros((b, b), complex)
        for j in range(b):
            T[j, j] = taus[j]
            if j:
                T[:j, j] = -taus[j] * (T[:j, :j] @ G[:j, j])
        Q = np.eye(m) - V @ T @ V.conj().T
        assert np.allclose(Q.conj().T @ A[r0:, c0:c0 + b], P, atol=1e-10)
        A[r0:, c0:c0 + b] = P
        A[c0:c0 + b, r0:] = P.conj().T
        A22 = A[r0:, r0:]
        X = A22 @ V @ T
        M = V.conj().T @ X
        W = X - 0.5 * V @ (T.conj().T @ M)
        A[r0:, r0:] = A22 - V @ W.conj().T - W @ V.conj().T
        panels.append((r0, V, T))
        p += 1
    return A, panels


def hb2st(Bfull, b):
    """Stage 2: Hermitian band (lower bandwidth b) -> real tridiagonal by bulge chasing.
    Tasks (s, t) run in the lockstep schedule of the kernel: at time step T, sweep s does
    task t = T - 3 s.  Returns d, e and the reflectors {(s, t): (j0, v, tau)}."""
    A = Bfull.copy()
    n = A.shape[0]
    refl = {}
    ntask = [0] * n
    for s in range(n - 1):
        t = 0
        while s + 1 + t * b < n:
            t += 1
        ntask[s] = t

    def task(s, t):
        if t == 0:
            j0 = s + 1
            L = min(b, n - 1 - s)
            beta, tau, v = zlarfg(A[j0:j0 + L, s].copy())
            A[j0:j0 + L, s] = 0
            A[j0, s] = beta
            A[s, j0:j0 + L] = A[j0:j0 + L, s].conj()
        else:
            jp, vp, taup = refl[(s, t - 1)]
            Lp = len(vp)
            j0 = s + 1 + t * b
            L = min(b, n - j0)
            E = A[j0:j0 + L, jp:jp + Lp]
            E = E - taup * np.outer(E @ vp, vp.conj())            # E H_prev
            beta, tau, v = zlarfg(E[:, 0].copy())
            E = E - np.conj(tau) * np.outer(v, v.conj() @ E)      # H^H E
            A[j0:j0 + L, jp:jp + Lp] = E
            A[jp:jp + Lp, j0:j0 + L] = E.conj().T
        D = A[j0:j0 + L, j0:j0 + L]
        y = D @ v
        gam = np.vdot(v, y).real
        w = tau * y - 0.5 * abs(tau) ** 2 * gam * v
        A[j0:j0 + L, j0:j0 + L] = D - np.outer(w, v.conj()) - np.outer(v, w.conj())
        refl[(s, t)] = (j0, v, tau)

    Tmax = 3 * (n - 1) + max(ntask) + 1
    for T in range(Tmax):
        for s in range(n - 1):
            t = T - 3 * s
            if 0 <= t < ntask[s]:
                task(s, t)
    # bandwidth check: out-of-band fill must be gone
    for i in range(n):
        for j in range(n):
            if abs(i - j) > 1:
                assert abs(A[i, j]) < 1e-9, (i, j, A[i, j])
    d = np.real(np.diag(A)).copy()
    e = np.array([A[i + 1, i] for i in range(n - 1)])
    assert np.allclose(e.imag, 0, atol=1e-12)
    return d, e.real, refl, ntask


def back_transform(Z, panels, refl, ntask, n):
    Y = Z.astype(complex).copy()
    for s in range(n - 2, -1, -1):
        for t in range(ntask[s] - 1, -1, -1):
            j0, v, tau = refl[(s, t)]
            L = len(v)
            Y[j0:j0 + L] -= tau * np.outer(v, v.conj() @ Y[j0:j0 + L])
    for r0, V, T in reversed(panels):
        Y[r0:] -= V @ (T @ (V.conj().T @ Y[r0:]))
    return Y


def main():
    rng = np.random.default_rng(0)
    for n, b in [(20, 4), (37, 8), (64, 16), (130, 16), (192, 16), (128, 16), (70, 8)]:
        X = rng.standard_normal((n + 7, n)) + 1j * rng.standard_normal((n + 7, n))
        A = X.conj().T @ X
        B, panels = he2hb(A, b)
        for i in range(n):
            for j in range(n):
                if i - j > b:
                    assert abs(B[i, j]) < 1e-9 * abs(A).max()
        d, e, refl, ntask = hb2st(B, b)
        Tm = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        lt, Zt = np.linalg.eigh(Tm)
        la = np.linalg.eigvalsh(A)
        assert np.allclose(lt, la, rtol=1e-10, atol=1e-10 * la.max()), np.abs(lt - la).max()
        k = min(32, n)
        Z = Zt[:, ::-1][:, :k]
        V = back_transform(Z, panels, refl, ntask, n)
        res = np.linalg.norm(A @ V - V * lt[::-1][:k]) / la.max()
        orth = np.linalg.norm(V.conj().T @ V - np.eye(k))
        print(f"n={n} b={b}: eig err {np.abs(lt - la).max() / la.max():.1e} residual {res:.1e} orth {orth:.1e} "
              f"reflectors {sum(ntask)} time steps {3 * (n - 2) + ntask[0]}")
        assert res < 1e-12 and orth < 1e-12


if __name__ == "__main__":
    main()
