"""The compress step's batched Hermitian eigensolver through the C ABI test hook
ttn_test_heev, against LAPACK (numpy.linalg.eigh) on the same matrices: the one-stage
tridiagonalisation (route 1) and the two-stage band reduction (route 2, 65 <= n <= 256,
csrc/heev2s.cu) over ragged orders, several matrices per launch, degenerate and
rank-deficient spectra, the zero matrix and tolerance truncation."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2601_19650_b200 as P
    c = P.Context(0)
    yield c
    c.close()


def wishart(rng, n, rows, nmat):
    X = (rng.standard_normal((nmat, rows, n)) + 1j * rng.standard_normal((nmat, rows, n))) / np.sqrt(2)
    return np.einsum("bki,bkj->bij", X.conj(), X)


def check_pairs(A, lam, vt, k, kmax, tol_rel=1e-11):
    n = A.shape[-1]
    ref = np.linalg.eigvalsh(A)[::-1]
    l1 = max(ref[0], 1e-300)
    assert np.all(np.abs(lam[:k] - ref[:k]) <= tol_rel * l1), np.abs(lam[:k] - ref[:k]).max() / l1
    V = vt[:k].T                                           # columns = eigenvectors
    res = np.linalg.norm(A @ V - V * lam[:k], axis=0).max() / l1
    orth = np.abs(V.conj().T @ V - np.eye(k)).max()
    assert res <= 1e-11 and orth <= 1e-11, (res, orth)
    assert np.all(vt[k:] == 0)


@pytest.mark.parametrize("n", [65, 72, 96, 127, 128, 130, 150, 192, 200, 255, 256])
@pytest.mark.parametrize("route", [1, 2])
def test_heev_routes_match_lapack(ctx, n, route):
    import paper_2601_19650_b200 as P
    rng = np.random.default_rng(1000 + n)
    nmat = 5
    A = wishart(rng, n, n + 37, nmat)
    kmax = min(32, n)
    lam, vt, k, w = P.ttn_test_heev(ctx, A, kmax, route=route)
    for i in range(nmat):
        assert k[i] == kmax
        check_pairs(A[i], lam[i], vt[i], k[i], kmax)
        ref = np.linalg.eigvalsh(A[i])[::-1]
        assert abs(w[i] - ref[kmax:].sum()) <= 1e-11 * np.trace(A[i]).real


@pytest.mark.parametrize("n", [96, 192])
def test_two_stage_equals_one_stage(ctx, n):
    """Same kept subspace from both routes (projector distance), larger kmax."""
    import paper_2601_19650_b200 as P
    rng = np.random.default_rng(7 + n)
    A = wishart(rng, n, 2 * n, 3)
    kmax = n // 2
    l1, v1, k1, w1 = P.ttn_test_heev(ctx, A, kmax, route=1)
    l2, v2, k2, w2 = P.ttn_test_heev(ctx, A, kmax, route=2)
    assert np.array_equal(k1, k2)
    for i in range(3):
        assert np.abs(l1[i] - l2[i]).max() <= 1e-12 * l1[i][0]
        P1 = v1[i].T @ v1[i].conj()
        P2 = v2[i].T @ v2[i].conj()
        assert np.abs(P1 - P2).max() <= 1e-9
        assert abs(w1[i] - w2[i]) <= 1e-11 * np.trace(A[i]).real


def test_two_stage_degenerate_and_rank_deficient(ctx):
    """Exactly degenerate kept eigenvalues (isometric circuit states give Gram = projector) and
    a rank-deficient Gram (fewer rows than columns): the kept subspace is unique only as a whole."""
    import paper_2601_19650_b200 as P
    rng = np.random.default_rng(3)
    n = 160
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    ev = np.concatenate([np.full(24, 2.0), np.full(24, 1.0), np.zeros(n - 48)])
    A0 = (Q * ev) @ Q.conj().T
    A0 = (A0 + A0.conj().T) / 2
    X = rng.standard_normal((40, n)) + 1j * rng.standard_normal((40, n))
    A1 = X.conj().T @ X
    A = np.stack([A0, A1])
    lam, vt, k, w = P.ttn_test_heev(ctx, A, 48, route=2)
    # degenerate: all 48 nonzero eigenvalues kept; subspace = span of the first 48 columns of Q
    assert k[0] == 48
    V = vt[0][:48].T
    Pk = V @ V.conj().T
    Pref = Q[:, :48] @ Q[:, :48].conj().T
    assert np.abs(Pk - Pref).max() <= 1e-10
    assert np.abs(np.sort(lam[0])[::-1] - ev[:48]).max() <= 1e-12 * 2
    # rank 40: the floor drops the 8 zero directions
    assert k[1] == 40
    check_pairs(A1, lam[1], vt[1], 40, 48)


def test_two_stage_zero_and_tolerance(ctx):
    import paper_2601_19650_b200 as P
    rng = np.random.default_rng(11)
    n = 100
    Z = np.zeros((1, n, n), np.complex128)
    lam, vt, k, w = P.ttn_test_heev(ctx, Z, 16, route=2)
    assert k[0] == 1 and w[0] == 0.0 and np.all(lam == 0)
    # prescribed spectrum, tol between sqrt(lam_5 / lam_1) and sqrt(lam_4 / lam_1)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    ev = np.concatenate([[1.0, 0.5, 0.3, 0.2], 0.01 * rng.random(n - 4)])
    A = ((Q * ev) @ Q.conj().T)[None]
    tol = np.sqrt(0.1)
    lam, vt, k, w = P.ttn_test_heev(ctx, A, 16, tol=tol, route=2)
    assert k[0] == 4
    assert abs(w[0] - ev[4:].sum()) <= 1e-12
    check_pairs(A[0], lam[0], vt[0], 4, 16)
