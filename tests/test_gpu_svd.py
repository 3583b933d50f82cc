"""GPU parity of the compress_svd error pass (compress.hpp:219-273):
kid_proj_gram (D = K C, G = D^T D, never materialised) against the CPU oracle, through the
C-ABI and through the C++ mirror (kernid_b200::compress_svd).

With C = V_perp (the trailing m - r right singular vectors of the sample),
||K - K V_r V_r^T||_2 = ||K V_perp||_2 = sqrt(lambda_max(G)).
Bars: rel_error within 1e-10 relative of the oracle's exact norm (or_svd_error_norm: QR + SVD of
the materialised difference), or the rounding floor of D where the error itself is rounding
noise (|dD_i| <~ m u ||K_i||: both sides form K V with independent rounding) -- floor =
10 m u ||K||_F / ||K||_2; Gram entries |dG_jk| <= 1e-10 sqrt(G_jj G_kk) + that floor's
square-root scale; ||K||_F^2 within 1e-12."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
U = 2.220446049250313e-16


@pytest.fixture(scope="module")
def dev():
    from paper_1409_2802_b200._lib import Device
    d = Device(0)
    yield d
    d.close()


def _svd_case(O, d, N, n, eps, xi=2.0, s=0.05, seed=0):
    t = O.prepare_trial(d, N, n, xi, O.derive_seed(1, seed, 0))
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    rows = O.sample_rows(O.SCHEME_UNIFORM, K.shape[0], s, O.derive_seed(3, seed, 1))
    sv, V = O.right_factor(K[rows])
    r = O.epsilon_rank(sv[: min(len(rows), n)], eps)
    return t, K, rows, V, r


def _check(O, dev, t, K, V, r, n):
    Vr, Vp = V[:, :r], V[:, r:]
    sd, sk, G = dev.proj_gram(t.h, Vp)
    Kg, skg = dev.gram(t.h)
    normK = O.spectral_norm_exact(K)
    fro = math.sqrt(np.sum(K * K))
    floor = 10 * n * U * fro / normK
    ref = O.svd_error_norm(K, Vr) / normK
    got = math.sqrt(max(np.linalg.eigvalsh(G)[-1], 0.0)) / math.sqrt(np.linalg.eigvalsh(Kg)[-1])
    assert abs(got - ref) <= max(1e-10 * ref, floor), (got, ref, floor)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)
    D = K @ Vp
    Gref = D.T @ D
    dg = np.sqrt(np.diag(Gref))
    tol = 1e-10 * np.outer(dg, dg) + 10 * n * U * fro * (dg[:, None] + dg[None, :] + 10 * n * U * fro)
    assert np.all(np.abs(G - Gref) <= tol)
    assert abs(sd - np.trace(Gref)) <= 1e-10 * np.trace(Gref) + 2 * np.sum(tol.diagonal())


@pytest.mark.parametrize("d,n,eps", [(3, 100, 1e-2), (2, 100, 1e-8), (1, 100, 1e-14), (5, 64, 1e-4), (8, 37, 1e-2),
                                     (3, 128, 1e-2), (4, 100, 1e-2)])
@pytest.mark.parametrize("large", [False, True])
def test_proj_gram_svd_error_vs_oracle(oracle, dev, d, n, eps, large):
    t, K, rows, V, r = _svd_case(oracle, d, 20_000, n, eps)
    assert 0 < r < n
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    dev.set_path(1 if large else 0)  # large: the 2-CTA cluster kernel (kid_fused.cu)
    try:
        _check(oracle, dev, t, K, V, r, n)
    finally:
        dev.set_path(0)


def test_proj_gram_edges(oracle, dev):
    from paper_1409_2802_b200._lib import KidError, KID_E_RANGE
    t, K, rows, V, r = _svd_case(oracle, 2, 5_000, 30, 1e-2)
    dev.set_points(t.points)
    dev.split(t.center, 30, 2.0)
    # C = I: G == K^T K of the Gram pass; one column; rank m - 1
    sd, sk, G = dev.proj_gram(t.h, np.eye(30))
    Kg, skg = dev.gram(t.h)
    assert np.allclose(G, Kg, rtol=1e-12, atol=1e-300) and sk == pytest.approx(skg, rel=1e-14)
    sd, sk, G = dev.proj_gram(t.h, V[:, :1])
    assert G.shape == (1, 1) and G[0, 0] == pytest.approx(np.sum((K @ V[:, 0]) ** 2), rel=1e-10)
    _check(oracle, dev, t, K, V, 29, 30)
    for bad in (np.zeros((30, 0)), np.zeros((30, 31))):
        with pytest.raises(KidError) as e:
            dev.proj_gram(t.h, bad)
        assert e.value.code == KID_E_RANGE
    # explicit blocks: one target, a ragged tile count (33 targets)
    for nt in (1, 33):
        dev.set_block(t.targets[:nt], t.sources)
        sd, sk, G = dev.proj_gram(t.h, V[:, r:])
        D = K[:nt] @ V[:, r:]
        assert np.allclose(G, D.T @ D, rtol=1e-10, atol=1e-13 * np.sum(K[:nt] ** 2))
        assert sk == pytest.approx(np.sum(K[:nt] ** 2), rel=1e-12)


@pytest.mark.parametrize("d,eps", [(2, 1e-8), (3, 1e-2), (1, 1e-4)])
def test_mirror_compress_svd(oracle, d, eps):
    """kernid_b200::compress_svd (host right factor + device error pass) vs the oracle pipeline."""
    from paper_1409_2802_b200 import kernid as H
    N, n, xi, s = 20_000, 100, 2.0, 0.02
    data_seed = oracle.derive_seed(1, 0, 0)
    sample_seed = oracle.derive_seed(data_seed, 0, 1)
    r, rel, fro, Vr = H.trial_svd(d, N, n, xi, data_seed, s, sample_seed, eps)
    t = oracle.prepare_trial(d, N, n, xi, data_seed)
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], s, sample_seed)
    sv, V = oracle.right_factor(K[rows])
    assert r == oracle.epsilon_rank(sv, eps)
    # the basis is unique up to signs / rotations inside repeated singular values: compare projectors
    assert np.allclose(Vr @ Vr.T, V[:, :r] @ V[:, :r].T, atol=1e-8)
    normK = oracle.spectral_norm_exact(K)
    ref = oracle.svd_error_norm(K, V[:, :r]) / normK
    floor = 10 * n * U * math.sqrt(np.sum(K * K)) / normK
    assert abs(rel - ref) <= max(1e-8 * ref, floor)
    D = K @ Vr @ Vr.T - K
    ref_fro = math.sqrt(np.sum(D * D) / np.sum(K * K))
    assert abs(fro - ref_fro) <= max(1e-8 * ref_fro, floor)
