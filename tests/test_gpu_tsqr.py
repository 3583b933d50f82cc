"""GPU parity of the TSQR spectrum: kid_tsqr_r's triangular factor R of
the full K (R^T R = K^T K) against the oracle's restatement of singular_values / right_factor
(lowrank.hpp:56-90: Householder QR + SVD of R), and the fold of per-block factors
(kid_tsqr_combine, the multi-rank step).

Bars: singular values within 1e-12 sigma_1 absolute -- the backward-stable floor of a
Householder QR, which the Gram route (sqrt(eig(K^T K)), ~1e-8 sigma_1) cannot reach; R^T R
within 1e-12 ||K||_2^2 of K^T K; right singular subspaces of well-separated leading sigmas
agree (projector difference <= 1e-9 / relative gap)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1409_2802_b200._lib import Device
    d = Device(0)
    yield d
    d.close()


def _block(O, d, N, n, xi=2.0, seed=0):
    t = O.prepare_trial(d, N, n, xi, O.derive_seed(1, seed, 0))
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    return t, K


def _check_R(O, R, K):
    m = K.shape[1]
    assert np.all(np.tril(R, -1) == 0.0)
    s1 = O.spectral_norm_exact(K)
    assert np.allclose(R.T @ R, K.T @ K, rtol=0, atol=1e-12 * s1 * s1)
    sv = np.linalg.svd(R, compute_uv=False)
    ref = O.singular_values(K)
    assert sv.shape == ref.shape == (m,)
    assert np.all(np.abs(sv - ref) <= 1e-12 * s1), np.max(np.abs(sv - ref)) / s1
    return sv, ref


@pytest.mark.parametrize("d,n,N", [(2, 100, 20_000), (3, 100, 30_000), (1, 100, 20_000), (5, 64, 20_000),
                                   (8, 37, 20_000), (3, 128, 20_000), (16, 100, 20_000)])
def test_tsqr_spectrum_vs_oracle(oracle, dev, d, n, N):
    t, K = _block(oracle, d, N, n)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    R = dev.tsqr_r(t.h)
    sv, ref = _check_R(oracle, R, K)
    # the Gram route cannot resolve the tail that TSQR does (where the spectrum reaches it)
    G, _ = dev.gram(t.h)
    sv_gram = np.sqrt(np.clip(np.linalg.eigvalsh(G)[::-1], 0.0, None))
    tail = ref < 1e-9 * ref[0]
    if np.any(tail):
        assert np.max(np.abs(sv_gram - ref)[tail]) > 10 * np.max(np.abs(sv - ref)[tail])
    # leading right singular subspaces (lowrank.hpp:81-86 right_factor) where the gap is clear
    _, V = oracle.right_factor(K)
    Vg = np.linalg.svd(R)[2].T
    for r in range(1, min(n, 12)):
        gap = (ref[r - 1] - ref[r]) / ref[0]
        if gap > 1e-3:
            P1, P2 = V[:, :r] @ V[:, :r].T, Vg[:, :r] @ Vg[:, :r].T
            assert np.max(np.abs(P1 - P2)) <= 1e-9 / gap


def test_tsqr_combine_and_edges(oracle, dev):
    from paper_1409_2802_b200._lib import KidError, KID_E_DIM
    t, K = _block(oracle, 3, 20_000, 100)
    nt = K.shape[0]
    # two blocks folded: the per-rank factors of a 2-way shard
    dev.set_block(t.targets[: nt // 3], t.sources)
    R1 = dev.tsqr_r(t.h)
    dev.set_block(t.targets[nt // 3:], t.sources)
    R2 = dev.tsqr_r(t.h)
    R = dev.tsqr_combine([R1, R2])
    _check_R(oracle, R, K)
    # fewer rows than one tile, one row, fewer rows than columns
    for rows in (1, 5, 63, 64, 65, 99):
        dev.set_block(t.targets[:rows], t.sources)
        R = dev.tsqr_r(t.h)
        Ks = K[:rows]
        assert np.all(np.tril(R, -1) == 0.0)
        assert np.allclose(R.T @ R, Ks.T @ Ks, rtol=0, atol=1e-13 * max(np.sum(Ks * Ks), 1e-300))
        assert np.all(np.abs(R[rows:, :]) <= 1e-13 * np.linalg.norm(Ks))  # rank <= rows: rounding only
    # m = 1
    dev.set_block(t.targets[:100], t.sources[:1])
    R = dev.tsqr_r(t.h)
    assert abs(abs(R[0, 0]) - np.linalg.norm(K[:100, 0])) <= 1e-14 * np.linalg.norm(K[:100, 0])
    # m > 128: the factor does not fit shared memory
    t2, _ = _block(oracle, 3, 5_000, 129)
    dev.set_points(t2.points)
    dev.split(t2.center, 129, 2.0)
    with pytest.raises(KidError) as e:
        dev.tsqr_r(t2.h)
    assert e.value.code == KID_E_DIM
