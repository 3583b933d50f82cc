"""GPU parity of SURVEY.md 8(f) rows against the CPU oracle: the skeleton matvec
apply_skeleton (compress.hpp:309-325, item 4) and the Monte Carlo error mc_error
(compress.hpp:279-305, item 3) through the row-subset view kid_select_rows, both through the
C-ABI and through the C++ mirror.

Bars: u within 1e-12 of sum_j |K_ij (P q)_j| per target (exp <= 1 ulp, different summation
rounding); mc_error estimates within 1e-10 relative of the oracle (exact norms on both sides)
or the D rounding floor of test_recon_error_vs_oracle."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1409_2802_b200._lib import Device
    d = Device(0)
    yield d
    d.close()


def _case(O, d, N, n, eps, xi=2.0, s=0.05):
    t = O.prepare_trial(d, N, n, xi, O.derive_seed(1, 0, 0))
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    rows = O.sample_rows(O.SCHEME_UNIFORM, K.shape[0], s, O.derive_seed(3, 0, 1))
    res = O.compress_id(K, rows, eps=eps)
    return t, K, res


@pytest.mark.parametrize("d,n,eps", [(2, 100, 1e-2), (3, 100, 1e-8), (5, 64, 1e-4), (8, 37, 1e-2), (1, 100, 1e-8)])
def test_apply_skeleton_vs_oracle(oracle, dev, d, n, eps):
    t, K, res = _case(oracle, d, 20_000, n, eps)
    q = np.random.default_rng(d).standard_normal(n)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    u = dev.apply_skeleton(t.h, res.skeleton, res.P, q)
    ref = oracle.apply_skeleton(t.targets, t.sources[res.skeleton], t.h, res.P, q)
    qs = res.P @ q
    scale = np.abs(K[:, res.skeleton]) @ np.abs(qs)
    assert u.shape == ref.shape
    assert np.all(np.abs(u - ref) <= 1e-12 * scale + 1e-300)


def test_apply_skeleton_edges(oracle, dev):
    from paper_1409_2802_b200._lib import KidError, KID_E_RANGE
    t, K, res = _case(oracle, 2, 5_000, 30, 1e-2)
    dev.set_points(t.points)
    dev.split(t.center, 30, 2.0)
    q = np.ones(30)
    # rank 0: u == 0; an explicit block with one target; out-of-range skeleton index
    assert np.all(dev.apply_skeleton(t.h, np.zeros(0, np.int64), np.zeros((0, 30)), q) == 0.0)
    with pytest.raises(KidError) as e:
        dev.apply_skeleton(t.h, np.array([30]), np.ones((1, 30)), q)
    assert e.value.code == KID_E_RANGE
    dev.set_block(t.targets[:1], t.sources)
    u = dev.apply_skeleton(t.h, res.skeleton, res.P, q)
    ref = oracle.apply_skeleton(t.targets[:1], t.sources[res.skeleton], t.h, res.P, q)
    assert abs(u[0] - ref[0]) <= 1e-12 * np.sum(np.abs(K[0, res.skeleton] * (res.P @ q)))


@pytest.mark.parametrize("d,n,eps,s_mc", [(2, 100, 1e-2, 0.1), (3, 64, 1e-4, 0.02), (2, 40, 1e-8, 0.5)])
def test_mc_error_vs_oracle(oracle, dev, d, n, eps, s_mc):
    t, K, res = _case(oracle, d, 20_000, n, eps)
    nt = K.shape[0]
    seed = 11
    ref = oracle.mc_error(K, res.skeleton, res.P, s_mc, 3, seed)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    for rep in range(3):
        rows = oracle.sample_rows(oracle.SCHEME_BERNOULLI, nt, s_mc, oracle.derive_seed(seed, rep, 0))
        dev.select_rows(rows)
        assert dev.nt == rows.size
        sd, sk, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
        G, _ = dev.gram(t.h)
        dev.select_rows(None)
        assert dev.nt == nt
        est = math.sqrt(max(np.linalg.eigvalsh(DtD)[-1], 0.0) / np.linalg.eigvalsh(G)[-1])
        Ks = K[rows]
        floor = 10 * math.sqrt(res.rank) * 2.2e-16 * np.abs(res.P).max() * math.sqrt(np.sum(Ks * Ks)) / \
            oracle.spectral_norm_exact(Ks)
        assert abs(est - ref[rep]) <= max(1e-10 * ref[rep], floor)


def test_select_rows_edges(oracle, dev):
    from paper_1409_2802_b200._lib import KidError, KID_E_RANGE
    t, K, res = _case(oracle, 2, 5_000, 30, 1e-2)
    dev.set_points(t.points)
    dev.split(t.center, 30, 2.0)
    nt = dev.nt
    rows = np.array([nt - 1, 0, 7, 7])  # any order, repeats allowed (gather_rows semantics)
    dev.select_rows(rows)
    G, sk = dev.gram(t.h)
    assert sk == pytest.approx(np.sum(K[rows] ** 2), rel=1e-12)
    assert np.allclose(dev.row_norms(t.h), oracle.row_norms(K[rows]), rtol=1e-12)
    with pytest.raises(KidError) as e:
        dev.select_rows(np.array([nt]))
    assert e.value.code == KID_E_RANGE
    dev.select_rows(np.zeros(0, np.int64))
    assert dev.nt == 0
    dev.select_rows(None)
    assert dev.nt == nt
    dev.split(t.center, 30, 2.0)  # a new split resets any subset
    assert dev.nt == nt


def test_mirror_next_rows(oracle):
    """mc_error + apply_skeleton through the C++ mirror (kernid_b200::mc_error / apply_skeleton)."""
    from paper_1409_2802_b200 import kernid as H
    d, N, n, xi, eps, s, s_mc, n_mc = 2, 20_000, 100, 2.0, 1e-4, 0.05, 0.1, 4
    data_seed = oracle.derive_seed(1, 0, 0)
    sample_seed = oracle.derive_seed(data_seed, 0, 1)
    q = np.linspace(-1.0, 2.0, n)
    nt, r, skel, P, mc, u = H.trial_next_rows(d, N, n, xi, data_seed, s, sample_seed, eps, s_mc, n_mc, 5, q)
    t = oracle.prepare_trial(d, N, n, xi, data_seed)
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], s, sample_seed)
    res = oracle.compress_id(K, rows, eps=eps)
    assert nt == K.shape[0] and r == res.rank and np.array_equal(skel, res.skeleton)
    assert np.array_equal(P, res.P)  # the host ID is bit-identical to the oracle's
    ref_mc = oracle.mc_error(K, res.skeleton, res.P, s_mc, n_mc, 5)
    floor = 10 * math.sqrt(r) * 2.2e-16 * np.abs(res.P).max() * math.sqrt(np.sum(K * K)) / oracle.spectral_norm_exact(K)
    assert np.all(np.abs(mc - ref_mc) <= np.maximum(1e-10 * ref_mc, 10 * floor))
    ref_u = oracle.apply_skeleton(t.targets, t.sources[res.skeleton], t.h, res.P, q)
    scale = np.abs(K[:, res.skeleton]) @ np.abs(res.P @ q)
    assert np.all(np.abs(u - ref_u) <= 1e-12 * scale + 1e-300)
