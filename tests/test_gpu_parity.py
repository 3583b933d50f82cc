"""GPU parity of the C-ABI (libkernid_cuda.so) against the CPU oracle.

Bars: split (sources, rho bits, targets) bit-exact; per-entry
passes (row norms, gathered rows) within 1e-12 relative (CUDA exp vs glibc exp differ
by <= 2 ulp); Grams |dG_jk| <= 1e-10 sqrt(G_jj G_kk) (hard part 2);
leverage within 1e-10 of the oracle; rel_error within 1e-10 relative (the
tolerance-ladder floor applies where D is rounding noise).
"""
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


def _trial(O, d, N, n, xi, seed=1, trial=0, scheme=0, h_value=1.0):
    data_seed = O.derive_seed(seed, trial, scheme)
    return O.prepare_trial(d, N, n, xi, data_seed, h_value)


@pytest.mark.parametrize("d,N,n,xi", [(2, 100_000, 100, 2.0), (1, 20_000, 100, 2.0), (3, 200_000, 100, 2.0),
                                      (5, 50_000, 100, 3.0), (8, 300_000, 512, 2.0), (16, 30_000, 256, 2.0),
                                      (3, 2_000, 40, 0.0), (4, 70_000, 1000, 1.0)])
def test_split_bit_exact(oracle, dev, d, N, n, xi):
    t = _trial(oracle, d, N, n, xi)
    dev.set_points(t.points)
    src, rho, nt = dev.split(t.center, n, xi)
    assert np.array_equal(src, t.split.source_indices)
    assert rho == t.split.rho  # bitwise (same double)
    assert nt == t.split.target_indices.size
    assert np.array_equal(dev.targets(), t.split.target_indices)


def test_split_ties_and_errors(oracle, dev):
    from paper_1409_2802_b200._lib import KidError, KID_E_NO_TARGETS, KID_E_RANGE, KID_E_DIM
    ps = np.array([[1.0], [-1.0], [1.0], [-1.0], [1.0], [5.0]])
    dev.set_points(ps)
    src, rho, nt = dev.split([0.0], 3, 1.0)
    ref = oracle.split_sources_targets(ps, [0.0], 3, 1.0)
    assert np.array_equal(src, ref.source_indices) and rho == ref.rho
    assert np.array_equal(dev.targets(), ref.target_indices)
    line = np.array([[0.0], [0.1], [-0.1], [0.5], [-0.5], [2.0], [-2.0], [3.0]])
    dev.set_points(line)
    src, rho, nt = dev.split([0.0], 3, 2.0)
    assert list(src) == [0, 1, 2] and list(dev.targets()) == [3, 4, 5, 6, 7]
    for args, code in ((([0.0], 3, 100.0), KID_E_NO_TARGETS), (([0.0], 0, 1.0), KID_E_RANGE),
                       (([0.0], 8, 1.0), KID_E_RANGE), (([0.0, 0.0], 3, 1.0), KID_E_DIM)):
        with pytest.raises(KidError) as e:
            dev.split(*args)
        assert e.value.code == code


def _block(oracle, d=3, N=20_000, n=100, xi=2.0, h_value=1.0):
    t = _trial(oracle, d, N, n, xi, h_value=h_value)
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    return t, K


@pytest.mark.parametrize("d", [2, 3, 5])
def test_row_norms_and_rows(oracle, dev, d):
    t, K = _block(oracle, d=d)
    dev.set_points(t.points)
    dev.split(t.center, 100, 2.0)
    w = dev.row_norms(t.h)
    ref = oracle.row_norms(K)
    nz = ref > 0
    assert np.all(np.abs(w[nz] - ref[nz]) <= 1e-12 * ref[nz])
    assert np.all(w[~nz] == 0.0)
    rows = np.array([0, 5, 17, K.shape[0] - 1])
    Ks = dev.eval_rows(t.h, rows)
    assert np.allclose(Ks, K[rows], rtol=1e-12, atol=0)


def _gram_ok(G, ref, tol=1e-10):
    dg = np.sqrt(np.abs(np.diag(ref)))
    bound = tol * np.outer(dg, dg) + 1e-300
    return np.all(np.abs(G - ref) <= bound)


@pytest.mark.parametrize("d,n", [(2, 100), (3, 100), (4, 37), (8, 64)])
def test_gram(oracle, dev, d, n):
    t, K = _block(oracle, d=d, n=n)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    G, sk = dev.gram(t.h)
    ref = K.T @ K
    assert _gram_ok(G, ref)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)
    assert np.array_equal(G, G.T)


@pytest.mark.parametrize("d,eps,n", [(2, 1e-2, 100), (2, 1e-8, 100), (3, 1e-8, 100), (4, 1e-4, 100),
                                     (3, 1e-4, 37), (1, 1e-8, 64), (8, 1e-2, 200)])
def test_recon_error_vs_oracle(oracle, dev, d, eps, n):
    t, K = _block(oracle, d=d, n=n)
    nt = K.shape[0]
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, nt, 0.02, oracle.derive_seed(7, 0, 1))
    res = oracle.compress_id(K, rows, eps=eps)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    sd, sk, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
    r_sd, r_sk, r_DtD, r_KtK = oracle.residual_stats(K, res.skeleton, res.P)
    assert sk == pytest.approx(r_sk, rel=1e-12)
    # tolerance ladder (hard part 2): D = K_N - K_S P carries rounding noise of
    # ~u (|K_N| + |K_S| |P|) per column, independent of the implementation's summation order
    u = 2.0 ** -53
    colnorm = np.sqrt((K * K).sum(0))
    noise = 8 * u * (colnorm + np.abs(res.P).T @ colnorm[res.skeleton])
    noise[res.skeleton] = 0.0
    dg = np.sqrt(np.abs(np.diag(r_DtD)))
    bound = 1e-10 * np.outer(dg, dg) + np.outer(noise, dg) + np.outer(dg, noise) + np.outer(noise, noise)
    assert np.all(np.abs(DtD - r_DtD) <= bound + 1e-300)
    assert abs(sd - r_sd) <= 1e-10 * r_sd + 2 * np.sum(noise * dg) + np.sum(noise ** 2)
    # spectral relative error: sqrt(lmax(D^T D) / lmax(K^T K)) vs the oracle's exact SVD path
    G, _ = dev.gram(t.h)
    rel = math.sqrt(np.linalg.eigvalsh(DtD)[-1] / np.linalg.eigvalsh(G)[-1])
    floor = 10 * math.sqrt(res.rank) * 2.2e-16 * np.abs(res.P).max() * math.sqrt(r_sk) / math.sqrt(np.linalg.eigvalsh(r_KtK)[-1])
    assert abs(rel - res.rel_error) <= max(1e-10 * res.rel_error, floor)


@pytest.mark.parametrize("d,n,rs", [(16, 256, (8, 64)), (8, 200, (30,))])
def test_leverage_large(oracle, dev, d, n, rs):
    """W beyond shared memory (c4-like m = 256, d = 16): the 2-CTA cluster kernel (K W on DMMA across
    the CTA pair, row sums of squares); the same bar as test_leverage."""
    t, K = _block(oracle, d=d, N=30_000, n=n)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    sv, V = oracle.right_factor(K)
    for r in rs:
        W = V[:, :r] / sv[:r]
        ref, _ = oracle.row_leverage_scores(K, r)
        got = dev.leverage(t.h, W)
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, ref.max())
    dev.set_path(1)  # small m through the cluster kernel too
    try:
        t, K = _block(oracle, d=3)
        dev.set_points(t.points)
        dev.split(t.center, 100, 2.0)
        sv, V = oracle.right_factor(K)
        W = V[:, :20] / sv[:20]
        ref, _ = oracle.row_leverage_scores(K, 20)
        assert np.max(np.abs(dev.leverage(t.h, W) - ref)) <= 1e-10 * max(1.0, ref.max())
    finally:
        dev.set_path(0)


def test_leverage(oracle, dev):
    t, K = _block(oracle, d=3)
    dev.set_points(t.points)
    dev.split(t.center, 100, 2.0)
    for r in (5, 20):
        sv, V = oracle.right_factor(K)
        W = V[:, :r] / sv[:r]
        ref, _ = oracle.row_leverage_scores(K, r)
        got = dev.leverage(t.h, W)
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, ref.max())
        assert got.sum() == pytest.approx(r, rel=1e-8)


def test_explicit_block(oracle, dev):
    tg = oracle.gen_normal(5, 333, 11) + 4.0
    sr = oracle.gen_normal(5, 21, 12)
    dev.set_block(tg, sr)
    K = oracle.kernel_matrix(tg, sr, 0.9)
    assert np.allclose(dev.row_norms(0.9), oracle.row_norms(K), rtol=1e-12, atol=0)
    G, _ = dev.gram(0.9)
    assert _gram_ok(G, K.T @ K)


def test_fast_exp_accuracy(dev):
    """exp_fast (the FP64 passes' exp) vs glibc exp: <= 1 ulp over the Gaussian argument range,
    exact 0 below the underflow threshold, correct subnormal scaling."""
    rng = np.random.default_rng(5)
    x = np.concatenate([-rng.random(1_000_000) * 760.0, -rng.random(100_000) * 1e-3, [0.0, -0.0, -745.13, -745.14,
                                                                                     -708.4, -709.0, -740.0, -800.0],
                        # far arguments: the clamp keeps them exact zeros (padding sources rely on it)
                        [-1.3e5, -1.4e6, -2.0e7, -1e12, -1e300, -np.inf]])
    y = dev.exp_check(x)
    ref = np.exp(x)
    normal = ref >= np.finfo(float).tiny
    ulp = np.abs(y[normal] - ref[normal]) / np.spacing(ref[normal])
    assert ulp.max() <= 1.0, ulp.max()
    sub = (ref < np.finfo(float).tiny) & (ref > 0)
    assert np.all(np.abs(y[sub] - ref[sub]) <= np.spacing(0.0) * 1.0)
    assert np.all(y[ref == 0.0] == 0.0)


@pytest.mark.parametrize("d,n,eps,force", [(16, 256, 1e-2, False), (8, 512, 1e-2, False), (3, 100, 1e-4, True)])
def test_recon_error_large_m_path(oracle, dev, d, n, eps, force):
    """m - r > 128 runs the 2-CTA cluster kernel (kid_fused.cu); kid_set_path routes a small case
    through it too so both kernel families are checked against the oracle."""
    dev.set_path(1 if force else 0)
    t, K = _block(oracle, d=d, N=12_000, n=n)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], 0.2, 5)
    res = oracle.compress_id(K, rows, eps=eps)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    sd, sk, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
    r_sd, r_sk, r_DtD, r_KtK = oracle.residual_stats(K, res.skeleton, res.P)
    assert sk == pytest.approx(r_sk, rel=1e-12)
    u = 2.0 ** -53
    colnorm = np.sqrt((K * K).sum(0))
    noise = 8 * u * (colnorm + np.abs(res.P).T @ colnorm[res.skeleton])
    noise[res.skeleton] = 0.0
    dg = np.sqrt(np.abs(np.diag(r_DtD)))
    bound = 1e-10 * np.outer(dg, dg) + np.outer(noise, dg) + np.outer(dg, noise) + np.outer(noise, noise)
    assert np.all(np.abs(DtD - r_DtD) <= bound + 1e-300)
    G, gsk = dev.gram(t.h)
    dev.set_path(0)
    assert _gram_ok(G, r_KtK)


def test_edge_cases(oracle, dev):
    """Degenerate shapes the reference handles: m = 1 source, full-rank skeleton (r = m: D == 0
    exactly), rank-1 skeleton, targets fewer than one tile, an empty explicit block, d = 64."""
    # m = 1
    t, K = _block(oracle, d=2, N=5000, n=1)
    dev.set_points(t.points)
    src, rho, nt = dev.split(t.center, 1, 2.0)
    assert np.array_equal(src, t.split.source_indices) and nt == K.shape[0]
    assert np.allclose(dev.row_norms(t.h), oracle.row_norms(K), rtol=1e-12, atol=0)
    G, sk = dev.gram(t.h)
    assert G.shape == (1, 1) and G[0, 0] == pytest.approx((K[:, 0] ** 2).sum(), rel=1e-12)
    # full-rank and rank-1 skeletons
    t, K = _block(oracle, d=3, N=8000, n=24)
    dev.set_points(t.points)
    dev.split(t.center, 24, 2.0)
    skel = np.arange(24)[::-1].copy()
    P = np.zeros((24, 24))
    P[np.arange(24), skel] = 1.0
    sd, sk, DtD, _ = dev.recon_error(t.h, skel, P)
    assert sd == 0.0 and np.all(DtD == 0.0) and sk == pytest.approx(np.sum(K * K), rel=1e-12)
    res = oracle.compress_id(K, np.arange(K.shape[0]), fixed_r=1)
    sd, sk, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
    r_sd, _, r_DtD, _ = oracle.residual_stats(K, res.skeleton, res.P)
    assert sd == pytest.approx(r_sd, rel=1e-9)
    # fewer targets than one 32-row tile, and no targets at all (explicit blocks)
    tg = oracle.gen_normal(3, 7, 3) + 5.0
    sr = oracle.gen_normal(3, 11, 4)
    dev.set_block(tg, sr)
    Kb = oracle.kernel_matrix(tg, sr, 1.3)
    G, sk = dev.gram(1.3)
    assert _gram_ok(G, Kb.T @ Kb)
    assert np.allclose(dev.row_norms(1.3), oracle.row_norms(Kb), rtol=1e-12, atol=0)
    dev.set_block(np.zeros((0, 3)), sr)
    G, sk = dev.gram(1.3)
    assert sk == 0.0 and np.all(G == 0.0)
    assert dev.row_norms(1.3).size == 0


def test_split_high_dimension(oracle, dev):
    """d = 64 (BASELINE c4): the generic-d kernels, bit-exact split and parity of the passes."""
    t, K = _block(oracle, d=64, N=3000, n=64, xi=1.0)
    dev.set_points(t.points)
    src, rho, nt = dev.split(t.center, 64, 1.0)
    assert np.array_equal(src, t.split.source_indices) and rho == t.split.rho
    assert np.array_equal(dev.targets(), t.split.target_indices)
    w = dev.row_norms(t.h)
    ref = oracle.row_norms(K)
    nz = ref > 0
    assert np.all(np.abs(w[nz] - ref[nz]) <= 1e-12 * ref[nz])
    G, _ = dev.gram(t.h)
    assert _gram_ok(G, K.T @ K)


@pytest.mark.parametrize("n", [1, 7, 100, 1024, 1025])
def test_split_lattice_ties_and_selection_paths(oracle, dev, n):
    """Many exactly equal distances (an integer lattice around its centre point) through the
    device-side selection (n <= 1024, one synchronisation) and the general path (n > 1024):
    sources, rho and targets bit-exact against nth_element's (dist, idx) order."""
    g = np.arange(-40, 41, dtype=np.float64)
    xx, yy = np.meshgrid(g, g, indexing="ij")
    ps = np.stack([xx.ravel(), yy.ravel()], axis=1)  # 6561 points, exact integer coordinates
    ps = ps[np.random.default_rng(n).permutation(ps.shape[0])]
    center = np.array([0.0, 0.0])
    dev.set_points(ps)
    src, rho, nt = dev.split(center, n, 1.5)
    ref = oracle.split_sources_targets(ps, center, n, 1.5)
    assert np.array_equal(src, ref.source_indices)
    assert rho == ref.rho
    assert np.array_equal(dev.targets(), ref.target_indices)


def test_generic_dimension_passes(oracle, dev):
    """d = 7 (not one of the compiled dimensions 1, 2, 3, 4, 5, 8, 16): every pass through the
    generic-d kernels against the oracle."""
    t, K = _block(oracle, d=7, N=12_000, n=60, xi=1.5)
    dev.set_points(t.points)
    src, rho, nt = dev.split(t.center, 60, 1.5)
    assert np.array_equal(src, t.split.source_indices) and rho == t.split.rho
    assert np.allclose(dev.row_norms(t.h), oracle.row_norms(K), rtol=1e-12, atol=0)
    G, sk = dev.gram(t.h)
    assert _gram_ok(G, K.T @ K) and sk == pytest.approx(np.sum(K * K), rel=1e-12)
    R = dev.tsqr_r(t.h)
    s1 = oracle.spectral_norm_exact(K)
    assert np.allclose(R.T @ R, K.T @ K, rtol=0, atol=1e-12 * s1 * s1)
    sv, V = oracle.right_factor(K)
    W = V[:, :10] / sv[:10]
    ref, _ = oracle.row_leverage_scores(K, 10)
    assert np.max(np.abs(dev.leverage(t.h, W) - ref)) <= 1e-10 * max(1.0, ref.max())


def test_full_rank_residual_device_pass(oracle, dev):
    """r = m through the device entry point (kid_recon_error_dev): D == 0 exactly and
    ||K||_F^2 from the reduction-only kernel."""
    import torch
    t, K = _block(oracle, d=3, N=20_000, n=40)
    dev.set_points(t.points)
    dev.split(t.center, 40, 2.0)
    skel = np.arange(40)
    dev.recon_prepare(skel, np.eye(40))
    out = torch.full((8,), -1.0, dtype=torch.float64, device="cuda")
    dev.recon_error_dev(t.h, out.data_ptr())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert o[0] == 0.0
    assert o[1] == pytest.approx(np.sum(K * K), rel=1e-12)


def test_empty_block_all_passes(oracle, dev):
    """A block with no targets (kid_set_block with nt = 0): every pass returns the empty result."""
    sr = oracle.gen_normal(3, 12, 5)
    dev.set_block(np.zeros((0, 3)), sr)
    assert dev.row_norms(0.5).size == 0
    G, sk = dev.gram(0.5)
    assert np.all(G == 0.0) and sk == 0.0
    skel, P = np.array([0, 3]), np.zeros((2, 12))
    P[:, skel] = np.eye(2)
    sd, sk, DtD, _ = dev.recon_error(0.5, skel, P)
    assert sd == 0.0 and sk == 0.0 and np.all(DtD == 0.0)
    sd, sk, Gp = dev.proj_gram(0.5, np.eye(12)[:, :5])
    assert sd == 0.0 and sk == 0.0 and np.all(Gp == 0.0)
    assert np.all(dev.tsqr_r(0.5) == 0.0)
    assert dev.leverage(0.5, np.eye(12)[:, :3]).size == 0
