"""GPU parity of the 2-CTA cluster kernel (kid_fused.cu) against the CPU oracle.

The kernel serves every Gram / leverage / projected pass whose operands do not fit one SM
(BASELINE c4: m = 256, d = 16; c5: m = 512, d = 8). kid_set_path(KID_PATH_CLUSTER) also routes
small blocks through it, so each pass is checked on both kernel families against the same
oracle restatement (compress.hpp:141-159, lowrank.hpp:56-90, 296-308, compress.hpp:243-257).
Bars as tests/test_gpu_parity.py: Grams |dG_jk| <= 1e-10 sqrt(G_jj G_kk) plus the rounding floor
of D = K_N - K_S P; ||K||_F^2 1e-12; leverage 1e-10 of max(1, max l).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def dev():
    from paper_1409_2802_b200._lib import Device
    d = Device(0)
    yield d
    d.close()


@pytest.fixture
def cluster(dev):
    dev.set_path(1)
    yield dev
    dev.set_path(0)


def _block(O, d, N, n, xi=2.0, seed=1, h_value=1.0):
    t = O.prepare_trial(d, N, n, xi, O.derive_seed(seed, 0, 0), h_value)
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    return t, K


def _gram_ok(G, ref, tol=1e-10):
    dg = np.sqrt(np.abs(np.diag(ref)))
    return np.all(np.abs(G - ref) <= tol * np.outer(dg, dg) + 1e-300)


def _resid_bound(K, res, r_DtD):
    colnorm = np.sqrt((K * K).sum(0))
    noise = 8 * U * (colnorm + np.abs(res.P).T @ colnorm[res.skeleton])
    noise[res.skeleton] = 0.0
    dg = np.sqrt(np.abs(np.diag(r_DtD)))
    return 1e-10 * np.outer(dg, dg) + np.outer(noise, dg) + np.outer(dg, noise) + np.outer(noise, noise), noise, dg


def _check_resid(O, dev, t, K, n, eps, s=0.05, seed=5):
    rows = O.sample_rows(O.SCHEME_UNIFORM, K.shape[0], s, seed)
    res = O.compress_id(K, rows, eps=eps)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    sd, sk, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
    r_sd, r_sk, r_DtD, r_KtK = O.residual_stats(K, res.skeleton, res.P)
    assert sk == pytest.approx(r_sk, rel=1e-12)
    bound, noise, dg = _resid_bound(K, res, r_DtD)
    assert np.all(np.abs(DtD - r_DtD) <= bound + 1e-300)
    assert abs(sd - r_sd) <= 1e-10 * r_sd + 2 * np.sum(noise * dg) + np.sum(noise ** 2) + 1e-300
    return res, DtD, r_KtK


@pytest.mark.parametrize("d,n", [(2, 100), (3, 37), (5, 64), (8, 100), (16, 48), (7, 30)])
def test_cluster_gram(oracle, cluster, d, n):
    t, K = _block(oracle, d, 20_000, n)
    cluster.set_points(t.points)
    cluster.split(t.center, n, 2.0)
    G, sk = cluster.gram(t.h)
    assert _gram_ok(G, K.T @ K)
    assert np.array_equal(G, G.T)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)


@pytest.mark.parametrize("d,n,eps", [(2, 100, 1e-2), (2, 100, 1e-8), (3, 100, 1e-4), (8, 64, 1e-2),
                                     (16, 48, 1e-6), (5, 90, 1e-12), (7, 30, 1e-3)])
@pytest.mark.parametrize("kern", [1, 2])
def test_cluster_residual(oracle, cluster, d, n, eps, kern):
    """kern 1: the warp-specialised k_fused; 2: the warp-tile k_fused_w where n - r <= 32 (else k_fused)."""
    t, K = _block(oracle, d, 20_000, n)
    cluster.set_option(3, kern)
    try:
        _check_resid(oracle, cluster, t, K, n, eps)
    finally:
        cluster.set_option(3, 0)


@pytest.mark.parametrize("d,n,r", [(8, 100, 80), (3, 64, 60), (16, 48, 17), (5, 40, 39), (8, 200, 175), (2, 100, 90),
                                   (4, 37, 30), (1, 16, 5), (7, 100, 70), (12, 40, 33)])
def test_warp_tile_kernel(oracle, dev, d, n, r):
    """k_fused_w (n - r <= 32 D columns: 1 to 4 column blocks, ragged tiles) in both forms -- one CTA per SM
    (the automatic choice here: M and the sources fit one SM) and the CTA pair with its DSMEM exchange --
    against the oracle, the same Grams from k_fused within the rounding ladder, bitwise reproducible run to
    run; the automatic path of kid_recon_error takes it for n <= 32."""
    t, K = _block(oracle, d, 15_000, n)
    dev.set_points(t.points)
    dev.split(t.center, n, 2.0)
    res = oracle.compress_id(K, np.arange(0, K.shape[0], 7), fixed_r=r)
    _, _, r_DtD, _ = oracle.residual_stats(K, res.skeleton, res.P)
    bound, _, _ = _resid_bound(K, res, r_DtD)
    out = {}
    try:
        auto = dev.recon_error(t.h, res.skeleton, res.P)
        assert dev.last_kernel() == "k_fused_w (solo)"
        out["auto"] = auto
        for form, warps in ((1, 0), (1, 8), (2, 0)):
            dev.set_option(5, form)
            dev.set_option(4, warps)
            got = dev.recon_error(t.h, res.skeleton, res.P)
            assert dev.last_kernel() == ("k_fused_w (solo)" if form == 1 else "k_fused_w")
            again = dev.recon_error(t.h, res.skeleton, res.P)
            assert np.array_equal(again[2], got[2]) and again[0] == got[0]
            out[(form, warps)] = got
        dev.set_option(5, 0)
        dev.set_option(4, 0)
        dev.set_path(1)
        dev.set_option(3, 1)
        out["k_fused"] = dev.recon_error(t.h, res.skeleton, res.P)
        assert dev.last_kernel() == "k_fused"
    finally:
        dev.set_option(3, 0)
        dev.set_option(4, 0)
        dev.set_option(5, 0)
        dev.set_path(0)
    assert np.array_equal(out["auto"][2], out[(1, 0)][2])
    for key, got in out.items():
        assert np.all(np.abs(got[2] - r_DtD) <= bound + 1e-300), key
        assert got[1] == pytest.approx(float(np.sum(K * K)), rel=1e-12), key


@pytest.mark.parametrize("d,n,r,form", [(16, 200, 160, "k_fused_w (solo)"), (8, 256, 210, "k_fused_w"),
                                        (5, 150, 108, "k_fused_w"), (8, 512, 478, "k_fused_w")])
def test_warp_tile_kernel_wide(oracle, dev, d, n, r, form):
    """5 / 6 column blocks (33 <= n - r <= 48) at m > 128: one CTA per SM up to 40 D columns, the CTA pair up
    to 48; against the oracle and against k_fused."""
    t, K = _block(oracle, d, 12_000, n, xi=1.0)
    dev.set_points(t.points)
    dev.split(t.center, n, 1.0)
    res = oracle.compress_id(K, np.arange(0, K.shape[0], 5), fixed_r=r)
    _, _, r_DtD, _ = oracle.residual_stats(K, res.skeleton, res.P)
    bound, _, _ = _resid_bound(K, res, r_DtD)
    try:
        dev.set_path(1)  # (m = 150 would otherwise fit k_gram)
        got = dev.recon_error(t.h, res.skeleton, res.P)
        assert dev.last_kernel() == form
        dev.set_option(3, 1)
        ref = dev.recon_error(t.h, res.skeleton, res.P)
        assert dev.last_kernel() == "k_fused"
    finally:
        dev.set_option(3, 0)
        dev.set_path(0)
    for g in (got, ref):
        assert np.all(np.abs(g[2] - r_DtD) <= bound + 1e-300)
        assert g[1] == pytest.approx(float(np.sum(K * K)), rel=1e-12)


def test_cluster_residual_rank_one_and_full(oracle, cluster):
    """rank 1 (one skeleton column: the A k-slice of CTA 1 is empty) and r = m - 1 (one D column)."""
    t, K = _block(oracle, 3, 10_000, 40)
    cluster.set_points(t.points)
    cluster.split(t.center, 40, 2.0)
    for r in (1, 39):
        res = oracle.compress_id(K, np.arange(0, K.shape[0], 3), fixed_r=r)
        sd, sk, DtD, _ = cluster.recon_error(t.h, res.skeleton, res.P)
        r_sd, r_sk, r_DtD, _ = oracle.residual_stats(K, res.skeleton, res.P)
        bound, noise, dg = _resid_bound(K, res, r_DtD)
        assert np.all(np.abs(DtD - r_DtD) <= bound + 1e-300)
        assert sk == pytest.approx(r_sk, rel=1e-12)


@pytest.mark.parametrize("d,n,k", [(3, 100, 17), (8, 64, 40), (2, 50, 50)])
def test_cluster_proj_gram(oracle, cluster, d, n, k):
    t, K = _block(oracle, d, 15_000, n)
    cluster.set_points(t.points)
    cluster.split(t.center, n, 2.0)
    C = np.linalg.qr(np.random.default_rng(k).standard_normal((n, k)))[0]
    sd, sk, G = cluster.proj_gram(t.h, C)
    KC = K @ C
    ref = KC.T @ KC
    dg = np.sqrt(np.abs(np.diag(ref)))
    floor = 4 * n * U * np.sqrt((K * K).sum()) * np.sqrt(np.abs(C).sum(0) ** 2)
    assert np.all(np.abs(G - ref) <= 1e-10 * np.outer(dg, dg) + np.outer(floor, floor) + np.outer(floor, dg) * 2 + 1e-300)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)


@pytest.mark.parametrize("d,n,rs", [(3, 100, (5, 20)), (8, 64, (64,)), (16, 40, (7,))])
def test_cluster_leverage(oracle, cluster, d, n, rs):
    t, K = _block(oracle, d, 15_000, n)
    cluster.set_points(t.points)
    cluster.split(t.center, n, 2.0)
    sv, V = oracle.right_factor(K)
    for r in rs:
        W = V[:, :r] / sv[:r]
        ref, _ = oracle.row_leverage_scores(K, r)
        got = cluster.leverage(t.h, W)
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, ref.max())


def test_cluster_small_blocks(oracle, cluster):
    """Fewer targets than one tile, a ragged last tile, and an empty block through the cluster kernel."""
    sr = oracle.gen_normal(3, 11, 4)
    for nt in (7, 33, 95):
        tg = oracle.gen_normal(3, nt, 3) * 0.5 + 1.0
        cluster.set_block(tg, sr)
        Kb = oracle.kernel_matrix(tg, sr, 1.3)
        G, sk = cluster.gram(1.3)
        assert _gram_ok(G, Kb.T @ Kb) and sk == pytest.approx(np.sum(Kb * Kb), rel=1e-12)
    cluster.set_block(np.zeros((0, 3)), sr)
    G, sk = cluster.gram(1.3)
    assert sk == 0.0 and np.all(G == 0.0)
    skel, P = np.array([0, 3]), np.zeros((2, 11))
    P[:, skel] = np.eye(2)
    P[:, [1, 2]] = 0.5
    sd, sk, DtD, _ = cluster.recon_error(1.3, skel, P)
    assert sd == 0.0 and sk == 0.0 and np.all(DtD == 0.0)


# --------------------------------------------------------------------------- the BASELINE large-m shapes
@pytest.mark.parametrize("d,n,eps", [(16, 256, 1e-2), (16, 256, 1e-8), (8, 512, 1e-2), (8, 512, 1e-12),
                                     (8, 256, 1e-4)])
def test_large_m_residual(oracle, dev, d, n, eps):
    """c4 (m = 256, d = 16) and c5 (m = 512, d = 8) shapes on 1.2e4 points: the cluster kernel is the
    only path (AUTO), so these run without kid_set_path."""
    t, K = _block(oracle, d, 12_000, n)
    res, DtD, r_KtK = _check_resid(oracle, dev, t, K, n, eps, s=0.2)
    G, gsk = dev.gram(t.h)
    assert _gram_ok(G, r_KtK)


@pytest.mark.parametrize("d,n", [(16, 256), (8, 512), (5, 300), (3, 129), (64, 256)])
def test_large_m_gram_parts(oracle, dev, d, n):
    """The m x m Gram for m > 128 does not fit one SM's registers: parts (grid.y), each evaluating only the
    columns of its blocks, every block written once. Both kernels -- the two-phase k_gram2 (the automatic
    choice; d = 64 falls back to the cluster kernel: shared memory) and the warp-specialised cluster kernel
    k_fused -- against the oracle; ragged column groups (m = 300, 129), run-to-run bitwise equality."""
    xi = 1.0 if d < 64 else 0.0
    t, K = _block(oracle, d, 9_000, n, xi=xi)
    dev.set_points(t.points)
    dev.split(t.center, n, xi)
    ref = K.T @ K
    try:
        for kern in (0, 1):
            dev.set_option(3, kern)
            G, sk = dev.gram(t.h)
            assert dev.last_kernel() == ("k_gram2" if kern == 0 and d < 64 else "k_fused")
            assert _gram_ok(G, ref), kern
            assert np.array_equal(G, G.T)
            assert sk == pytest.approx(np.sum(K * K), rel=1e-12)
            G2, sk2 = dev.gram(t.h)
            assert np.array_equal(G, G2) and sk == sk2
    finally:
        dev.set_option(3, 0)


@pytest.mark.parametrize("d,n,N", [(2, 100, 20_000), (3, 37, 5_000), (8, 16, 40), (16, 130, 4_000), (7, 8, 1_000), (1, 20, 3_000)])
def test_gram2_small_and_ragged(oracle, dev, d, n, N):
    """k_gram2 forced (KID_OPT_KERNEL = 3) on small / ragged blocks: one diagonal part with padded warp tiles,
    fewer targets than one tile, m not a multiple of 8, generic d."""
    t, K = _block(oracle, d, N, n, xi=1.0)
    dev.set_points(t.points)
    dev.split(t.center, n, 1.0)
    try:
        dev.set_path(1)
        dev.set_option(3, 3)
        G, sk = dev.gram(t.h)
        assert dev.last_kernel() == "k_gram2"
    finally:
        dev.set_option(3, 0)
        dev.set_path(0)
    assert _gram_ok(G, K.T @ K)
    assert np.array_equal(G, G.T)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)


@pytest.mark.parametrize("d,n,r", [(16, 256, 86), (8, 512, 300), (8, 512, 20)])
def test_large_m_leverage(oracle, dev, d, n, r):
    t, K = _block(oracle, d, 9_000, n, xi=1.0)
    dev.set_points(t.points)
    dev.split(t.center, n, 1.0)
    sv, V = oracle.right_factor(K)
    W = V[:, :r] / sv[:r]
    ref, _ = oracle.row_leverage_scores(K, r)
    got = dev.leverage(t.h, W)
    assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, ref.max())


def test_cluster_matches_single_cta(oracle, dev):
    """Same block, both kernel families: residual Grams agree to the rounding ladder and the
    cluster kernel is bitwise reproducible run to run."""
    t, K = _block(oracle, 3, 30_000, 100)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], 0.05, 9)
    res = oracle.compress_id(K, rows, eps=1e-6)
    dev.set_points(t.points)
    dev.split(t.center, 100, 2.0)
    a = dev.recon_error(t.h, res.skeleton, res.P)
    dev.set_path(1)
    try:
        b = dev.recon_error(t.h, res.skeleton, res.P)
        b2 = dev.recon_error(t.h, res.skeleton, res.P)
    finally:
        dev.set_path(0)
    assert np.array_equal(b[2], b2[2]) and b[0] == b2[0] and b[1] == b2[1]
    _, _, r_DtD, _ = oracle.residual_stats(K, res.skeleton, res.P)
    bound, _, _ = _resid_bound(K, res, r_DtD)
    assert np.all(np.abs(a[2] - b[2]) <= 2 * bound + 1e-300)
    assert a[1] == pytest.approx(b[1], rel=1e-13)
