"""GPU parity at the BASELINE configs' real sizes (the reported configs must be the
tested ones). Each case generates the config's seeded N(0, I_d) point set with the oracle (RNG pinned
to the reference's rng.hpp), runs the device split and the fused error pass, and compares with the
oracle restatement of the reference path:

  c1     (d=2, N=1e5, m=100)        whole trial: split bits, EuclideanNorm sample + ID (oracle), the
                                    residual Grams, rel_error against the oracle's exact QR+SVD norms
  c2-d3  (d=3, N=1e6, m=100)        the bench's own trial (999,058 targets), same checks
  c4-d16 (d=16, N=1.2e7, m=256)     split bits at full size; the error pass on a 1e6-row slice
  c5     (d=8, N=1.0012e8, m=512)   split bits at full size (1e8 points); the error pass on a 4e5-row
                                    slice (the dense K of the full block is 410 GB)

Bars: split bit-exact; ||K||_F^2 1e-12; Grams |dG_jk| <= 1e-10 sqrt(G_jj G_kk) plus the rounding
floor of D = K_N - K_S P (tests/test_gpu_parity.py); rel_error 1e-10 relative (or that floor).
The Gram references of the slices are BLAS products of the oracle's K and D (the oracle's scalar
O(N m^2) loops would take minutes at m = 512).
"""
import math

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
U = 2.0 ** -53


@pytest.fixture(scope="module")
def dev():
    from paper_1409_2802_b200._lib import Device
    d = Device(0)
    yield d
    d.close()


def _trial(O, d, N, m, xi=2.0):
    return O.prepare_trial(d, N, m, xi, O.derive_seed(1, 0, 0))


def _check_split(dev, t, m, xi=2.0):
    dev.set_points(t.points)
    src, rho, nt = dev.split(t.center, m, xi)
    assert np.array_equal(src, t.split.source_indices)
    assert rho == t.split.rho
    assert nt == t.split.target_indices.size
    assert np.array_equal(dev.targets(), t.split.target_indices)


def _ladder(K, skel, P, DtD_ref):
    colnorm = np.sqrt((K * K).sum(0))
    noise = 8 * U * (colnorm + np.abs(P).T @ colnorm[skel])
    noise[skel] = 0.0
    dg = np.sqrt(np.abs(np.diag(DtD_ref)))
    return 1e-10 * np.outer(dg, dg) + np.outer(noise, dg) + np.outer(dg, noise) + np.outer(noise, noise), noise, dg


def _device_vs(O, dev, K, skel, P, h, r_sd, r_sk, r_DtD, r_KtK):
    sd, sk, DtD, _ = dev.recon_error(h, skel, P)
    # a sum of 1e7..5e10 positive terms: the oracle's own sequential sum carries ~sqrt(N) u ~ 1e-12, so
    # the full-size bar for the Frobenius sums is the Gram bar
    assert sk == pytest.approx(r_sk, rel=1e-10)
    bound, noise, dg = _ladder(K, skel, P, r_DtD)
    assert np.all(np.abs(DtD - r_DtD) <= bound + 1e-300)
    assert abs(sd - r_sd) <= 1e-10 * r_sd + 2 * np.sum(noise * dg) + np.sum(noise ** 2) + 1e-300
    G, gsk = dev.gram(h)
    dk = np.sqrt(np.abs(np.diag(r_KtK)))
    assert np.all(np.abs(G - r_KtK) <= 1e-10 * np.outer(dk, dk) + 1e-300)
    return DtD, G


@pytest.mark.parametrize("cfg,d,N,eps", [("c1", 2, 100_000, 1e-2), ("c1", 2, 100_000, 1e-8),
                                         ("c2-d3", 3, 1_000_000, 1e-2), ("c2-d3", 3, 1_000_000, 1e-8)])
def test_whole_trial(oracle, dev, cfg, d, N, eps):
    """c1 / c2-d3 end to end at full size: the oracle's trial (EuclideanNorm sample of 2% of the rows,
    ID, exact rel_error) against the device split + error pass + the host mirror's error pass."""
    from paper_1409_2802_b200 import kernid as H
    O = oracle
    t = _trial(O, d, N, 100)
    _check_split(dev, t, 100)
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    w = O.row_norms(K)
    # 1e-12 relative, plus the subnormal floor: rows whose every entry is below ~1e-154 sum subnormal
    # squares, each rounded to 2^-1075 absolute by any implementation (the oracle's own sum included)
    floor = 100 * 2.0 ** -1074 / (2.0 * np.maximum(w, 1e-300))
    assert np.all(np.abs(dev.row_norms(t.h) - w) <= 1e-12 * w + floor)
    rows = O.sample_rows(O.SCHEME_EUCLIDEAN, K.shape[0], 0.02, O.derive_seed(O.derive_seed(1, 0, 0), 0, 1), w)
    res = O.compress_id(K, rows, eps=eps)
    r_sd, r_sk, r_DtD, r_KtK = O.residual_stats(K, res.skeleton, res.P)
    DtD, G = _device_vs(O, dev, K, res.skeleton, res.P, t.h, r_sd, r_sk, r_DtD, r_KtK)
    rel, fro, knorm = H.error_pass(dev, t.h, res.skeleton, res.P)
    floor = 10 * math.sqrt(res.rank) * 2.2e-16 * np.abs(res.P).max() * math.sqrt(r_sk) / knorm
    assert abs(rel - res.rel_error) <= max(1e-10 * res.rel_error, floor), (rel, res.rel_error)
    assert knorm == pytest.approx(O.matrix_norm(K), rel=1e-10)


@pytest.mark.parametrize("cfg,d,N,m,rows,eps", [("c4-d16", 16, 12_000_000, 256, 1_000_000, 1e-2),
                                                ("c4-d16", 16, 12_000_000, 256, 1_000_000, 1e-8),
                                                ("c5", 8, 100_120_000, 512, 400_000, 1e-2)])
def test_large_config_slice(oracle, dev, cfg, d, N, m, rows, eps):
    """c4 / c5 at full size: the split of all N points bit-exact, then the fused error pass (the 2-CTA
    cluster kernel) on the first `rows` targets (kid_select_rows) against BLAS Grams of the oracle's
    K slice and D; the ID from a uniform sample of 4000 rows of the slice."""
    O = oracle
    t = _trial(O, d, N, m)
    _check_split(dev, t, m)
    tg = np.ascontiguousarray(t.targets[:rows])
    del t.targets
    K = O.kernel_matrix(tg, t.sources, t.h)
    smp = O.sample_rows(O.SCHEME_UNIFORM, rows, 4000.0 / rows, 11)
    res = O.compress_id(K[smp], np.arange(smp.size), eps=eps)
    skel, P = res.skeleton, res.P
    D = K - K[:, skel] @ P
    D[:, skel] = 0.0
    r_DtD, r_KtK = D.T @ D, K.T @ K
    r_sd, r_sk = float(np.sum(D * D)), float(np.sum(K * K))
    dev.select_rows(np.arange(rows, dtype=np.int64))
    try:
        _device_vs(O, dev, K, skel, P, t.h, r_sd, r_sk, r_DtD, r_KtK)
        assert dev.last_kernel() in ("k_fused", "k_gram2")  # the last pass of _device_vs: K^T K (m > 128)
    finally:
        dev.select_rows(None)
