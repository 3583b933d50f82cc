"""GPU parity of the remaining SURVEY.md 8f item-4 callers: interaction_fractions
(compress.hpp:327-378, block Grams on the device) and bandwidth_search (harness.hpp:330-438,
one device TSQR spectrum per evaluated h), against the oracle restatements and the reference's
own known answers (test_compress.cpp:180-190, test_harness.cpp:244-280, acceptance.cpp:78-98)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_interaction_fractions_constant_kernel(oracle):
    from paper_1409_2802_b200 import kernid as H
    from paper_1409_2802_b200._lib import KID_E_RANGE
    f = H.interaction_fractions(3, 160, 71, 1e100, np.zeros(3), 40)  # K == 1 exactly
    assert f[0] == pytest.approx(0.5, rel=1e-10)
    assert f[1] == pytest.approx(0.5, rel=1e-10)
    assert f[2] == pytest.approx(math.sqrt(0.5), rel=1e-10)
    with pytest.raises(H.KidError) as e:
        H.interaction_fractions(3, 160, 71, 1e100, np.zeros(3), 81)
    assert e.value.code == KID_E_RANGE


@pytest.mark.parametrize("d,N,n", [(3, 4000, 100), (2, 3000, 37), (5, 2000, 64)])
def test_interaction_fractions_vs_oracle(oracle, d, N, n):
    from paper_1409_2802_b200 import kernid as H
    seed = oracle.derive_seed(20240601, d, 0xF4)
    h = oracle.silverman_bandwidth(d, N)
    got = H.interaction_fractions(d, N, seed, h, np.zeros(d), n)
    ref = oracle.interaction_fractions(oracle.gen_normal(d, N, seed), h, np.zeros(d), n)
    for g, r in zip(got, ref):
        assert g == pytest.approx(r, rel=1e-10, abs=1e-15)


@pytest.mark.parametrize("d,expect,tol", [(4, (84.44, 40.52, 38.09), 5.0), (64, (100.0, 0.0, 0.0), 1.0)])
def test_interaction_fractions_acceptance(oracle, d, expect, tol):
    """acceptance.cpp criterion 3: N = 1e5 N(0, I_d) points, n = 500, h_S, center 0."""
    from paper_1409_2802_b200 import kernid as H
    N, n = 100_000, 500
    f = H.interaction_fractions(d, N, oracle.derive_seed(20240601, d, 0xF4), oracle.silverman_bandwidth(d, N),
                                np.zeros(d), n)
    for g, e in zip(f, expect):
        assert abs(100.0 * g - e) <= tol, (d, f)


@pytest.mark.parametrize("large_h", [False, True])
def test_bandwidth_search_vs_oracle(oracle, large_h):
    from paper_1409_2802_b200 import kernid as H
    seed = oracle.derive_seed(3, 0, 0xB5)
    got = H.bandwidth_search(2, 4000, 100, 1.0, seed, kappa=0.2, large_h=large_h, eps=1e-2, tol_rows=2)
    h_abs, ratio, rank, evals, conv, prof = oracle.bandwidth_search(2, 4000, 100, 1.0, seed, kappa=0.2,
                                                                     large_h=large_h, eps=1e-2, tol_rows=2)
    assert [r for _, r in got["profile"]] == [r for _, r in prof]
    assert np.allclose([h for h, _ in got["profile"]], [h for h, _ in prof], rtol=1e-15)
    assert got["h_abs"] == pytest.approx(h_abs, rel=1e-15) and got["rank"] == rank
    assert got["evaluations"] == evals and got["converged"] == conv
    assert conv and abs(rank - 20) <= 2  # test_harness.cpp:259-260


def test_bandwidth_search_degenerate_budget(oracle):
    """test_harness.cpp:267-280: full rank at eps = 1e-14 either fails to bracket (profile kept)
    or lands where the rank saturates near n."""
    from paper_1409_2802_b200 import kernid as H
    seed = oracle.derive_seed(3, 0, 0xB5)
    try:
        r = H.bandwidth_search(2, 4000, 100, 1.0, seed, kappa=1.0, eps=1e-14)
        assert r["rank"] >= 90
    except H.SearchFailure as e:
        assert len(e.profile) > 0


def test_bandwidth_search_acceptance(oracle):
    """acceptance.cpp criterion 2: d = 4, N = 1e5, n = 500, xi = 1, kappa = 0.2, eps = 1e-2, seed
    20240601; mean h / h_S over 5 seeds: small_h branch 0.1656 +- 0.024, large_h 1.1719 +- 0.05
    (m = 500: the Gram route, eigenvalues by the tridiagonal QL solver)."""
    from paper_1409_2802_b200 import kernid as H
    ratios = {False: [], True: []}
    for large in (False, True):
        for seed_idx in range(5):
            r = H.bandwidth_search(4, 100_000, 500, 1.0, oracle.derive_seed(20240601, seed_idx, 0xB5), kappa=0.2,
                                   large_h=large, eps=1e-2, max_iters=40, tol_rows=2)
            ratios[large].append(r["h_over_hs"])
    small, large_ = np.mean(ratios[False]), np.mean(ratios[True])
    assert abs(small - 0.1656) <= 0.024, ratios
    assert abs(large_ - 1.1719) <= 0.05, ratios
