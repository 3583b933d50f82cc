"""GPU tests of the host C++ mirror (libkernid_host.so): whole compress trials and the
run_experiment CSV sweep through the device path, checked against the oracle pipeline
(prepare_trial -> kernel_matrix -> sample_rows -> compress_id, compress.hpp:168-215)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle_trial(O, d, N, n, xi, data_seed, scheme, s, sample_seed, eps, lev_rank=0):
    t = O.prepare_trial(d, N, n, xi, data_seed)
    K = O.kernel_matrix(t.targets, t.sources, t.h)
    w = None
    if scheme == O.SCHEME_EUCLIDEAN:
        w = O.row_norms(K)
    elif scheme == O.SCHEME_LEVERAGE:
        if lev_rank <= 0:  # auto rank from the full spectrum (harness.hpp:176-184)
            lev_rank = max(1, O.epsilon_rank(O.singular_values(K), eps))
        w, _ = O.row_leverage_scores(K, lev_rank)
    rows = O.sample_rows(scheme, K.shape[0], s, sample_seed, w)
    res = O.compress_id(K, rows, eps=eps)
    return t, K, rows, res


@pytest.mark.parametrize("d,scheme,eps,lev", [(2, 2, 1e-8, 0), (3, 2, 1e-2, 0), (2, 0, 1e-8, 0), (3, 4, 1e-4, 8),
                                              (1, 2, 1e-8, 0), (3, 4, 1e-6, 0), (2, 4, 1e-9, 0)])
def test_compress_trial_matches_oracle(oracle, d, scheme, eps, lev):
    from paper_1409_2802_b200 import kernid as H
    N, n, xi = 20000, 100, 2.0
    data_seed = oracle.derive_seed(1, 0, 0)
    sample_seed = oracle.derive_seed(data_seed, 0, 1)
    s = 0.02
    got = H.compress_trial(d, N, n, xi, data_seed, scheme, s, sample_seed, eps, lev_rank=lev)
    t, K, rows, res = _oracle_trial(oracle, d, N, n, xi, data_seed, scheme, s, sample_seed, eps, lev)
    assert got.n_targets == K.shape[0]
    assert np.array_equal(got.sample, rows)
    assert got.rank == res.rank
    assert np.array_equal(got.skeleton, res.skeleton)
    floor = 10 * math.sqrt(max(res.rank, 1)) * 2.2e-16 * (np.abs(res.P).max() if res.rank else 1.0) * \
        math.sqrt(np.sum(K * K)) / oracle.spectral_norm_exact(K)
    assert abs(got.rel_error - res.rel_error) <= max(1e-10 * res.rel_error, floor)
    if res.rank:
        D = K[:, res.skeleton] @ res.P - K
        fro = math.sqrt(np.sum(D * D) / np.sum(K * K))
        assert abs(got.rel_error_fro - fro) <= max(1e-10 * fro, floor)


def test_compress_trial_errors(oracle):
    from paper_1409_2802_b200 import kernid as H
    from paper_1409_2802_b200._lib import KidError, KID_E_NO_TARGETS, KID_E_RANGE
    with pytest.raises(KidError) as e:
        H.compress_trial(2, 5000, 100, 1000.0, 7, 0, 0.1, 3, 1e-2)
    assert e.value.code == KID_E_NO_TARGETS
    with pytest.raises(KidError) as e:
        H.compress_trial(2, 5000, 100, 2.0, 7, 0, 1.5, 3, 1e-2)
    assert e.value.code == KID_E_RANGE


def test_run_experiment_csv_matches_oracle(oracle, tmp_path):
    from paper_1409_2802_b200 import kernid as H
    d, N, n, xi, eps, trials = 2, 20000, 100, 2.0, 1e-8, 2
    s_grid = [0.01, 0.05]
    csv = H.run_experiment(str(tmp_path / "out.csv"), d, N, n, xi, H.EUCLIDEAN_NORM, s_grid, eps, trials=trials, seed=1)
    lines = csv.strip().splitlines()
    assert lines[0] == ("dataset,d,N,n,xi,kernel,h,method,scheme,s,trial,seed,rank,rel_error,mc_error,bound_id,"
                        "bound_sampling,elapsed_ms")
    rows = [l.split(",") for l in lines[1:]]
    body = [r for r in rows if r[10] not in ("mean", "std")]
    assert len(body) == len(s_grid) * trials
    for r in body:
        # the reference prints the seed through static_cast<long long> (harness.hpp:227)
        s, trial, seed = float(r[9]), int(r[10]), int(r[11]) % (1 << 64)
        data_seed = oracle.derive_seed(1, trial, 0)
        assert seed == oracle.derive_seed(data_seed, s_grid.index(s), 1)
        t, K, rws, res = _oracle_trial(oracle, d, N, n, xi, data_seed, oracle.SCHEME_EUCLIDEAN, s, seed, eps)
        assert int(r[12]) == res.rank
        assert float(r[13]) == pytest.approx(res.rel_error, rel=1e-8)
        assert float(r[6]) == t.h
    stats = [r for r in rows if r[10] in ("mean", "std")]
    assert len(stats) == 2 * len(s_grid)


def test_run_experiment_methods_and_mc(oracle, tmp_path):
    """methods ["id", "svd"] with an mc_error block (harness.hpp:211-289): per row the ID / SVD
    rel_error and the mean Monte Carlo estimate (seed derive_seed(data_seed, s_idx, 2)) against
    the oracle pipeline; summary rows per (scheme, s, method)."""
    from paper_1409_2802_b200 import kernid as H
    d, N, n, xi, eps, trials, s_mc, n_mc = 2, 20000, 100, 2.0, 1e-4, 2, 0.1, 2
    s_grid = [0.02]
    csv = H.run_experiment(str(tmp_path / "m.csv"), d, N, n, xi, H.EUCLIDEAN_NORM, s_grid, eps, trials=trials, seed=1,
                           methods=("id", "svd"), s_mc=s_mc, n_mc=n_mc)
    rows = [l.split(",") for l in csv.strip().splitlines()[1:]]
    body = [r for r in rows if r[10] not in ("mean", "std")]
    assert [(r[10], r[7]) for r in body] == [("0", "id"), ("0", "svd"), ("1", "id"), ("1", "svd")]
    U = 2.220446049250313e-16
    for r in body:
        trial, seed = int(r[10]), int(r[11]) % (1 << 64)
        data_seed = oracle.derive_seed(1, trial, 0)
        t, K, rws, res = _oracle_trial(oracle, d, N, n, xi, data_seed, oracle.SCHEME_EUCLIDEAN, 0.02, seed, eps)
        normK = oracle.spectral_norm_exact(K)
        floor = 10 * n * U * math.sqrt(np.sum(K * K)) / normK
        mc_seed = oracle.derive_seed(data_seed, 0, 2)
        if r[7] == "id":
            assert int(r[12]) == res.rank
            assert float(r[13]) == pytest.approx(res.rel_error, rel=1e-8)
            ref_mc = float(np.mean(oracle.mc_error(K, res.skeleton, res.P, s_mc, n_mc, mc_seed)))
        else:
            sv, V = oracle.right_factor(K[rws])
            rank = oracle.epsilon_rank(sv, eps)
            Vr = V[:, :rank]
            assert int(r[12]) == rank
            ref = oracle.svd_error_norm(K, Vr) / normK
            assert abs(float(r[13]) - ref) <= max(1e-8 * ref, floor)
            ests = []
            for rep in range(n_mc):
                sel = oracle.sample_rows(oracle.SCHEME_BERNOULLI, K.shape[0], s_mc, oracle.derive_seed(mc_seed, rep, 0))
                Ks = K[sel]
                ests.append(np.linalg.norm(Ks @ Vr @ Vr.T - Ks, 2) / np.linalg.norm(Ks, 2))
            ref_mc = float(np.mean(ests))
        assert abs(float(r[14]) - ref_mc) <= max(1e-8 * ref_mc, 10 * floor)
    stats = [r for r in rows if r[10] in ("mean", "std")]
    assert [(r[7], r[10]) for r in stats] == [("id", "mean"), ("id", "std"), ("svd", "mean"), ("svd", "std")]
    assert all(r[14] != "" for r in stats)
