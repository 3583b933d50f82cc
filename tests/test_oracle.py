"""Pins the CPU oracle (oracle/kernid_oracle.c) before it is trusted as the checker.

1. RNG streams: bit-exact against tests/golden/rng_ref.json, produced by the
   REFERENCE's own rng.hpp compiled into oracle/_ref (make_rng_golden.py).
2. The reference's known-answer / property tests for the hot path
   (proj/tests/test_geometry.cpp, test_kernel.cpp, test_sampling.cpp,
   test_lowrank.cpp, test_compress.cpp), ported case by case.
3. Independent LAPACK (numpy) cross-checks of the QR/SVD stand-ins.
"""
import json
import math
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _hex2d(h):
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


def random_matrix(O, m, n, seed):
    # proj/tests/test_lowrank.cpp:12-18: a(i, j) = rng.normal(), i outer
    return O.gen_normal(n, m, seed)


# ---------------------------------------------------------------- RNG pin
def test_rng_streams_bit_exact_vs_reference_build(oracle):
    gold = json.load(open(os.path.join(HERE, "golden", "rng_ref.json")))
    assert len(gold["streams"]) >= 4
    for st in gold["streams"]:
        seed = st["seed"]
        n = len(st["u64"])
        u64, un, nm, bl = oracle.rng_dump(seed, n)
        assert [int(x) for x in u64] == st["u64"]
        assert [struct.pack("<d", x) for x in un] == [struct.pack("<d", _hex2d(h)) for h in st["uniform01"]]
        assert [struct.pack("<d", x) for x in nm] == [struct.pack("<d", _hex2d(h)) for h in st["normal"]]
        assert [int(x) for x in bl] == st["below_1000003"]
        for a, b, v in st["derive_seed"]:
            assert oracle.derive_seed(seed, a, b) == v
        assert oracle.derive_seed(seed, 0xDA7A) == st["derive_special"][0]
        assert oracle.derive_seed(seed, 0xCE) == st["derive_special"][1]
        pts = oracle.gen_normal(3, n, oracle.derive_seed(seed, 0xDA7A))
        flat = pts.T.ravel()  # col-major
        assert [struct.pack("<d", x) for x in flat] == [struct.pack("<d", _hex2d(h)) for h in st["gen_normal_d3"]]


def test_mt19937_64_standard_check_value(oracle):
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64 (seed 5489)
    u64, _, _, _ = oracle.rng_dump(5489, 10000)
    assert int(u64[-1]) == 9981545732273789042


# ------------------------------------------------------- test_geometry.cpp
LINE = np.array([[0.0], [0.1], [-0.1], [0.5], [-0.5], [2.0], [-2.0], [3.0]])


def test_split_line_example(oracle):  # test_geometry.cpp:17-24
    s = oracle.split_sources_targets(LINE, [0.0], 3, 2.0)
    assert list(s.source_indices) == [0, 1, 2]
    assert s.rho == pytest.approx(0.1)
    assert list(s.target_indices) == [3, 4, 5, 6, 7]


def test_split_xi_zero_keeps_all_nonsources(oracle):  # :26-30
    ps = oracle.gen_normal(3, 200, 5)
    s = oracle.split_sources_targets(ps, np.zeros(3), 40, 0.0)
    assert s.target_indices.size == 160


def test_split_errors(oracle):  # :32-39
    with pytest.raises(oracle.OracleError) as e:
        oracle.split_sources_targets(LINE, [0.0], 3, 100.0)
    assert e.value.code == oracle.E_NO_TARGETS
    for n in (0, 8):
        with pytest.raises(oracle.OracleError) as e:
            oracle.split_sources_targets(LINE, [0.0], n, 1.0)
        assert e.value.code == oracle.E_RANGE
    with pytest.raises(oracle.OracleError) as e:
        oracle.split_sources_targets(LINE, [0.0, 0.0], 3, 1.0)
    assert e.value.code == oracle.E_DIM


def test_split_deterministic_disjoint(oracle):  # :41-52
    ps = oracle.gen_normal(4, 500, 9)
    a = oracle.split_sources_targets(ps, np.zeros(4), 50, 1.0)
    b = oracle.split_sources_targets(ps, np.zeros(4), 50, 1.0)
    assert np.array_equal(a.source_indices, b.source_indices)
    assert np.array_equal(a.target_indices, b.target_indices)
    assert not set(a.source_indices) & set(a.target_indices)
    nrm = np.sqrt((ps ** 2).sum(1))
    assert np.all(nrm[a.source_indices] <= a.rho * (1 + 1e-15))
    assert np.all(nrm[a.target_indices] >= a.xi * a.rho * (1 - 1e-15))


def test_split_survival_collapses_with_dimension(oracle):  # :54-69
    def survival(d, xi):
        ps = oracle.gen_normal(d, 20000, 13 + d)
        return oracle.split_sources_targets(ps, np.zeros(d), 200, xi).target_indices.size

    d2 = survival(2, 1.0) / survival(2, 2.0)
    d8 = survival(8, 1.0) / survival(8, 2.0)
    d32 = survival(32, 1.0) / survival(32, 2.0)
    assert d2 < d8 < d32 and d32 > 10.0


def test_split_ties_break_by_index(oracle):
    # every point equidistant: nth_element with (dist, idx) keeps the lowest indices
    ps = np.array([[1.0], [-1.0], [1.0], [-1.0], [1.0], [5.0]])
    s = oracle.split_sources_targets(ps, [0.0], 3, 1.0)
    assert list(s.source_indices) == [0, 1, 2]
    assert list(s.target_indices) == [3, 4, 5]


# --------------------------------------------------------- test_kernel.cpp
def test_gaussian_closed_forms(oracle):  # test_kernel.cpp:17-29
    x = np.array([0.3, -1.2, 0.7])
    assert oracle.eval_gaussian(x, x, 1.0) == 1.0
    assert oracle.eval_gaussian([0.0], [2.0], 2.0) == pytest.approx(math.exp(-0.5), rel=1e-12)


def test_silverman_table(oracle):  # :50-63
    assert oracle.silverman_bandwidth(4, 100000) == pytest.approx(0.2143, abs=5e-5)
    assert oracle.silverman_bandwidth(16, 100000) == pytest.approx(0.5060, abs=5e-5)
    assert oracle.silverman_bandwidth(64, 100000) == pytest.approx(0.8022, abs=5e-5)
    for d in (1, 4, 12):
        prev = oracle.silverman_bandwidth(d, 10)
        for N in (100, 10000, 1000000):
            h = oracle.silverman_bandwidth(d, N)
            assert h < prev
            prev = h
    with pytest.raises(oracle.OracleError):
        oracle.silverman_bandwidth(0, 10)


def test_kernel_matrix_examples(oracle):  # :65-84
    t = np.array([[0.1, 0.2, 0.3]])
    s = np.array([[-0.4, 0.0, 1.0]])
    K = oracle.kernel_matrix(t, s, 0.7)
    assert K.shape == (1, 1) and K[0, 0] == oracle.eval_gaussian(t[0], s[0], 0.7)
    K = oracle.kernel_matrix(np.array([[1.0, 0, 0], [2.0, 0, 0]]), np.zeros((1, 3)), 1.0)
    assert K[0, 0] == pytest.approx(math.exp(-0.5), rel=1e-14)
    assert K[1, 0] == pytest.approx(math.exp(-2.0), rel=1e-14)


def test_kernel_matrix_entrywise_exact_and_symmetric(oracle):  # :86-107
    tg = oracle.gen_normal(5, 20, 11)
    sr = oracle.gen_normal(5, 5, 12)
    K = oracle.kernel_matrix(tg, sr, 0.8)
    for i in range(20):
        for j in range(5):
            assert K[i, j] == oracle.eval_gaussian(tg[i], sr[j], 0.8)
    a = oracle.gen_normal(4, 13, 21)
    b = oracle.gen_normal(4, 7, 22)
    assert np.array_equal(oracle.kernel_matrix(a, b, 0.5).T, oracle.kernel_matrix(b, a, 0.5))
    # threaded row-block assembly is bitwise independent of the thread count
    big_t = oracle.gen_normal(3, 5000, 3)
    assert np.array_equal(oracle.kernel_matrix(big_t, sr[:, :3], 0.4, threads=1),
                          oracle.kernel_matrix(big_t, sr[:, :3], 0.4, threads=7))


def test_gaussian_range_and_monotone(oracle):  # :109-121
    prev = 2.0
    for r in (0.0, 0.1, 0.5, 1.0, 2.5, 7.0):
        v = oracle.eval_gaussian(np.zeros(3), [r, 0.0, 0.0], 0.9)
        assert 0.0 < v <= 1.0 and v < prev
        if r == 0.0:
            assert v == 1.0
        prev = v


# ------------------------------------------------------- test_sampling.cpp
def test_uniform_counts_and_determinism(oracle):  # test_sampling.cpp:19-43
    a = oracle.sample_rows(oracle.SCHEME_UNIFORM, 10, 0.3, 5)
    assert a.size == 3 and len(set(a)) == 3 and a.min() >= 0 and a.max() < 10
    full = oracle.sample_rows(oracle.SCHEME_UNIFORM, 10, 1.0, 6)
    assert sorted(full) == list(range(10))
    for s in (0.0, 1.5):
        with pytest.raises(oracle.OracleError):
            oracle.sample_rows(oracle.SCHEME_UNIFORM, 10, s, 7)
    x = oracle.sample_rows(oracle.SCHEME_UNIFORM, 1000, 0.1, 42)
    assert np.array_equal(x, oracle.sample_rows(oracle.SCHEME_UNIFORM, 1000, 0.1, 42))
    assert not np.array_equal(x, oracle.sample_rows(oracle.SCHEME_UNIFORM, 1000, 0.1, 43))


def test_with_replacement_duplicates(oracle):  # :45-56
    dup = False
    for seed in range(30):
        s = oracle.sample_rows(oracle.SCHEME_UNIFORM, 5, 1.0, seed, replacement=True)
        assert s.size == 5
        dup = dup or len(set(s)) < 5
    assert dup


def test_euclidean_dominant_row(oracle):  # :73-87
    K = np.full((100, 2), 1e-6)
    K[17] = 1e6
    w = oracle.row_norms(K)
    hits = sum(int(oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, 100, 0.01, seed, w)[0] == 17)
               for seed in range(1000))
    assert hits >= 999


def test_weighted_marginals(oracle):  # :89-107
    K = (np.arange(10, dtype=float) + 1.0).reshape(10, 1)
    w = oracle.row_norms(K)
    counts = np.zeros(10)
    trials = 20000  # reference uses 1e5 at tolerance 0.01; 2e4 keeps the CPU suite fast (3 sigma < 0.01)
    for t in range(trials):
        counts[oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, 10, 0.05, oracle.derive_seed(777, t), w,
                                  replacement=True)[0]] += 1
    assert np.all(np.abs(counts / trials - (np.arange(10) + 1.0) / 55.0) < 0.01)


def test_leverage_lone_row(oracle):  # :109-131
    m = 40
    K = np.zeros((m, 6))
    K[0, 0] = 1.0
    K[1:, 1] = 1.0
    sc, _ = oracle.row_leverage_scores(K, 2)
    hits = sum(int(oracle.sample_rows(oracle.SCHEME_LEVERAGE, m, 1.0 / m, oracle.derive_seed(888, t), sc)[0] == 0)
               for t in range(2000))
    assert hits / 2000 >= 0.45


def test_zero_weight_is_error(oracle):  # :160-167
    w = oracle.row_norms(np.zeros((6, 3)))
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, 6, 0.5, 3, w)
    assert e.value.code == oracle.E_ERROR


def test_without_replacement_distinct_every_scheme(oracle):  # :226-247
    ps = oracle.gen_normal(3, 150, 2024)
    sp = oracle.split_sources_targets(ps, np.zeros(3), 30, 1.0)
    K = oracle.kernel_matrix(ps[sp.target_indices], ps[sp.source_indices], 0.8)
    m = K.shape[0]
    lev, _ = oracle.row_leverage_scores(K, 5)
    for kind, w in ((oracle.SCHEME_UNIFORM, None), (oracle.SCHEME_EUCLIDEAN, oracle.row_norms(K)),
                    (oracle.SCHEME_LEVERAGE, lev)):
        s = oracle.sample_rows(kind, m, 0.33, 9, w)
        assert s.size == (m * 33 + 99) // 100 and len(set(s)) == s.size


# -------------------------------------------------------- test_lowrank.cpp
def test_singular_values_vs_lapack(oracle):  # :22-76 (QR-reduction vs direct SVD, 1e-10 sigma1)
    for shape, seed in (((3000, 25), 8), ((12, 7), 5), ((7, 12), 6), ((40, 40), 7)):
        a = random_matrix(oracle, *shape, seed)
        sv = oracle.singular_values(a)
        ref = np.linalg.svd(a, compute_uv=False)
        assert np.max(np.abs(sv - ref)) <= 1e-10 * ref[0]
    a = np.diag([3.0, 2.0, 1.0])
    assert np.allclose(oracle.singular_values(a), [3, 2, 1], rtol=1e-14)


def test_epsilon_rank(oracle):  # :89-101
    sv = np.array([1.0, 0.5, 1e-3])
    assert oracle.epsilon_rank(sv, 1e-2) == 2
    assert oracle.epsilon_rank(np.ones(5), 0.5) == 5
    assert oracle.epsilon_rank(np.array([1.0, 1e-3, 1e-4]), 1e-2) == 1
    assert oracle.epsilon_rank(np.zeros(4), 0.5) == 0
    assert oracle.epsilon_rank(sv, 1e-2, 200.0) == 0
    assert oracle.epsilon_rank(sv, 1e-2, 10.0) == 2
    with pytest.raises(oracle.OracleError):
        oracle.epsilon_rank(sv, 1.5)


def test_id_known_answers(oracle):  # :141-198
    skel, P = oracle.interpolative_decomposition(np.ones((4, 3)), 1)
    assert list(skel) == [0] and np.allclose(P, 1.0, rtol=1e-13)
    a = random_matrix(oracle, 10, 6, 61)
    skel, P = oracle.interpolative_decomposition(a, 6)
    assert np.linalg.norm(a[:, skel] @ P - a) < 1e-10 * np.linalg.norm(a)
    assert sorted(skel) == list(range(6))
    a = random_matrix(oracle, 20, 12, 81)
    for r in (1, 4, 9):
        skel, P = oracle.interpolative_decomposition(a, r)
        assert np.array_equal(P[:, skel], np.eye(r))  # exact identity submatrix
    u = random_matrix(oracle, 8, 1, 91)
    v = random_matrix(oracle, 5, 1, 92)
    with pytest.raises(oracle.OracleError) as e:
        oracle.interpolative_decomposition(u @ v.T, 3)
    assert e.value.code == oracle.E_ILLCOND
    with pytest.raises(oracle.OracleError) as e:
        oracle.interpolative_decomposition(u @ v.T, 0)
    assert e.value.code == oracle.E_RANGE


def test_id_error_bound_random(oracle):  # :200-225
    for t in range(30):
        rng = np.random.default_rng(t)
        n = 3 + int(rng.integers(25))
        m = n + int(rng.integers(30))
        r = 1 + int(rng.integers(n))
        a = random_matrix(oracle, m, n, oracle.derive_seed(2000, t))
        sv = np.linalg.svd(a, compute_uv=False)
        try:
            skel, P = oracle.interpolative_decomposition(a, r)
        except oracle.OracleError:
            continue
        err = np.linalg.norm(a - a[:, skel] @ P, 2)
        s1 = sv[r] if r < sv.size else 0.0
        assert err <= math.sqrt(1 + n * r * (n - r)) * s1 + 1e-8 * sv[0]


def test_row_leverage(oracle):  # :227-246
    a = random_matrix(oracle, 18, 7, 131)
    for r in (1, 4, 7):
        sc, _ = oracle.row_leverage_scores(a, r)
        assert sc.sum() == pytest.approx(r, rel=1e-10)
        U = np.linalg.svd(a, full_matrices=False)[0][:, :r]
        assert np.allclose(sc, (U ** 2).sum(1), atol=1e-10)
    # Gram-eigen route (proj/tests/oracles.hpp:68-83)
    ev, V = oracle.jacobi_eigen(a.T @ a)
    W = V[:, :4] / np.sqrt(ev[:4])
    assert np.allclose(((a @ W) ** 2).sum(1), oracle.row_leverage_scores(a, 4)[0], atol=1e-8)
    _, gap = oracle.row_leverage_scores(np.eye(5), 2)
    assert gap


def test_power_iteration_matches_exact(oracle):  # :285-288
    a = random_matrix(oracle, 60, 25, 171)
    assert oracle.power_iteration_norm(a) == pytest.approx(oracle.spectral_norm_exact(a), rel=1e-5)


# ------------------------------------------------------- test_compress.cpp
def test_rank_one_compresses_exactly(oracle):  # test_compress.cpp:37-48
    u = np.abs(random_matrix(oracle, 60, 1, 1))
    v = np.abs(random_matrix(oracle, 12, 1, 2))
    K = u @ v.T
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, 60, 0.1, 3)
    res = oracle.compress_id(K, rows, eps=1e-2)
    assert res.rank == 1 and res.rel_error < 1e-10


def test_rank_zero_and_empty(oracle):  # :82-95
    K = np.zeros((40, 10))
    res = oracle.compress_id(K, oracle.sample_rows(oracle.SCHEME_UNIFORM, 40, 0.25, 5), eps=1e-2)
    assert res.rank == 0 and res.rank_zero and res.rel_error == 1.0
    with pytest.raises(oracle.OracleError):
        oracle.compress_id(random_matrix(oracle, 10, 4, 6), np.zeros(0, np.int64), eps=1e-2)


def test_precomputed_norm_shortcut(oracle):  # :218-226
    K = np.abs(random_matrix(oracle, 80, 25, 81))
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, 80, 0.5, 9)
    a = oracle.compress_id(K, rows, eps=1e-3)
    b = oracle.compress_id(K, rows, eps=1e-3, k_norm=oracle.spectral_norm_exact(K))
    assert a.rel_error == pytest.approx(b.rel_error, rel=1e-12)


def test_full_sampling_obeys_id_bound(oracle):  # :50-66
    K = random_matrix(oracle, 90, 30, 11)
    sv = np.linalg.svd(K, compute_uv=False)
    res = oracle.compress_id(K, np.arange(90), eps=1e-2)
    r = res.rank
    s1 = sv[r] if r < sv.size else 0.0
    assert res.rel_error <= math.sqrt(1 + 30.0 * r * (30.0 - r)) * s1 / sv[0] + 1e-8


def test_gaussian_instance_error_and_norm_paths(oracle):  # :119-141 fixture (d=3, N=3000, n=100, xi=1, h=0.6)
    ps = oracle.gen_normal(3, 3000, 41)
    sp = oracle.split_sources_targets(ps, np.zeros(3), 100, 1.0)
    K = oracle.kernel_matrix(ps[sp.target_indices], ps[sp.source_indices], 0.6)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], 0.2, 3)
    res = oracle.compress_id(K, rows, eps=1e-4)
    assert res.rank > 0
    # exact path vs numpy, and the power-iteration path vs the exact path (1e-5)
    D = K[:, res.skeleton] @ res.P - K
    ref = np.linalg.norm(D, 2) / np.linalg.norm(K, 2)
    assert res.rel_error == pytest.approx(ref, rel=1e-9)
    pw = oracle.compress_id(K, rows, eps=1e-4, budget=1.0)
    assert pw.rel_error == pytest.approx(res.rel_error, rel=1e-5)
    # residual-Gram route (the fused pass' math) agrees with the exact spectral norm
    sd, sk, DtD, KtK = oracle.residual_stats(K, res.skeleton, res.P)
    lam_d = np.linalg.eigvalsh(DtD)[-1]
    lam_k = np.linalg.eigvalsh(KtK)[-1]
    assert math.sqrt(lam_d / lam_k) == pytest.approx(res.rel_error, rel=1e-8)
    assert sd == pytest.approx(np.sum(D * D), rel=1e-12)
    assert sk == pytest.approx(np.sum(K * K), rel=1e-12)


# ---------------------------------------------------------------- SURVEY.md 8(f) rows
def test_oracle_bernoulli_draw(oracle):
    """Bernoulli (sampling.hpp:183-188): i kept iff uniform01 < s, in row order; s outside (0, 1]
    is a RangeError."""
    seed = oracle.derive_seed(4, 2, 0)
    got = oracle.sample_rows(oracle.SCHEME_BERNOULLI, 500, 0.3, seed)
    _, unif, _, _ = oracle.rng_dump(seed, 500)
    assert np.array_equal(got, np.nonzero(unif < 0.3)[0])
    assert oracle.sample_rows(oracle.SCHEME_BERNOULLI, 50, 1.0, seed).size == 50
    with pytest.raises(oracle.OracleError):
        oracle.sample_rows(oracle.SCHEME_BERNOULLI, 50, 0.0, seed)


def test_oracle_apply_skeleton_and_errors(oracle):
    """apply_skeleton equals K[:, skel] (P q); mc_error with s_mc = 1 equals the full relative
    error; the SVD-path numerator equals ||K V V^T - K|| (compress.hpp:243-325)."""
    t = oracle.prepare_trial(2, 3000, 30, 2.0, oracle.derive_seed(1, 0, 0))
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], 0.1, 3)
    res = oracle.compress_id(K, rows, eps=1e-4)
    q = np.linspace(-1.0, 1.0, K.shape[1])
    u = oracle.apply_skeleton(t.targets, t.sources[res.skeleton], t.h, res.P, q)
    assert np.allclose(u, K[:, res.skeleton] @ (res.P @ q), rtol=1e-13, atol=1e-15)
    est = oracle.mc_error(K, res.skeleton, res.P, 1.0, 2, 7)
    assert np.allclose(est, res.rel_error, rtol=1e-12)
    _, _, Vt = np.linalg.svd(K[rows], full_matrices=True)
    Vr = np.ascontiguousarray(Vt.T[:, : res.rank])
    assert oracle.svd_error_norm(K, Vr) == pytest.approx(np.linalg.norm(K @ Vr @ Vr.T - K, 2), rel=1e-12)
    with pytest.raises(oracle.OracleError):
        oracle.mc_error(K, res.skeleton, res.P, 1.5, 2, 7)


def test_interaction_fractions_constant_kernel(oracle):  # test_compress.cpp:180-190
    """A kernel that evaluates to exactly one (Gaussian with an enormous bandwidth stands in for
    the reference's polynomial kernel): fractions 1/2, 1/2, sqrt(1/2) for N = 4n."""
    n = 40
    ps = oracle.gen_normal(3, 4 * n, 71)
    f = oracle.interaction_fractions(ps, 1e100, np.zeros(3), n)
    assert f[0] == pytest.approx(0.5, rel=1e-10)
    assert f[1] == pytest.approx(0.5, rel=1e-10)
    assert f[2] == pytest.approx(math.sqrt(0.5), rel=1e-10)
    with pytest.raises(oracle.OracleError):
        oracle.interaction_fractions(ps, 1e100, np.zeros(3), 2 * n + 1)


def test_bandwidth_search_brackets_both_branches(oracle):  # test_harness.cpp:244-266
    seed = oracle.derive_seed(3, 0, 0xB5)
    small = oracle.bandwidth_search(2, 4000, 100, 1.0, seed, kappa=0.2, eps=1e-2, tol_rows=2)
    assert small[4] and abs(small[2] - 20) <= 2
    large = oracle.bandwidth_search(2, 4000, 100, 1.0, seed, kappa=0.2, eps=1e-2, tol_rows=2, large_h=True)
    assert large[4] and large[0] > small[0]
