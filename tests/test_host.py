"""CPU tests of the product's host side (libkernid_host.so) and of the C-ABI library.

The host steps the north star keeps on the host (K_s rows, epsilon-rank, CPQR/ID,
weighted draws, Gram eigen-solve) are checked against the oracle: draws and the ID
skeleton must be bit-identical given identical inputs.
No GPU is needed here.
"""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    from paper_1409_2802_b200 import kernid
    kernid.host_lib()
    return kernid


def test_cuda_library_exports_every_declared_symbol():
    from paper_1409_2802_b200 import _lib
    header = open(os.path.join(ROOT, "include", "kernid_cuda.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(kid_\w+)\s*\(", header, re.M))
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.CUDA_SO], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kid_\w+)", out))
    assert declared <= exported, declared - exported
    assert set(_lib.SYMBOLS) <= exported
    L = _lib.cuda_lib()  # loads without a GPU (cudart is linked statically)
    assert L.kid_abi_version() == 1


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1409_2802_b200._lib import Device, KidError
    with pytest.raises(KidError):
        Device(0)


def test_host_rng_and_points_match_oracle(H, oracle):
    for seed in (1, 42, 2**63 + 5):
        assert H.derive_seed(seed, 3, 1) == oracle.derive_seed(seed, 3, 1)
    a = H.gen_normal(3, 1000, 77)
    b = oracle.gen_normal(3, 1000, 77)
    assert np.array_equal(a, b)


def test_host_draws_match_oracle(H, oracle):
    rng = np.random.default_rng(0)
    w = rng.random(5000) ** 4
    for seed in range(5):
        for s in (0.001, 0.02, 0.3):
            assert np.array_equal(H.draw(H.UNIFORM, 5000, s, seed), oracle.sample_rows(oracle.SCHEME_UNIFORM, 5000, s, seed))
            assert np.array_equal(H.draw(H.EUCLIDEAN_NORM, 5000, s, seed, w),
                                  oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, 5000, s, seed, w))
            assert np.array_equal(H.draw(H.EUCLIDEAN_NORM, 5000, s, seed, w, replacement=True),
                                  oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, 5000, s, seed, w, replacement=True))


def test_host_kernel_rows_bit_exact(H, oracle):
    t = oracle.prepare_trial(3, 5000, 50, 2.0, oracle.derive_seed(1, 0, 0))
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    rows = np.array([0, 3, 99, K.shape[0] - 1])
    pts = np.ascontiguousarray(t.points.T).ravel()
    Ks = H.kernel_rows(pts, t.points.shape[0], 3, t.split.target_indices, rows, t.split.source_indices, t.h)
    assert np.array_equal(Ks, K[rows])


@pytest.mark.parametrize("d,eps", [(2, 1e-2), (2, 1e-8), (3, 1e-8), (3, 1e-14), (5, 1e-4)])
def test_host_id_skeleton_identical_to_oracle(H, oracle, d, eps):
    t = oracle.prepare_trial(d, 20000, 100, 2.0, oracle.derive_seed(1, 0, 0))
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    rows = oracle.sample_rows(oracle.SCHEME_UNIFORM, K.shape[0], 0.05, 11)
    sub = K[rows]
    sv_h = H.singular_values(sub)
    sv_o = oracle.singular_values(sub)
    assert np.all(np.abs(sv_h - sv_o) <= 1e-13 * sv_o[0])
    r = oracle.epsilon_rank(sv_o, eps)
    assert H.epsilon_rank(sv_h, eps) == r
    try:
        skel_o, P_o = oracle.interpolative_decomposition(sub, r)
    except oracle.OracleError as e:
        from paper_1409_2802_b200._lib import KidError
        with pytest.raises(KidError) as ee:
            H.interpolative_decomposition(sub, r)
        assert ee.value.code == e.code
        return
    skel_h, P_h = H.interpolative_decomposition(sub, r)
    assert np.array_equal(skel_h, skel_o)
    assert np.array_equal(P_h, P_o)


def test_host_sym_eig(H):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((60, 40))
    G = A.T @ A
    ev, V = H.sym_eig(G)
    ref = np.linalg.eigvalsh(G)[::-1]
    assert np.allclose(ev, ref, rtol=1e-12, atol=1e-12 * ref[0])
    assert np.allclose(V.T @ V, np.eye(40), atol=1e-12)


def test_host_errors_mirror_reference(H):
    from paper_1409_2802_b200._lib import KidError, KID_E_RANGE, KID_E_ILLCOND
    with pytest.raises(KidError) as e:
        H.epsilon_rank([1.0, 0.5], 1.5)
    assert e.value.code == KID_E_RANGE
    u = np.arange(1.0, 9.0).reshape(8, 1)
    v = np.arange(1.0, 6.0).reshape(5, 1)
    with pytest.raises(KidError) as e:
        H.interpolative_decomposition(u @ v.T, 3)
    assert e.value.code == KID_E_ILLCOND


def test_sym_eigvals_vs_lapack():
    """The eigenvalue-only host solver (Householder tridiagonalisation + implicit QL) used for the
    m > 128 spectra, against LAPACK: random PSD, a Gaussian-kernel Gram with a fast-decaying
    spectrum, repeated eigenvalues and the 1 x 1 case."""
    import numpy as np
    from paper_1409_2802_b200 import kernid as H
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 64, 300):
        X = rng.standard_normal((n + 5, n))
        A = X.T @ X
        ref = np.linalg.eigvalsh(A)[::-1]
        assert np.max(np.abs(H.sym_eigvals(A) - ref)) <= 1e-13 * ref[0]
    x = np.linspace(0.0, 1.0, 257)
    K = np.exp(-(x[:, None] - x[None, :]) ** 2 / 0.01)
    ref = np.linalg.eigvalsh(K)[::-1]
    assert np.max(np.abs(H.sym_eigvals(K) - ref)) <= 1e-13 * ref[0]
    assert np.allclose(H.sym_eigvals(np.eye(9) * 3.0), 3.0, rtol=0, atol=1e-15)


def test_sym_eig_vectors_large():
    """sym_eig for n > 128 (tridiagonal + QL with accumulated vectors): eigenpairs of a
    Gaussian-kernel Gram against LAPACK -- residual ||A V - V L|| and orthogonality at ~u."""
    import numpy as np
    from paper_1409_2802_b200 import kernid as H
    rng = np.random.default_rng(1)
    n = 200
    x = np.sort(rng.standard_normal(n))
    K = np.exp(-(x[:, None] - x[None, :]) ** 2 / 0.1)
    A = K.T @ K
    ev, V = H.sym_eig(A)
    ref = np.linalg.eigvalsh(A)[::-1]
    assert np.max(np.abs(ev - ref)) <= 1e-13 * ref[0]
    assert np.max(np.abs(A @ V - V * ev)) <= 1e-13 * ref[0]
    assert np.max(np.abs(V.T @ V - np.eye(n))) <= 1e-12


@pytest.mark.parametrize("n,kind", [(50, "rand"), (200, "rand"), (512, "rand"), (300, "cluster"), (256, "lowrank"),
                                    (129, "gram")])
def test_host_lambda_max(n, kind):
    """lambda_max (Jacobi for n <= 128, Lanczos with full reorthogonalisation above) against LAPACK:
    the spectral norms of compress_id at c4 / c5 (m = 256 / 512) come from it."""
    from paper_1409_2802_b200 import kernid as H
    rng = np.random.default_rng(n)
    if kind == "rand":
        X = rng.standard_normal((n + 7, n))
        A = X.T @ X
    elif kind == "cluster":  # top eigenvalues nearly equal: slow Lanczos convergence, exact at k = n
        Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        ev = np.concatenate([[1.0, 1.0 - 1e-9, 1.0 - 2e-9], rng.random(n - 3) * 0.5])
        A = (Q * ev) @ Q.T
    elif kind == "lowrank":  # rank 5 PSD, the numerically rank-deficient Gram of a far-field block
        X = rng.standard_normal((5, n)) * np.array([1e-3, 1e-7, 1e-11, 1e-15, 1e-20])[:, None]
        A = X.T @ X
    else:
        t = rng.standard_normal((4000, 3))
        s = rng.standard_normal((n, 3)) * 0.3
        K = np.exp(-((t[:, None, :] - s[None, :, :]) ** 2).sum(-1))
        A = K.T @ K
    A = 0.5 * (A + A.T)
    ref = np.linalg.eigvalsh(A)[-1]
    got = H.lambda_max(A)
    assert abs(got - ref) <= 1e-12 * ref, (got, ref)


def test_host_id_vs_lapack_cpqr(H):
    """An independent pin of the ID restatement (lowrank.hpp:135-262: column-pivoted Householder QR,
    P = R11^-1 [R11 R12] Pi^T): LAPACK's dgeqp3 (scipy) on sampled Gaussian-kernel rows. Both pick the
    largest remaining column norm at every step, so wherever that choice is not a near-tie the pivot
    sequences -- hence the skeletons -- must coincide, and the projections agree to the conditioning of R11."""
    import scipy.linalg as sla
    from oracle import oracle as O
    checked = 0
    for d, N, n, s, eps in [(2, 20_000, 100, 0.02, 1e-6), (3, 20_000, 100, 0.02, 1e-4), (5, 20_000, 64, 0.03, 1e-8),
                            (8, 30_000, 200, 0.02, 1e-2), (1, 10_000, 100, 0.05, 1e-10)]:
        t = O.prepare_trial(d, N, n, 2.0, O.derive_seed(1, 0, 0))
        K = O.kernel_matrix(t.targets, t.sources, t.h)
        rows = O.sample_rows(O.SCHEME_UNIFORM, K.shape[0], s, O.derive_seed(3, 0, 1))
        A = K[rows]
        r = int(H.epsilon_rank(H.singular_values(A), eps))
        if r < 1 or r >= n:
            continue
        skel, P = H.interpolative_decomposition(A, r)
        Q, R, piv = sla.qr(A, mode="economic", pivoting=True)
        # pivot steps with a clear winner: replay LAPACK's sequence and measure the margin of each choice
        W = A.copy()
        clear = True
        for k in range(r):
            nr = np.sqrt((W ** 2).sum(0))
            nr[piv[:k]] = -1.0
            order = np.argsort(nr)[::-1]
            if nr[order[1]] > (1.0 - 1e-6) * nr[order[0]]:
                clear = False
                break
            assert order[0] == piv[k]
            q = Q[:, k]
            W = W - np.outer(q, q @ W)
        if not clear:
            continue
        checked += 1
        assert np.array_equal(np.sort(skel), np.sort(piv[:r]))
        # P against LAPACK's: columns piv[:r] carry the identity, the rest R11^-1 R12
        T = sla.solve_triangular(R[:r, :r], R[:r, r:])
        P_ref = np.zeros((r, n))
        P_ref[np.arange(r), piv[:r]] = 1.0
        P_ref[:, piv[r:]] = T
        # rows of P follow the skeleton order of the ID; map both to ascending column index
        o1, o2 = np.argsort(skel), np.argsort(piv[:r])
        cond = np.linalg.cond(R[:r, :r])
        assert np.max(np.abs(P[o1] - P_ref[o2])) <= 1e-13 * cond * max(1.0, np.abs(P_ref).max())
        assert np.linalg.norm(A[:, skel] @ P - A, 2) <= 10 * np.linalg.norm(A[:, piv[:r]] @ P_ref - A, 2) + 1e-14
    assert checked >= 3


def test_host_library_then_torch_in_one_process():
    """libkernid_host.so links NCCL (kernid_multi.cpp); loading it before PyTorch must not pin an older system
    libnccl.so.2 under torch's feet (kernid._preload_nccl loads the copy torch bundles first)."""
    code = ("import sys; sys.path.insert(0, %r); from paper_1409_2802_b200 import kernid as H; H.host_lib(); "
            "import torch; import torch.distributed; print('ok', torch.distributed.is_nccl_available())" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stderr[-2000:]
