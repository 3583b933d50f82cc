"""One small invocation of every device pass (K1 split, K2 row norms, K3 Gram, K4 leverage, K5 residual
Gram on both kernel families and the warp-tile kernel, compress_svd's projected Gram, TSQR, the skeleton
matvec, gathered rows), each checked against the oracle -- run under compute-sanitizer (memcheck /
racecheck / synccheck) by tools/gpu/r02_sanitize.sh. Sizes are small: the tools slow kernels ~100x."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1409_2802_b200._lib import Device  # noqa: E402


def close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(1e-300, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) <= tol * scale


def main():
    dev = Device(0)
    ok = True
    for d, N, n in [(3, 4000, 40), (8, 3000, 100)]:
        t = O.prepare_trial(d, N, n, 2.0, O.derive_seed(1, 0, 0))
        K = O.kernel_matrix(t.targets, t.sources, t.h)
        dev.set_points(t.points)
        src, rho, nt = dev.split(t.center, n, 2.0)
        ok &= bool(np.array_equal(src, t.split.source_indices) and rho == t.split.rho)
        ok &= close(dev.row_norms(t.h), O.row_norms(K), 1e-12)
        G, sk = dev.gram(t.h)
        ok &= close(G, K.T @ K, 1e-10)
        res = O.compress_id(K, np.arange(0, K.shape[0], 5), eps=1e-6)
        _, _, r_DtD, _ = O.residual_stats(K, res.skeleton, res.P)
        for path, kern in ((0, 0), (1, 1), (1, 2)):
            dev.set_path(path)
            dev.set_option(3, kern)
            sd, sk2, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
            ok &= close(DtD, r_DtD, 1e-6)
            sv, V = O.right_factor(K)
            W = V[:, :5] / sv[:5]
            ok &= close(dev.leverage(t.h, W), O.row_leverage_scores(K, 5)[0], 1e-8)
        dev.set_path(0)
        dev.set_option(3, 0)
        C = np.linalg.qr(np.random.default_rng(0).standard_normal((n, 7)))[0]
        _, _, Gp = dev.proj_gram(t.h, C)
        ok &= close(Gp, (K @ C).T @ (K @ C), 1e-8)
        if n <= 128:
            R = dev.tsqr_r(t.h)
            ok &= close(R.T @ R, K.T @ K, 1e-10)
        q = np.random.default_rng(1).standard_normal(n)
        u = dev.apply_skeleton(t.h, res.skeleton, res.P, q)
        ok &= close(u, O.apply_skeleton(t.targets, t.sources[res.skeleton], t.h, res.P, q), 1e-10)
        rows = np.array([0, 3, K.shape[0] - 1])
        ok &= close(dev.eval_rows(t.h, rows), K[rows], 1e-12)
    print("sanitize cases:", "PASS" if ok else "FAIL")
    dev.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
