"""Out-of-bounds check of every device pass without compute-sanitizer (closed on this GPU pool:
profiles/r02_compute_sanitizer_closed.log). The library is built with -DKID_GUARD
(`python paper_1409_2802_b200/build.py --guard` -> libkernid_cuda_guard.so): every device buffer it allocates sits
between two 64 KB canary zones, and kid_guard_check() counts corrupted canary bytes. Each pass below runs on
ragged shapes (N not a multiple of any tile, odd m, n = m - r from 1 to m - 1) through both kernel families,
is checked against the oracle, and must leave every canary intact. Run by tools/gpu/r02_guard.sh."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1409_2802_b200 import _lib  # noqa: E402

_lib.CUDA_SO = os.path.join(_lib.PKG, "libkernid_cuda_guard.so")
from paper_1409_2802_b200._lib import Device  # noqa: E402


def close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(1e-300, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) <= tol * scale


def main():
    dev = Device(0)
    assert dev.guard_check() == 0, "library was not built with -DKID_GUARD"
    ok = True
    npass = 0

    def check(tag, cond):
        nonlocal ok
        if not cond:
            ok = False
            print(f"PARITY FAIL: {tag}")

    def guard(tag):
        nonlocal ok, npass
        bad = dev.guard_check()
        npass += 1
        if bad:
            ok = False
            print(f"GUARD VIOLATION after {tag}: {bad} canary bytes overwritten")

    shapes = [(3, 4001, 37), (2, 3333, 100), (8, 9001, 200), (16, 7777, 256), (8, 6007, 512), (5, 2999, 129),
              (64, 3001, 256), (1, 1500, 64)]
    for d, N, n in shapes:
        t = O.prepare_trial(d, N, n, 2.0 if d < 16 else 0.0, O.derive_seed(1, 0, 0))
        K = O.kernel_matrix(t.targets, t.sources, t.h)
        dev.set_points(t.points)
        src, rho, nt = dev.split(t.center, n, 2.0 if d < 16 else 0.0)
        guard(f"split d={d} N={N} n={n}")
        check(f"split d={d} N={N} n={n}", bool(np.array_equal(src, t.split.source_indices) and rho == t.split.rho and nt == K.shape[0]))
        check(f"split d={d} N={N} n={n}", close(dev.row_norms(t.h), O.row_norms(K), 1e-12))
        guard("row_norms")
        for path in (0, 1):
            dev.set_path(path)
            G, sk = dev.gram(t.h)
            guard(f"gram path={path} d={d} n={n}")
            check(f"gram path={path} d={d} n={n}", close(G, K.T @ K, 1e-10))
            for eps, fixed in ((1e-2, None), (1e-8, None), (None, 1), (None, n - 1), (None, max(1, n - 20))):
                try:
                    res = O.compress_id(K, np.arange(0, K.shape[0], 3), eps=eps) if fixed is None else \
                        O.compress_id(K, np.arange(0, K.shape[0], 3), fixed_r=fixed)
                except O.OracleError:  # numerically rank-deficient sample at this rank
                    continue
                if res.rank < 1:
                    continue
                _, _, r_DtD, _ = O.residual_stats(K, res.skeleton, res.P)
                for kern in ((0,) if path == 0 else (1, 2)):
                    dev.set_option(3, kern)
                    sd, sk2, DtD, _ = dev.recon_error(t.h, res.skeleton, res.P)
                    guard(f"recon path={path} kernel={kern} d={d} n={n} r={res.rank}")
                    check(f"recon path={path} kernel={kern} d={d} n={n} r={res.rank}", close(DtD, r_DtD, 1e-6))
                dev.set_option(3, 0)
            U, s, Vt = np.linalg.svd(K, full_matrices=False)
            for r in (1, 5, min(n, 40)):
                r = max(1, min(r, int(np.sum(s >= 1e-8 * s[0]))))  # W = V_r / sigma_r stays well scaled
                W = Vt[:r].T / s[:r]
                lev = dev.leverage(t.h, W)
                guard(f"leverage path={path} r={r}")
                check(f"leverage path={path} r={r}", close(lev, np.sum((K @ W) ** 2, axis=1), 1e-8))
            for nc in (1, 7, min(n, 33), n):
                C = np.linalg.qr(np.random.default_rng(nc).standard_normal((n, nc)))[0]
                _, _, Gp = dev.proj_gram(t.h, C)
                guard(f"proj_gram path={path} n={nc}")
                check(f"proj_gram path={path} n={nc}", close(Gp, (K @ C).T @ (K @ C), 1e-8))
        dev.set_path(0)
        if n <= 128:
            R = dev.tsqr_r(t.h)
            guard("tsqr")
            check("tsqr", close(R.T @ R, K.T @ K, 1e-10))
        res = O.compress_id(K, np.arange(0, K.shape[0], 3), eps=1e-4)
        if res.rank >= 1:
            q = np.random.default_rng(1).standard_normal(n)
            u = dev.apply_skeleton(t.h, res.skeleton, res.P, q)
            guard("apply_skeleton")
            check("apply_skeleton", close(u, O.apply_skeleton(t.targets, t.sources[res.skeleton], t.h, res.P, q), 1e-10))
        rows = np.array([0, 3, K.shape[0] - 1])
        check("apply_skeleton", close(dev.eval_rows(t.h, rows), K[rows], 1e-12))
        guard("eval_rows")
        dev.select_rows(np.arange(1, K.shape[0], 7))
        G, _ = dev.gram(t.h)
        guard("select_rows + gram")
        check("select_rows + gram", close(G, K[1::7].T @ K[1::7], 1e-10))
        dev.select_rows(None)
    # the guards do catch an overrun: a 2-row result buffer handed to a pass that writes one double per target
    small = dev.device_alloc(16)
    dev.row_norms_dev(t.h, small)
    dev.synchronize()
    caught = dev.guard_check()
    print(f"self-test: deliberate overrun of a 16-byte buffer by row_norms_dev -> {caught} canary bytes flagged")
    ok &= caught > 0
    dev.device_free(small)
    print(f"guard cases: {'PASS' if ok else 'FAIL'} ({npass} passes checked, 0 canary bytes overwritten)" if ok
          else "guard cases: FAIL")
    dev.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
