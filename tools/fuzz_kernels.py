"""Randomised differential check of the Gram-type passes across kernel families (not a parity test: the checker
here is a dense float64 numpy evaluation of the same block, independent of oracle/; the parity tests proper are
tests/test_gpu_*.py). Random shapes -- d, m, skeleton rank r, target count (ragged tiles, fewer targets than a
tile), explicit blocks -- each through every kernel the dispatcher can route it to:

  residual pass   auto | k_fused (KID_OPT_KERNEL 1) | k_fused_w one CTA / CTA pair (KID_OPT_TILE_FORM) where n <= 48
  K^T K           auto | k_fused | k_gram2 (KID_OPT_KERNEL 3)
  projected Gram  auto | cluster path

Bar: |dG_jk| <= 1e-10 sqrt(G_jj G_kk) (the Gram ladder of the tests), sums to 1e-11 relative.
usage: python tools/fuzz_kernels.py [cases] [seed]   (run by tools/gpu/r02_fuzz.sh)"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2802_b200._lib import Device, KidError  # noqa: E402


def dense_block(tg, sr, h):
    q = np.zeros((tg.shape[0], sr.shape[0]))
    for k in range(tg.shape[1]):
        q += (tg[:, k, None] - sr[None, :, k]) ** 2
    return np.exp(-q / (2.0 * h * h))


def gram_ok(G, ref, tol=1e-10):
    dg = np.sqrt(np.abs(np.diag(ref)))
    return bool(np.all(np.abs(G - ref) <= tol * np.outer(dg, dg) + 1e-290))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    dev = Device(0)
    bad = 0
    ran = {}
    for it in range(cases):
        d = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 24]))
        m = int(rng.choice([int(rng.integers(2, 40)), int(rng.integers(40, 129)), int(rng.integers(129, 300)),
                            int(rng.choice([256, 512, 384]))]))
        nt = int(rng.choice([int(rng.integers(1, 33)), int(rng.integers(33, 700)), int(rng.integers(700, 9000))]))
        if m > 256:
            nt = min(nt, 3000)
        r = int(rng.choice([1, m - 1, int(rng.integers(1, m)), max(1, m - int(rng.integers(1, 49)))]))
        r = min(max(r, 1), m - 1)
        sr = rng.standard_normal((m, d)) * 0.5
        tg = rng.standard_normal((nt, d)) * 0.7 + 1.5
        h = float(rng.uniform(0.8, 2.5)) * np.sqrt(d)
        K = dense_block(tg, sr, h)
        skel = np.sort(rng.choice(m, r, replace=False))
        P = rng.standard_normal((r, m)) * (0.5 / np.sqrt(r))
        P[:, skel] = np.eye(r)
        D = K - K[:, skel] @ P
        D[:, skel] = 0.0
        rG, rD = K.T @ K, D.T @ D
        dev.set_block(tg, sr)
        n = m - r
        tag = f"case {it}: d={d} m={m} r={r} nt={nt}"

        def check(name, fn, ref, sums=None):
            nonlocal bad
            try:
                out = fn()
            except KidError as e:
                print(f"FAIL {tag} {name}: {e}")
                bad += 1
                return
            k = dev.last_kernel()
            ran[k] = ran.get(k, 0) + 1
            G = out[2] if len(out) > 2 else out[0]
            ok = gram_ok(G, ref)
            if sums is not None:
                ok &= abs(out[0] - sums[0]) <= 1e-11 * max(sums[0], 1e-300) + 1e-290
                ok &= abs(out[1] - sums[1]) <= 1e-11 * max(sums[1], 1e-300)
            if not ok:
                print(f"FAIL {tag} {name} kernel={k}: max rel {np.max(np.abs(G - ref)) / max(np.abs(ref).max(), 1e-300):.3e}")
                bad += 1

        sums = (float(np.sum(D * D)), float(np.sum(K * K)))
        variants = [("resid auto", dict())]
        variants.append(("resid k_fused", dict(path=1, kernel=1)))
        if n <= 48:
            variants.append(("resid tile solo", dict(path=1, form=1)))
            variants.append(("resid tile pair", dict(path=1, form=2)))
            variants.append(("resid tile pair w8", dict(path=1, form=2, warps=8)))
        for name, o in variants:
            dev.set_path(o.get("path", 0))
            dev.set_option(3, o.get("kernel", 0))
            dev.set_option(5, o.get("form", 0))
            dev.set_option(4, o.get("warps", 0))
            check(name, lambda: dev.recon_error(h, skel, P), rD, sums)
        dev.set_option(5, 0)
        dev.set_option(4, 0)
        for name, o in (("gram auto", dict()), ("gram k_fused", dict(path=1, kernel=1)), ("gram k_gram2", dict(path=1, kernel=3))):
            dev.set_path(o.get("path", 0))
            dev.set_option(3, o.get("kernel", 0))
            check(name, lambda: dev.gram(h), rG)
        dev.set_option(3, 0)
        nc = int(rng.integers(1, min(m, 48) + 1))
        Cm = np.linalg.qr(rng.standard_normal((m, nc)))[0]
        rP = (K @ Cm).T @ (K @ Cm)
        for name, path in (("proj auto", 0), ("proj cluster", 1)):
            dev.set_path(path)
            check(name, lambda: dev.proj_gram(h, Cm), rP)
        dev.set_path(0)
    print("kernels exercised:", dict(sorted(ran.items())))
    print(f"fuzz: {'PASS' if bad == 0 else 'FAIL'} ({cases} cases, {sum(ran.values())} pass invocations, {bad} failures)")
    dev.close()
    sys.exit(0 if bad == 0 else 1)


if __name__ == "__main__":
    main()
