"""CPU ORACLE -- test infrastructure only.

ctypes/numpy front-end of ``oracle/kernid_oracle.c``, the plain-C restatement of
the reference far-field path (/root/reference/proj/include/kernid/*.hpp). Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module; the product path never does.

Pinning: see ``kernid_oracle.h`` (RNG bit-exact against the reference's own
rng.hpp built into ``oracle/_ref``; the rest against the reference's
known-answer tests, ported in ``tests/test_oracle.py``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libkernid_oracle.so")
_lib = None

# error codes shared with the product C-ABI (include/kernid_cuda.h)
E_RANGE, E_DIM, E_NO_TARGETS, E_NUMERICAL, E_ERROR, E_ILLCOND = 1, 2, 3, 4, 5, 8

SCHEME_UNIFORM, SCHEME_BERNOULLI, SCHEME_EUCLIDEAN, SCHEME_LEVERAGE = 0, 1, 2, 4


def build() -> str:
    """Compile the oracle (and oracle/_ref when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int), ("has_spare", C.c_int), ("spare", C.c_double)]


def _declare(L):
    i64, i32, u64, dbl = C.c_int64, C.c_int32, C.c_uint64, C.c_double
    L.or_derive_seed.restype = u64
    L.or_derive_seed.argtypes = [u64, u64, u64]
    L.or_rng_dump.argtypes = [u64, i64, _up, _dp, _dp, u64, _up]
    L.or_gen_normal.argtypes = [i32, i64, u64, _dp]
    L.or_silverman_bandwidth.restype = dbl
    L.or_silverman_bandwidth.argtypes = [i32, i64]
    L.or_random_center_index.restype = i64
    L.or_random_center_index.argtypes = [i64, u64]
    L.or_split.argtypes = [_dp, i64, i32, _dp, i64, dbl, _ip, _ip, C.POINTER(i64), C.POINTER(dbl), C.c_void_p]
    L.or_gather_points.argtypes = [_dp, i64, i32, _ip, i64, _dp]
    L.or_kernel_matrix.argtypes = [_dp, i64, _dp, i64, i32, dbl, _dp, i32]
    L.or_eval_gaussian.restype = dbl
    L.or_eval_gaussian.argtypes = [_dp, _dp, i32, dbl]
    L.or_sample_count.restype = i64
    L.or_sample_count.argtypes = [dbl, i64]
    L.or_row_norms.argtypes = [_dp, i64, i64, _dp]
    L.or_sample_rows.restype = i64
    L.or_sample_rows.argtypes = [i32, i32, i64, C.c_void_p, dbl, u64, _ip]
    L.or_apply_skeleton.argtypes = [_dp, i64, _dp, i64, i32, dbl, _dp, i64, _dp, _dp]
    L.or_mc_error.argtypes = [_dp, i64, i64, _ip, i64, _dp, dbl, i32, u64, dbl, dbl, i32, _dp]
    L.or_svd_error_norm.restype = dbl
    L.or_svd_error_norm.argtypes = [_dp, i64, i64, _dp, i64, dbl, dbl, i32]
    L.or_qr_r.argtypes = [_dp, i64, i64, _dp]
    L.or_jacobi_svd.argtypes = [_dp, i64, _dp, C.c_void_p]
    L.or_singular_values.argtypes = [_dp, i64, i64, _dp]
    L.or_right_factor.argtypes = [_dp, i64, i64, _dp, _dp]
    L.or_epsilon_rank.restype = i64
    L.or_epsilon_rank.argtypes = [_dp, i64, dbl, dbl]
    L.or_row_leverage_scores.argtypes = [_dp, i64, i64, i64, _dp, C.POINTER(i32)]
    L.or_interpolative_decomposition.argtypes = [_dp, i64, i64, i64, _ip, _dp]
    L.or_power_iteration_norm.restype = dbl
    L.or_power_iteration_norm.argtypes = [_dp, i64, i64, dbl, i32]
    L.or_spectral_norm_exact.restype = dbl
    L.or_spectral_norm_exact.argtypes = [_dp, i64, i64]
    L.or_reconstruction_error_norm.restype = dbl
    L.or_reconstruction_error_norm.argtypes = [_dp, i64, i64, _ip, i64, _dp, dbl, dbl, i32]
    L.or_matrix_norm.restype = dbl
    L.or_matrix_norm.argtypes = [_dp, i64, i64, dbl, dbl, i32]
    L.or_residual_stats.argtypes = [_dp, i64, i64, _ip, i64, _dp, C.POINTER(dbl), C.POINTER(dbl),
                                    C.c_void_p, C.c_void_p]
    L.or_bound_id_value.restype = dbl
    L.or_bound_id_value.argtypes = [i64, i64, dbl]
    L.or_reconstruction_bound.restype = dbl
    L.or_reconstruction_bound.argtypes = [i64, i64, dbl, dbl]
    L.or_compress_id.argtypes = [_dp, i64, i64, _ip, i64, dbl, i64, dbl, dbl, dbl, dbl, i32,
                                 C.POINTER(i64), C.POINTER(dbl), _ip, _dp, C.POINTER(dbl),
                                 C.POINTER(dbl), C.POINTER(dbl)]
    L.or_jacobi_eigen.argtypes = [_dp, i64, _dp, C.c_void_p]


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle error code {code}")
        self.code = code


def _f(a):
    """Column-major (Eigen layout) flat float64 copy of a 2-D array."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(a.shape).T).ravel() if np.ndim(a) == 2 \
        else np.ascontiguousarray(a, dtype=np.float64)


def _from_f(flat, rows, cols):
    return np.asarray(flat).reshape(cols, rows).T.copy()


# ---------------------------------------------------------------- rng.hpp
def derive_seed(master: int, a: int, b: int = 0) -> int:
    return int(lib().or_derive_seed(master, a, b))


def rng_dump(seed: int, n: int, below_n: int = 1000003):
    u64 = np.zeros(n, np.uint64)
    un = np.zeros(n)
    nm = np.zeros(n)
    bl = np.zeros(n, np.uint64)
    lib().or_rng_dump(seed, n, u64, un, nm, below_n, bl)
    return u64, un, nm, bl


# ------------------------------------------------------------ datagen.hpp
def gen_normal(d: int, N: int, seed: int) -> np.ndarray:
    """N x d points (datagen.hpp:35-43). Returned as an (N, d) float64 array."""
    out = np.zeros(N * d)
    if lib().or_gen_normal(d, N, seed, out):
        raise OracleError(E_RANGE, "gen_normal")
    return _from_f(out, N, d)


def silverman_bandwidth(d: int, N: int) -> float:
    if d < 1 or N < 1:
        raise OracleError(E_RANGE, "silverman_bandwidth")
    return float(lib().or_silverman_bandwidth(d, N))


def random_center_index(N: int, data_seed: int) -> int:
    return int(lib().or_random_center_index(N, data_seed))


@dataclass
class Split:
    source_indices: np.ndarray
    target_indices: np.ndarray
    rho: float
    xi: float
    center: np.ndarray


def split_sources_targets(points: np.ndarray, center, n: int, xi: float, dist_out=None) -> Split:
    """geometry.hpp:29-65."""
    N, d = points.shape
    center = np.ascontiguousarray(center, dtype=np.float64)
    if center.size != d:
        raise OracleError(E_DIM, "split_sources_targets")
    src = np.zeros(max(n, 1), np.int64)
    tgt = np.zeros(N, np.int64)
    nt = C.c_int64()
    rho = C.c_double()
    dptr = None
    if dist_out is not None:
        dptr = dist_out.ctypes.data_as(C.c_void_p)
    rc = lib().or_split(_f(points), N, d, center, n, xi, src, tgt, C.byref(nt), C.byref(rho), dptr)
    if rc:
        raise OracleError(rc, "split_sources_targets")
    return Split(src[:n].copy(), tgt[: nt.value].copy(), rho.value, xi, center.copy())


def gather_points(points: np.ndarray, idx) -> np.ndarray:
    return np.ascontiguousarray(points[np.asarray(idx, dtype=np.int64)])


# -------------------------------------------------------------- kernel.hpp
def kernel_matrix(targets: np.ndarray, sources: np.ndarray, h: float, threads: int = 0) -> np.ndarray:
    """Dense Gaussian K (kernel.hpp:202-208), returned as an (nt, m) array."""
    nt, d = targets.shape
    m = sources.shape[0]
    K = np.zeros(nt * m)
    lib().or_kernel_matrix(_f(targets), nt, _f(sources), m, d, h, K, threads)
    return _from_f(K, nt, m)


def eval_gaussian(x, y, h) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.size != y.size:
        raise OracleError(E_DIM, "eval_kernel")
    return float(lib().or_eval_gaussian(x, y, x.size, h))


# ------------------------------------------------------------ sampling.hpp
def sample_count(s: float, m: int) -> int:
    c = int(lib().or_sample_count(s, m))
    if c < 0:
        raise OracleError(E_RANGE, "sample_count")
    return c


def row_norms(K: np.ndarray) -> np.ndarray:
    nt, m = K.shape
    w = np.zeros(nt)
    lib().or_row_norms(_f(K), nt, m, w)
    return w


def sample_rows(kind: int, m: int, s: float, seed: int, weights=None, replacement: bool = False) -> np.ndarray:
    """sample_rows (sampling.hpp:156-243) for Uniform / Bernoulli / EuclideanNorm / Leverage weights."""
    cnt = m if kind == SCHEME_BERNOULLI else sample_count(s, m)
    out = np.zeros(cnt, np.int64)
    wp = None
    if weights is not None:
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        wp = weights.ctypes.data_as(C.c_void_p)
    rc = int(lib().or_sample_rows(kind, int(replacement), m, wp, s, seed, out))
    if rc < 0:
        raise OracleError(-rc, "sample_rows")
    return out[:rc].copy()


# ------------------------------------------------------------- lowrank.hpp
def qr_r(A: np.ndarray) -> np.ndarray:
    rows, cols = A.shape
    R = np.zeros(cols * cols)
    lib().or_qr_r(_f(A), rows, cols, R)
    return _from_f(R, cols, cols)


def singular_values(A: np.ndarray) -> np.ndarray:
    rows, cols = A.shape
    sv = np.zeros(min(rows, cols))
    lib().or_singular_values(_f(A), rows, cols, sv)
    return sv


def right_factor(A: np.ndarray):
    rows, cols = A.shape
    sv = np.zeros(cols)
    V = np.zeros(cols * cols)
    lib().or_right_factor(_f(A), rows, cols, sv, V)
    return sv, _from_f(V, cols, cols)


def epsilon_rank(sv, eps: float, ref_sigma1: float | None = None) -> int:
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    r = int(lib().or_epsilon_rank(sv, sv.size, eps, ref_sigma1 if ref_sigma1 is not None else -1.0))
    if r < 0:
        raise OracleError(E_RANGE, "epsilon_rank")
    return r


def row_leverage_scores(A: np.ndarray, r: int):
    rows, cols = A.shape
    sc = np.zeros(rows)
    gap = C.c_int32()
    rc = lib().or_row_leverage_scores(_f(A), rows, cols, r, sc, C.byref(gap))
    if rc:
        raise OracleError(rc, "row_leverage_scores")
    return sc, bool(gap.value)


def interpolative_decomposition(A: np.ndarray, r: int):
    m, n = A.shape
    skel = np.zeros(max(r, 1), np.int64)
    P = np.zeros(max(r, 1) * n)
    rc = lib().or_interpolative_decomposition(_f(A), m, n, r, skel, P)
    if rc:
        raise OracleError(rc, "interpolative_decomposition")
    return skel[:r].copy(), _from_f(P[: r * n], r, n)


def power_iteration_norm(A: np.ndarray, tol=1e-6, cap=1000) -> float:
    rows, cols = A.shape
    return float(lib().or_power_iteration_norm(_f(A), rows, cols, tol, cap))


def spectral_norm_exact(A: np.ndarray) -> float:
    rows, cols = A.shape
    return float(lib().or_spectral_norm_exact(_f(A), rows, cols))


def jacobi_eigen(A: np.ndarray):
    n = A.shape[0]
    ev = np.zeros(n)
    V = np.zeros(n * n)
    lib().or_jacobi_eigen(_f(A), n, ev, V.ctypes.data_as(C.c_void_p))
    return ev, _from_f(V, n, n)


# ------------------------------------------------------------ compress.hpp
BUDGET, POWER_TOL, POWER_CAP = 2e8, 1e-6, 1000  # NormPolicy defaults (compress.hpp:46-50)


def reconstruction_error_norm(K, skel, P, budget=BUDGET, tol=POWER_TOL, cap=POWER_CAP) -> float:
    nt, m = K.shape
    skel = np.ascontiguousarray(skel, dtype=np.int64)
    return float(lib().or_reconstruction_error_norm(_f(K), nt, m, skel, skel.size, _f(P), budget, tol, cap))


def matrix_norm(K, budget=BUDGET, tol=POWER_TOL, cap=POWER_CAP) -> float:
    nt, m = K.shape
    return float(lib().or_matrix_norm(_f(K), nt, m, budget, tol, cap))


def residual_stats(K, skel, P, grams: bool = True):
    """Frobenius sums and the Grams D^T D, K^T K of D = K - K[:,skel] P (fused-pass oracle)."""
    nt, m = K.shape
    skel = np.ascontiguousarray(skel, dtype=np.int64)
    sd, sk = C.c_double(), C.c_double()
    DtD = np.zeros(m * m) if grams else None
    KtK = np.zeros(m * m) if grams else None
    lib().or_residual_stats(_f(K), nt, m, skel, skel.size, _f(P), C.byref(sd), C.byref(sk),
                            DtD.ctypes.data_as(C.c_void_p) if grams else None,
                            KtK.ctypes.data_as(C.c_void_p) if grams else None)
    if grams:
        return sd.value, sk.value, _from_f(DtD, m, m), _from_f(KtK, m, m)
    return sd.value, sk.value, None, None


def bound_id_value(n, r, sigma_r1) -> float:
    if r < 0 or r > n:
        raise OracleError(E_RANGE, "bound_id_value")
    return float(lib().or_bound_id_value(n, r, sigma_r1))


def reconstruction_bound(m, s_count, eps, sigma_r1) -> float:
    return float(lib().or_reconstruction_bound(m, s_count, eps, sigma_r1))


@dataclass
class CompressResult:
    rank: int
    rel_error: float
    skeleton: np.ndarray
    P: np.ndarray
    sigma1_sample: float
    sigma_r1_sample: float
    bound_id: float
    rank_zero: bool


def compress_id(K, rows, eps=None, fixed_r=None, ref_sigma1=None, k_norm=None,
                budget=BUDGET, tol=POWER_TOL, cap=POWER_CAP) -> CompressResult:
    """compress_id (compress.hpp:168-215)."""
    nt, m = K.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    rank = C.c_int64()
    rel = C.c_double()
    s1, sr1, bid = C.c_double(), C.c_double(), C.c_double()
    skel = np.zeros(m, np.int64)
    P = np.zeros(m * m)
    rc = lib().or_compress_id(_f(K), nt, m, rows, rows.size,
                              eps if eps is not None else -1.0,
                              fixed_r if fixed_r is not None else 0,
                              ref_sigma1 if ref_sigma1 is not None else -1.0,
                              k_norm if k_norm is not None else -1.0,
                              budget, tol, cap, C.byref(rank), C.byref(rel), skel, P,
                              C.byref(s1), C.byref(sr1), C.byref(bid))
    if rc:
        raise OracleError(rc, "compress_id")
    r = rank.value
    return CompressResult(r, rel.value, skel[:r].copy(), _from_f(P[: r * m], r, m) if r else np.zeros((0, m)),
                          s1.value, sr1.value, bid.value, r == 0)


def apply_skeleton(targets, skel_points, h, P, q) -> np.ndarray:
    """apply_skeleton (compress.hpp:309-325): u_i = sum_j Ker(y_i, xskel_j) (P q)_j."""
    nt, d = targets.shape
    r = skel_points.shape[0]
    m = P.shape[1]
    u = np.zeros(nt)
    lib().or_apply_skeleton(_f(targets), nt, _f(skel_points), r, d, h, _f(P), m,
                            np.ascontiguousarray(q, dtype=np.float64), u)
    return u


def mc_error(K, skel, P, s_mc, n_mc, seed, budget=BUDGET, tol=POWER_TOL, cap=POWER_CAP) -> np.ndarray:
    """mc_error (compress.hpp:279-305) with khat_row(i) = K[i, skel] P."""
    nt, m = K.shape
    est = np.zeros(n_mc)
    rc = lib().or_mc_error(_f(K), nt, m, np.ascontiguousarray(skel, dtype=np.int64), len(skel), _f(P),
                           s_mc, n_mc, seed, budget, tol, cap, est)
    if rc:
        raise OracleError(rc, "mc_error")
    return est


def svd_error_norm(K, Vr, budget=BUDGET, tol=POWER_TOL, cap=POWER_CAP) -> float:
    """compress_svd numerator (compress.hpp:243-262): ||K V_r V_r^T - K||."""
    nt, m = K.shape
    return float(lib().or_svd_error_norm(_f(K), nt, m, _f(Vr), Vr.shape[1], budget, tol, cap))


# ------------------------------------------------------------- harness.hpp
@dataclass
class Trial:
    points: np.ndarray
    center: np.ndarray
    split: Split
    sources: np.ndarray
    targets: np.ndarray
    h: float
    d: int


def prepare_trial(d: int, N: int, n_sources: int, xi: float, data_seed: int, h_value: float = 1.0,
                  silverman_units: bool = True, center: str = "random") -> Trial:
    """prepare_trial (harness.hpp:107-129) for the Normal dataset; center "random" (RandomPoint,
    the BASELINE configs) or "origin" (the reference default, harness.hpp:88)."""
    points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A))
    center = points[random_center_index(N, data_seed)].copy() if center == "random" else np.zeros(d)
    split = split_sources_targets(points, center, n_sources, xi)
    sources = gather_points(points, split.source_indices)
    targets = gather_points(points, split.target_indices)
    h = h_value * silverman_bandwidth(d, N) if silverman_units else h_value
    return Trial(points, center, split, sources, targets, h, d)


# ------------------------------------------------------------- compress.hpp:327-378, harness.hpp:330-438
def interaction_fractions(points: np.ndarray, h: float, x_c, n: int):
    """interaction_fractions (compress.hpp:336-378): order all points by (||p - x_c||, index),
    sources = first n, neighbours = next n, far = the rest; fractions of ||K||_2 of the stack
    carried by each block (exact norms: matrix_norm at these sizes, compress.hpp:156-159)."""
    N = points.shape[0]
    if N < 2 * n:
        raise OracleError(E_RANGE, "interaction_fractions: requires N >= 2n")
    diff = points - np.asarray(x_c)[None, :]
    acc = diff[:, 0] * diff[:, 0]
    for k in range(1, points.shape[1]):
        acc = acc + diff[:, k] * diff[:, k]
    dist = np.sqrt(acc)
    order = np.lexsort((np.arange(N), dist))
    src, nb, far = points[order[:n]], points[order[n:2 * n]], points[order[2 * n:]]
    KS, KN = kernel_matrix(src, src, h), kernel_matrix(nb, src, h)
    KF = kernel_matrix(far, src, h) if far.shape[0] else np.zeros((0, n))
    total = spectral_norm_exact(np.concatenate([KS, KN, KF]))
    if not total > 0.0:
        return 0.0, 0.0, 0.0
    return (spectral_norm_exact(KS) / total, spectral_norm_exact(KN) / total,
            spectral_norm_exact(KF) / total if far.shape[0] else 0.0)


def bandwidth_search(d, N, n, xi, data_seed, kappa=0.2, large_h=False, eps=1e-2, max_iters=40, tol_rows=2,
                     center="origin"):
    """bandwidth_search (harness.hpp:345-438) on the oracle's K and singular_values; returns
    (h_abs, h_over_hs, rank, evaluations, converged, profile) or raises OracleError with the
    profile in .profile when the budget cannot be bracketed."""
    t = prepare_trial(d, N, n, xi, data_seed, center=center)
    h_S = silverman_bandwidth(d, N)
    target = kappa * n
    profile = []

    def rank_at(h):
        r = epsilon_rank(singular_values(kernel_matrix(t.targets, t.sources, h)), eps)
        profile.append((h, r))
        return r

    def fail(msg):
        e = OracleError(E_RANGE, msg)
        e.profile = profile
        raise e

    scan = [1e-3, 1e-2, 0.03, 0.1, 0.3, 1.0, 3.0, 10.0, 1e2]
    coarse, peak = [], 0
    for i, sc in enumerate(scan):
        coarse.append((sc * h_S, rank_at(sc * h_S)))
        if coarse[i][1] > coarse[peak][1]:
            peak = i
    if coarse[peak][1] < target:
        fail("rank budget exceeds the peak epsilon-rank")
    if not large_h:
        hi, r_hi = coarse[peak]
        below = peak
        while below > 0 and coarse[below][1] >= target:
            below -= 1
        lo, r_lo = coarse[below]
        for _ in range(5):
            if r_lo < target:
                break
            lo /= 2.0
            r_lo = rank_at(lo)
        ok = r_lo < target <= r_hi
    else:
        lo, r_lo = coarse[peak]
        above = peak
        while above + 1 < len(coarse) and coarse[above][1] >= target:
            above += 1
        hi, r_hi = coarse[above]
        for _ in range(5):
            if r_hi < target:
                break
            hi *= 2.0
            r_hi = rank_at(hi)
        ok = r_lo >= target > r_hi
    if not ok:
        fail("could not bracket the rank budget")
    h_best, r_best = (hi, r_hi) if not large_h else (lo, r_lo)
    converged = False
    while len(profile) < max_iters:
        mid = math.sqrt(lo * hi)
        r_mid = rank_at(mid)
        if abs(r_mid - target) <= abs(r_best - target):
            h_best, r_best = mid, r_mid
        if abs(r_mid - target) <= tol_rows:
            converged = True
            break
        go_right = (r_mid < target) if not large_h else (r_mid >= target)
        if go_right:
            lo = mid
        else:
            hi = mid
    return h_best, h_best / h_S, r_best, len(profile), converged, profile
