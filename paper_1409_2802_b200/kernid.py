"""Python front-end of the host C++ mirror (libkernid_host.so, include/kernid_b200.hpp).

Names follow the reference `kernid::` API (/root/reference/proj/include/kernid/) so the
parity tests read like the reference's own tests. Device work goes through
libkernid_cuda.so; there is no CPU fallback for the O(N_T m) passes.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import ERROR_NAMES, KidError, cuda_lib  # noqa: F401  (cuda_lib loads libkernid_cuda.so first)

PKG = os.path.dirname(os.path.abspath(__file__))
HOST_SO = os.path.join(PKG, "libkernid_host.so")
_host = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")

UNIFORM, BERNOULLI, EUCLIDEAN_NORM, LEVERAGE = 0, 1, 2, 4


def _preload_nccl():
    """libkernid_host.so needs libnccl.so.2 (kernid_multi.cpp). When PyTorch is installed, load the NCCL it
    bundles first: the loader then binds the host library to that copy (same soname), and a later
    `import torch` in the same process finds the symbols of its own NCCL instead of an older system one."""
    try:
        import glob
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for loc in (spec.submodule_search_locations if spec else []) or []:
            for so in sorted(glob.glob(os.path.join(loc, "lib", "libnccl.so.*"))):
                C.CDLL(so, mode=C.RTLD_GLOBAL)
                return
    except (ImportError, OSError, ValueError):
        pass


def host_lib():
    global _host
    if _host is None:
        cuda_lib()
        if not os.path.exists(HOST_SO):
            raise OSError(f"{HOST_SO} missing: run __graft_entry__.build()")
        _preload_nccl()
        L = C.CDLL(HOST_SO)
        i64, i32, u64, dbl, P = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.POINTER
        L.kidh_last_error.restype = C.c_char_p
        L.kidh_derive_seed.restype = u64
        L.kidh_derive_seed.argtypes = [u64, u64, u64]
        L.kidh_center_index.restype = i64
        L.kidh_center_index.argtypes = [i64, u64]
        L.kidh_gen_normal.argtypes = [i32, i64, u64, _dp]
        L.kidh_singular_values.argtypes = [_dp, i64, i64, _dp]
        L.kidh_epsilon_rank.argtypes = [_dp, i64, dbl, dbl, P(i64)]
        L.kidh_interpolative_decomposition.argtypes = [_dp, i64, i64, i64, _ip, _dp]
        L.kidh_sym_eig.argtypes = [_dp, i64, _dp, C.c_void_p]
        L.kidh_sym_eigvals.argtypes = [_dp, i64, _dp]
        L.kidh_lambda_max.argtypes = [_dp, i64, P(dbl)]
        L.kidh_draw.argtypes = [i32, i32, i64, C.c_void_p, dbl, u64, _ip, P(i64)]
        L.kidh_kernel_rows.argtypes = [_dp, i64, i32, _ip, _ip, i64, _ip, i64, dbl, _dp]
        L.kidh_error_pass.argtypes = [C.c_void_p, dbl, _ip, i64, _dp, dbl, P(dbl), P(dbl), P(dbl)]
        L.kidh_trial_next_rows.argtypes = [i32, i32, i64, i64, dbl, dbl, u64, dbl, u64, dbl, dbl, i32, u64, _dp,
                                           P(i64), P(i64), _ip, _dp, _dp, _dp, i64]
        L.kidh_sharded_compress_trial.argtypes = [C.c_void_p, i32, i32, i64, i64, dbl, dbl, u64, dbl, u64, dbl,
                                                  P(i64), P(i64), P(dbl), P(dbl), _ip, _ip, P(i64), P(i32)]
        L.kidh_compress_trial.argtypes = [i32, i32, i64, i64, dbl, dbl, u64, i32, i64, dbl, u64, dbl, P(i64), P(i64),
                                          P(dbl), P(dbl), _ip, _ip, P(i64)]
        L.kidh_trial_spectrum.argtypes = [i32, i32, i64, i64, dbl, dbl, u64, dbl, i64, P(i64), _dp, _dp, _dp, i64]
        L.kidh_trial_svd.argtypes = [i32, i32, i64, i64, dbl, dbl, u64, dbl, u64, dbl, P(i64), P(dbl), P(dbl), _dp]
        L.kidh_interaction_fractions.argtypes = [i32, i32, i64, u64, dbl, _dp, i64, _dp]
        L.kidh_bandwidth_search.argtypes = [i32, i32, i64, i64, dbl, dbl, i32, dbl, i32, i32, u64, _dp, _dp, i32,
                                            P(i32), i32]
        L.kidh_run_experiment.argtypes = [i32, i32, i64, i64, dbl, dbl, i32, i64, _dp, i32, dbl, i32, u64, C.c_char_p,
                                          i32, dbl, i32]
        _host = L
    return _host


def _ck(rc, what):
    if rc:
        raise KidError(rc, f"{what}: {host_lib().kidh_last_error().decode(errors='replace')}")


def _cm(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).ravel()


def _uncm(flat, rows, cols):
    return np.asarray(flat).reshape(cols, rows).T.copy()


def derive_seed(master: int, a: int, b: int = 0) -> int:
    return int(host_lib().kidh_derive_seed(master, a, b))


def center_index(N: int, data_seed: int) -> int:
    """RandomPoint center row (harness.hpp:95-100)."""
    return int(host_lib().kidh_center_index(N, data_seed))


def gen_normal(d: int, N: int, seed: int) -> np.ndarray:
    out = np.zeros(N * d)
    _ck(host_lib().kidh_gen_normal(d, N, seed, out), "gen_normal")
    return _uncm(out, N, d)


def singular_values(A) -> np.ndarray:
    A = np.asarray(A, dtype=np.float64)
    sv = np.zeros(min(A.shape))
    _ck(host_lib().kidh_singular_values(_cm(A), A.shape[0], A.shape[1], sv), "singular_values")
    return sv


def epsilon_rank(sv, eps: float, ref_sigma1: float | None = None) -> int:
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    r = C.c_int64()
    _ck(host_lib().kidh_epsilon_rank(sv, sv.size, eps, ref_sigma1 or -1.0, C.byref(r)), "epsilon_rank")
    return r.value


def interpolative_decomposition(A, r: int):
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    skel = np.zeros(max(r, 1), np.int64)
    P = np.zeros(max(r, 1) * n)
    _ck(host_lib().kidh_interpolative_decomposition(_cm(A), m, n, r, skel, P), "interpolative_decomposition")
    return skel[:r].copy(), _uncm(P[: r * n], r, n)


def sym_eigvals(A):
    """Eigenvalues (descending) of a symmetric matrix: Householder tridiagonalisation + QL."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    ev = np.zeros(n)
    _ck(host_lib().kidh_sym_eigvals(_cm(A), n, ev), "sym_eigvals")
    return ev


def lambda_max(A) -> float:
    """Largest eigenvalue of a symmetric PSD matrix (Jacobi for n <= 128, Lanczos above)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    if n == 0:
        return 0.0
    v = C.c_double()
    _ck(host_lib().kidh_lambda_max(_cm(A), n, C.byref(v)), "lambda_max")
    return v.value


def sym_eig(A):
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    ev = np.zeros(n)
    V = np.zeros(n * n)
    _ck(host_lib().kidh_sym_eig(_cm(A), n, ev, V.ctypes.data), "sym_eig")
    return ev, _uncm(V, n, n)


def draw(kind: int, m: int, s: float, seed: int, weights=None, replacement: bool = False) -> np.ndarray:
    """sample_rows' draw step (sampling.hpp:156-243) for given weights (host)."""
    out = np.zeros(max(m, 1), np.int64)
    cnt = C.c_int64()
    wp = None
    if weights is not None:
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        wp = weights.ctypes.data
    _ck(host_lib().kidh_draw(kind, int(replacement), m, wp, s, seed, out, C.byref(cnt)), "sample_rows")
    return out[: cnt.value].copy()


def kernel_rows(points_colmajor: np.ndarray, N: int, d: int, tgt_idx, rows, src_idx, h: float) -> np.ndarray:
    """Host K rows with the reference arithmetic (gather_rows of kernel_matrix)."""
    tgt_idx = np.ascontiguousarray(tgt_idx, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    src_idx = np.ascontiguousarray(src_idx, dtype=np.int64)
    out = np.zeros(max(rows.size * src_idx.size, 1))
    _ck(host_lib().kidh_kernel_rows(points_colmajor, N, d, tgt_idx, rows, rows.size, src_idx, src_idx.size, h, out),
        "kernel_rows")
    return _uncm(out[: rows.size * src_idx.size], rows.size, src_idx.size)


def error_pass(dev, h: float, skel, P, k_norm: float = 0.0):
    """compress_id's error pass (compress.hpp:178-206) through the host mirror on the block held by
    the C-ABI Device `dev`: (rel_error, rel_error_fro, ||K||_2). k_norm > 0 skips the K^T K pass."""
    skel = np.ascontiguousarray(skel, dtype=np.int64)
    Pc = _cm(np.asarray(P, dtype=np.float64))
    rel, fro, kn = C.c_double(), C.c_double(), C.c_double()
    _ck(host_lib().kidh_error_pass(dev.h, h, skel, skel.size, Pc, k_norm, C.byref(rel), C.byref(fro), C.byref(kn)),
        "error_pass")
    return rel.value, fro.value, kn.value


@dataclass
class TrialResult:
    n_targets: int
    rank: int
    rel_error: float
    rel_error_fro: float
    skeleton: np.ndarray
    sample: np.ndarray


def compress_trial(d, N, n, xi, data_seed, scheme, s, sample_seed, eps, h_value=1.0, lev_rank=0, device=0):
    """prepare_trial + sample_rows + compress_id through the C++ mirror on the GPU."""
    nt, rank, cnt = C.c_int64(), C.c_int64(), C.c_int64()
    rel, relf = C.c_double(), C.c_double()
    skel = np.zeros(n, np.int64)
    sample = np.zeros(N, np.int64)
    _ck(host_lib().kidh_compress_trial(device, d, N, n, xi, h_value, data_seed, scheme, lev_rank, s, sample_seed, eps,
                                       C.byref(nt), C.byref(rank), C.byref(rel), C.byref(relf), skel, sample,
                                       C.byref(cnt)), "compress_trial")
    return TrialResult(nt.value, rank.value, rel.value, relf.value, skel[: rank.value].copy(), sample[: cnt.value].copy())


def sharded_compress_trial(devices, d, N, n, xi, data_seed, s, sample_seed, eps, h_value=1.0):
    """compress_trial (EuclideanNorm) with the targets sharded over `devices` by the C++ multi-GPU mirror
    (DeviceGroup / ShardedBlock, NCCL reductions for distinct devices). Returns (TrialResult, used_nccl)."""
    dv = np.ascontiguousarray(devices, dtype=np.int32)
    nt, rank, cnt, nccl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    rel, fro = C.c_double(), C.c_double()
    skel = np.zeros(n, np.int64)
    smp = np.zeros(max(N, 1), np.int64)
    _ck(host_lib().kidh_sharded_compress_trial(dv.ctypes.data, dv.size, d, N, n, xi, h_value, data_seed, s, sample_seed,
                                               eps, C.byref(nt), C.byref(rank), C.byref(rel), C.byref(fro), skel, smp,
                                               C.byref(cnt), C.byref(nccl)), "sharded_compress_trial")
    return TrialResult(nt.value, rank.value, rel.value, fro.value, skel[: rank.value].copy(),
                       smp[: cnt.value].copy()), bool(nccl.value)


def trial_next_rows(d, N, n, xi, data_seed, s, sample_seed, eps, s_mc, n_mc, mc_seed, q, h_value=1.0, device=0):
    """A uniform-sampling compress trial through the C++ mirror, then mc_error (compress.hpp:279-305)
    and apply_skeleton (compress.hpp:309-325) on its ID. Returns (n_targets, rank, skeleton, P
    (rank x n), mc estimates, u)."""
    nt, rank = C.c_int64(), C.c_int64()
    skel = np.zeros(n, np.int64)
    P = np.zeros(n * n)
    mc = np.zeros(n_mc)
    u = np.zeros(N)
    q = np.ascontiguousarray(q, dtype=np.float64)
    _ck(host_lib().kidh_trial_next_rows(device, d, N, n, xi, h_value, data_seed, s, sample_seed, eps, s_mc, n_mc,
                                        mc_seed, q, C.byref(nt), C.byref(rank), skel, P, mc, u, N), "trial_next_rows")
    r = rank.value
    return (nt.value, r, skel[:r].copy(), P[: r * n].reshape(n, r).T.copy() if r else np.zeros((0, n)), mc,
            u[: nt.value].copy())


def trial_spectrum(d, N, n, xi, data_seed, resolve=0.0, lev_rank=0, h_value=1.0, device=0):
    """singular_values / right_factor of a trial's full block K(T, S) (lowrank.hpp:56-90) through the C++
    mirror: device TSQR for n <= 128, the Gram route plus its preconditioned second pass above that
    (`resolve`: the relative level the spectrum is needed to; 0 = all). With lev_rank > 0 also
    row_leverage_scores(K, lev_rank). Returns (n_targets, sv, V, scores or None)."""
    nt = C.c_int64()
    sv = np.zeros(n)
    V = np.zeros(n * n)
    scores = np.zeros(N if lev_rank > 0 else 1)
    _ck(host_lib().kidh_trial_spectrum(device, d, N, n, xi, h_value, data_seed, resolve, lev_rank, C.byref(nt), sv, V,
                                       scores, scores.size), "trial_spectrum")
    return nt.value, sv, _uncm(V, n, n), (scores[: nt.value].copy() if lev_rank > 0 else None)


def trial_svd(d, N, n, xi, data_seed, s, sample_seed, eps, h_value=1.0, device=0):
    """A uniform-sampling compress_svd trial (compress.hpp:219-273) through the C++ mirror.
    Returns (rank, rel_error, rel_error_fro, V_r (n x rank))."""
    rank, rel, fro = C.c_int64(), C.c_double(), C.c_double()
    V = np.zeros(n * n)
    _ck(host_lib().kidh_trial_svd(device, d, N, n, xi, h_value, data_seed, s, sample_seed, eps, C.byref(rank),
                                  C.byref(rel), C.byref(fro), V), "trial_svd")
    r = rank.value
    return r, rel.value, fro.value, _uncm(V[: n * r], n, r)


def run_experiment(path: str, d, N, n, xi, scheme, s_grid, eps, trials=1, seed=1, h_value=1.0, lev_rank=0, device=0,
                   methods=("id",), s_mc=None, n_mc=1):
    """kernid_b200::run_experiment (harness.hpp:143-328): the compress sweep CSV. `methods` in
    {"id", "svd"} (config "methods"); `s_mc` / `n_mc` the config's mc_error block."""
    s_grid = np.ascontiguousarray(s_grid, dtype=np.float64)
    mask = (1 if "id" in methods else 0) | (2 if "svd" in methods else 0)
    _ck(host_lib().kidh_run_experiment(device, d, N, n, xi, h_value, scheme, lev_rank, s_grid, s_grid.size, eps, trials,
                                       seed, path.encode(), mask, s_mc if s_mc else 0.0, n_mc), "run_experiment")
    with open(path) as f:
        return f.read()


def interaction_fractions(d, N, seed, h, x_c, n, device=0):
    """interaction_fractions (compress.hpp:327-378) over gen_normal(d, N, seed); (self, nn, far)."""
    f = np.zeros(3)
    _ck(host_lib().kidh_interaction_fractions(device, d, N, seed, h, np.ascontiguousarray(x_c, dtype=np.float64), n, f),
        "interaction_fractions")
    return tuple(float(x) for x in f)


class SearchFailure(KidError):
    def __init__(self, code, msg, profile):
        super().__init__(code, msg)
        self.profile = profile


def bandwidth_search(d, N, n, xi, data_seed, kappa=0.2, large_h=False, eps=1e-2, max_iters=40, tol_rows=2, device=0,
                     center="origin"):
    """bandwidth_search (harness.hpp:330-438) through the mirror (center: "origin", the reference
    default, or "random"): dict(h_abs, h_over_hs, rank,
    evaluations, converged, profile); raises SearchFailure (with the profile) when it cannot bracket."""
    out = np.zeros(5)
    prof = np.zeros(2 * 256)
    npf = C.c_int32()
    rc = host_lib().kidh_bandwidth_search(device, d, N, n, xi, kappa, int(large_h), eps, max_iters, tol_rows, data_seed,
                                          out, prof, 256, C.byref(npf), int(center == "random"))
    profile = [(float(prof[2 * i]), int(prof[2 * i + 1])) for i in range(npf.value)]
    if rc:
        raise SearchFailure(rc, f"bandwidth_search: {host_lib().kidh_last_error().decode(errors='replace')}", profile)
    return dict(h_abs=float(out[0]), h_over_hs=float(out[1]), rank=int(out[2]), evaluations=int(out[3]),
                converged=bool(out[4]), profile=profile)
