"""ctypes binding of libkernid_cuda.so (include/kernid_cuda.h).

The product path has no fallback: if the CUDA library is missing or no device is
present, calls fail loudly (KidError / OSError). The oracle is never imported here.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
CUDA_SO = os.path.join(PKG, "libkernid_cuda.so")

KID_OK, KID_E_RANGE, KID_E_DIM, KID_E_NO_TARGETS, KID_E_NUMERICAL = 0, 1, 2, 3, 4
KID_E_ERROR, KID_E_CUDA, KID_E_OOM, KID_E_ILLCOND, KID_E_CONFIG = 5, 6, 7, 8, 9
KID_RECON_DTD, KID_RECON_KTK = 1, 2

ERROR_NAMES = {1: "RangeError", 2: "DimensionError", 3: "NoTargetsError", 4: "NumericalError", 5: "Error",
               6: "Error(CUDA)", 7: "Error(OOM)", 8: "IllConditionedSkeletonError", 9: "ConfigError"}


class KidError(RuntimeError):
    """Mirror of the reference exception taxonomy (errors.hpp:11-77); .code is the kid status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, 'Error')}: {msg}")
        self.code = code


_cuda = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")

SYMBOLS = ["kid_abi_version", "kid_host_alloc", "kid_host_free", "kid_create", "kid_destroy", "kid_last_error", "kid_set_stream", "kid_synchronize",
           "kid_set_points", "kid_set_points_device", "kid_split", "kid_split_candidates", "kid_split_finish",
           "kid_get_targets", "kid_set_block", "kid_block_shape", "kid_row_norms", "kid_row_norms_dev", "kid_gram",
           "kid_gram_dev", "kid_leverage", "kid_leverage_dev", "kid_recon_error", "kid_recon_prepare",
           "kid_recon_error_dev", "kid_eval_rows", "kid_apply_skeleton", "kid_apply_skeleton_dev", "kid_select_rows",
           "kid_launch_count", "kid_profile", "kid_profile_read", "kid_exp_check", "kid_set_path", "kid_last_kernel", "kid_set_option",
           "kid_device_id", "kid_stream", "kid_device_alloc", "kid_device_free", "kid_memcpy_dtoh", "kid_guard_check"]


def cuda_lib():
    """Load libkernid_cuda.so (raises OSError if it was not built)."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_SO):
            raise OSError(f"{CUDA_SO} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(CUDA_SO)
        i64, i32, dbl, vp, u32 = C.c_int64, C.c_int32, C.c_double, C.c_void_p, C.c_uint32
        P = C.POINTER
        L.kid_abi_version.restype = C.c_int
        L.kid_host_alloc.restype = vp
        L.kid_host_alloc.argtypes = [C.c_size_t]
        L.kid_host_free.argtypes = [vp]
        L.kid_host_free.restype = None
        L.kid_create.argtypes = [P(vp), i32]
        L.kid_destroy.argtypes = [vp]
        L.kid_destroy.restype = None
        L.kid_last_error.argtypes = [vp]
        L.kid_last_error.restype = C.c_char_p
        L.kid_set_stream.argtypes = [vp, vp]
        L.kid_synchronize.argtypes = [vp]
        L.kid_set_path.argtypes = [vp, i32]
        L.kid_last_kernel.argtypes = [vp]
        L.kid_set_option.argtypes = [vp, i32, i64]
        L.kid_last_kernel.restype = C.c_char_p
        L.kid_set_points.argtypes = [vp, vp, i64, i32, i64]
        L.kid_set_points_device.argtypes = [vp, vp, i64, i32, i64]
        L.kid_split.argtypes = [vp, _dp, i64, dbl, _ip, P(dbl), P(i64)]
        L.kid_split_candidates.argtypes = [vp, _dp, i64, _dp, _ip]
        L.kid_split_finish.argtypes = [vp, _ip, i64, vp, dbl, dbl, P(i64)]
        L.kid_get_targets.argtypes = [vp, _ip, i64]
        L.kid_set_block.argtypes = [vp, _dp, i64, _dp, i64, i32]
        L.kid_block_shape.argtypes = [vp, P(i64), P(i64), P(i32)]
        L.kid_row_norms.argtypes = [vp, dbl, _dp]
        L.kid_row_norms_dev.argtypes = [vp, dbl, vp]
        L.kid_gram.argtypes = [vp, dbl, _dp, P(dbl)]
        L.kid_gram_dev.argtypes = [vp, dbl, vp, vp]
        L.kid_leverage.argtypes = [vp, dbl, _dp, i64, _dp]
        L.kid_leverage_dev.argtypes = [vp, dbl, vp, i64, vp]
        L.kid_recon_error.argtypes = [vp, dbl, _ip, i64, _dp, u32, P(dbl), P(dbl), vp, vp]
        L.kid_recon_prepare.argtypes = [vp, _ip, i64, _dp]
        L.kid_recon_error_dev.argtypes = [vp, dbl, u32, vp]
        L.kid_eval_rows.argtypes = [vp, dbl, _ip, i64, _dp]
        L.kid_tsqr_r.argtypes = [vp, dbl, _dp]
        L.kid_tsqr_r_dev.argtypes = [vp, dbl, vp]
        L.kid_tsqr_combine.argtypes = [vp, _dp, i64, i64, _dp]
        L.kid_proj_gram.argtypes = [vp, dbl, _dp, i64, P(dbl), P(dbl), vp]
        L.kid_proj_gram_dev.argtypes = [vp, dbl, vp, i64, vp]
        L.kid_apply_skeleton.argtypes = [vp, dbl, _ip, i64, _dp, _dp, _dp]
        L.kid_apply_skeleton_dev.argtypes = [vp, dbl, _ip, i64, _dp, vp]
        L.kid_select_rows.argtypes = [vp, vp, i64]
        L.kid_launch_count.argtypes = [vp]
        L.kid_launch_count.restype = i64
        L.kid_profile.argtypes = [vp, i32]
        L.kid_exp_check.argtypes = [vp, _dp, i64, _dp]
        L.kid_guard_check.argtypes = [vp]
        L.kid_device_alloc.argtypes = [vp, C.c_size_t]
        L.kid_device_alloc.restype = vp
        L.kid_device_free.argtypes = [vp, vp]
        L.kid_device_free.restype = None
        L.kid_guard_check.restype = i64
        L.kid_profile_read.argtypes = [vp, vp, i64, P(i64)]
        _cuda = L
    return _cuda


def _colmajor(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(a.T).ravel()


class Device:
    """One kid_ctx (one CUDA device, one stream). Methods mirror the C-ABI 1:1 with numpy I/O."""

    def __init__(self, device: int = 0):
        self.L = cuda_lib()
        h = C.c_void_p()
        rc = self.L.kid_create(C.byref(h), device)
        if rc:
            raise KidError(rc, f"kid_create(device={device}) failed (no CUDA device?)")
        self.h = h
        self._pinned = None  # (ptr, bytes) reusable page-locked buffer
        self.N = 0
        self.d = 0
        self.m = 0
        self.nt = 0

    def close(self):
        if self._pinned:
            self.L.kid_host_free(self._pinned[0])
            self._pinned = None
        if self.h:
            self.L.kid_destroy(self.h)
            self.h = None

    def pinned(self, nbytes: int) -> int:
        """A reusable page-locked host buffer of at least nbytes (freed with the Device)."""
        if not self._pinned or self._pinned[1] < nbytes:
            if self._pinned:
                self.L.kid_host_free(self._pinned[0])
            ptr = self.L.kid_host_alloc(max(nbytes, 1))
            if not ptr:
                raise KidError(KID_E_OOM, "kid_host_alloc failed")
            self._pinned = (ptr, nbytes)
        return self._pinned[0]

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc, what=""):
        if rc:
            raise KidError(rc, f"{what}: {self.L.kid_last_error(self.h).decode(errors='replace')}")

    @property
    def launches(self) -> int:
        return int(self.L.kid_launch_count(self.h))

    def profile(self, enable: bool):
        self._ck(self.L.kid_profile(self.h, int(enable)), "kid_profile")

    def profile_read(self) -> np.ndarray:
        cap = 1 << 16
        buf = np.zeros(cap)
        n = C.c_int64()
        self._ck(self.L.kid_profile_read(self.h, buf.ctypes.data, cap, C.byref(n)), "kid_profile_read")
        return buf[: min(n.value, cap)].copy()

    def device_alloc(self, nbytes: int) -> int:
        p = self.L.kid_device_alloc(self.h, nbytes)
        if not p:
            raise KidError(KID_E_OOM, "kid_device_alloc failed")
        return int(p)

    def device_free(self, p: int):
        self.L.kid_device_free(self.h, p)

    def guard_check(self) -> int:
        """Corrupted canary bytes around the library's device buffers (-DKID_GUARD build); -1 without guards."""
        return int(self.L.kid_guard_check(self.h))

    def exp_check(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(max(x.size, 1))
        self._ck(self.L.kid_exp_check(self.h, x, x.size, y), "kid_exp_check")
        return y[: x.size].copy()

    def recon_prepare(self, skel, P):
        skel = np.ascontiguousarray(skel, dtype=np.int64)
        self._ck(self.L.kid_recon_prepare(self.h, skel, skel.size, _colmajor(P)), "kid_recon_prepare")

    def recon_error_dev(self, h: float, out_ptr: int, flags: int = KID_RECON_DTD):
        self._ck(self.L.kid_recon_error_dev(self.h, h, flags, out_ptr), "kid_recon_error_dev")

    def set_stream(self, stream_ptr: int | None):
        self._ck(self.L.kid_set_stream(self.h, stream_ptr or None), "kid_set_stream")

    def set_path(self, path: int):
        """KID_PATH_AUTO (0) or KID_PATH_CLUSTER (1): force the 2-CTA cluster kernel (kid_set_path)."""
        self._ck(cuda_lib().kid_set_path(self.h, int(path)), "kid_set_path")

    def set_option(self, key: int, value: int):
        """kid_set_option: KID_OPT_EVAL_WARPS (1) = 0 (auto), 8 or 12."""
        self._ck(cuda_lib().kid_set_option(self.h, int(key), int(value)), "kid_set_option")

    def last_kernel(self) -> str:
        return cuda_lib().kid_last_kernel(self.h).decode()

    def synchronize(self):
        self._ck(self.L.kid_synchronize(self.h), "kid_synchronize")

    # -- points / split
    def set_points(self, points: np.ndarray, index_offset: int = 0):
        """points: (N, d) array (any layout); uploaded column-major."""
        N, d = points.shape
        buf = _colmajor(points)
        self._ck(self.L.kid_set_points(self.h, buf.ctypes.data, N, d, index_offset), "kid_set_points")
        self.synchronize()
        self.N, self.d = N, d

    def set_points_colmajor_ptr(self, ptr: int, N: int, d: int, index_offset: int = 0, device: bool = False):
        f = self.L.kid_set_points_device if device else self.L.kid_set_points
        self._ck(f(self.h, ptr, N, d, index_offset), "kid_set_points")
        self.N, self.d = N, d

    def split(self, center, n: int, xi: float):
        center = np.ascontiguousarray(center, dtype=np.float64)
        if center.size != self.d:
            raise KidError(KID_E_DIM, "split_sources_targets: center dimension mismatch")
        src = np.zeros(max(n, 1), np.int64)
        rho = C.c_double()
        nt = C.c_int64()
        self._ck(self.L.kid_split(self.h, center, n, xi, src, C.byref(rho), C.byref(nt)), "kid_split")
        self.nt, self.m = nt.value, n
        return src[:n].copy(), rho.value, nt.value

    def split_candidates(self, center, n: int):
        center = np.ascontiguousarray(center, dtype=np.float64)
        k = min(n, self.N)
        cd = np.zeros(k)
        ci = np.zeros(k, np.int64)
        self._ck(self.L.kid_split_candidates(self.h, center, n, cd, ci), "kid_split_candidates")
        return cd, ci

    def split_finish(self, src_idx, rho: float, xi: float, src_points=None):
        src_idx = np.ascontiguousarray(src_idx, dtype=np.int64)
        nt = C.c_int64()
        sp = None
        if src_points is not None:
            sp_buf = _colmajor(src_points)
            sp = sp_buf.ctypes.data
        self._ck(self.L.kid_split_finish(self.h, src_idx, src_idx.size, sp, rho, xi, C.byref(nt)), "kid_split_finish")
        self.nt, self.m = nt.value, src_idx.size
        return nt.value

    def targets(self, view: bool = False) -> np.ndarray:
        """Target indices (geometry.hpp:58-60). view=True returns a view of the Device's pinned
        buffer (no host copy; valid until the next pinned-buffer use)."""
        if view:
            ptr = self.pinned(8 * max(self.nt, 1))
            out = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_int64)), shape=(max(self.nt, 1),))
            self._ck(self.L.kid_get_targets.__call__(self.h, out, self.nt), "kid_get_targets")
            return out[: self.nt]
        out = np.zeros(max(self.nt, 1), np.int64)
        self._ck(self.L.kid_get_targets(self.h, out, self.nt), "kid_get_targets")
        return out[: self.nt].copy()

    def set_block(self, targets: np.ndarray, sources: np.ndarray):
        nt, d = targets.shape
        m = sources.shape[0]
        self._ck(self.L.kid_set_block(self.h, _colmajor(targets) if nt else np.zeros(1), nt, _colmajor(sources), m, d),
                 "kid_set_block")
        self.nt, self.m, self.d = nt, m, d

    # -- passes
    def row_norms(self, h: float) -> np.ndarray:
        w = np.zeros(max(self.nt, 1))
        self._ck(self.L.kid_row_norms(self.h, h, w), "kid_row_norms")
        return w[: self.nt].copy()

    def row_norms_dev(self, h: float, d_w: int):
        self._ck(self.L.kid_row_norms_dev(self.h, h, d_w), "kid_row_norms_dev")

    def gram(self, h: float):
        G = np.zeros(self.m * self.m)
        sk = C.c_double()
        self._ck(self.L.kid_gram(self.h, h, G, C.byref(sk)), "kid_gram")
        return G.reshape(self.m, self.m).T.copy(), sk.value

    def gram_dev(self, h: float, d_out: int):
        """d_out (device) <- [sumsq_K, sumsq_K, K^T K (m x m)] (kid_gram_dev)."""
        self._ck(self.L.kid_gram_dev(self.h, h, d_out, None), "kid_gram_dev")

    def leverage_dev(self, h: float, d_W: int, r: int, d_scores: int):
        self._ck(self.L.kid_leverage_dev(self.h, h, d_W, r, d_scores), "kid_leverage_dev")

    def leverage(self, h: float, W: np.ndarray) -> np.ndarray:
        r = W.shape[1]
        out = np.zeros(max(self.nt, 1))
        self._ck(self.L.kid_leverage(self.h, h, _colmajor(W), r, out), "kid_leverage")
        return out[: self.nt].copy()

    def recon_error(self, h: float, skel, P: np.ndarray, flags: int = KID_RECON_DTD, grams: bool = True):
        skel = np.ascontiguousarray(skel, dtype=np.int64)
        r = skel.size
        m = self.m
        sd, sk = C.c_double(), C.c_double()
        DtD = np.zeros(m * m) if grams else None
        KtK = np.zeros(m * m) if (grams and flags & KID_RECON_KTK) else None
        Pf = _colmajor(P) if r else np.zeros(1)
        self._ck(self.L.kid_recon_error(self.h, h, skel if r else np.zeros(1, np.int64), r, Pf, flags,
                                        C.byref(sd), C.byref(sk),
                                        DtD.ctypes.data if DtD is not None else None,
                                        KtK.ctypes.data if KtK is not None else None), "kid_recon_error")
        return (sd.value, sk.value, DtD.reshape(m, m).T.copy() if DtD is not None else None,
                KtK.reshape(m, m).T.copy() if KtK is not None else None)

    def tsqr_r(self, h: float) -> np.ndarray:
        """Upper-triangular R with R^T R = K^T K (kid_tsqr_r, Householder TSQR over all targets)."""
        R = np.zeros(max(self.m * self.m, 1))
        self._ck(self.L.kid_tsqr_r(self.h, h, R), "kid_tsqr_r")
        return R[: self.m * self.m].reshape(self.m, self.m).T.copy()

    def tsqr_r_dev(self, h: float, d_R: int):
        self._ck(self.L.kid_tsqr_r_dev(self.h, h, d_R), "kid_tsqr_r_dev")

    def tsqr_combine(self, Rs) -> np.ndarray:
        """Fold stacked m x m factors into one (kid_tsqr_combine)."""
        Rs = [np.asarray(R, dtype=np.float64) for R in Rs]
        m = Rs[0].shape[0]
        flat = np.concatenate([_colmajor(R) for R in Rs])
        out = np.zeros(m * m)
        self._ck(self.L.kid_tsqr_combine(self.h, flat, len(Rs), m, out), "kid_tsqr_combine")
        return out.reshape(m, m).T.copy()

    def proj_gram(self, h: float, Cm: np.ndarray):
        """(||K C||_F^2, ||K||_F^2, (K C)^T (K C)) for an m x n coefficient matrix C
        (kid_proj_gram: the compress_svd error pass with C = V_perp)."""
        n = Cm.shape[1]
        sd, sk = C.c_double(), C.c_double()
        G = np.zeros(n * n)
        self._ck(self.L.kid_proj_gram(self.h, h, _colmajor(Cm), n, C.byref(sd), C.byref(sk), G.ctypes.data),
                 "kid_proj_gram")
        return sd.value, sk.value, G.reshape(n, n).T.copy()

    def proj_gram_dev(self, h: float, d_C: int, n: int, d_out: int):
        self._ck(self.L.kid_proj_gram_dev(self.h, h, d_C, n, d_out), "kid_proj_gram_dev")

    def apply_skeleton(self, h: float, skel, P: np.ndarray, q) -> np.ndarray:
        """u = K(T, S[skel]) (P q) over the block's targets (kid_apply_skeleton)."""
        skel = np.ascontiguousarray(skel, dtype=np.int64)
        r = skel.size
        q = np.ascontiguousarray(q, dtype=np.float64)
        u = np.zeros(max(self.nt, 1))
        Pf = _colmajor(P) if r else np.zeros(1)
        self._ck(self.L.kid_apply_skeleton(self.h, h, skel if r else np.zeros(1, np.int64), r, Pf, q, u),
                 "kid_apply_skeleton")
        return u[: self.nt].copy()

    def apply_skeleton_dev(self, h: float, skel, q_skel, d_u: int):
        skel = np.ascontiguousarray(skel, dtype=np.int64)
        self._ck(self.L.kid_apply_skeleton_dev(self.h, h, skel, skel.size,
                                               np.ascontiguousarray(q_skel, dtype=np.float64), d_u),
                 "kid_apply_skeleton_dev")

    def select_rows(self, rows=None):
        """Restrict the block's targets to rows of the full list (None: restore it)."""
        if rows is None:
            self._ck(self.L.kid_select_rows(self.h, None, -1), "kid_select_rows")
        else:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            self._ck(self.L.kid_select_rows(self.h, rows.ctypes.data if rows.size else None, rows.size),
                     "kid_select_rows")
        nt, m, d = C.c_int64(), C.c_int64(), C.c_int32()
        self._ck(self.L.kid_block_shape(self.h, C.byref(nt), C.byref(m), C.byref(d)), "kid_block_shape")
        self.nt = nt.value

    def eval_rows(self, h: float, rows) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros(max(rows.size * self.m, 1))
        self._ck(self.L.kid_eval_rows(self.h, h, rows, rows.size, out), "kid_eval_rows")
        return out[: rows.size * self.m].reshape(self.m, rows.size).T.copy()
